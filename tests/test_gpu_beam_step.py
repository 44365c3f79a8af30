"""GPU vs oracle: trie_beam_step (log-softmax + global top-b, Alg. 2 l.9) on identical fp32
logits.  Near-tie protocol: where the oracle's gap between rank b-1 and
rank b exceeds tau = 1e-5 * max(1, |score|) the selection (parents, tokens, ORDER) must be
identical; otherwise the GPU's set must be tau-valid.  Scores within 1e-4 relative
(BASELINE.json north_star fp32 tolerance, reading R24/R25)."""
import numpy as np
import pytest
import torch

import synth
from oracle.kernels_ref import beam_step_ref
from tests.gpu_util import need_gpu

pytestmark = pytest.mark.gpu


def _check(logits, scores, b, par, tok, sc):
    """Near-tie protocol + R3 validity.  Always: b distinct (j, v) pairs in range; the set is
    a tau-valid top-b (every selected score >= every unselected score - tau); ranks are
    non-increasing within tau; where two candidates tie EXACTLY in fp64 (same beam and equal
    logits, e.g. quantised logits) their relative order -- inside the selection and across
    the rank-b boundary -- is R3's (token asc, then beam asc; Alg. 2 l.9 argsort_b P:146).
    Where the oracle's rank-b gap exceeds tau the selection must equal the oracle's,
    order included, up to adjacent ranks that are themselves near-tied."""
    refp, reft, refs, gap, lp = beam_step_ref(logits, scores, b)
    J, V = lp.shape
    k = min(b, J * V)
    tau = 1e-5 * max(1.0, float(np.abs(refs).max()))
    par, tok = np.asarray(par)[:k], np.asarray(tok)[:k]
    assert ((par >= 0) & (par < J)).all() and ((tok >= 0) & (tok < V)).all(), "index out of range"
    pairs = list(zip(par.tolist(), tok.tolist()))
    assert len(set(pairs)) == k, f"duplicate selections: {pairs}"
    cs_all = np.asarray(scores, np.float64)[:, None] + lp            # [J][V] fp64
    cs = np.array([cs_all[j, v] for j, v in pairs])
    sel = np.zeros((J, V), bool)
    sel[par, tok] = True
    rest = cs_all[~sel]
    rest = rest[np.isfinite(rest)]
    if rest.size:
        assert cs.min() >= rest.max() - tau, "selected set is not a tau-valid top-b"
        # exact fp64 ties across the rank-b boundary resolve by (v asc, j asc)
        worst = cs.min()
        for jj, vv in zip(*np.nonzero((cs_all == worst) & ~sel)):
            for (j, v), c in zip(pairs, cs):
                if c == worst:
                    assert (v, j) < (vv, jj), f"R3 boundary order: ({j},{v}) selected over ({jj},{vv})"
    for i in range(k - 1):
        assert cs[i] >= cs[i + 1] - tau, "ranks out of order"
        if cs[i] == cs[i + 1]:
            assert (pairs[i][1], pairs[i][0]) < (pairs[i + 1][1], pairs[i + 1][0]), "R3 tie order"
    if gap > tau:
        # identical except where adjacent ranks are themselves near-tied (order only)
        same = (np.array_equal(par, refp) and np.array_equal(tok, reft))
        if not same:
            ranks_ok = all(abs(refs[i] - refs[i + 1]) <= tau for i in range(len(refs) - 1)
                           if (par[i], tok[i]) != (refp[i], reft[i]))
            assert ranks_ok, f"selection differs: {pairs} vs {list(zip(refp, reft))}"
            assert set(pairs) == set(zip(refp.tolist(), reft.tolist()))
    assert np.all(np.abs(sc[:k] - cs) <= 1e-4 * np.maximum(1.0, np.abs(cs)))
    return gap <= tau


@pytest.mark.parametrize("R,b,V,kappa", [(2, 3, 256, 4.0), (3, 4, 32064, 3.0), (2, 8, 128256, 3.0),
                                         (1, 32, 131072, 2.0), (4, 1, 5000, 1.0), (2, 16, 4097, 5.0),
                                         (2, 5, 5, 1.0), (2, 8, 40000, -2.0),
                                         (1, 32, 131072, -1.0), (2, 4, 32064, -0.25)])
def test_beam_step_matches_oracle(R, b, V, kappa):
    """kappa < 0: logits quantised to multiples of |kappa| -- thousands of exact ties per
    chunk overflow the kernel's candidate buffer and exercise its arg-max fallback."""
    need_gpu()
    from paper_2502_00085_b200.trie import TrieState
    seed = b * 7 + V
    prompts, lens = synth.prompts(seed, R, 6, V)
    st = TrieState(R, b, 6, 6 + 4 * b + b, 0, 1, 1, 16, V, prompts, lens, dtype=torch.float32)
    scores = np.zeros((R, 1))
    near = 0
    for step in range(3):
        b_live = 1 if step == 0 else b
        logits = synth.normal(seed, 10 + step, (R, b_live, V)) * abs(kappa)
        if kappa < 0:
            logits = np.round(logits / abs(kappa)) * abs(kappa)
        logits = logits.astype(np.float32)
        lt = torch.as_tensor(logits, device="cuda")
        par = torch.empty(R, b, dtype=torch.int32, device="cuda")
        tok = torch.empty_like(par)
        sc = torch.empty(R, b, dtype=torch.float32, device="cuda")
        st.beam_step(lt, par, tok, sc)
        par, tok, sc = par.cpu().numpy(), tok.cpu().numpy(), sc.cpu().numpy()
        for r in range(R):
            near += _check(logits[r], scores[r], b, par[r], tok[r], sc[r])
            if kappa < 0 and step == 0:  # one row: exact ties resolve by token asc (R3)
                refp, reft, _, _, _ = beam_step_ref(logits[r], scores[r], b)
                assert tok[r].tolist() == list(reft) and par[r].tolist() == list(refp)
        # the trie grew by the selections: leaves are the new slots, depth t + step
        leaf = st.leaf.cpu().numpy()[:, :b]
        N = st.n_nodes.cpu().numpy()
        assert np.array_equal(leaf, N[:, None] - b + np.arange(b))
        scores = sc.astype(np.float64)  # lockstep on the GPU's own choice (protocol)
    assert st.status() == 0
    assert near <= 1 or kappa < 0


def test_beam_step_exact_ties_follow_total_order():
    """Reading R3: equal cumulative scores -> token asc, then beam asc."""
    need_gpu()
    from paper_2502_00085_b200.trie import TrieState
    V, b = 64, 6
    prompts, lens = synth.prompts(3, 1, 4, V)
    st = TrieState(1, b, 4, 40, 0, 1, 1, 16, V, prompts, lens, dtype=torch.float32)
    st.beam_step(torch.zeros(1, 1, V, device="cuda"))
    lt = torch.zeros(1, b, V, device="cuda")  # all candidates tie exactly
    par = torch.empty(1, b, dtype=torch.int32, device="cuda")
    tok = torch.empty_like(par)
    st.beam_step(lt, par, tok)
    assert tok.cpu().numpy()[0].tolist() == [0] * 6
    assert par.cpu().numpy()[0].tolist() == [0, 1, 2, 3, 4, 5]



@pytest.mark.parametrize("R,b,V", [(2, 4, 256), (2, 8, 32064), (1, 16, 128256), (2, 3, 4097)])
def test_beam_step_absorbing_eos_matches_oracle(R, b, V):
    """NEXT-3 (reading R5b): finished beams (last token = EOS) continue only with EOS at
    log-prob 0.  Step 1 is steered so EOS is selected; later steps are checked against
    beam_step_ref on the absorbed logits (finished rows one-hot at EOS), and the device
    finished flags against the selected tokens."""
    need_gpu()
    from paper_2502_00085_b200.trie import TrieState
    seed, eos = b * 13 + V, V // 3
    prompts, lens = synth.prompts(seed, R, 6, V)
    st = TrieState(R, b, 6, 6 + 5 * b + b, 0, 1, 1, 16, V, prompts, lens, dtype=torch.float32)
    st.set_eos(eos)
    scores = np.zeros((R, 1))
    fin = np.zeros((R, 1), bool)
    near = absorbed_rows = done_seen = 0
    for step in range(5):
        b_live = 1 if step == 0 else b
        logits = (synth.normal(seed, 20 + step, (R, b_live, V)) * 3.0).astype(np.float32)
        if step in (0, 1, 2):  # EOS is every row's argmax at steps 1-3
            logits[:, :, eos] = logits.max(axis=-1) + 30.0
        lt = torch.as_tensor(logits, device="cuda")
        par = torch.empty(R, b, dtype=torch.int32, device="cuda")
        tok = torch.empty_like(par)
        sc = torch.empty(R, b, dtype=torch.float32, device="cuda")
        n_before = st.n_nodes.cpu().numpy().copy()
        st.beam_step(lt, par, tok, sc)
        par, tok, sc = par.cpu().numpy(), tok.cpu().numpy(), sc.cpu().numpy()
        n_after = st.n_nodes.cpu().numpy()
        for r in range(R):
            if b_live == b and fin[r].all():  # done (R5b): identity selection, trie frozen
                done_seen += 1
                assert par[r].tolist() == list(range(b)) and (tok[r] == eos).all()
                assert np.array_equal(sc[r], scores[r].astype(np.float32)) and n_after[r] == n_before[r]
            absorbed = logits[r].astype(np.float64).copy()
            for j in range(b_live):
                if fin[r, j]:
                    absorbed[j] = -np.inf
                    absorbed[j, eos] = 0.0
                    absorbed_rows += 1
            near += _check(absorbed, scores[r], b, par[r], tok[r], sc[r])
            for q in range(b):  # a finished parent continues with EOS at its own score
                if fin[r, par[r, q]]:
                    assert tok[r, q] == eos and abs(sc[r, q] - scores[r, par[r, q]]) <= 1e-6 * max(1, abs(sc[r, q]))
        fin = tok == eos
        assert np.array_equal(st.finished.cpu().numpy()[:, :b] != 0, fin)
        scores = sc.astype(np.float64)
    assert absorbed_rows > 0  # finished beams were carried through later steps
    assert done_seen > 0      # and some request finished all its beams
    assert st.status() == 0
    assert near <= 1
