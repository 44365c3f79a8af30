"""Pins for oracle/select.py and oracle/decode.py: SPEC's hand logit table, brute-force
exhaustive search, greedy collapse, trie == batch (bitwise in float64), GC-schedule
invariance, memory dominance, fault injection."""
import itertools
import json
import math
import os

import numpy as np
import pytest

import synth
from oracle.decode import batch_beam_search, greedy_decode, trie_beam_search
from oracle.kernels_ref import beam_step_ref
from oracle.model import Model, ModelConfig
from oracle.select import select_topb, select_topb_np
from oracle.trie import unique_prefix_count


def _model(seed, Hkv=4, kappa=4.0, V=256):
    cfg = ModelConfig(L=2, d=64, Hq=4, Hkv=Hkv, D=16, ffn=256, V=V, kappa=kappa)
    return Model(synth.tiny_weights(seed, cfg.L, cfg.d, cfg.Hq, cfg.Hkv, cfg.D, cfg.ffn, cfg.V), cfg)


class TableModel:
    """Stub LM whose next-token distribution is a lookup on the generated suffix.  It
    stores its token id as its 'key' and reads the allowed rows back, so the prefix it
    sees is exactly the row set the decoder lets it attend to (tests the mask too)."""

    class cfg:
        L = 1

    def __init__(self, table, t):
        self.table, self.t = table, t

    def forward(self, token, pos, ctx):
        K, _ = ctx(0, np.array([[float(token)]]), np.zeros((1, 1)))
        prefix = [int(x) for x in K[:, 0, 0]]
        key = "".join("ABC"[x] for x in prefix[self.t:])
        return np.log(np.array(self.table[key], dtype=np.float64))


@pytest.fixture(scope="module")
def hand(golden_dir):
    return json.load(open(os.path.join(golden_dir, "spec_hand_logit_table.json")))


@pytest.mark.parametrize("decoder", ["batch", "trie"])
def test_hand_logit_table(hand, decoder):
    m = TableModel(hand["table"], t=1)
    if decoder == "batch":
        res = batch_beam_search(m, [2], hand["b"], hand["steps"])
    else:
        res = trie_beam_search(m, [2], hand["b"], hand["steps"], g=1)
    got = [("".join("ABC"[x] for x in toks[1:]), math.exp(sc)) for toks, sc in res.hyps]
    for (s, p), (es, ep) in zip(got, hand["expected_beams"]):
        assert s == es and abs(p - ep) < 1e-12
    # exhaustive enumeration of all 9 sequences agrees on the best one
    best = max(itertools.product(range(3), repeat=2),
               key=lambda sq: hand["table"][""][sq[0]] * hand["table"]["ABC"[sq[0]]][sq[1]])
    assert "".join("ABC"[x] for x in best) == got[0][0]


def test_select_ties_total_order():
    """Reading R3: score desc, token asc, beam asc."""
    sel = select_topb([0.0, 0.0], [np.zeros(3), np.zeros(3)], 4)
    assert [(v, j) for _, v, j in sel] == [(0, 0), (0, 1), (1, 0), (1, 1)]
    cs, vv, jj = select_topb_np([0.0, 0.0], np.zeros((2, 3)), 4)
    assert list(zip(vv, jj)) == [(0, 0), (0, 1), (1, 0), (1, 1)]


def test_select_np_equals_python_sort():
    for seed in range(20):
        J, V, b = 1 + seed % 4, 37, 1 + seed % 7
        lp = np.round(synth.normal(seed, 1, (J, V)), 1)   # coarse -> many exact ties
        sc = np.round(synth.normal(seed, 2, (J,)), 1)
        a = select_topb(list(sc), list(lp), b)
        cs, vv, jj = select_topb_np(sc, lp, b)
        assert [(v, j) for _, v, j in a] == list(zip(vv.tolist(), jj.tolist()))


def test_beam_step_ref_brute_force():
    """Kernel-level ref == brute force over every (j, v) candidate."""
    for seed in range(10):
        J, V, b = 3, 50, 4
        logits = synth.normal(seed, 3, (J, V)) * 3
        sc = synth.normal(seed, 4, (J,))
        par, tok, ns, gap, _ = beam_step_ref(logits, sc, b)
        lse = [max(x) + math.log(sum(math.exp(y - max(x)) for y in x)) for x in logits]
        cands = sorted(((sc[j] + logits[j][v] - lse[j], v, j) for j in range(J) for v in range(V)),
                       key=lambda c: (-c[0], c[1], c[2]))
        assert [(c[2], c[1]) for c in cands[:b]] == list(zip(par.tolist(), tok.tolist()))
        np.testing.assert_allclose(ns, [c[0] for c in cands[:b]], atol=1e-12)
        assert abs(gap - (cands[b - 1][0] - cands[b][0])) < 1e-12


def test_exhaustive_search_special_case():
    """b >= V^(s-1) keeps every sequence, so beam search == argmax over all V^s."""
    m = _model(3, V=4, kappa=3.0)
    prompt, s, V = [1, 2, 0], 3, 4
    res = trie_beam_search(m, prompt, V ** (s - 1), s, g=1)
    best_sc, best_seq = -np.inf, None
    for seq in itertools.product(range(V), repeat=s):
        full = m.forward_full_causal(prompt + list(seq[:-1]))
        sc = sum(full[len(prompt) - 1 + i][seq[i]] for i in range(s))
        if sc > best_sc:
            best_sc, best_seq = sc, list(seq)
    assert res.best[0][len(prompt):] == best_seq
    assert abs(res.best[1] - best_sc) < 1e-9


@pytest.mark.parametrize("seed", range(8))
def test_b1_collapse_to_greedy(seed):
    m = _model(seed)
    prompt = [int(x) for x in synth.randint(seed, 5, 8, 256)]
    gt, gs = greedy_decode(m, prompt, 10)
    for res in (batch_beam_search(m, prompt, 1, 10), trie_beam_search(m, prompt, 1, 10, g=None)):
        assert res.best[0] == gt and abs(res.best[1] - gs) < 1e-12


CASES = [(seed, Hkv, b, W) for seed in range(6) for (Hkv, b, W) in
         [(4, 3, 0), (2, 3, 0), (4, 5, 0), (1, 2, 0), (4, 3, 5), (2, 4, 3)]]


@pytest.mark.parametrize("seed,Hkv,b,W", CASES)
def test_trie_equals_batch_bitwise(seed, Hkv, b, W):
    """trie decoding == batch beam search.  float64, identical per-query row
    lists -> bitwise equal scores and log-prob rows; SWA by depth (reading R14) too."""
    m = _model(100 + seed, Hkv=Hkv)
    prompt = [int(x) for x in synth.randint(seed, 6, 8, 256)]
    s = 12
    bt = batch_beam_search(m, prompt, b, s, window=W)
    tr = trie_beam_search(m, prompt, b, s, g=1, window=W)
    assert bt.hyps == tr.hyps
    for sb, st in zip(bt.steps, tr.steps):
        assert sb["sel"] == st["sel"]
        for x, y in zip(sb["lp_rows"], st["lp_rows"]):
            assert np.array_equal(x, y)
        assert st["entries"] <= sb["entries"]          # memory dominance
    assert bt.steps[-1]["entries"] == len(bt.hyps) * (len(prompt) + s)


@pytest.mark.parametrize("seed", range(5))
def test_gc_schedule_invariance(seed):
    """g in {1, 4, 15, inf} -> identical outputs."""
    m = _model(200 + seed, Hkv=2)
    prompt = [int(x) for x in synth.randint(seed, 7, 8, 256)]
    ref = trie_beam_search(m, prompt, 4, 16, g=None)
    for g in (1, 4, 15):
        res = trie_beam_search(m, prompt, 4, 16, g=g)
        assert res.hyps == ref.hyps
        for a, c in zip(res.steps, ref.steps):
            for x, y in zip(a["lp_rows"], c["lp_rows"]):
                assert np.array_equal(x, y)


def test_unique_prefix_invariant_real_beams():
    for seed in range(4):
        m = _model(300 + seed)
        prompt = [int(x) for x in synth.randint(seed, 8, 8, 256)]
        res = trie_beam_search(m, prompt, 3, 16, g=1, final_gc=True)
        assert res.trie.N == unique_prefix_count(res.trie)
        assert res.trie.N <= 3 * (8 + 16)


def test_fault_injection_corrupted_mask_bit_is_detected():
    """a corrupted mask bit (cross-branch leak) must change the log-probs
    by more than 1e-3 (softmax-normalised), i.e. the mask bits are live."""
    import oracle.decode as dec
    m = _model(7)
    prompt = [int(x) for x in synth.randint(7, 9, 8, 256)]
    clean = trie_beam_search(m, prompt, 3, 6, g=None)
    orig = dec.update_mask

    def leaky(M, T, sel):
        M2 = orig(M, T, sel)
        if M2.shape[1] > T.t + 4:
            cross = [n for n in range(T.t, M2.shape[1]) if not M2[0, n]]
            if cross:
                M2[0, cross[0]] = True
        return M2
    dec.update_mask = leaky
    try:
        dirty = trie_beam_search(m, prompt, 3, 6, g=None)
    finally:
        dec.update_mask = orig
    div = max(np.abs(np.exp(x) - np.exp(y)).max()
              for a, c in zip(clean.steps, dirty.steps) for x, y in zip(a["lp_rows"], c["lp_rows"]))
    assert div > 1e-3


def test_memory_ratio_direction_and_bound():
    """b(t+s)/(t+s+b-1) bound and ratio decreasing in b on a convergent workload."""
    t, s = 8, 12
    ratios = []
    for b in (2, 3, 5):
        m = _model(400, kappa=8.0)
        prompt = [int(x) for x in synth.randint(1, 10, t, 256)]
        tr = trie_beam_search(m, prompt, b, s, g=1, final_gc=True)
        batch = b * (t + s)
        assert batch / tr.trie.N <= b * (t + s) / (t + s + b - 1) + 1e-12
        ratios.append(tr.trie.N / batch)
    assert ratios[0] > ratios[1] > ratios[2]



# ---- NEXT-3: EOS as an absorbing token (reading R5b) ----------------------------------
def _eos_seen(m, prompt, b, s):
    """A token the no-EOS search selects at step 2 or 3 (so that EOS really occurs)."""
    res = trie_beam_search(m, prompt, b, s, g=1)
    return res.steps[2]["sel"][1][1]


@pytest.mark.parametrize("seed", range(6))
def test_eos_trie_equals_batch_bitwise(seed):
    """With EOS, trie decoding still equals batch beam search bitwise (float64)."""
    m = _model(200 + seed, kappa=6.0, V=64)
    prompt = [int(x) for x in synth.randint(seed, 7, 6, 64)]
    b, s = 4, 9
    eos = _eos_seen(m, prompt, b, s)
    bt = batch_beam_search(m, prompt, b, s, eos=eos)
    tr = trie_beam_search(m, prompt, b, s, g=1, eos=eos)
    assert bt.hyps == tr.hyps
    for sb, st in zip(bt.steps, tr.steps):
        assert sb["sel"] == st["sel"]
    # EOS occurred, and a finished beam only ever continues with EOS at an unchanged score
    assert any(v == eos for (_, v, _) in tr.steps[2]["sel"] + tr.steps[3]["sel"])
    for k in range(1, s):
        prev = tr.steps[k - 1]["sel"]
        for (sc, v, j) in tr.steps[k]["sel"]:
            if prev[j][1] == eos:
                assert v == eos and sc == prev[j][0]


@pytest.mark.parametrize("seed", range(3))
def test_eos_never_selected_changes_nothing(seed):
    m = _model(300 + seed, V=64)
    prompt = [int(x) for x in synth.randint(seed, 8, 6, 64)]
    b, s = 3, 8
    ref = trie_beam_search(m, prompt, b, s, g=1)
    used = {v for st in ref.steps for (_, v, _) in st["sel"]}
    eos = min(set(range(64)) - used)
    res = trie_beam_search(m, prompt, b, s, g=1, eos=eos)
    assert res.hyps == ref.hyps


def _eos_exhaustive(s, eos_ids):
    """b >= V^(s-1) keeps every sequence: beam search with an absorbing EOS == argmax over
    all sequences of the absorbing chain (tokens after the first EOS are EOS, log-prob 0)."""
    m = _model(5, V=4, kappa=3.0)
    prompt, V = [1, 2, 0], 4
    for eos in eos_ids:
        res = trie_beam_search(m, prompt, V ** (s - 1), s, g=1, eos=eos)
        best_sc, best_seq = -np.inf, None
        for seq in itertools.product(range(V), repeat=s):
            if eos in seq:
                e = seq.index(eos)
                if any(x != eos for x in seq[e:]):
                    continue  # not a sequence of the absorbing chain
                n = e + 1      # log-probs up to and including the first EOS
            else:
                n = s
            full = m.forward_full_causal(prompt + list(seq[: max(n - 1, 0)]))
            sc = sum(full[len(prompt) - 1 + i][seq[i]] for i in range(n))
            if sc > best_sc + 1e-12:
                best_sc, best_seq = sc, list(seq)
        assert abs(res.best[1] - best_sc) < 1e-9
        assert res.best[0][len(prompt):] == best_seq


def test_eos_exhaustive_special_case():
    _eos_exhaustive(3, (0, 2, 3))


@pytest.mark.slow
def test_eos_exhaustive_special_case_s4_all_ids():
    """The full pin (s = 4, b = V^3 = 64, every token id as EOS): ~40 s of CPU."""
    _eos_exhaustive(4, range(4))


def test_eos_all_finished_is_stable():
    """Once every beam is finished, further steps leave the hypotheses unchanged."""
    m = _model(12, kappa=8.0, V=32)
    prompt = [3, 1, 4, 1, 5]
    b = 2
    ref = trie_beam_search(m, prompt, b, 6, g=1)
    eos = ref.steps[1]["sel"][0][1]   # the best continuation at step 2: finishes early
    short = trie_beam_search(m, prompt, b, 10, g=1, eos=eos)
    longer = trie_beam_search(m, prompt, b, 14, g=1, eos=eos)
    assert all(tok[-1] == eos for tok, _ in short.hyps)  # every beam finished by step 10
    assert longer.hyps == short.hyps                     # decoding stopped: nothing changes
    assert len(longer.steps) == len(short.steps) < 10
