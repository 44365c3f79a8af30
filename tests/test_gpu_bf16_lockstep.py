"""Model-driven bf16 lockstep decode: the production bf16 kernels (fused RoPE + append +
trie attention -- narrow / wide / tcgen05 --
the beam step and GC) run for >= 16 steps inside a random-init decoder, and after every
step every layer is checked against the oracle on the SAME inputs (SURVEY §8(c)
"snapshot-differential" checks; the lockstep protocol: the oracle follows the GPU's own
selections, so bf16 rounding never lets the two drift apart):

* trie metadata (token / parent / depth / N / leaves) == the oracle trie grown by
  update_trie (Alg. 2 l.10) + garbage_collect (§3.5) with the GPU's selections
  -- bit-exact;
* the K/V pool rows [0, N) == the rows the oracle trie carries (its GC moves them; the
  appended leaf rows enter it after the next check) -- bit-exact;
* the appended leaf rows == rotate-half RoPE of the model's k at the leaf depth (§3.4
  P:202-209, reading R16), fp64, within bf16 rounding;
* attention outputs == attn_ref (§3.3) with q rotated in fp64 at the leaf
  depth over the oracle's rows -- <= 2e-2 per row (BASELINE.json north_star bf16
  tolerance, reading R24);
* the selection == beam_step_ref on the GPU's own fp32 logits (near-tie protocol).
"""
import numpy as np
import pytest
import torch

import synth
from oracle.kernels_ref import attn_ref, beam_step_ref
from oracle.numerics import rope_rotate_half
from oracle.trie import Trie, garbage_collect
from tests.gpu_util import need_gpu, rel_err

pytestmark = pytest.mark.gpu

# name, D, Hq, Hkv, b, R, t_max, s, W, expected attention path (trie_attn_plan_info)
CASES = [
    ("narrow-mha", 64, 4, 4, 4, 3, 150, 18, 0, ("narrow-mma.sync",)),
    ("narrow-gqa", 64, 8, 2, 2, 3, 140, 17, 0, ("narrow-mma.sync",)),
    ("wide1-gqa", 128, 8, 2, 4, 3, 150, 17, 0, ("wide-mma.sync",)),   # Qg = 16: one m-tile
    ("wide1-swa", 96, 8, 4, 8, 2, 130, 17, 100, ("wide-mma.sync",)),   # Qg = 16, D = 96
    ("wide", 128, 8, 2, 8, 3, 150, 17, 0, ("wide-mma.sync",)),
    ("wide-swa", 128, 8, 2, 8, 2, 130, 17, 100, ("wide-mma.sync",)),
    ("tcgen05", 128, 8, 1, 8, 2, 150, 17, 0, ("tcgen05-tmem",)),
]


def _bf16_np(t):
    return t.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("paged", [False, True], ids=["dense", "paged"])
@pytest.mark.parametrize("name,D,Hq,Hkv,b,R,t_max,s,W,paths", CASES)
def test_bf16_lockstep_decode(name, D, Hq, Hkv, b, R, t_max, s, W, paths, paged):
    """paged: the same decode over paged pools (pages mapped as the
    trie grows, returned by GC)."""
    need_gpu()
    if paged and name not in ("narrow-gqa", "wide-swa", "wide1-gqa", "tcgen05"):
        pytest.skip("paged pools: a subset of the shapes")
    from paper_2502_00085_b200 import _lib
    from paper_2502_00085_b200.model import TinyModel
    from paper_2502_00085_b200.trie import TrieState
    seed, L, V, ffn, base = 40 + D + Hkv + b, 2, 512, 256, 10000.0
    lens = synth.ragged_lens(seed, R, t_max, t_min=t_max // 2)
    prompts, lens = synth.prompts(seed, R, t_max, V, lens)
    cap = (t_max + b * s + b + 63) // 64 * 64
    gm = TinyModel(seed, L=L, d=Hq * D, Hq=Hq, Hkv=Hkv, D=D, ffn=ffn, V=V, rope_base=base,
                   kappa=4.0, dtype=torch.bfloat16)
    st = TrieState(R, b, t_max, cap, L, Hq, Hkv, D, V, prompts, lens, window=W,
                   dtype=torch.bfloat16, n_pages=R * cap // 64 if paged else 0)
    path = _lib.trie_attn_plan_info(st.cfg, b, 0)["path"]
    assert path in paths, f"{name}: planned path {path}"
    kp, vp = st.new_pools()
    if paged:  # prefill into dense rows, then through the page table
        kd = torch.zeros(L, R, Hkv, cap, D, dtype=torch.bfloat16, device="cuda")
        vd = torch.zeros_like(kd)
        logits = gm.prefill(prompts, lens, kd, vd, window=W)
        for l in range(L):
            st.write_rows(kp[l], kd[l][:, :, :t_max])
            st.write_rows(vp[l], vd[l][:, :, :t_max])
    else:
        logits = gm.prefill(prompts, lens, kp, vp, window=W)
    dense = lambda pool: st.dense_view(pool)  # noqa: E731  slot-order rows (paged or not)
    # the oracle's tries, carrying the K/V rows (as bf16 values in float64) per slot
    tries = [Trie([int(x) for x in prompts[r][: lens[r]]], n_layers=L) for r in range(R)]
    for r, T in enumerate(tries):
        for l in range(L):
            K, Vv = _bf16_np(dense(kp[l])[r]), _bf16_np(dense(vp[l])[r])
            T.kv[l] = [(K[:, n], Vv[:, n]) for n in range(T.t)]
    checked_rows = 0
    for k in range(1, s + 1):
        lg = logits.float().cpu().numpy()
        sp = torch.empty(R, b, dtype=torch.int32, device="cuda")
        tk = torch.empty_like(sp)
        sc = torch.empty(R, b, dtype=torch.float32, device="cuda")
        st.beam_step(logits.float().contiguous(), sp, tk, sc)
        st.prune_compact(kp, vp)
        sp, tk, sc = sp.cpu().numpy(), tk.cpu().numpy(), sc.cpu().numpy()
        for r, T in enumerate(tries):
            refp, reft, refs, gap, _ = beam_step_ref(lg[r][: len(T.leaves)], np.asarray(T.scores), b)
            tau = 1e-5 * max(1.0, float(np.abs(refs).max()))
            if gap > tau:
                assert sp[r].tolist() == refp.tolist() and tk[r].tolist() == reft.tolist(), \
                    f"{name} step {k} r={r}: selection differs from beam_step_ref"
            T.update_trie([(float(sc[r, i]), int(tk[r, i]), int(sp[r, i])) for i in range(b)])
            garbage_collect(T)
        # trie metadata, bit-exact
        N = st.n_nodes.cpu().numpy()
        tok, par, dep = st.token.cpu().numpy(), st.parent.cpu().numpy(), st.depth.cpu().numpy()
        leaf = st.leaf.cpu().numpy()[:, :b]
        for r, T in enumerate(tries):
            assert N[r] == T.N
            assert tok[r, : T.N].tolist() == T.token and par[r, : T.N].tolist() == T.parent
            assert dep[r, : T.N].tolist() == T.depth and leaf[r].tolist() == T.leaves
        # the K/V rows the pools hold for every slot with K/V (pending leaves excluded)
        KD = [_bf16_np(dense(kp[l])) for l in range(L)]
        VD = [_bf16_np(dense(vp[l])) for l in range(L)]
        for r, T in enumerate(tries):
            for l in range(L):
                K, Vv = KD[l][r], VD[l][r]
                for n in range(T.N):
                    if T.kv[l][n] is not None:
                        assert np.array_equal(K[:, n], T.kv[l][n][0]) and \
                            np.array_equal(Vv[:, n], T.kv[l][n][1]), \
                            f"{name} step {k}: K/V of slot {n} (layer {l}, r={r}) moved wrongly"
        if k == s:
            break
        rec = {}

        def hook(l, q, kk, vv, o):
            rec[l] = tuple(_bf16_np(x) for x in (q, kk, vv, o)) + (_bf16_np(dense(kp[l])), _bf16_np(dense(vp[l])))
        logits = gm.step(st, kp, vp, fused=True, hook=hook)
        torch.cuda.synchronize()
        for l in range(L):
            q, kn, vn, o, K, Vv = rec[l]
            for r, T in enumerate(tries):
                pos = T.depth[T.leaves[0]]
                assert all(T.depth[x] == pos for x in T.leaves)
                for j, lf in enumerate(T.leaves):
                    krot = rope_rotate_half(kn[r, j], pos, base)      # [Hkv][D]
                    assert rel_err(K[r][:, lf], krot) <= 1.6e-2, f"{name}: leaf K row (l={l}, r={r})"
                    assert np.array_equal(Vv[r][:, lf], vn[r, j]), f"{name}: leaf V row"
                    T.kv[l][lf] = (K[r][:, lf].copy(), Vv[r][:, lf].copy())
                Kr = np.stack([T.kv[l][n][0] for n in range(T.N)], axis=1)   # [Hkv][N][D]
                Vr = np.stack([T.kv[l][n][1] for n in range(T.N)], axis=1)
                # the oracle's own leaf rows (fp64 RoPE of the model's k) for the attention
                for j, lf in enumerate(T.leaves):
                    Kr[:, lf] = rope_rotate_half(kn[r, j], pos, base)
                qr = np.stack([rope_rotate_half(q[r, j], pos, base) for j in range(b)])
                o_ref, _ = attn_ref(qr, Kr, Vr, T, window=W)
                err = rel_err(o[r], o_ref)
                assert err <= 2e-2, f"{name} step {k} layer {l} r={r}: attention rel err {err:.3g}"
                checked_rows += b * Hq
    assert st.status() == 0
    assert checked_rows >= 16 * L * R * b * Hq // 2
