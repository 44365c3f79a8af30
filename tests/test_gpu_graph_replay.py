"""The CUDA-graph contract of include/triedecode.h ("CUDA graphs"): all trie state lives on
the device, so one steady-state step (L fused RoPE + attention calls, trie_beam_step,
trie_prune_compact) captured ONCE after the first beam step and replayed for every later
step gives, bit for bit, what eager calls give on a second handle fed the same inputs --
selections, scores, trie metadata, attention outputs and the K/V pools.  The first step of
the job (b_live = 1) is its own graph, as bench.py's "first" graph.  GPU vs
GPU (same kernels, same inputs): exact equality is the bar; the numerics themselves are
pinned to the oracle by the other -m gpu tests."""
import numpy as np
import pytest
import torch

import synth
from tests.gpu_util import need_gpu

pytestmark = pytest.mark.gpu

# name, R, b, Hq, Hkv, D, t_max, steps: Qg = 16 (wide, one m-tile), 32 (wide), 8 (narrow)
CASES = [
    ("wide1", 2, 4, 8, 2, 64, 40, 12),
    ("wide", 2, 8, 8, 2, 128, 70, 10),
    ("narrow-paged", 3, 2, 4, 1, 96, 33, 12),
]


def _inputs(seed, steps, R, b, Hq, Hkv, D, L, V):
    """Per step: logits [R][b_live][V] and per layer (q, k_new, v_new), b_live = 1 at step 0."""
    out = []
    for k in range(steps):
        bl = 1 if k == 0 else b
        lg = torch.as_tensor(synth.normal(seed + k, 1, (R, bl, V)) * 3.0, dtype=torch.float32).cuda()
        lay = []
        for l in range(L):
            q = torch.as_tensor(synth.normal(seed + k, 10 + 3 * l, (R, bl, Hq, D)), dtype=torch.float32)
            kk = torch.as_tensor(synth.normal(seed + k, 11 + 3 * l, (R, bl, Hkv, D)), dtype=torch.float32)
            vv = torch.as_tensor(synth.normal(seed + k, 12 + 3 * l, (R, bl, Hkv, D)), dtype=torch.float32)
            lay.append(tuple(x.to(torch.bfloat16).cuda() for x in (q, kk, vv)))
        out.append((lg, lay))
    return out


@pytest.mark.parametrize("name,R,b,Hq,Hkv,D,t_max,steps", CASES)
def test_graph_replay_equals_eager(name, R, b, Hq, Hkv, D, t_max, steps):
    need_gpu()
    from paper_2502_00085_b200.trie import TrieState
    L, V, theta, seed = 2, 300, 10000.0, 17 + D
    lens = synth.ragged_lens(seed, R, t_max, t_min=t_max // 2)
    prompts, lens = synth.prompts(seed, R, t_max, V, lens)
    cap = (t_max + b * (steps + 2) + 63) // 64 * 64
    paged = name.endswith("paged")
    sts = [TrieState(R, b, t_max, cap, L, Hq, Hkv, D, V, prompts, lens, dtype=torch.bfloat16,
                     n_pages=R * cap // 64 if paged else 0) for _ in range(2)]
    from paper_2502_00085_b200 import _lib
    for st in sts:  # attention scratch allocated up front (no allocation inside a capture)
        need = max(_lib.trie_attn_scratch_bytes(st.cfg, bl, 0) for bl in (1, b))
        st.attn_scratch = torch.zeros(need, dtype=torch.uint8, device="cuda")
    pools = []
    for st in sts:  # identical prefill (prompt rows) on both handles
        kp, vp = st.new_pools()
        g = torch.Generator(device="cpu").manual_seed(seed)
        kd = torch.randn(L, R, Hkv, t_max, D, generator=g).to(torch.bfloat16).cuda()
        vd = torch.randn(L, R, Hkv, t_max, D, generator=g).to(torch.bfloat16).cuda()
        for l in range(L):
            st.write_rows(kp[l], kd[l])
            st.write_rows(vp[l], vd[l])
        pools.append((kp, vp))
    inp = _inputs(seed, steps, R, b, Hq, Hkv, D, L, V)

    def step(st, kp, vp, lg, lay, outs, sel):
        for l, (q, kk, vv) in enumerate(lay):
            st.attn_decode_rope(q, kk, vv, kp[l], vp[l], theta, outs[l])
        st.beam_step(lg, *sel)
        st.prune_compact(kp, vp)

    def new_sel():
        return (torch.empty(R, b, dtype=torch.int32, device="cuda"),
                torch.empty(R, b, dtype=torch.int32, device="cuda"),
                torch.empty(R, b, dtype=torch.float32, device="cuda"))

    # eager reference on handle 0
    st0, (kp0, vp0) = sts[0], pools[0]
    eager = []
    for k, (lg, lay) in enumerate(inp):
        outs = [torch.empty_like(q) for q, _, _ in lay]
        sel = new_sel()
        step(st0, kp0, vp0, lg, lay, outs, sel)
        torch.cuda.synchronize()
        eager.append(([o.clone() for o in outs], [s.clone() for s in sel]))

    # handle 1: step 0 as a "first" graph (captured right after trie_create's state, i.e.
    # b_live = 1), then ONE steady graph captured at step 1 and replayed for steps 1..
    st1, (kp1, vp1) = sts[1], pools[1]
    s_stream = torch.cuda.Stream()

    def capture(k):
        lg, lay = inp[k]
        st_lg = lg.clone()
        st_lay = [tuple(x.clone() for x in t) for t in lay]
        st_outs = [torch.empty_like(q) for q, _, _ in lay]
        st_sel = new_sel()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s_stream):
            step(st1, kp1, vp1, st_lg, st_lay, st_outs, st_sel)
        return gr, st_lg, st_lay, st_outs, st_sel

    # capturing does not execute: the "first" graph is captured at b_live = 1 and replayed
    g0 = capture(0)
    g0[0].replay()
    torch.cuda.synchronize()
    got = [([o.clone() for o in g0[3]], [s.clone() for s in g0[4]])]
    gs = capture(1)  # b_live = b from here on
    for k in range(1, steps):
        lg, lay = inp[k]
        gs[1].copy_(lg)
        for dst, src in zip(gs[2], lay):
            for a, bsrc in zip(dst, src):
                a.copy_(bsrc)
        gs[0].replay()
        torch.cuda.synchronize()
        got.append(([o.clone() for o in gs[3]], [s.clone() for s in gs[4]]))

    for k in range(steps):
        (eo, es), (go, gsel) = eager[k], got[k]
        for a, bb in zip(es, gsel):
            assert torch.equal(a, bb), f"{name} step {k}: selections differ (graph vs eager)"
        for l, (a, bb) in enumerate(zip(eo, go)):
            assert torch.equal(a, bb), f"{name} step {k} layer {l}: attention output differs"
    for attr in ("n_nodes", "token", "parent", "depth", "beam_mask", "leaf", "score"):
        assert torch.equal(getattr(st0, attr), getattr(st1, attr)), f"{name}: {attr} differs"
    N = st0.n_nodes.cpu().numpy()
    for l in range(L):
        for pa, pb in ((kp0, kp1), (vp0, vp1)):
            da, db = st0.dense_view(pa[l]), st1.dense_view(pb[l])
            for r in range(R):
                assert torch.equal(da[r, :, : N[r]], db[r, :, : N[r]]), f"{name}: pool rows differ"
    assert st0.status() == 0 and st1.status() == 0
