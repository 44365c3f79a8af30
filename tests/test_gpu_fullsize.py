"""GPU vs oracle at BASELINE.json's FULL sizes, in the launch configuration bench.py times
(its HotPath: the same buffers, plans, fused / unfused kernel choice and step order).

Per workload, a few beam-decode steps run through the C ABI; on SAMPLED requests the
oracle then checks, one by one:
  * the beam step (a-4): selections vs oracle.kernels_ref.beam_step_ref on the step's own
    fp32 logits and the scores before the step, under the near-tie protocol;
  * the trie (a-2, a-5, a-6): bit-exact token / parent / depth / beam-mask / leaves / N vs
    oracle build_tries teacher-forced with the GPU's selections (prune every step, g = 1);
  * the attention (a-1 + a-3) of the first and last layer: one extra launch of the step's
    attention call on the current trie, output vs attn_ref on the pool rows of the sampled
    requests (bf16 tolerance 2e-2, reading R24), the appended leaf K rows vs the oracle's
    rotate-half RoPE at the leaf depth and the V rows bit-exact.
"""
import numpy as np
import pytest
import torch

import synth
from oracle.kernels_ref import attn_ref, beam_step_ref, build_tries, soa
from oracle.numerics import rope_rotate_half
from tests.gpu_util import need_gpu, rel_err
from tests.test_gpu_beam_step import _check

pytestmark = pytest.mark.gpu

STEPS = 5


@pytest.mark.parametrize("paged", [0.5, 0.0], ids=["paged", "dense"])
@pytest.mark.parametrize("wl_name,beam", [("phi", 0), ("llama", 0), ("sweep", 16), ("mistral-shard", 0)])
def test_fullsize_sampled_parity(wl_name, beam, paged):
    """paged = 0.5: bench.py's default pools (NEXT-2 pages: prompt + half the no-GC
    generated pages); 0: dense pools sized for the no-GC worst case."""
    need_gpu()
    import bench
    from paper_2502_00085_b200 import _lib
    from paper_2502_00085_b200.build import build
    build()
    _lib.load()
    wl = dict(bench.WORKLOADS[wl_name])
    if beam:
        wl["b"] = beam
    wl["paged"] = paged
    hp = bench.HotPath(wl, 0, torch.device("cuda", 0))
    st, R, b, t, V, L = hp.st, hp.R, hp.b, hp.t, hp.V, hp.L
    rs = sorted({0, R // 2, R - 1})
    prompts, lens = synth.prompts(10_000, R, t, V)  # HotPath's rank-0 / shared prompts
    sels = []
    near = 0
    for k in range(STEPS):
        var, slot = ("first" if k == 0 else "steady"), k % 2
        b_live = 1 if k == 0 else b
        scores_before = st.score.cpu().numpy()[:, :b_live].astype(np.float64) if k else np.zeros((R, 1))
        hp.step_ops(var, slot)
        torch.cuda.synchronize()
        assert st.status() == 0
        par, tok, sc = hp.sel_p.cpu().numpy(), hp.sel_t.cpu().numpy(), hp.sel_s.cpu().numpy()
        logits = hp.inp[(var, slot)]["logits"].float().cpu().numpy()
        for r in rs:  # a-4 on this step's logits
            near += _check(logits[r], scores_before[r], b, par[r], tok[r], sc[r])
        sels.append((par[rs], tok[rs]))
    assert near <= 1
    # a-2 / a-5 / a-6: the sampled requests' tries, teacher-forced with the GPU's choices
    tries = build_tries(prompts[rs], lens[rs], sels, b, g=1, final_gc=True)
    ref = soa(tries, hp.cap, b)
    got = {k: getattr(st, k).cpu().numpy()[rs] for k in ("token", "parent", "depth", "beam_mask")}
    assert np.array_equal(st.n_nodes.cpu().numpy()[rs], ref["N"])
    for i, T in enumerate(tries):
        N = T.N
        assert np.array_equal(got["token"][i, :N], ref["token"][i, :N])
        assert np.array_equal(got["parent"][i, :N], ref["parent"][i, :N])
        assert np.array_equal(got["depth"][i, :N], ref["depth"][i, :N])
        assert np.array_equal(got["beam_mask"][i, :N].view(np.uint32), ref["mask"][i, :N])
        assert np.array_equal(st.leaf.cpu().numpy()[rs[i], :b], ref["leaf"][i])
    # a-1 + a-3 on the first and last layer: the step's attention call on the current trie
    d = hp.inp[("steady", 0)]
    W, theta = hp.W, wl["theta"]
    for l in (0, L - 1):
        q, kn, vn = d["views"][l]
        q0 = q.float().cpu().numpy().astype(np.float64)
        k0 = kn.float().cpu().numpy().astype(np.float64)
        v0 = vn.float().cpu().numpy().astype(np.float64)
        out = torch.empty_like(q)
        if hp.fused["steady"]:
            st.attn_decode_rope(q, kn, vn, hp.kp[l], hp.vp[l], theta, out, rows_hint=hp.rows_hint)
        else:  # two launches; rope_kv_append rotates q in place
            st.rope_kv_append(q, kn, vn, hp.kp[l], hp.vp[l], theta)
            st.attn_decode(q, hp.kp[l], hp.vp[l], out, rows_hint=hp.rows_hint)
        torch.cuda.synchronize()
        assert st.status() == 0
        o = out.float().cpu().numpy()
        for i, r in enumerate(rs):
            T = tries[i]
            Kp = st.dense_view(hp.kp[l], T.N, [r])[0].float().cpu().numpy().astype(np.float64)
            Vp = st.dense_view(hp.vp[l], T.N, [r])[0].float().cpu().numpy().astype(np.float64)
            qr = np.zeros_like(q0[r])
            for j, leaf in enumerate(T.leaves):
                pos = int(T.depth[leaf])
                for hh in range(q0.shape[2]):
                    qr[j, hh] = rope_rotate_half(q0[r, j, hh], pos, theta)
                for hk in range(k0.shape[2]):  # the appended leaf rows (write-before-read)
                    krot = rope_rotate_half(k0[r, j, hk], pos, theta)
                    assert rel_err(Kp[hk, leaf], krot) <= 1e-2
                    assert np.array_equal(Vp[hk, leaf], v0[r, j, hk])
                    Kp[hk, leaf] = krot  # the reference attends over the oracle's own leaf rows
            o_ref, _ = attn_ref(qr, Kp, Vp, T, window=W)
            err = rel_err(o[r], o_ref)
            assert err <= 2e-2, f"{wl_name} layer {l} request {r}: rel err {err}"
