"""GPU vs oracle: trie_attn_decode and trie_rope_kv_append.

Each side builds its own trie from the same seeded selection sequence (GPU: trie_append +
trie_prune_compact; oracle: build_tries), the integer states are checked equal, then the
GPU kernel and oracle.kernels_ref.attn_ref run on the same seeded Q/K/V.  Tolerances
(BASELINE.json north_star, reading R24): 1e-4 relative for fp32, 2e-2 for bf16; lse
absolute 1e-4 / 2e-2.  Shapes span several tiles, ragged prompt lengths, GQA groups,
windows, b_live = 1, and the beam_mask == NULL (Alg. 3 walk) variant."""
import zlib

import numpy as np
import pytest
import torch

import synth
from oracle.kernels_ref import attn_ref, build_tries, soa
from oracle.numerics import rope_rotate_half
from tests.gpu_util import need_gpu, per_request_selections, rel_err

pytestmark = pytest.mark.gpu

CASES = [
    # name, R, b, t_max, ragged, steps, rho, Hq, Hkv, D, window, dtype, use_mask
    ("tiny", 2, 3, 8, False, 16, 0.5, 4, 4, 16, 0, "f32", True),
    ("tiny-walk", 3, 3, 8, True, 16, 0.5, 4, 2, 16, 0, "f32", False),
    ("phi-like", 2, 4, 800, False, 12, 0.5, 32, 32, 96, 0, "bf16", True),
    ("phi-f32", 1, 4, 300, False, 9, 0.3, 8, 8, 96, 0, "f32", True),
    ("llama-like", 2, 8, 150, True, 40, 0.5, 32, 8, 128, 0, "bf16", True),
    ("llama-f32", 2, 8, 150, False, 20, 0.5, 8, 2, 128, 0, "f32", True),
    ("swa", 2, 4, 300, False, 20, 0.5, 8, 2, 128, 64, "bf16", True),
    ("swa-w1", 1, 4, 50, False, 6, 0.5, 4, 1, 64, 1, "f32", True),
    ("b32", 1, 32, 500, False, 10, 0.9, 8, 2, 128, 0, "bf16", True),
    ("b16-g4", 1, 16, 700, False, 8, 0.0, 16, 4, 128, 0, "bf16", True),
    # tcgen05 path: ragged + window, head_dim 64, and Qg = 48 (a live warp with padding rows)
    ("b16-swa-ragged", 2, 16, 600, True, 8, 0.5, 16, 4, 128, 200, "bf16", True),
    ("b32-d64", 1, 32, 300, False, 6, 0.5, 4, 2, 64, 0, "bf16", True),
    ("b12-g4", 2, 12, 400, True, 6, 0.5, 8, 2, 128, 0, "bf16", True),
    ("b1", 3, 1, 40, True, 5, 0.0, 4, 4, 32, 0, "f32", True),
    # long tries at Qg = 16 / 32 take the tcgen05 kernel by the default plan (>= 1024 rows)
    ("llama-long-qg32", 1, 8, 1200, True, 12, 0.5, 32, 8, 128, 0, "bf16", True),
    ("qg16-swa-long", 2, 4, 1100, True, 10, 0.5, 16, 4, 128, 300, "bf16", True),
    ("d256", 1, 2, 70, False, 4, 0.5, 2, 1, 256, 0, "f32", True),
]


@pytest.mark.parametrize("name,R,b,t_max,ragged,steps,rho,Hq,Hkv,D,W,dt,use_mask", CASES,
                         ids=[c[0] for c in CASES])
def test_attn_matches_oracle(name, R, b, t_max, ragged, steps, rho, Hq, Hkv, D, W, dt, use_mask):
    need_gpu()
    from paper_2502_00085_b200.trie import TrieState
    seed = zlib.crc32(name.encode()) % 1000
    V = 500
    lens = synth.ragged_lens(seed, R, t_max) if ragged else None
    prompts, lens = synth.prompts(seed, R, t_max, V, lens)
    sels = per_request_selections(seed, R, steps, b, V, rho)
    cap = t_max + b * steps + b
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    st = TrieState(R, b, t_max, cap, 1, Hq, Hkv, D, V, prompts, lens, window=W, dtype=dtype)
    kp0, vp0 = st.new_pools()
    for k, (par, tok) in enumerate(sels, 1):
        st.append(torch.as_tensor(par, device="cuda"), torch.as_tensor(tok, device="cuda"))
        st.prune_compact(kp0, vp0)
    tries = build_tries(prompts, lens, sels, b, g=1, final_gc=True)
    ref = soa(tries, cap, b)
    assert np.array_equal(st.n_nodes.cpu().numpy(), ref["N"])
    # seeded K/V for every slot and Q for the b leaves, rounded to the kernel's dtype
    K = synth.normal(seed, 1, (R, Hkv, cap, D))
    Vv = synth.normal(seed, 2, (R, Hkv, cap, D))
    Q = synth.normal(seed, 3, (R, b, Hq, D))
    tK, tV, tQ = (torch.as_tensor(x, dtype=torch.float32).to(dtype).cuda() for x in (K, Vv, Q))
    K, Vv, Q = (x.float().cpu().numpy().astype(np.float64) for x in (tK, tV, tQ))
    out = torch.empty_like(tQ)
    lse = torch.empty(R, b, Hq, dtype=torch.float32, device="cuda")
    st.attn_decode(tQ, tK, tV, out, lse, rows_hint=int(ref["N"].max()), use_mask=use_mask)
    torch.cuda.synchronize()
    o = out.float().cpu().numpy()
    l = lse.cpu().numpy()
    tol = 1e-4 if dt == "f32" else 2e-2
    for r in range(R):
        N = tries[r].N
        o_ref, lse_ref = attn_ref(Q[r], K[r][:, :N], Vv[r][:, :N], tries[r], window=W)
        assert rel_err(o[r], o_ref) <= tol, f"{name} r={r}: rel err {rel_err(o[r], o_ref)}"
        assert np.abs(l[r] - lse_ref).max() <= tol * max(1.0, np.abs(lse_ref).max())
    assert st.status() == 0


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_rope_kv_append_matches_oracle(dt):
    """a-1: RoPE at depth (§3.4) + write-before-read append, vs oracle rope_rotate_half."""
    need_gpu()
    from paper_2502_00085_b200.trie import TrieState
    R, b, t_max, Hq, Hkv, D, V, base = 2, 4, 700, 8, 2, 128, 100, 500000.0
    prompts, lens = synth.prompts(5, R, t_max, V, [700, 333])
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    st = TrieState(R, b, t_max, t_max + 20, 1, Hq, Hkv, D, V, prompts, lens, dtype=dtype)
    sels = per_request_selections(5, R, 2, b, V, 0.5)
    for par, tok in sels:
        st.append(torch.as_tensor(par, device="cuda"), torch.as_tensor(tok, device="cuda"))
    q = torch.as_tensor(synth.normal(6, 1, (R, b, Hq, D)), dtype=torch.float32).to(dtype).cuda()
    k = torch.as_tensor(synth.normal(6, 2, (R, b, Hkv, D)), dtype=torch.float32).to(dtype).cuda()
    v = torch.as_tensor(synth.normal(6, 3, (R, b, Hkv, D)), dtype=torch.float32).to(dtype).cuda()
    q0, k0, v0 = (x.float().cpu().numpy().astype(np.float64) for x in (q, k, v))
    kp, vp = st.new_pools()
    st.rope_kv_append(q, k, v, kp[0], vp[0], base)
    torch.cuda.synchronize()
    tol = 1e-5 if dt == "f32" else 1e-2
    leaf = st.leaf.cpu().numpy()
    depth = st.depth.cpu().numpy()
    for r in range(R):
        for j in range(b):
            pos = int(depth[r, leaf[r, j]])
            assert pos == int(lens[r]) + 1           # two appends: depth t + 1 (§3.4)
            qr = rope_rotate_half(q0[r, j], pos, base)
            kr = rope_rotate_half(k0[r, j], pos, base)
            assert rel_err(q[r, j].float().cpu().numpy(), qr) <= tol
            assert rel_err(kp[0, r, :, leaf[r, j]].float().cpu().numpy(), kr) <= tol
            assert np.array_equal(vp[0, r, :, leaf[r, j]].float().cpu().numpy(), v0[r, j])


@pytest.mark.parametrize("name,R,b,t_max,Hq,Hkv,D,W", [
    ("paged-narrow", 3, 4, 300, 8, 8, 96, 0),
    ("paged-gqa-swa", 2, 4, 200, 8, 2, 128, 60),
    ("paged-wide", 2, 8, 150, 32, 8, 128, 0),
    ("paged-umma", 2, 16, 400, 8, 2, 128, 0),
    ("paged-split", 1, 2, 1500, 2, 2, 128, 0),
])
def test_fused_paged_pools_match_oracle(name, R, b, t_max, Hq, Hkv, D, W):
    """the same fused RoPE + append + attention over PAGED pools
    ([n_pages][Hkv][64][D], 64-slot pages mapped through the page table as N grows,
    returned by GC) -- identical results to the oracle as with dense pools."""
    _fused_case(name, R, b, t_max, Hq, Hkv, D, W, paged=True)


@pytest.mark.parametrize("name,R,b,t_max,Hq,Hkv,D,W,steps", [
    ("evict-narrow", 2, 4, 300, 8, 2, 128, 100, 8),
    ("evict-umma", 2, 16, 600, 8, 2, 128, 200, 6),
    ("evict-d64", 1, 4, 500, 4, 1, 64, 64, 10),
])
def test_swa_eviction_frees_prompt_pages_and_matches_oracle(name, R, b, t_max, Hq, Hkv, D, W, steps):
    """with paged pools and a window, trie_swa_evict returns the pages
    of prompt blocks below every live beam's window to the free queue (later appends reuse
    them); attention over the remaining pages still equals the oracle (reading R14)."""
    _fused_case(name, R, b, t_max, Hq, Hkv, D, W, steps=steps, paged=True, evict=True)


@pytest.mark.parametrize("name,R,b,t_max,Hq,Hkv,D,W", [
    ("phi-fused", 2, 4, 300, 8, 8, 96, 0),
    ("gqa-fused", 2, 4, 200, 8, 2, 128, 0),
    ("swa-fused", 1, 4, 150, 4, 1, 64, 40),
    ("split-fused", 1, 2, 1500, 2, 2, 128, 0),
    ("wide-fused", 1, 8, 130, 8, 2, 128, 0),      # Qg = 32: wide kernel, fused
    ("wide-fused-llama", 2, 8, 150, 32, 8, 128, 0),
    ("wide-fused-split", 1, 6, 1000, 16, 4, 64, 0),  # Qg = 24, D = 64, split K
    ("wide1-fused-split", 1, 4, 1500, 8, 2, 64, 0),  # Qg = 16: one m-tile, 4 row slices, split K
    ("wide1-fused-q12", 2, 3, 300, 8, 2, 96, 0),     # Qg = 12: padded query rows
    ("umma-fused", 1, 16, 130, 8, 2, 128, 0),     # Qg = 64: tcgen05, fused
    ("umma-fused-swa", 2, 16, 400, 8, 2, 128, 100),
    ("umma-fused-d96", 1, 12, 300, 8, 2, 96, 0),  # Qg = 48
    ("umma-fused-d64-split", 1, 32, 1500, 4, 2, 64, 0),  # Qg = 64, split K: leaves in the last split
])
def test_fused_rope_attention_matches_oracle(name, R, b, t_max, Hq, Hkv, D, W):
    """trie_attn_decode_rope == RoPE at depth (§3.4) + write-before-read append + trie
    attention, vs the oracle (rope_rotate_half + attn_ref on its own trie)."""
    _fused_case(name, R, b, t_max, Hq, Hkv, D, W)


@pytest.mark.parametrize("name,R,b,t_max,Hq,Hkv,D", [
    ("wide-ragged", 6, 8, 1500, 32, 8, 128),   # Llama shape, requests of 1-24 tiles
    ("wide-ragged-many", 40, 8, 700, 8, 2, 128),
    ("wide-ragged-d96", 3, 6, 900, 12, 3, 96),  # Qg = 24, D = 96
    ("wide1-ragged", 6, 4, 1500, 32, 8, 128),  # Mistral-like Qg = 16, requests of 1-24 tiles
])
def test_fused_ragged_matches_oracle(name, R, b, t_max, Hq, Hkv, D):
    """Fused RoPE + wide attention on requests of very different lengths, vs the oracle."""
    _fused_case(name, R, b, t_max, Hq, Hkv, D, 0, ragged=True)


def _fused_case(name, R, b, t_max, Hq, Hkv, D, W, ragged=False, steps=6, rho=0.5, paged=False,
                evict=False):
    need_gpu()
    from paper_2502_00085_b200.trie import TrieState
    seed = zlib.crc32(name.encode()) % 1000
    V, base = 300, 500000.0
    lens = synth.ragged_lens(seed, R, t_max) if ragged else None
    prompts, lens = synth.prompts(seed, R, t_max, V, lens)
    sels = per_request_selections(seed, R, steps, b, V, rho)
    cap = (t_max + b * steps + b + 63) // 64 * 64
    st = TrieState(R, b, t_max, cap, 1, Hq, Hkv, D, V, prompts, lens, window=W, dtype=torch.bfloat16,
                   n_pages=R * cap // 64 if paged else 0)
    kp, vp = st.new_pools()
    for par, tok in sels:
        st.append(torch.as_tensor(par, device="cuda"), torch.as_tensor(tok, device="cuda"))
        st.prune_compact(kp, vp)
        if evict:  # NEXT-3: free the prompt pages below every live beam's window
            st.swa_evict()
    tries = build_tries(prompts, lens, sels, b, g=1, final_gc=True)
    if evict:  # every block of prompt rows below min_j (depth[leaf_j] - W + 1) is unmapped
        pt = st.page_table.cpu().numpy()
        for r, T in enumerate(tries):
            lo = min(T.depth[x] for x in T.leaves) - W + 1
            nblk = min(lo, T.t) // 64
            assert nblk > 0 and np.all(pt[r, :nblk] == -1) and np.all(pt[r, nblk:(T.N + 63) // 64] >= 0)
    K = synth.normal(seed, 1, (R, Hkv, cap, D))
    Vv = synth.normal(seed, 2, (R, Hkv, cap, D))
    tK = torch.as_tensor(K, dtype=torch.float32).to(torch.bfloat16).cuda()
    tV = torch.as_tensor(Vv, dtype=torch.float32).to(torch.bfloat16).cuda()
    st.write_rows(kp[0], tK)  # dense copy, or through the page table (NEXT-2)
    st.write_rows(vp[0], tV)
    q = torch.as_tensor(synth.normal(seed, 3, (R, b, Hq, D)), dtype=torch.float32).to(torch.bfloat16).cuda()
    kn = torch.as_tensor(synth.normal(seed, 4, (R, b, Hkv, D)), dtype=torch.float32).to(torch.bfloat16).cuda()
    vn = torch.as_tensor(synth.normal(seed, 5, (R, b, Hkv, D)), dtype=torch.float32).to(torch.bfloat16).cuda()
    q0, k0, v0 = (x.float().cpu().numpy().astype(np.float64) for x in (q, kn, vn))
    Kh, Vh = tK.float().cpu().numpy().astype(np.float64), tV.float().cpu().numpy().astype(np.float64)
    out = torch.empty_like(q)
    lse = torch.empty(R, b, Hq, dtype=torch.float32, device="cuda")
    st.attn_decode_rope(q, kn, vn, kp[0], vp[0], base, out, lse, rows_hint=t_max + steps)
    torch.cuda.synchronize()
    assert st.status() == 0
    o, l = out.float().cpu().numpy(), lse.cpu().numpy()
    kpool_after = st.dense_view(kp[0]).float().cpu().numpy()
    vpool_after = st.dense_view(vp[0]).float().cpu().numpy()
    for r in range(R):
        T = tries[r]
        Kr, Vr = Kh[r].copy(), Vh[r].copy()
        qr = np.zeros((b, Hq, D))
        for j, leaf in enumerate(T.leaves):
            pos = T.depth[leaf]
            qr[j] = rope_rotate_half(q0[r, j], pos, base)
            Kr[:, leaf] = rope_rotate_half(k0[r, j], pos, base)
            Vr[:, leaf] = v0[r, j]
            assert rel_err(kpool_after[r, :, leaf], Kr[:, leaf]) <= 1e-2   # appended, rotated
            assert np.array_equal(vpool_after[r, :, leaf], Vr[:, leaf])
        o_ref, lse_ref = attn_ref(qr, Kr[:, :T.N], Vr[:, :T.N], T, window=W)
        assert rel_err(o[r], o_ref) <= 2e-2, f"{name} r={r}: {rel_err(o[r], o_ref)}"
        assert np.abs(l[r] - lse_ref).max() <= 2e-2 * max(1.0, np.abs(lse_ref).max())


def test_attention_plan_paths():
    """The kernel choice the bench relies on: narrow (Qg <= 8), wide (Qg 9..32; one query
    m-tile over 4 row slices for Qg <= 16, r2z3), tcgen05 (Qg >= 33) -- round 2: mma.sync
    with split-K also for long tries at Qg <= 32 (r2r)."""
    need_gpu()
    from paper_2502_00085_b200 import _lib
    import os
    if os.environ.get("TRIE_UMMA_MIN_QG") or os.environ.get("TRIE_ATTN_PERSIST"):
        pytest.skip("plan overridden by environment")

    def path(b, Hq, Hkv, D, cap, rows):
        cfg = _lib.make_cfg(2, b, 8, cap, 1, Hq, Hkv, D, 1000, 0, 1, _lib.TRIE_BF16)
        return _lib.trie_attn_plan_info(cfg, b, rows)["path"]
    assert path(4, 32, 32, 96, 1088, 864).startswith("narrow")         # Phi, Qg = 4
    assert path(8, 32, 8, 128, 448, 406).startswith("wide")            # Llama t=150, Qg = 32
    assert path(8, 32, 8, 128, 8448, 8320).startswith("wide")          # sweep t=8192, Qg = 32
    assert path(4, 32, 8, 128, 8448, 8320).startswith("wide")          # sweep, Qg = 16 (r2z3)
    assert path(4, 32, 8, 128, 4224, 4100).startswith("wide")          # Mistral shard, Qg = 16
    assert path(32, 32, 8, 128, 8448, 8320).startswith("tcgen05")      # sweep, Qg = 128
    assert path(16, 32, 8, 128, 448, 406).startswith("tcgen05")        # Qg = 64
    assert path(2, 32, 8, 128, 8448, 8320).startswith("narrow")        # Qg = 8


def _fuzz_cases(n=24, seed=2502):
    """Seeded random shapes for the fused path (the call bench.py times): ragged prompts
    from 1 row to several tiles (pre-wait prefetch from 0 to many tiles, prompts that end on
    and off tile boundaries), b in 1..16, GQA groups 1..8, D in {64, 96, 128}, windows
    shorter and longer than the tries, narrow / wide / tcgen05 kernels."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        D = int(rng.choice([64, 96, 128]))
        Hkv = int(rng.choice([1, 2, 4]))
        g = int(rng.choice([1, 2, 4, 8]))
        b = int(rng.choice([1, 2, 3, 4, 5, 8, 12, 16]))
        t_max = int(rng.choice([1, 17, 64, 65, 128, 150, 300, 513]))
        W = int(rng.choice([0, 0, 1, 7, 64, 200]))
        out.append((f"fuzz{i}", int(rng.integers(1, 5)), b, t_max, g * Hkv, Hkv, D, W,
                    bool(rng.integers(0, 2)), int(rng.integers(1, 9)), float(rng.choice([0.0, 0.5, 1.0]))))
    return out


@pytest.mark.parametrize("name,R,b,t_max,Hq,Hkv,D,W,ragged,steps,rho", _fuzz_cases(),
                         ids=[c[0] for c in _fuzz_cases()])
def test_fused_fuzz_matches_oracle(name, R, b, t_max, Hq, Hkv, D, W, ragged, steps, rho):
    """trie_attn_decode_rope on seeded random shapes vs the oracle (bf16, 2e-2)."""
    _fused_case(name, R, b, t_max, Hq, Hkv, D, W, ragged=ragged, steps=steps, rho=rho)


@pytest.mark.parametrize("Hq,Hkv,D", [(8, 8, 96), (32, 4, 128), (32, 2, 128)])  # narrow, wide, tcgen05
def test_fused_skips_finished_requests(Hq, Hkv, D):
    """NEXT-3 (reading R5b): with an EOS id set, trie_attn_decode_rope skips a request whose
    beams are all finished (no append, output rows untouched); the other requests are
    computed as usual (vs the oracle)."""
    need_gpu()
    from paper_2502_00085_b200.trie import TrieState
    R, b, t, V, steps, eos, base = 3, 4, 200, 300, 4, 7, 500000.0
    seed = 4242 + D
    prompts, lens = synth.prompts(seed, R, t, V)
    sels = per_request_selections(seed, R, steps, b, V, 0.5)
    # request 1 finishes every beam at the last step: tokens = eos
    sels[-1][1][1, :] = eos
    for k in range(steps - 1):
        sels[k][1][sels[k][1] == eos] = eos + 1
    cap = (t + b * steps + b + 63) // 64 * 64
    st = TrieState(R, b, t, cap, 1, Hq, Hkv, D, V, prompts, lens, dtype=torch.bfloat16)
    st.set_eos(eos)
    kp, vp = st.new_pools()
    for par, tok in sels:
        st.append(torch.as_tensor(par, device="cuda"), torch.as_tensor(tok, device="cuda"))
        st.prune_compact(kp, vp)
    fin = st.finished.cpu().numpy()[:, :b] != 0
    assert fin[1].all() and not fin[0].all() and not fin[2].all()
    tries = build_tries(prompts, lens, sels, b, g=1, final_gc=True)
    K = torch.as_tensor(synth.normal(seed, 1, (R, Hkv, cap, D)), dtype=torch.float32).to(torch.bfloat16).cuda()
    Vv = torch.as_tensor(synth.normal(seed, 2, (R, Hkv, cap, D)), dtype=torch.float32).to(torch.bfloat16).cuda()
    kp[0].copy_(K)
    vp[0].copy_(Vv)
    q = torch.as_tensor(synth.normal(seed, 3, (R, b, Hq, D)), dtype=torch.float32).to(torch.bfloat16).cuda()
    kn = torch.as_tensor(synth.normal(seed, 4, (R, b, Hkv, D)), dtype=torch.float32).to(torch.bfloat16).cuda()
    vn = torch.as_tensor(synth.normal(seed, 5, (R, b, Hkv, D)), dtype=torch.float32).to(torch.bfloat16).cuda()
    out = torch.full_like(q, 123.0)
    st.attn_decode_rope(q, kn, vn, kp[0], vp[0], base, out, rows_hint=t + steps)
    torch.cuda.synchronize()
    assert st.status() == 0
    o = out.float().cpu().numpy()
    assert (o[1] == 123.0).all()                               # skipped: output untouched
    assert torch.equal(kp[0][1].cpu(), K[1].cpu())             # and nothing appended
    Kh, Vh = K.float().cpu().numpy().astype(np.float64), Vv.float().cpu().numpy().astype(np.float64)
    q0, k0, v0 = (x.float().cpu().numpy().astype(np.float64) for x in (q, kn, vn))
    for r in (0, 2):
        T = tries[r]
        Kr, Vr = Kh[r].copy(), Vh[r].copy()
        qr = np.zeros((b, Hq, D))
        for j, leaf in enumerate(T.leaves):
            pos = T.depth[leaf]
            qr[j] = rope_rotate_half(q0[r, j], pos, base)
            Kr[:, leaf] = rope_rotate_half(k0[r, j], pos, base)
            Vr[:, leaf] = v0[r, j]
        o_ref, _ = attn_ref(qr, Kr[:, :T.N], Vr[:, :T.N], T)
        assert rel_err(o[r], o_ref) <= 2e-2


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_empty_row_latches_status(dt):
    """TRIE_ST_EMPTY_ROW ("an all-blocked row signals a trie/mask construction bug"):
    a beam whose own mask bit is missing, under a window of 1 key (self only, reading R14),
    has no allowed key -- the pure trie_attn_decode latches the bit in the caller's status
    word, the row's lse is -inf and its output row 0; the other beam's row is unaffected."""
    need_gpu()
    from paper_2502_00085_b200 import _lib
    t, b, Hq, Hkv, D = 4, 2, 4, 2, 64
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    cfg = _lib.make_cfg(1, b, t, 64, 1, Hq, Hkv, D, 100, 1, 1,
                        _lib.TRIE_BF16 if dt == "bf16" else _lib.TRIE_F32)
    cu = lambda x: torch.as_tensor(np.asarray(x), device="cuda")  # noqa: E731
    parent = cu(np.array([[-1, 0, 1, 2, 3, 3] + [-1] * 58], np.int32))
    depth = cu(np.array([[0, 1, 2, 3, 4, 4] + [0] * 58], np.int32))
    mask = cu(np.array([[0, 0, 0, 0, 1, 0] + [0] * 58], np.int32))  # slot 5: beam 1's bit missing
    leaf = cu(np.array([[4, 5] + [0] * 30], np.int32))
    K = torch.randn(1, Hkv, 64, D, device="cuda").to(dtype)
    Vv = torch.randn(1, Hkv, 64, D, device="cuda").to(dtype)
    Q = torch.randn(1, b, Hq, D, device="cuda").to(dtype)
    out = torch.full_like(Q, 7.0)
    lse = torch.zeros(1, b, Hq, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    scratch = torch.zeros(_lib.trie_attn_scratch_bytes(cfg, b, 6), dtype=torch.uint8, device="cuda")
    _lib.trie_attn_decode(cfg, b, Q, K, Vv, cu(np.array([t], np.int32)), parent, depth, leaf,
                          cu(np.array([6], np.int32)), mask, 1, 6, out, lse, scratch, status=status)
    torch.cuda.synchronize()
    assert int(status.item()) & _lib.TRIE_ST_EMPTY_ROW
    l = lse.cpu().numpy()
    assert np.isneginf(l[0, 1]).all() and np.isfinite(l[0, 0]).all()
    assert (out[0, 1].float() == 0).all()
    # beam 0 (window 1: itself only) reads exactly V[slot 4]
    ref = Vv[0, :, 4].float().repeat_interleave(Hq // Hkv, dim=0)
    assert torch.allclose(out[0, 0].float(), ref, atol=1e-2 if dt == "bf16" else 1e-5)


def test_leaf_latch_and_reset_clears_status():
    """TRIE_ST_LEAF: a leaf id outside [0, N) (a corrupted handle) latches on the next beam
    step; trie_reset starts a new job with a clear status word."""
    need_gpu()
    from paper_2502_00085_b200 import _lib
    from paper_2502_00085_b200.trie import TrieState
    prompts, lens = synth.prompts(5, 1, 6, 50)
    st = TrieState(1, 3, 6, 40, 0, 1, 1, 16, 50, prompts, lens, dtype=torch.float32)
    lg1 = torch.zeros(1, 1, 50, device="cuda")
    lg1[0, 0, :3] = 10.0  # three equal-score beams
    st.beam_step(lg1)
    assert st.status() == 0
    st.leaf[0, 1] = 9999
    lg = torch.zeros(1, 3, 50, device="cuda")
    lg[0, 1, 5] = 50.0  # beam 1's continuation (log-prob ~0) outranks the flat rows (-log 50)
    st.beam_step(lg)
    assert st.status() & _lib.TRIE_ST_LEAF
    st.reset()
    assert st.status() == 0
