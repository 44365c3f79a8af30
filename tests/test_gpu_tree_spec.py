"""GPU: trie_attn_decode on speculative draft trees ("multi-token
branches").

A draft tree of depth > 1 hangs off the prompt; EVERY draft node is a query (verification
of all branches in one pass) and attends to the prompt and to its own ancestors-or-self.
That is Alg. 3's mask with one walker per query node, so the unchanged
attention entry point covers it: leaf_ids = the query nodes (interior ones included),
beam_mask bit j = node on query j's root path.  The oracle is attn_ref on an oracle Trie
whose `leaves` are the query nodes (build_mask walks from each)."""
import zlib

import numpy as np
import pytest
import torch

import synth
from oracle.kernels_ref import attn_ref, mask_bits
from oracle.trie import Trie
from tests.gpu_util import need_gpu, rel_err

pytestmark = pytest.mark.gpu


def _draft_tree(T: Trie, branching):
    """Append a draft tree level by level (BFS slot order, so parent < child)."""
    frontier = [T.t - 1]
    nodes = []
    for lvl, k in enumerate(branching):
        nxt = []
        for p in frontier:
            for c in range(k):
                T.token.append(7 * lvl + c)
                T.parent.append(p)
                T.depth.append(T.depth[p] + 1)
                nxt.append(T.N - 1)
        nodes += nxt
        frontier = nxt
    T.leaves = nodes  # every draft node is a query
    return nodes


@pytest.mark.parametrize("name,R,t,branching,Hq,Hkv,D,W,dt", [
    ("mha-d96", 2, 300, (2, 2, 2), 4, 4, 96, 0, "bf16"),        # 14 queries, Qg = 14: narrow
    ("gqa-d128", 2, 500, (3, 2, 2), 8, 2, 128, 0, "bf16"),      # 21 queries, Qg = 84: tcgen05
    ("gqa-wide", 1, 200, (2, 3, 1), 8, 2, 64, 0, "bf16"),       # 14 queries, Qg = 56
    ("swa", 1, 260, (2, 2, 2), 4, 2, 128, 100, "bf16"),         # window by depth
    ("f32", 1, 90, (4, 2), 4, 2, 64, 0, "f32"),                 # 12 queries, CUDA-core path
    ("deep-chain", 1, 64, (1,) * 20 + (2,), 2, 1, 128, 0, "bf16"),  # 22 queries, one long branch
])
def test_draft_tree_attention_matches_oracle(name, R, t, branching, Hq, Hkv, D, W, dt):
    need_gpu()
    from paper_2502_00085_b200 import _lib
    seed = zlib.crc32(name.encode()) % 1000
    V = 100
    prompts, lens = synth.prompts(seed, R, t, V)
    tries = []
    for r in range(R):
        T = Trie(prompts[r][: lens[r]])
        _draft_tree(T, branching)
        tries.append(T)
    nq = len(tries[0].leaves)
    assert nq <= 32
    N = tries[0].N
    cap = (max(N, t + 32) + 63) // 64 * 64  # cfg: capacity >= t_max + beam_width (32)
    meta = {k: np.zeros((R, cap), np.int32) for k in ("parent", "depth")}
    mask = np.zeros((R, cap), np.uint32)
    leaf = np.zeros((R, 32), np.int32)
    for r, T in enumerate(tries):
        meta["parent"][r, :N] = T.parent
        meta["depth"][r, :N] = T.depth
        mask[r, :N] = mask_bits(T)
        leaf[r, :nq] = T.leaves
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    K = torch.as_tensor(synth.normal(seed, 1, (R, Hkv, cap, D)), dtype=torch.float32).to(dtype).cuda()
    Vv = torch.as_tensor(synth.normal(seed, 2, (R, Hkv, cap, D)), dtype=torch.float32).to(dtype).cuda()
    Q = torch.as_tensor(synth.normal(seed, 3, (R, nq, Hq, D)), dtype=torch.float32).to(dtype).cuda()
    cfg = _lib.make_cfg(R, 32, t, cap, 1, Hq, Hkv, D, V, W, 1,
                        _lib.TRIE_BF16 if dt == "bf16" else _lib.TRIE_F32)
    scratch = torch.zeros(_lib.trie_attn_scratch_bytes(cfg, nq, N), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(Q)
    lse = torch.empty(R, nq, Hq, dtype=torch.float32, device="cuda")
    cu = lambda x: torch.as_tensor(x, device="cuda")  # noqa: E731
    _lib.trie_attn_decode(cfg, nq, Q, K, Vv, cu(np.asarray(lens, np.int32)), cu(meta["parent"]),
                          cu(meta["depth"]), cu(leaf), cu(np.full(R, N, np.int32)),
                          cu(mask.view(np.int32)), W, N, out, lse, scratch)
    torch.cuda.synchronize()
    tol = 1e-4 if dt == "f32" else 2e-2
    Kh, Vh, Qh = (x.float().cpu().numpy().astype(np.float64) for x in (K, Vv, Q))
    o, l = out.float().cpu().numpy(), lse.cpu().numpy()
    for r, T in enumerate(tries):
        o_ref, lse_ref = attn_ref(Qh[r], Kh[r][:, :N], Vh[r][:, :N], T, window=W)
        assert rel_err(o[r], o_ref) <= tol, f"{name} r={r}: {rel_err(o[r], o_ref)}"
        assert np.abs(l[r] - lse_ref).max() <= tol * max(1.0, np.abs(lse_ref).max())
