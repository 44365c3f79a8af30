"""Multi-GPU plumbing; one process per GPU.

Request data parallelism: each rank owns a contiguous block of independent requests
("distinct sessions may run in parallel").  No per-step collective: ranks decode
their own requests; the only collectives are the end-of-job gather of the hypotheses and
the max-over-ranks timing reduction.

KV-head sharding (BASELINE.json configs[3], the 24B shape): every rank holds the SAME
requests and trie metadata but only its slice of the KV heads (Hkv / world KV heads and
their Hq / world query heads, GQA groups kept whole).  Per layer each rank runs
trie_attn_decode on its slice and the attention outputs are all-gathered so that the
replicated O-projection / MLP / LM head (model context) see every head; identical logits
then give identical beam-step choices and identical trie metadata on every rank, and each
rank prunes / compacts only its own KV slice.

Works with any torch.distributed backend (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def partition(n_requests: int, world: int, rank: int):
    """Contiguous, balanced block [start, start + count) of the global request ids."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(n_requests, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def gather_hyps(start: int, tokens: np.ndarray, lens: np.ndarray, scores: np.ndarray, dst: int = 0):
    """Gather per-rank hypotheses ([r][b][max_len] tokens, [r][b] lens, [r][b] scores) to
    rank `dst`, ordered by global request id.  Returns the concatenation on dst, else None."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    payload = (int(start), np.asarray(tokens), np.asarray(lens), np.asarray(scores))
    if world == 1:
        return payload[1:]
    objs = [None] * world if dist.get_rank() == dst else None
    dist.gather_object(payload, objs, dst=dst)
    if dist.get_rank() != dst:
        return None
    objs.sort(key=lambda p: p[0])
    return (np.concatenate([o[1] for o in objs if len(o[1])]),
            np.concatenate([o[2] for o in objs if len(o[2])]),
            np.concatenate([o[3] for o in objs if len(o[3])]))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank timing (the bench reports the slowest rank)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def kv_head_shard(n_q_heads: int, n_kv_heads: int, world: int, rank: int):
    """This rank's KV heads [kv0, kv0 + n_kv) and query heads [q0, q0 + n_q): contiguous
    blocks of whole GQA groups (query head h uses KV head h // (Hq / Hkv))."""
    if n_q_heads % n_kv_heads:
        raise ValueError("n_q_heads must be a multiple of n_kv_heads")
    if world < 1 or not (0 <= rank < world) or n_kv_heads % world:
        raise ValueError(f"{n_kv_heads} KV heads cannot be split over {world} ranks")
    n_kv = n_kv_heads // world
    g = n_q_heads // n_kv_heads
    return rank * n_kv, n_kv, rank * n_kv * g, n_kv * g


def gather_heads(out_local: torch.Tensor, gathered: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather of the per-rank attention outputs [R][b][Hq/world][D] into the rank-major
    buffer [world][R][b][Hq/world][D] (one collective per layer; CUDA-graph capturable
    under NCCL).  `gathered` may be preallocated (the bench captures it in its graphs)."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    if gathered is None:
        gathered = out_local.new_empty((world,) + tuple(out_local.shape))
    if world == 1:
        gathered[0].copy_(out_local)
        return gathered
    if gathered.is_cuda:
        dist.all_gather_into_tensor(gathered, out_local.contiguous())
    else:  # gloo (CPU tests): list form
        dist.all_gather(list(gathered.unbind(0)), out_local.contiguous())
    return gathered


def heads_view(gathered: torch.Tensor) -> torch.Tensor:
    """[world][R][b][Hq/world][D] -> [R][b][Hq][D] in global head order (a copy)."""
    w, R, b, hl, D = gathered.shape
    return gathered.permute(1, 2, 0, 3, 4).reshape(R, b, w * hl, D)


class FusedGather:
    """the KV-head shard's per-layer all-gather fused into the attention
    kernels (include/triedecode.h trie_gather_setup).  Every rank allocates its gather buffer
    [2][R][b][world*Hq_local][D] bf16 and flag array [world] uint32 with CUDA IPC, the
    handles are exchanged once over the process group (any backend: plumbing, not data
    path), every rank maps every peer's buffers and registers them with its trie handle.
    Then each trie_attn_decode_rope stores its output rows straight into every rank's
    buffer from the kernel epilogue, and wait(dst) = trie_gather_wait copies the completed
    call's [R][b_live][world*Hq_local][D] into dst once every rank has published it."""

    def __init__(self, st, world: int, rank: int):
        from . import _lib as L
        self.L, self.st, self.world, self.rank = L, st, world, rank
        half = st.R * st.b * world * st.Hq * st.D
        self.out_ptr, h_out = L.trie_ipc_alloc(2 * half * 2)
        self.flag_ptr, h_flag = L.trie_ipc_alloc(64)
        handles = [None] * world
        dist.all_gather_object(handles, (h_out, h_flag))
        self.peer_out, self.peer_flags, self.opened = [], [], []
        for q, (ho, hf) in enumerate(handles):
            if q == rank:
                self.peer_out.append(self.out_ptr)
                self.peer_flags.append(self.flag_ptr)
                continue
            po, pf = L.trie_ipc_open(ho), L.trie_ipc_open(hf)
            self.opened += [po, pf]
            self.peer_out.append(po)
            self.peer_flags.append(pf)
        L.trie_gather_setup(st.h, world, rank, self.peer_out, self.peer_flags)
        dist.barrier()  # every rank registered before anyone stores into a peer

    def wait(self, dst=None, stream=None):
        """Enqueue the wait for the last call's gather; copy it into dst [R][b_live][world*Hq][D]."""
        self.L.trie_gather_wait(self.st.h, dst, stream)
        return dst

    def close(self):
        torch.cuda.synchronize()
        dist.barrier()  # no rank still stores into our buffers
        for p in self.opened:
            self.L.trie_ipc_close(p)
        self.opened = []
        dist.barrier()
        self.L.trie_ipc_free(self.out_ptr)
        self.L.trie_ipc_free(self.flag_ptr)
