"""Request data parallelism: one process per GPU, each owning a
contiguous block of independent requests ("distinct sessions may run in parallel").
There is no per-step collective: ranks decode their own requests; the only collectives are
the end-of-job gather of the hypotheses and the max-over-ranks timing reduction.
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
