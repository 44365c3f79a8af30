"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 host logic: request
partitioning, per-rank decoding of its own block, gather ordered by request id, and the
max-over-ranks timing reduction.  Per-rank 'decoding' here runs the CPU oracle (test
infrastructure) so the gathered result can be compared with a single-process run."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_00085_b200.dist import (gather_heads, gather_hyps, heads_view, kv_head_shard,
                                        max_over_ranks, partition)


def test_partition_covers_all_requests():
    for n in (1, 7, 8, 64, 65):
        for world in (1, 2, 3, 8):
            seen = []
            for rank in range(world):
                s, c = partition(n, world, rank)
                seen += list(range(s, s + c))
            assert seen == list(range(n))
            counts = [partition(n, world, r)[1] for r in range(world)]
            assert max(counts) - min(counts) <= 1


def _decode_block(start, count, b=3, s=6):
    import synth
    from oracle.decode import trie_beam_search
    from oracle.model import Model, ModelConfig
    om = Model(synth.tiny_weights(0, 2, 64, 4, 4, 16, 256, 256), ModelConfig())
    prompts, _ = synth.prompts(42, 16, 8, 256)
    toks = np.full((count, b, 8 + s), -1, np.int32)
    lens = np.zeros((count, b), np.int32)
    scores = np.zeros((count, b))
    for i in range(count):
        res = trie_beam_search(om, [int(x) for x in prompts[start + i]], b, s, g=1)
        for j, (h, sc) in enumerate(res.hyps):
            toks[i, j, : len(h)] = h
            lens[i, j] = len(h)
            scores[i, j] = sc
    return toks, lens, scores


def _worker(rank, world, port, n_req, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, count = partition(n_req, world, rank)
    toks, lens, scores = _decode_block(start, count)
    out = gather_hyps(start, toks, lens, scores)
    t = max_over_ranks(1.0 + rank)
    if rank == 0:
        q.put((out[0], out[1], out[2], t))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n_req", [5, 4])
def test_two_rank_gloo_decode_equals_single_process(n_req):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_req, q)) for r in range(2)]
    for p in procs:
        p.start()
    toks, lens, scores, t = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = _decode_block(0, n_req)
    assert np.array_equal(toks, ref[0]) and np.array_equal(lens, ref[1])
    assert np.array_equal(scores, ref[2])
    assert t == 2.0  # max over ranks


def test_kv_head_shard_blocks():
    for Hq, Hkv in ((32, 8), (4, 4), (8, 1)):
        for world in (1, 2, 4, 8):
            if Hkv % world:
                with pytest.raises(ValueError):
                    kv_head_shard(Hq, Hkv, world, 0)
                continue
            kv_seen, q_seen = [], []
            for r in range(world):
                kv0, nkv, q0, nq = kv_head_shard(Hq, Hkv, world, r)
                kv_seen += list(range(kv0, kv0 + nkv))
                q_seen += list(range(q0, q0 + nq))
                g = Hq // Hkv
                assert all(h // g in range(kv0, kv0 + nkv) for h in range(q0, q0 + nq))
            assert kv_seen == list(range(Hkv)) and q_seen == list(range(Hq))


def _shard_case():
    """One request of the 24B-like GQA shape in miniature: Hq = 8, Hkv = 4, D = 16, a
    random trie (b = 3) with a window; q, K, V seeded."""
    import synth
    from oracle.kernels_ref import build_tries
    rng = np.random.default_rng(5)
    b, t, steps, V = 3, 12, 5, 50
    prompts, lens = synth.prompts(7, 1, t, V)
    sel = [(np.zeros((1, b), np.int32), rng.choice(V, (1, b), replace=False).astype(np.int32))]
    sel += [(rng.integers(0, b, (1, b)).astype(np.int32), rng.integers(0, V, (1, b)).astype(np.int32))
            for _ in range(steps - 1)]
    T = build_tries(prompts, lens, sel, b)[0]
    q = rng.standard_normal((b, 8, 16))
    K = rng.standard_normal((4, T.N, 16))
    Vv = rng.standard_normal((4, T.N, 16))
    return T, q, K, Vv


def _shard_worker(rank, world, port, q_out):
    import torch
    from oracle.kernels_ref import attn_ref
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    T, q, K, Vv = _shard_case()
    kv0, nkv, q0, nq = kv_head_shard(8, 4, world, rank)
    o, _ = attn_ref(q[:, q0:q0 + nq], K[kv0:kv0 + nkv], Vv[kv0:kv0 + nkv], T, window=6)
    g = gather_heads(torch.as_tensor(o)[None])  # [world][1][b][nq][D]
    full = heads_view(g)[0].numpy()
    if rank == 0:
        q_out.put(full)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_kv_head_shard_gather_equals_full_attention():
    """configs[3] host logic: per-rank attention over its KV-head slice + the all-gather
    of the outputs == attention over all heads in one process (oracle as the per-rank
    compute, test infrastructure)."""
    from oracle.kernels_ref import attn_ref
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    T, qq, K, Vv = _shard_case()
    ref, _ = attn_ref(qq, K, Vv, T, window=6)
    assert np.array_equal(full, ref)
