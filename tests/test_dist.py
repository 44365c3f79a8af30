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

from paper_2502_00085_b200.dist import gather_hyps, max_over_ranks, partition


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
