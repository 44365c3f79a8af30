"""CPU checks of bench.py's host logic (no GPU): the roofline's algorithmic bytes against the
oracle's own definition of the rows a launch must read, and the GC schedule against the
oracle's Alg. 2 schedule."""
import types

import numpy as np
import pytest

import bench
import synth
from oracle.kernels_ref import build_tries
from oracle.trie import build_mask, window_allow


def _fake(wl, R):
    return types.SimpleNamespace(t=wl["t"], b=wl["b"], W=wl["W"], R=R, Hq=wl["Hq"], Hkv=wl["Hkv"],
                                 D=wl["D"], g=1, s=wl["s"])


@pytest.mark.parametrize("W", [0, 40, 140])
def test_attn_bytes_counts_the_union_of_visible_rows(W):
    """bench.HotPath.attn_bytes: unique rows U_r = rows visible to SOME beam
    (Alg. 3 mask rows, windowed by depth, reading R14), x 2*Hkv*D*2 B, + Q/O + 8 B per
    generated row -- checked against the oracle's masks on teacher-forced tries (prune
    every step), in the bench's regime (window lower bound <= t)."""
    R, b, t, V, steps = 3, 4, 150, 50, 7
    wl = dict(t=t, b=b, W=W, Hq=8, Hkv=2, D=64, s=64)
    prompts, lens = synth.prompts(5, R, t, V)
    sels = []
    rng = np.random.default_rng(7)
    for k in range(steps):
        bl = 1 if k == 0 else b
        sels.append((rng.integers(0, bl, (R, b)).astype(np.int32), rng.integers(0, V, (R, b)).astype(np.int32)))
    tries = build_tries(prompts, lens, sels, b, g=1, final_gc=True)
    N = np.array([T.N for T in tries])
    U = 0
    for T in tries:
        M = build_mask(T)
        vis = np.zeros(T.N, bool)
        for j, leaf in enumerate(T.leaves):
            vis |= window_allow(T, leaf, M[j], W)
        U += int(vis.sum())
    want = U * 2 * wl["Hkv"] * wl["D"] * 2 + R * b * wl["Hq"] * wl["D"] * 2 * 2 + int((N - t).sum()) * 8
    got = bench.HotPath.attn_bytes(_fake(wl, R), steps, N)
    assert got == want


@pytest.mark.parametrize("g", [1, 3, 4, 15])
def test_gc_schedule_matches_the_oracle(g):
    """bench.HotPath.gc_now (0-based job step k) == the oracle's build_tries schedule
    ((t + k) mod g == 0 after the append of 1-based step k, readings R7/R8)."""
    t, s = 150, 40
    hp = types.SimpleNamespace(g=g, t=t)
    for k0 in range(s):
        assert bench.HotPath.gc_now(hp, k0) == ((t + (k0 + 1)) % g == 0)


def test_reference_arm_shares_the_gpu_arm_config():
    """--impl reference reports the GPU arm's exact `config` (same workload, shape, parallelism)."""
    args = types.SimpleNamespace(workload="phi", beam=0, requests=0, gc_interval=1, eos_frac=0.0)
    wl = bench._workload(args)
    cfg = bench.bench_config(wl, 1)
    assert cfg["workload"] == bench.WORKLOADS["phi"]["name"] and cfg["requests_per_gpu"] == 64
    assert cfg["parallelism"] == "request-dp1"
    shard = bench.bench_config(dict(bench.WORKLOADS["mistral-shard"], g=1), 8)
    assert shard["kv_heads_per_gpu"] == 1 and shard["q_heads_per_gpu"] == 4


def test_cpu_oracle_run_is_measured_per_step():
    """The CPU oracle leg times every layer for real: 2 worker processes, a tiny workload,
    and a wall clock per step that covers L x attn_ref (no extrapolation)."""
    wl = dict(name="tiny", L=2, Hq=4, Hkv=2, D=16, V=64, t=20, b=3, s=6, R=2, W=0)
    v, d = bench.cpu_oracle_run(wl, steps=3, warmup=1, workers=2)
    assert d["workers"] == 2 and d["steps"] == 3 and v > 0
    assert abs(v - 2 * 3 / (d["ms_per_step"] * 3e-3)) <= 1e-2 * v
    assert d["per_request_step_s"] * 1e3 <= d["ms_per_step"] * 1.5
