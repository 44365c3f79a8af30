"""Experiment: per-launch time of trie_attn_decode alone (graph of L back-to-back
launches) vs inside the full step, and of the other step kernels alone.
    python scripts/attn_only.py [--workload phi]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402


def time_graph(fn, reps=20):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="phi")
    ap.add_argument("--beam", type=int, default=0)
    ap.add_argument("--requests", type=int, default=0)
    a = ap.parse_args()
    from paper_2502_00085_b200 import _lib
    from paper_2502_00085_b200.build import build
    build()
    _lib.load()
    wl = dict(bench.WORKLOADS[a.workload])
    if a.beam:
        wl["b"] = a.beam
    if a.requests:
        wl["R"] = a.requests
    dev = torch.device("cuda", 0)
    hp = bench.HotPath(wl, 0, dev)
    for i in range(8):  # advance into a job (steady state)
        hp.step_ops("first" if i == 0 else "steady", i % 2)
    torch.cuda.synchronize()
    st, L = hp.st, hp.L
    d = hp.inp[("steady", 0)]
    res = {}
    res["attn_only_per_launch_us"] = 1e3 * time_graph(
        lambda: [st.attn_decode(d["views"][l][0], hp.kp[l], hp.vp[l], d["out"], rows_hint=hp.rows_hint)
                 for l in range(L)]) / L
    res["rope_only_per_launch_us"] = 1e3 * time_graph(
        lambda: [st.rope_kv_append(*d["views"][l], hp.kp[l], hp.vp[l], wl["theta"]) for l in range(L)]) / L
    res["rope_attn_per_layer_us"] = 1e3 * time_graph(
        lambda: [(st.rope_kv_append(*d["views"][l], hp.kp[l], hp.vp[l], wl["theta"]),
                  st.attn_decode(d["views"][l][0], hp.kp[l], hp.vp[l], d["out"], rows_hint=hp.rows_hint))
                 for l in range(L)]) / L
    res["fused_per_launch_us"] = 1e3 * time_graph(
        lambda: [st.attn_decode_rope(*d["views"][l], hp.kp[l], hp.vp[l], wl["theta"], d["out"],
                                     rows_hint=hp.rows_hint) for l in range(L)]) / L
    N = st.n_nodes.cpu().numpy()
    res["attn_bytes_per_launch"] = hp.attn_bytes(8, N)
    res["attn_only_GBps"] = res["attn_bytes_per_launch"] / (res["attn_only_per_launch_us"] * 1e-6) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
