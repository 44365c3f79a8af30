"""Experiment: isolated per-CTA streaming rate of trie_attn_decode (a few items, unloaded
memory system).  R requests x Hkv heads = CTAs (one split each); prompt t rows + `steps`
appends of b beams (random parents, no GC) -> tiles per item.  Prints us per launch and
us per tile per CTA for the kernel the plan picks (set TRIE_WIDE_RS / TRIE_WIDE1_MIN_QG to
compare variants).
    python scripts/attn_single.py --b 8 --hq 32 --hkv 8 --R 1
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2502_00085_b200 import _lib  # noqa: E402
from paper_2502_00085_b200.build import build  # noqa: E402
from paper_2502_00085_b200.trie import TrieState  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--R", type=int, default=1)
    ap.add_argument("--b", type=int, default=8)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--D", type=int, default=128)
    ap.add_argument("--t", type=int, default=256)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    build()
    _lib.load()
    R, b, t, V = a.R, a.b, a.t, 1000
    cap = (t + b * (a.steps + 2) + 63) // 64 * 64
    prompts, lens = synth.prompts(1, R, t, V, np.full(R, t))
    st = TrieState(R, b, t, cap, 1, a.hq, a.hkv, a.D, V, prompts, lens)
    kp, vp = st.new_pools()
    kp.normal_()
    vp.normal_()
    rng = np.random.default_rng(0)
    st.append(torch.zeros(R, b, dtype=torch.int32, device="cuda"),
              torch.as_tensor(rng.integers(0, V, (R, b)), dtype=torch.int32, device="cuda"))
    for _ in range(a.steps):
        par = torch.as_tensor(np.sort(rng.integers(0, b, (R, b)), axis=1), dtype=torch.int32, device="cuda")
        tok = torch.as_tensor(rng.integers(0, V, (R, b)), dtype=torch.int32, device="cuda")
        st.append(par, tok)
    q = torch.randn(R, b, a.hq, a.D, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    N = int(st.n_nodes.max().item())
    plan = _lib.trie_attn_plan_info(st.cfg, b, N)
    st.attn_decode(q, kp[0], vp[0], out, rows_hint=N)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(a.reps):
            st.attn_decode(q, kp[0], vp[0], out, rows_hint=N)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (5 * a.reps)
    tiles = (N + 63) // 64
    print(json.dumps(dict(R=R, b=b, Hq=a.hq, Hkv=a.hkv, D=a.D, N=N, tiles=tiles, plan=plan,
                          us=round(us, 2), us_per_tile=round(us / tiles, 3),
                          env={k: v for k, v in os.environ.items() if k.startswith("TRIE_")})))


if __name__ == "__main__":
    main()
