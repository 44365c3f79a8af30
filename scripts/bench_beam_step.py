"""Experiment: trie_beam_step alone (steady state, b live beams) at the bench shapes.
Times a CUDA graph of REPS back-to-back beam steps (the trie is reset between graphs;
capacity covers REPS appends) and reports us per launch and GB/s over the fp32 logits.
    python scripts/bench_beam_step.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_00085_b200 import _lib  # noqa: E402
from paper_2502_00085_b200.build import build  # noqa: E402
from paper_2502_00085_b200.trie import TrieState  # noqa: E402
import synth  # noqa: E402

SHAPES = [("phi", 64, 4, 32064), ("llama", 32, 8, 128256), ("sweep-b16", 16, 16, 128256),
          ("sweep-b32", 16, 32, 128256), ("mistral", 16, 4, 131072)]
REPS = 16


def main():
    build()
    _lib.load()
    out = {}
    only = sys.argv[1:]
    for name, R, b, V in SHAPES:
        if only and name not in only:
            continue
        t = 8
        prompts, lens = synth.prompts(1, R, t, V)
        st = TrieState(R, b, t, t + b * (REPS + 2) + 64, 0, 1, 1, 16, V, prompts, lens,
                       dtype=torch.float32)
        # distinct logits buffers per step: > L2 in total for the big shapes
        lg = [torch.randn(R, b, V, device="cuda") * 3.0 for _ in range(4)]
        st.beam_step(torch.randn(R, 1, V, device="cuda"))  # first step: b live beams after
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(REPS):
                st.beam_step(lg[i % 4])
        ts = []
        for _ in range(5):
            st.reset()
            st.beam_step(torch.randn(R, 1, V, device="cuda"))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / REPS * 1e3)
        us = sorted(ts)[len(ts) // 2]
        out[name] = dict(R=R, b=b, V=V, us=round(us, 2), GBps=round(R * b * V * 4 / us / 1e3, 1),
                         status=st.status())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
