"""Experiment: in-step cost of trie_prune_compact at a BASELINE shape, without event nodes.
Two CUDA graphs of REPS steady steps each -- [beam_step] x REPS and [beam_step + prune_compact]
x REPS -- replayed on identical mid-job tries (two handles, same random logits); the time
difference per step is the GC's cost inside the step sequence (PDL-chained launches).
    python scripts/gc_cost.py [llama|phi]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2502_00085_b200 import _lib  # noqa: E402
from paper_2502_00085_b200.build import build  # noqa: E402
from paper_2502_00085_b200.trie import TrieState  # noqa: E402

REPS, WARM = 16, 64


def main():
    build()
    _lib.load()
    name = sys.argv[1] if len(sys.argv) > 1 else "llama"
    wl = dict(bench.WORKLOADS[name])
    R, b, t, L, Hq, Hkv, D, V = (wl[k] for k in ("R", "b", "t", "L", "Hq", "Hkv", "D", "V"))
    cap = (t + b * (WARM + 3 * REPS + 4) + 63) // 64 * 64
    prompts, lens = synth.prompts(7, R, t, V)
    g = torch.Generator(device="cuda").manual_seed(3)
    logits = [torch.randn(R, b, V, device="cuda", generator=g) * 3.0 for _ in range(4)]
    first = torch.randn(R, 1, V, device="cuda", generator=g) * 3.0
    res = {"workload": name, "R": R, "b": b, "L": L, "cap": cap}
    times = {}
    for gc in (False, True):
        st = TrieState(R, b, t, cap, L, Hq, Hkv, D, V, prompts, lens, dtype=torch.bfloat16)
        kp, vp = st.new_pools()
        st.beam_step(first)
        for i in range(WARM):  # mid-job trie with GC every step
            st.beam_step(logits[i % 4])
            st.prune_compact(kp, vp)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for i in range(REPS):
                st.beam_step(logits[i % 4])
                if gc:
                    st.prune_compact(kp, vp)
        gr.replay()  # warm
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        times[gc] = e0.elapsed_time(e1) * 1e3 / REPS
        res["rows_mean" + ("_gc" if gc else "_nogc")] = float(st.n_nodes.float().mean())
        assert st.status() == 0
        del st, kp, vp
        torch.cuda.empty_cache()
    res["beam_step_us"] = round(times[False], 2)
    res["beam_step_plus_gc_us"] = round(times[True], 2)
    res["gc_us"] = round(times[True] - times[False], 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
