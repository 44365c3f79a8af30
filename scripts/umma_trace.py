"""Experiment: per-tile clock() trace of one tcgen05 attention CTA (trace build only).
    TRIE_BUILD_DEFINES="TRIE_UMMA_TRACE=1" python -m paper_2502_00085_b200.build --force
    python scripts/umma_trace.py --beam 16
Columns per tile: softmax warp 2 [wait start, s_full seen, full seen, P ready, p_full
arrived], MMA warp [QK issued, p_full seen], producer [empty seen, TMA issued]."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="sweep")
    ap.add_argument("--beam", type=int, default=16)
    a = ap.parse_args()
    from paper_2502_00085_b200 import _lib
    _lib.load()
    wl = dict(bench.WORKLOADS[a.workload])
    wl["b"] = a.beam
    hp = bench.HotPath(wl, 0, torch.device("cuda", 0))
    for i in range(8):
        hp.step_ops("first" if i == 0 else "steady", i % 2)
    torch.cuda.synchronize()
    d = hp.inp[("steady", 0)]
    for _ in range(3):  # warm, then the traced launch
        hp.st.attn_decode(d["views"][0][0], hp.kp[0], hp.vp[0], d["out"], rows_hint=hp.rows_hint)
    torch.cuda.synchronize()
    t = d["out"].view(-1).view(torch.int32)[: 400 * 16].cpu().numpy().astype(np.int64).reshape(400, 16)
    t = t - t[0, 0]
    n = 1
    while n < 400 and 0 < t[n, 4] - t[n - 1, 4] < 10 ** 6:  # the traced CTA's tiles only
        n += 1
    t = t[:n]
    np.set_printoptions(linewidth=200)
    print("tiles traced", n)
    print("   i  wait  sfull  full  Pready arrive | qk_iss pfull | empty tma_iss | ld  max  exp")
    for i in list(range(0, 12)) + list(range(n // 2, n // 2 + 12)):
        if i < n:
            print(f"{i:4d} " + " ".join(f"{x:7d}" for x in t[i]))
    dt = np.diff(t[:, 4])
    print("per-tile period (clk): median", np.median(dt), "mean", dt.mean())
    print("softmax wait s_full (clk) median", np.median(t[:, 1] - t[:, 0]),
          "wait full", np.median(t[:, 2] - t[:, 1]), "compute", np.median(t[:, 3] - t[:, 2]),
          "store+arrive", np.median(t[:, 4] - t[:, 3]))
    print("tma issue -> softmax sees full (latency) median", np.median(t[:, 2] - t[:, 8]))
    print("p_full arrive -> mma sees", np.median(t[:, 6] - t[:, 4]))
    print("compute split: S load", np.median(t[:, 9] - t[:, 2]), "mask+max+exchange", np.median(t[:, 10] - t[:, 9]),
          "rescale+exp+pack", np.median(t[:, 11] - t[:, 10]), "O rescale", np.median(t[:, 3] - t[:, 11]))
    print("V: issue -> PV warp sees fullV", np.median(t[:, 14] - t[:, 13]),
          "| p_full seen -> fullV seen", np.median(t[:, 14] - t[:, 6]),
          "| V issue lag behind K issue", np.median(t[:, 13] - t[:, 8]))
    print("K: issue -> QK issued", np.median(t[:, 5] - t[:, 8]))


if __name__ == "__main__":
    main()
