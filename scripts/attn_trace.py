"""Experiment: per-CTA %globaltimer timeline of one narrow / wide attention launch
(trace build only).
    TRIE_BUILD_DEFINES="TRIE_ATTN_TRACE=1" python -m paper_2502_00085_b200.build --force
    python scripts/attn_trace.py --workload llama --step 131
Prints, over the launch's CTAs, the distribution (us, relative to the first CTA start) of:
start, setup done, first tile seen, last tile done, epilogue done, producer done."""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama")
    ap.add_argument("--step", type=int, default=131)
    ap.add_argument("--beam", type=int, default=0)
    ap.add_argument("--requests", type=int, default=0)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    from paper_2502_00085_b200 import _lib
    lib = _lib.load()
    fn = lib.trie_debug_attn_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    wl = dict(bench.WORKLOADS[a.workload])
    if a.beam:
        wl["b"] = a.beam
    if a.requests:
        wl["R"] = a.requests
    hp = bench.HotPath(wl, 0, torch.device("cuda", 0))
    hp.capture()
    for _ in range(a.step):
        hp.replay(0)
    torch.cuda.synchronize()
    st, d = hp.st, hp.inp[("steady", 0)]
    q, k, v = d["views"][0]
    n = hp.R * hp.Hkv * max(1, hp.plan["steady"]["splits"])
    buf = (ctypes.c_ulonglong * (8 * n))()
    for rep in range(3):
        if rep == 2:
            assert fn(buf, n) == 0  # clears the trace
        for l in (0, 1):  # the second launch runs right behind the first (PDL overlap)
            if hp.fused["steady"]:
                st.attn_decode_rope(q, k, v, hp.kp[l], hp.vp[l], wl["theta"], d["out"], rows_hint=hp.rows_hint)
            else:
                st.attn_decode(q, hp.kp[l], hp.vp[l], d["out"], rows_hint=hp.rows_hint)
        torch.cuda.synchronize()
    assert fn(buf, n) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(n, 8).astype(np.int64)
    keep = (t[:, 0] != 0) & (t[:, 4] != 0)  # CTAs that ran an item (idle ones exit early)
    cta_id = np.nonzero(keep)[0]
    t = t[keep]
    n = len(t)
    t0 = t[:, 0].min()
    names = ["start", "setup", "first_tile", "last_tile", "epilogue", "producer_done"]
    rel = {nm: (t[:, i] - t0) / 1e3 for i, nm in enumerate(names)}
    print(json.dumps({"workload": wl["name"], "step": a.step, "ctas": n, "plan": hp.plan["steady"],
                      "N": hp.st.n_nodes.cpu().tolist()[:8]}))
    for nm in names:
        x = rel[nm]
        print(f"{nm:14s} min {x.min():7.2f} p10 {np.percentile(x, 10):7.2f} p50 {np.median(x):7.2f} "
              f"p90 {np.percentile(x, 90):7.2f} max {x.max():7.2f} us")
    dur = {"setup-start": rel["setup"] - rel["start"], "first-setup": rel["first_tile"] - rel["setup"],
           "tiles": rel["last_tile"] - rel["first_tile"], "epi": rel["epilogue"] - rel["last_tile"],
           "cta": rel["epilogue"] - rel["start"]}
    for nm, x in dur.items():
        print(f"{nm:14s} p10 {np.percentile(x, 10):7.2f} p50 {np.median(x):7.2f} p90 {np.percentile(x, 90):7.2f} us")
    ntl = t[:, 7]
    print("tiles per CTA: min", ntl.min(), "median", np.median(ntl), "max", ntl.max(),
          "| per-tile p50 us", np.median(dur["tiles"] / np.maximum(ntl - 1, 1)))
    sm = t[:, 6]
    print("CTAs per SM: max", np.bincount(sm).max(), "SMs used", len(np.unique(sm)))
    # per-SM load: tiles of the SM's CTAs vs when its last CTA finished; CTA -> SM placement
    sms = np.unique(sm)
    load = np.array([ntl[sm == x].sum() for x in sms])
    fin = np.array([rel["epilogue"][sm == x].max() for x in sms])
    cnt = np.array([(sm == x).sum() for x in sms])
    print("per-SM tiles: min", load.min(), "median", np.median(load), "max", load.max(),
          "| corr(tiles, finish)", round(float(np.corrcoef(load, fin)[0, 1]), 3))
    for c in (1, 2, 3, 4):
        if (cnt == c).any():
            print(f"  SMs with {c} CTA(s): {int((cnt == c).sum())}, tiles median {np.median(load[cnt == c]):.1f},"
                  f" finish median {np.median(fin[cnt == c]):.2f} us")
    gaps = [int(np.diff(np.sort(cta_id[sm == x]))[0]) for x in sms if (sm == x).sum() == 2]
    if gaps:
        u, c = np.unique(gaps, return_counts=True)
        top = np.argsort(-c)[:5]
        print("  CTA-index gap between the two CTAs of an SM (top):", [(int(u[i]), int(c[i])) for i in top])
    per_tile = dur["tiles"] / np.maximum(ntl - 1, 1)
    shared = np.array([cnt[np.searchsorted(sms, x)] for x in sm])
    for c in (1, 2):
        if (shared == c).any():
            print(f"  per-tile us on SMs with {c} CTA(s): median {np.median(per_tile[shared == c]):.2f}")
    # occupancy over time: CTAs resident (start..epilogue) and streaming (first..last tile)
    end = rel["epilogue"].max()
    bins = np.linspace(0, end, 21)
    res = [int(((rel["start"] <= b) & (rel["epilogue"] > b)).sum()) for b in bins[:-1]]
    stream = [int(((rel["first_tile"] <= b) & (rel["last_tile"] > b)).sum()) for b in bins[:-1]]
    print("t(us)    ", " ".join(f"{b:5.0f}" for b in bins[:-1]))
    print("resident ", " ".join(f"{x:5d}" for x in res))
    print("streaming", " ".join(f"{x:5d}" for x in stream))
    if a.out:
        np.save(a.out, t)


if __name__ == "__main__":
    main()
