"""Summarise ncu captures (run here, on the CPU box) into profiles/.

    python scripts/ncu_summary.py <tag> <workload> <launches.csv> <attn.ncu-rep> [aux.ncu-rep]
        [--requests R --beam b]   (recorded with the dram bytes; bench.py uses them only
                                   for the same workload, requests and beam width)

Writes profiles/<tag>_<workload>_launches.md (per-kernel share of the step from the
gpu__time_duration launch list), profiles/<tag>_<workload>_ncu.md (key --set full metrics
per captured kernel) and merges dram bytes per attention launch into
profiles/ncu_attn_summary.json (read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__inst_executed.sum", "launch__occupancy_limit_shared_mem"]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], rows[i + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in data:
        v = float(r[vi])
        if r[ui] == "usecond":
            v *= 1000
        elif r[ui] == "msecond":
            v *= 1e6
        agg[r[ki].split("(")[0][:70]].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean (us) | share of captured launches |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1000:.2f} | {100 * sum(v) / tot:.1f}% |")
    return "\n".join(out), agg


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?")
        m = {k: (d.get(k), units[hdr.index(k)] if k in hdr else "") for k in KEYS if k in hdr}
        out.append((name, m))
    return out


def to_bytes(v, u):
    v = float(v)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    argv = list(sys.argv[1:])
    opts = {}
    for key in ("--requests", "--beam"):
        if key in argv:
            i = argv.index(key)
            opts[key[2:]] = int(argv[i + 1])
            del argv[i:i + 2]
    tag, wl, lcsv, attn = argv[:4]
    aux = argv[4] if len(argv) > 4 else None
    os.makedirs(PROF, exist_ok=True)
    table = launches(lcsv)[0] if lcsv != "-" else None
    if table is not None:
        with open(os.path.join(PROF, f"{tag}_{wl}_launches.md"), "w") as f:
            f.write(f"# {tag} {wl}: launch list (ncu --metrics gpu__time_duration.sum --clock-control none)\n\n")
            f.write("Cold-cache, serialised per-launch times (compare shares, not absolutes).\n\n" + table + "\n")
    lines = [f"# {tag} {wl}: ncu --set full captures\n"]
    dram = []
    for rep in [attn] + ([aux] if aux else []):
        for name, m in raw(rep):
            lines.append(f"\n## `{name[:110]}`\n\n| metric | value |\n|---|---|")
            for k, (v, u) in m.items():
                lines.append(f"| {k} | {v} {u} |")
            if "attn" in name and "dram__bytes_read.sum" in m:
                rb = to_bytes(*m["dram__bytes_read.sum"])
                wb = to_bytes(*m["dram__bytes_write.sum"])
                dram.append(rb + wb)
    with open(os.path.join(PROF, f"{tag}_{wl}_ncu.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    js = os.path.join(PROF, "ncu_attn_summary.json")
    d = json.load(open(js)) if os.path.exists(js) else {}
    if dram:
        d[wl] = {"tag": tag, "dram_bytes_per_launch": sum(dram) / len(dram), "captures": len(dram), **opts}
    json.dump(d, open(js, "w"), indent=1)
    print("wrote", tag, wl, "attn dram/launch", d.get(wl))


if __name__ == "__main__":
    main()
