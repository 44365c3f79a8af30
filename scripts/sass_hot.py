"""Summarise an ncu --page source --print-source sass CSV: instructions executed and stall
samples per SASS line, top N, plus totals by opcode.
    ncu -i rep --page source --csv --print-source sass > x.csv; python scripts/sass_hot.py x.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iex, ist = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for k, r in enumerate(rows[2:]):
    if len(r) < len(hdr) or not r[iex].strip().isdigit():
        continue
    data.append((k, r[isrc].strip(), int(r[iex]), int(r[ist] or 0)))
tot_i = sum(d[2] for d in data) or 1
tot_s = sum(d[3] for d in data) or 1
print(f"total inst {tot_i}, stall samples {tot_s}")
op = collections.Counter()
ops = collections.Counter()
for k, src, ex, stl in data:
    o = src.split()[0] if not src.startswith("@") else src.split()[1]
    op[o.split(".")[0]] += ex
    ops[o.split(".")[0]] += stl
print("by opcode (inst%, stall%):", ", ".join(f"{o} {100*v/tot_i:.1f}/{100*ops[o]/tot_s:.1f}" for o, v in op.most_common(20)))
print("top lines by stall samples:")
for k, src, ex, stl in sorted(data, key=lambda d: -d[3])[:N]:
    print(f"{k:5d} {100*stl/tot_s:5.1f}% stall {100*ex/tot_i:5.1f}% inst  {src[:90]}")
