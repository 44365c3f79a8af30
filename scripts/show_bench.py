"""Print the key numbers of bench JSON lines: python scripts/show_bench.py gpurun_out/<tag>_bench_*.json"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    r = d.get("roofline", {})
    e2e = d.get("e2e") or {}
    print(f"{f.split('/')[-1]:40s} value {d['value']:>10.1f} ms/step {d['ms_per_step']:.3f} attn {r.get('achieved')} GB/s "
          f"frac {r.get('frac')} launch {r.get('avg_launch_us')} us share {r.get('attn_share_of_step')} "
          f"path {d['config'].get('attention', {}).get('path')} e2e {e2e.get('value')} "
          f"kv {d.get('kv_memory', {}).get('ratio_batch_over_trie')}")
