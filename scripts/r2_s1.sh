#!/bin/bash
# isolated per-CTA streaming rate of the attention kernels (scripts/attn_single.py)
TAG=${1:-r2s1}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
O=gpurun_out/${TAG}_single.jsonl; : > $O
for st in 100 400; do
for rs in 2 4 1; do
  TRIE_WIDE_RS=$rs timeout 120 python scripts/attn_single.py --R 1 --hq 4 --hkv 1 --b 8 --steps $st >> $O 2>&1
done
timeout 120 python scripts/attn_single.py --R 1 --hq 4 --hkv 1 --b 4 --steps $st >> $O 2>&1
TRIE_WIDE1_MIN_QG=16 timeout 120 python scripts/attn_single.py --R 1 --hq 4 --hkv 1 --b 4 --steps $st >> $O 2>&1
timeout 120 python scripts/attn_single.py --R 1 --hq 1 --hkv 1 --b 4 --D 96 --steps $st >> $O 2>&1
timeout 120 python scripts/attn_single.py --R 1 --hq 32 --hkv 8 --b 8 --steps $st >> $O 2>&1
timeout 120 python scripts/attn_single.py --R 32 --hq 32 --hkv 8 --b 8 --steps $st >> $O 2>&1
timeout 120 python scripts/attn_single.py --R 16 --hq 32 --hkv 8 --b 4 --steps $st >> $O 2>&1
done
cat $O
