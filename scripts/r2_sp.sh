#!/bin/bash
# split count for the one-m-tile kernel (Mistral shard, sweep b=4): plan (2) vs forced 3 / 4
TAG=${1:-r2sp}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
for rep in 1 2; do
for sp in 0 3 4; do
  if [ $sp = 0 ]; then unset TRIE_ATTN_SPLITS; else export TRIE_ATTN_SPLITS=$sp; fi
  timeout 300 python bench.py --workload mistral-shard --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_mis_s${sp}_$rep.json
  timeout 300 python bench.py --workload sweep --beam 4 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw4_s${sp}_$rep.json
done
done
unset TRIE_ATTN_SPLITS
