#!/bin/bash
# tcgen05 investigation: narrow vs tcgen05 at Qg=16 (mid-job), then per-tile clock() traces
TAG=${1:-r2n}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
for mq in 17 -1; do
  TRIE_UMMA_MIN_QG=$mq timeout 300 python bench.py --workload sweep --beam 4 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw4_mq$mq.json
  TRIE_UMMA_MIN_QG=$mq timeout 300 python bench.py --workload mistral-shard --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_mis_mq$mq.json
done
TRIE_BUILD_DEFINES="TRIE_UMMA_TRACE=1" python -m paper_2502_00085_b200.build --force > /dev/null 2>&1
for b in 4 16 32; do echo "== sweep b $b"; timeout 120 python scripts/umma_trace.py --beam $b 2>&1 | tail -22; done > gpurun_out/${TAG}_trace.txt 2>&1
echo "== mistral" >> gpurun_out/${TAG}_trace.txt; timeout 120 python scripts/umma_trace.py --workload mistral-shard --beam 4 2>&1 | tail -22 >> gpurun_out/${TAG}_trace.txt
