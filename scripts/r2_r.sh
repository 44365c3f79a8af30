#!/bin/bash
# which kernel for Qg = 16 / 32 mid-job: tcgen05 (default rule) vs mma.sync narrow / wide
TAG=${1:-r2r}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
for rep in 1 2; do
  for mq in -1 33; do
    for b in 4 8; do
      TRIE_UMMA_MIN_QG=$mq timeout 300 python bench.py --workload sweep --beam $b --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_mq${mq}_b${b}_$rep.json
    done
    TRIE_UMMA_MIN_QG=$mq timeout 300 python bench.py --workload mistral-shard --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_mq${mq}_mis_$rep.json
  done
done
timeout 900 python bench.py --impl reference --units > gpurun_out/${TAG}_units.json 2>gpurun_out/${TAG}_units.err
