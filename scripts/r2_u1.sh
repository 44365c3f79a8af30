#!/bin/bash
# Qg = 64 / 128 (sweep b = 16 / 32): tcgen05 (default) vs the mma.sync wide kernel
# (TRIE_UMMA_MIN_QG above Qg), after round 2's softmax diet of the mma.sync kernels
TAG=${1:-r2u1}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
for rep in 1 2; do
  timeout 300 python bench.py --workload sweep --beam 16 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_b16_umma_$rep.json
  TRIE_UMMA_MIN_QG=65 timeout 300 python bench.py --workload sweep --beam 16 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_b16_wide_$rep.json
  timeout 300 python bench.py --workload sweep --beam 32 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_b32_umma_$rep.json
  TRIE_UMMA_MIN_QG=129 timeout 300 python bench.py --workload sweep --beam 32 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_b32_wide_$rep.json
done
