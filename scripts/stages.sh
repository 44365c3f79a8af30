#!/bin/bash
# stage-count experiment for the narrow kernel on the sweep shape (b = 2, 4) and Phi
for st in 2 3 4; do
  for b in 2 4; do
    TRIE_NARROW_STAGES=$st python bench.py --workload sweep --beam $b --steps 16 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/st${st}_b${b}.json
  done
  TRIE_NARROW_STAGES=$st python bench.py --steps 32 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/st${st}_phi.json
done
