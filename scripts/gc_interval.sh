#!/bin/bash
# the GC interval g of Alg. 2 (Fig. 4 uses g = 15).
#   bash scripts/gc_interval.sh <tag> [workload]   -> gpurun_out/<tag>_gc<g>_<wl>.json
TAG=${1:-gc}; WL=${2:-llama}
mkdir -p gpurun_out
for g in 1 4 15 0; do
  timeout 600 python bench.py --workload $WL --gc-interval $g --no-cpu-baseline --no-e2e 2>gpurun_out/${TAG}_gc${g}_${WL}.err | tail -1 > gpurun_out/${TAG}_gc${g}_${WL}.json
done
