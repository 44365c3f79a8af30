#!/bin/bash
# BASELINE.json configs[4]: beam-width sweep at t = 8192 on the Llama-3.1-8B shape.
# bash scripts/sweep.sh <tag>   (under gpurun) -> gpurun_out/sweep_<tag>_b<b>.json
TAG=${1:-r02}
for b in 2 4 8 16 32; do
  python bench.py --workload sweep --beam $b --steps 16 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/sweep_${TAG}_b${b}.json
done
