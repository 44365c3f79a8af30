#!/bin/bash
# All bench workloads, one JSON line each -> gpurun_out/<tag>_bench_<wl>.json
TAG=${1:-r}
mkdir -p gpurun_out
for wl in phi llama mistral-shard; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline 2>gpurun_out/${TAG}_bench_${wl}.err | tail -1 > gpurun_out/${TAG}_bench_${wl}.json
done
for b in 2 4 8 16 32; do
  timeout 300 python bench.py --workload sweep --beam $b --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_bench_sweep_b${b}.json
done
