#!/bin/bash
# Launch list (ncu gpu__time_duration, cold-cache serialised) for several workloads.
#   bash scripts/launches.sh <tag> "<bench args 1>" "<bench args 2>" ...
TAG=$1; shift
mkdir -p gpurun_out
i=0
for a in "$@"; do
  /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_|trie" -c 400 --csv \
     --log-file gpurun_out/launches_${TAG}_${i}.csv python bench.py $a --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
     > gpurun_out/launches_${TAG}_${i}.log 2>&1
  echo "$a" > gpurun_out/launches_${TAG}_${i}.args
  i=$((i+1))
done
