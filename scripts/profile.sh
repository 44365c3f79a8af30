#!/bin/bash
# Profiling recipe (B200_PROFILING.md) for the bench workload; run under gpurun.
#   bash scripts/profile.sh <tag> [bench args...]
set -u
TAG=${1:-r01}; shift || true
ARGS=${@:---steps 4 --warmup 3 --no-cpu-baseline --no-e2e}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
# 1) every launch with its device time (cold-cache, serialised: compare shares)
$NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_|trie" -c 600 --csv \
     --log-file gpurun_out/launches_${TAG}.csv python bench.py $ARGS > gpurun_out/launches_${TAG}.log 2>&1
# 2) one full capture of the dominant kernel
$NCU --set full --clock-control none --import-source on -k regex:k_attn -s 200 -c 2 \
     -o gpurun_out/attn_${TAG} -f python bench.py $ARGS > gpurun_out/attn_${TAG}.log 2>&1
# 3) beam-step and prune kernels, one capture each
$NCU --set full --clock-control none -k regex:"k_beam_step|k_prune_scan|k_kv_compact|k_rope" -s 20 -c 5 \
     -o gpurun_out/aux_${TAG} -f python bench.py $ARGS > gpurun_out/aux_${TAG}.log 2>&1
ls -la gpurun_out/
