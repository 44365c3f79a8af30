#!/bin/bash
# ncu --set full of the attention kernels (+ combine) in one bench workload (1 GPU).
#   bash scripts/ncu_attn.sh <tag> <workload> [extra bench args]
TAG=$1; WL=$2; shift 2
mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"k_attn" -s 300 -c 4 \
   -o gpurun_out/attn_${TAG}_${WL} -f python bench.py --workload $WL --steps 4 --warmup 3 --no-cpu-baseline --no-e2e "$@" \
   > gpurun_out/attn_${TAG}_${WL}.log 2>&1
