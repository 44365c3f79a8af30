#!/bin/bash
# ncu --set full of the non-attention hot-path kernels (beam step, GC scan / compaction,
# RoPE table) in one bench workload, steady steps (one GPU).
#   bash scripts/ncu_aux.sh <tag> <workload>
TAG=$1; WL=$2; shift 2
mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --set full --clock-control none -k regex:"k_beam_step|k_prune_scan|k_kv_compact|k_rope_table" \
   -s 40 -c 4 -o gpurun_out/aux_${TAG}_${WL} -f python bench.py --workload $WL --steps 8 --warmup 3 \
   --no-cpu-baseline --no-e2e "$@" > gpurun_out/aux_${TAG}_${WL}.log 2>&1
