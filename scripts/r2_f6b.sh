#!/bin/bash
# round-2 final ncu captures (second call of r2f6: the reps exceed one call's
# 64 MiB gpurun_out): region C of mistral-shard and llama + the aux kernels on llama
TAG=${1:-r2f6}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
bash scripts/ncu_region_c.sh $TAG mistral-shard
bash scripts/ncu_region_c.sh $TAG llama
bash scripts/ncu_aux.sh $TAG llama 2>/dev/null || true
ls gpurun_out | grep $TAG; du -sh gpurun_out
