#!/bin/bash
# ncu --set full of exactly the attention launches that bench.py's roofline times (region
# C: one replay of the step's L launches at the middle of the timed window), selected with
# cudaProfilerStart/Stop (BENCH_PROFILE_REGION_C=1, ncu --profile-from-start off), so
# roofline.traffic and roofline.achieved describe the same launches (same trie state).
# Also the launch list (gpu__time_duration.sum) of the same command.  One GPU.
#   bash scripts/ncu_region_c.sh <tag> <workload> [extra bench args]
TAG=$1; WL=$2; shift 2
STEPS=${STEPS:-20}; WARM=${WARM:-5}
mkdir -p gpurun_out
BENCH_PROFILE_REGION_C=1 /usr/local/cuda/bin/ncu --profile-from-start off --set full --clock-control none \
   --import-source on -k regex:"k_attn_(narrow|wide|umma|v1)" -c 2 \
   -o gpurun_out/ncuc_${TAG}_${WL} -f python bench.py --workload $WL --steps $STEPS --warmup $WARM \
   --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncuc_${TAG}_${WL}.log 2>&1
# launch list of the whole default command (cold, serialised: only shares are comparable)
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
   --log-file gpurun_out/launches_${TAG}_${WL}.csv python bench.py --workload $WL --steps $STEPS \
   --warmup $WARM --no-cpu-baseline --no-e2e "$@" > gpurun_out/launches_${TAG}_${WL}.log 2>&1
