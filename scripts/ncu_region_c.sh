#!/bin/bash
# ncu --set full of the attention launches that bench.py's roofline times (region C: the
# step's L launches replayed after the timed steps), so roofline.traffic and
# roofline.achieved describe the same launch (same trie state).  One GPU.
#   bash scripts/ncu_region_c.sh <tag> <workload> [extra bench args]
TAG=$1; WL=$2; shift 2
STEPS=${STEPS:-64}; WARM=${WARM:-3}
mkdir -p gpurun_out
# attention launches before region C's graph replays: 2 eager warm-up steps, W warm-up and
# 2K timed step replays (regions A and B), one extra step if the job wrapped to k = 0, and
# region C's first (untimed) graph replay -- L launches each
SKIP=$(python - "$WL" "$STEPS" "$WARM" <<'EOF'
import sys
sys.path.insert(0, ".")
import bench
wl = bench.WORKLOADS[sys.argv[1]]
K, W = int(sys.argv[2]), int(sys.argv[3])
L, s = wl["L"], wl["s"]
k_end = (W + 2 * K) % s
print((2 + W + 2 * K + (1 if k_end == 0 else 0) + 1) * L)
EOF
)
echo "skip $SKIP attention launches" > gpurun_out/ncuc_${TAG}_${WL}.log
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
   -k regex:"k_attn_(narrow|wide|umma|v1)" -s $SKIP -c 2 \
   -o gpurun_out/ncuc_${TAG}_${WL} -f python bench.py --workload $WL --steps $STEPS --warmup $WARM \
   --no-cpu-baseline --no-e2e "$@" >> gpurun_out/ncuc_${TAG}_${WL}.log 2>&1
