#!/bin/bash
# A/B: round-1 build (wt_r1, its own bench) vs HEAD on mistral-shard and sweep b=16 (tcgen05 path)
TAG=${1:-r2i}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
for rep in 1 2; do
  (cd wt_r1 && timeout 600 python bench.py --workload mistral-shard --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1) > gpurun_out/${TAG}_old_mis_$rep.json
  timeout 600 python bench.py --workload mistral-shard --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_new_mis_$rep.json
  (cd wt_r1 && timeout 600 python bench.py --workload sweep --beam 16 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1) > gpurun_out/${TAG}_old_sw16_$rep.json
  timeout 600 python bench.py --workload sweep --beam 16 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_new_sw16_$rep.json
done
