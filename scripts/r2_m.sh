#!/bin/bash
# current numbers: beam sweep (tcgen05), ncu region C captures + launch lists, aux kernels
TAG=${1:-r2m}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
for b in 2 4 8 16 32; do
  timeout 300 python bench.py --workload sweep --beam $b --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sweep_b$b.json
done
for wl in phi llama mistral-shard; do bash scripts/ncu_region_c.sh $TAG $wl; done
STEPS=16 WARM=3 bash scripts/ncu_region_c.sh $TAG sweep --beam 16
bash scripts/ncu_aux.sh $TAG llama 2>/dev/null || true
ls gpurun_out | grep $TAG
