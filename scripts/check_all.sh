#!/bin/bash
# Round check under gpurun: GPU tests, smoke, default bench, beam sweep.
#   bash scripts/check_all.sh <tag>
TAG=${1:-chk}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
for b in 2 4 8 16 32; do
  timeout 300 python bench.py --workload sweep --beam $b --steps 16 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/${TAG}_sweep_b${b}.json
done
tail -n 3 gpurun_out/${TAG}_*.log
