#!/bin/bash
TAG=${1:-r2b}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
nproc > gpurun_out/${TAG}_host.txt; lscpu >> gpurun_out/${TAG}_host.txt
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2>gpurun_out/${TAG}_ref.err
timeout 900 python bench.py --impl reference --units > gpurun_out/${TAG}_units.json 2>gpurun_out/${TAG}_units.err
bash scripts/sanitize.sh $TAG
tail -n 3 gpurun_out/${TAG}_pytest.log
