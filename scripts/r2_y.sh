#!/bin/bash
# re-entry baseline: GPU tests, default + llama bench, beam-step microbench, ncu (source)
# of the llama wide launch and the aux kernels
TAG=${1:-r2y}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_phi.json 2>gpurun_out/${TAG}_phi.err
timeout 600 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_llama.json 2>gpurun_out/${TAG}_llama.err
timeout 300 python scripts/bench_beam_step.py > gpurun_out/${TAG}_beam.json 2>&1
bash scripts/ncu_region_c.sh $TAG llama
bash scripts/ncu_aux.sh $TAG llama 2>/dev/null || true
ls gpurun_out | grep $TAG
