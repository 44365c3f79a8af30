#!/bin/bash
# beam step: rank counting in shared memory for the chunk / row / request top-b (vs the
# bitonic shuffle sort / merge trees): parity + microbench + llama / phi bench
TAG=${1:-r2s5}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 900 python -m pytest tests/test_gpu_beam_step.py tests/test_gpu_integer_path.py tests/test_gpu_e2e_tiny.py tests/test_gpu_bf16_lockstep.py tests/test_gpu_batch_baseline.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python scripts/bench_beam_step.py > gpurun_out/${TAG}_beam.json 2>&1
timeout 300 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_llama.json
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_phi.json
tail -3 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_beam.json
