#!/bin/bash
# NEXT-4 fused all-gather: two-rank one-GPU parity (host vs fused), bench at N = 2, all GPU
# tests (the epilogue changes touch every attention kernel), synccheck/memcheck of the kv-shard test
TAG=${1:-r2h}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 900 python -m pytest tests/test_gpu_kv_shard.py -q -x > gpurun_out/${TAG}_kvshard.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_kvshard.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for wl in phi llama mistral-shard; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${wl}.json 2>gpurun_out/${TAG}_${wl}.err
done
tail -n 3 gpurun_out/${TAG}_*.log
