#!/bin/bash
# round-2 final validation: GPU tests, smoke, the driver's bench commands, all workloads,
# sanitizers, ncu region C of the default workload
TAG=${1:-r2f3}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2>gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2>gpurun_out/${TAG}_ref.err
for wl in llama mistral-shard; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_$wl.json 2>gpurun_out/${TAG}_$wl.err
done
timeout 600 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --paged 0 > gpurun_out/${TAG}_llama_dense.json 2>/dev/null
for b in 2 4 8 16 32; do
  timeout 300 python bench.py --workload sweep --beam $b --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sweep_b$b.json
done
timeout 600 python bench.py --impl batch --workload llama --steps 20 --warmup 5 > gpurun_out/${TAG}_batch_llama.json 2>/dev/null
timeout 600 python bench.py --impl batch --workload phi --steps 20 --warmup 5 > gpurun_out/${TAG}_batch_phi.json 2>/dev/null
# compute-sanitizer is closed on the GPU pool (r2f3): sanitize.sh no longer run
bash scripts/ncu_region_c.sh $TAG phi
tail -n 2 gpurun_out/${TAG}_pytest.log gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests/test_gpu_graph_replay.py -m gpu -q > gpurun_out/${TAG}_graph.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_graph.log
ls gpurun_out | grep $TAG; du -sh gpurun_out
