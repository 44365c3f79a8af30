#!/bin/bash
# re-validation after the one-m-tile kernel's software pipeline: GPU tests + smoke, the
# driver's default bench, the BASELINE workloads and the sweep
TAG=${1:-r2f6}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2>gpurun_out/${TAG}_bench.err
for wl in llama mistral-shard; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_$wl.json 2>gpurun_out/${TAG}_$wl.err
done
for b in 2 4 8 16 32; do
  timeout 300 python bench.py --workload sweep --beam $b --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sweep_b$b.json
done
tail -n 2 gpurun_out/${TAG}_pytest.log gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2>gpurun_out/${TAG}_ref.err
timeout 600 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --paged 0 > gpurun_out/${TAG}_llama_dense.json 2>/dev/null
timeout 600 python bench.py --impl batch --workload llama --steps 20 --warmup 5 > gpurun_out/${TAG}_batch_llama.json 2>/dev/null
timeout 600 python bench.py --impl batch --workload phi --steps 20 --warmup 5 > gpurun_out/${TAG}_batch_phi.json 2>/dev/null
bash scripts/ncu_region_c.sh $TAG phi
ls gpurun_out | grep $TAG; du -sh gpurun_out
