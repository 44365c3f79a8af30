#!/bin/bash
# Round-2 validation: GPU tests, smoke, driver-style default bench + reference arm, Llama,
# NEXT-1 experiments (--series): tab:ablation (Phi b=3 t=150, GC every step vs never) and
# Fig. 4 (Llama b=30, 1,000 tokens, GC every 15 steps).
TAG=${1:-r2f}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2>gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2>gpurun_out/${TAG}_ref.err
timeout 600 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_llama.json 2>gpurun_out/${TAG}_llama.err
for g in 1 0; do
  timeout 900 python bench.py --workload phi --beam 3 --prompt-len 150 --new-tokens 256 --gc-interval $g --steps 16 --series \
     --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ablation_g$g.json 2>gpurun_out/${TAG}_ablation_g$g.err
done
timeout 1500 python bench.py --workload llama --beam 30 --new-tokens 1000 --requests 4 --gc-interval 15 --steps 16 --series \
   --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_fig4.json 2>gpurun_out/${TAG}_fig4.err
tail -n 2 gpurun_out/${TAG}_*.log; tail -n 3 gpurun_out/${TAG}_*.err
