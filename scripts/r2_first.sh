#!/bin/bash
# Round-2 first GPU check: full GPU tests, smoke, llama with/without stream-K, phi default.
TAG=${1:-r2a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
for sk in 1 0; do
  TRIE_ATTN_STREAMK=$sk timeout 600 python bench.py --workload llama --no-cpu-baseline --no-e2e 2>gpurun_out/${TAG}_llama_sk${sk}.err | tail -1 > gpurun_out/${TAG}_llama_sk${sk}.json
done
timeout 600 python bench.py --workload phi --no-cpu-baseline --no-e2e 2>gpurun_out/${TAG}_phi.err | tail -1 > gpurun_out/${TAG}_phi.json
tail -n 3 gpurun_out/${TAG}_*.log
