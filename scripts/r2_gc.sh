#!/bin/bash
# in-step GC cost without event nodes (scripts/gc_cost.py) + model-context refresh
TAG=${1:-r2gc}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
for wl in llama phi; do timeout 600 python scripts/gc_cost.py $wl >> gpurun_out/${TAG}_gc.jsonl 2>&1; done
for wl in phi llama mistral-shard; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --model-context 2>/dev/null | tail -1 > gpurun_out/${TAG}_mc_$wl.json
done
cat gpurun_out/${TAG}_gc.jsonl
