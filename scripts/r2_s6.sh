#!/bin/bash
# beam step: L2 bulk prefetch of the chunk one wave ahead (TRIE_BEAM_L2_AHEAD sweep)
TAG=${1:-r2s6}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 600 python -m pytest tests/test_gpu_beam_step.py tests/test_gpu_integer_path.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for a in 0 592 1184 296 2368; do
  TRIE_BEAM_L2_AHEAD=$a timeout 300 python scripts/bench_beam_step.py > gpurun_out/${TAG}_beam_a$a.json 2>&1
done
for a in 0 592; do
  TRIE_BEAM_L2_AHEAD=$a timeout 300 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_llama_a$a.json
done
tail -2 gpurun_out/${TAG}_pytest.log; for f in gpurun_out/${TAG}_beam_a*.json; do echo $f; cat $f; done
