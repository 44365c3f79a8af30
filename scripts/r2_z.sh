#!/bin/bash
# wide kernel: lazy rescale (RS=2) vs RS=4 with Q staged in shared memory (112-reg cap)
TAG=${1:-r2z}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
for rs in 4 2; do
  TRIE_WIDE_RS=$rs timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/${TAG}_pytest_rs$rs.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_rs$rs.log
done
for rep in 1 2; do
for rs in 2 4; do
  TRIE_WIDE_RS=$rs timeout 300 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_llama_rs${rs}_$rep.json
  TRIE_WIDE_RS=$rs timeout 300 python bench.py --workload sweep --beam 8 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw8_rs${rs}_$rep.json
done
done
ls gpurun_out | grep $TAG
