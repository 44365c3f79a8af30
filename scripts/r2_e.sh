#!/bin/bash
TAG=${1:-r2e}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
for cfg in "0 3" "1 2" "1 3" "0 3"; do
  set -- $cfg
  TRIE_ATTN_STREAMK=$1 TRIE_SK_STAGES=$2 timeout 600 python bench.py --workload llama --steps 32 --no-cpu-baseline --no-e2e 2>gpurun_out/${TAG}_llama_sk$1_st$2.err | tail -1 >> gpurun_out/${TAG}_llama_sk$1_st$2.json
done
TRIE_ATTN_STREAMK=1 timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py -q -x > gpurun_out/${TAG}_pytest_sk.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_sk.log
tail -n 2 gpurun_out/${TAG}_*.log
