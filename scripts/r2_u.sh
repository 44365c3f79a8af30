#!/bin/bash
# adaptive split v2 (exact grid): parity + Llama A/B
TAG=${1:-r2u}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 1200 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fullsize.py tests/test_gpu_bf16_lockstep.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
  for ad in 1 0; do
    TRIE_ADAPTIVE_SPLIT=$ad timeout 300 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_llama_ad${ad}_$rep.json
  done
done
TRIE_BUILD_DEFINES="TRIE_ATTN_TRACE=1" python -m paper_2502_00085_b200.build --force > /dev/null 2>&1
timeout 300 python scripts/attn_trace.py --workload llama --step 128 > gpurun_out/${TAG}_trace_llama.txt 2>&1
tail -n 3 gpurun_out/${TAG}_pytest.log
