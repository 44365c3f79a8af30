#!/bin/bash
# Llama launch trace after the softmax diet (trace build)
TAG=${1:-r2t2}
mkdir -p gpurun_out
TRIE_BUILD_DEFINES="TRIE_ATTN_TRACE=1" python -m paper_2502_00085_b200.build --force > /dev/null 2>&1
for st in 40 128 200; do timeout 300 python scripts/attn_trace.py --workload llama --step $st; done > gpurun_out/${TAG}_trace_llama.txt 2>&1
timeout 300 python scripts/attn_trace.py --workload phi --step 32 > gpurun_out/${TAG}_trace_phi.txt 2>&1
python -m paper_2502_00085_b200.build --force > /dev/null 2>&1
