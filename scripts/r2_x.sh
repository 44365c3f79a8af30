#!/bin/bash
TAG=${1:-r2x}
mkdir -p gpurun_out
TRIE_BUILD_DEFINES="TRIE_UMMA_TRACE=1" python -m paper_2502_00085_b200.build --force > /dev/null 2>&1
for sk in 1 0; do echo "== SK $sk"; TRIE_UMMA_SK=$sk timeout 120 python scripts/umma_trace.py --beam 16 2>&1 | tail -12; done > gpurun_out/${TAG}_trace.txt 2>&1
python -m paper_2502_00085_b200.build --force > /dev/null 2>&1
