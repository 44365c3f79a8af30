#!/bin/bash
# tcgen05 attention experiment round (under gpurun): parity tests, per-launch time at
# b = 16 / 32 (sweep shape) for V-ring depths, then a clock() trace build.
timeout 300 python -m pytest tests/test_gpu_attn.py tests/test_gpu_e2e_tiny.py -x -q 2>&1 | tail -3
for st in ${STS:-6 8 4}; do TRIE_UMMA_ST=$st SWS=x DBGS="0" bash scripts/umma_dbg.sh gpurun_out/dbg_st$st.txt; done
TRIE_BUILD_DEFINES="TRIE_UMMA_TRACE=1" python -m paper_2502_00085_b200.build --force > /dev/null
for b in 16 32; do echo "== b $b"; timeout 120 python scripts/umma_trace.py --beam $b | tail -8; done > gpurun_out/trace.txt 2>&1
python -m paper_2502_00085_b200.build --force > /dev/null
