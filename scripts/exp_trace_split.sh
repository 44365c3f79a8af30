TRIE_BUILD_DEFINES="TRIE_ATTN_TRACE=1" python -m paper_2502_00085_b200.build --force >/dev/null
python scripts/attn_trace.py --workload phi --step 30 > gpurun_out/trace44_phi_s1.txt 2>&1
TRIE_ATTN_SPLITS=2 python scripts/attn_trace.py --workload phi --step 30 > gpurun_out/trace44_phi_s2.txt 2>&1
python -m paper_2502_00085_b200.build --force >/dev/null
