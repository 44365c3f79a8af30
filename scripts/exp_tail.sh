timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fullsize.py tests/test_gpu_e2e_tiny.py -x -q > gpurun_out/t45.log 2>&1; tail -3 gpurun_out/t45.log
for i in 1 2; do
timeout 300 python bench.py --workload phi --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e45_phi_tail_$i.json
TRIE_TAIL_SPLIT=0 timeout 300 python bench.py --workload phi --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e45_phi_notail_$i.json
done
TRIE_BUILD_DEFINES="TRIE_ATTN_TRACE=1" python -m paper_2502_00085_b200.build --force >/dev/null
python scripts/attn_trace.py --workload phi --step 30 > gpurun_out/trace45_phi.txt 2>&1
python -m paper_2502_00085_b200.build --force >/dev/null
