timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t39.log 2>&1; tail -3 gpurun_out/t39.log
for sp in 1 2 3; do TRIE_ATTN_SPLITS=$sp timeout 300 python bench.py --workload phi --no-cpu-baseline --no-e2e --steps 32 2>/dev/null | tail -1 > gpurun_out/e39_phi_s$sp.json; done
for sp in 1 4 8; do TRIE_ATTN_SPLITS=$sp timeout 300 python bench.py --workload mistral-shard --no-cpu-baseline --no-e2e --steps 32 2>/dev/null | tail -1 > gpurun_out/e39_mis_s$sp.json; done
for sp in 1 4 8; do TRIE_ATTN_SPLITS=$sp timeout 300 python bench.py --workload sweep --beam 16 --no-cpu-baseline --no-e2e --steps 16 2>/dev/null | tail -1 > gpurun_out/e39_sw16_s$sp.json; done
