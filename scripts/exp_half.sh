timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t47.log 2>&1; tail -3 gpurun_out/t47.log
for i in 1 2; do for v in 1 0; do
TRIE_HALF_TILE=$v timeout 300 python bench.py --workload phi --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e47_phi_h${v}_$i.json
TRIE_HALF_TILE=$v timeout 300 python bench.py --workload llama --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e47_llama_h${v}_$i.json
done; done
