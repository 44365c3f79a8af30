timeout 300 python bench.py --workload mistral-shard --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e56_mis_umma.json
TRIE_UMMA_MIN_QG=17 timeout 300 python bench.py --workload mistral-shard --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e56_mis_narrow.json
TRIE_UMMA_MIN_QG=17 timeout 300 python bench.py --workload sweep --beam 4 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e56_sw4_narrow.json
timeout 300 python bench.py --workload sweep --beam 4 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e56_sw4_umma.json
