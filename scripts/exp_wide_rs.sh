for rs in 2 1 4; do
  TRIE_WIDE_RS=$rs timeout 300 python bench.py --workload llama --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e71_llama_rs$rs.json
done
