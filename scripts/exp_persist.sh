for sp in 0 2 3 4; do
  if [ $sp = 0 ]; then unset TRIE_ATTN_SPLITS; else export TRIE_ATTN_SPLITS=$sp; fi
  TRIE_ATTN_PERSIST=1 timeout 300 python bench.py --workload phi --no-cpu-baseline --no-e2e --steps 32 2>gpurun_out/e42_phi_p$sp.err | tail -1 > gpurun_out/e42_phi_p$sp.json
done
unset TRIE_ATTN_SPLITS
timeout 300 python bench.py --workload phi --no-cpu-baseline --no-e2e --steps 32 2>/dev/null | tail -1 > gpurun_out/e42_phi_base.json
TRIE_ATTN_PERSIST=1 timeout 300 python bench.py --workload llama --no-cpu-baseline --no-e2e --steps 32 2>/dev/null | tail -1 > gpurun_out/e42_llama_p0.json
TRIE_ATTN_PERSIST=1 TRIE_ATTN_SPLITS=2 timeout 300 python bench.py --workload llama --no-cpu-baseline --no-e2e --steps 32 2>/dev/null | tail -1 > gpurun_out/e42_llama_p2.json
timeout 300 python bench.py --workload llama --no-cpu-baseline --no-e2e --steps 32 2>/dev/null | tail -1 > gpurun_out/e42_llama_base.json
