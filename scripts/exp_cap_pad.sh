# (the TRIE_BENCH_CAP_PAD knob was removed after this experiment; results in profiles/r08_experiments/e70_*)
for pad in 0 4 8 12 36; do
  TRIE_BENCH_CAP_PAD=$pad timeout 300 python bench.py --workload phi --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e70_phi_pad$pad.json
done
for pad in 0 8; do
  TRIE_BENCH_CAP_PAD=$pad timeout 300 python bench.py --workload llama --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e70_llama_pad$pad.json
done
