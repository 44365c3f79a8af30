for st in 2 3 4; do
  TRIE_NARROW_STAGES=$st timeout 300 python bench.py --workload phi --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e73_phi_st$st.json
done
