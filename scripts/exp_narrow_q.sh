for i in 1 2; do for v in base nq; do
  if [ $v = base ]; then unset TRIE_LIB; else export TRIE_LIB=$PWD/paper_2502_00085_b200/libtriedecode_nq.so; fi
  timeout 300 python bench.py --workload phi --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e72_phi_${v}_$i.json
done; done
