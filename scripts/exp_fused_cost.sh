for v in base NOQROT NOAPPEND; do
  if [ $v = base ]; then unset TRIE_LIB; else export TRIE_LIB=$PWD/paper_2502_00085_b200/libtriedecode_$v.so; fi
  timeout 300 python bench.py --workload phi --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e83_phi_$v.json
done
