for v in base ws2 ws4; do
  if [ $v = base ]; then unset TRIE_LIB; else export TRIE_LIB=$PWD/paper_2502_00085_b200/libtriedecode_$v.so; fi
  timeout 300 python bench.py --workload llama --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e65_llama_$v.json
done
