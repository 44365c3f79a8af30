for v in base minb3 minb2; do
  if [ $v = base ]; then unset TRIE_LIB; else export TRIE_LIB=$PWD/paper_2502_00085_b200/libtriedecode_$v.so; fi
  python scripts/bench_beam_step.py > gpurun_out/e64_beam_$v.json 2>&1
done
