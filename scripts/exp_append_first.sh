timeout 1200 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fullsize.py -q -x > gpurun_out/t81.log 2>&1; tail -2 gpurun_out/t81.log
for wl in phi llama; do
  timeout 300 python bench.py --workload $wl --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e81_${wl}.json
  TRIE_BENCH_FUSED=0 timeout 300 python bench.py --workload $wl --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e81_${wl}_unfused.json
done
