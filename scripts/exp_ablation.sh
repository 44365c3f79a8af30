# Ablation of the launch-overlap / data-movement features on the final build (one box)
for wl in phi llama; do
  timeout 300 python bench.py --workload $wl --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e80_${wl}_base.json
  TRIE_PDL=0 timeout 300 python bench.py --workload $wl --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e80_${wl}_nopdl.json
  TRIE_PREFETCH=0 timeout 300 python bench.py --workload $wl --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e80_${wl}_noprefetch.json
  TRIE_HALF_TILE=0 timeout 300 python bench.py --workload $wl --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e80_${wl}_nohalf.json
  TRIE_BENCH_FUSED=0 timeout 300 python bench.py --workload $wl --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e80_${wl}_unfused.json
done
