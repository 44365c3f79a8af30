timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t40.log 2>&1; tail -3 gpurun_out/t40.log
timeout 300 python bench.py --workload mistral-shard --no-cpu-baseline --no-e2e --steps 32 2>/dev/null | tail -1 > gpurun_out/e40_mis.json
TRIE_BENCH_FUSED=0 timeout 300 python bench.py --workload mistral-shard --no-cpu-baseline --no-e2e --steps 32 2>/dev/null | tail -1 > gpurun_out/e40_mis_unfused.json
for b in 4 16; do timeout 300 python bench.py --workload sweep --beam $b --no-cpu-baseline --no-e2e --steps 16 2>/dev/null | tail -1 > gpurun_out/e40_sw$b.json; TRIE_BENCH_FUSED=0 timeout 300 python bench.py --workload sweep --beam $b --no-cpu-baseline --no-e2e --steps 16 2>/dev/null | tail -1 > gpurun_out/e40_sw${b}_unfused.json; done
