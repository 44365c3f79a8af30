timeout 1200 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fullsize.py tests/test_gpu_tree_spec.py -q -x > gpurun_out/t84.log 2>&1; tail -2 gpurun_out/t84.log
for i in 1 2; do timeout 300 python bench.py --workload phi --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/e84_phi_$i.json; done
