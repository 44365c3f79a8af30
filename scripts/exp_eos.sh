for f in 0 0.5 0.75; do
  timeout 300 python bench.py --workload phi --steps 32 --no-cpu-baseline --no-e2e --eos-frac $f 2>gpurun_out/e67_phi_$f.err | tail -1 > gpurun_out/e67_phi_$f.json
  timeout 300 python bench.py --workload llama --steps 32 --no-cpu-baseline --no-e2e --eos-frac $f 2>/dev/null | tail -1 > gpurun_out/e67_llama_$f.json
done
