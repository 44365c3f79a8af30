#!/bin/bash
# model context (random-init shaped decoder + the hot path), kappa sweep, Fig. 4 with dead-tile counts
TAG=${1:-r2g}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
for wl in phi llama mistral-shard; do
  timeout 900 python bench.py --workload $wl --steps 16 --warmup 3 --no-cpu-baseline --no-e2e --model-context \
     > gpurun_out/${TAG}_mc_${wl}.json 2>gpurun_out/${TAG}_mc_${wl}.err
done
for kap in 0.5 1 2 3 5; do
  timeout 600 python bench.py --workload phi --steps 16 --warmup 3 --no-cpu-baseline --no-e2e --logit-scale $kap --series \
     > gpurun_out/${TAG}_kappa_phi_$kap.json 2>gpurun_out/${TAG}_kappa_phi_$kap.err
  timeout 600 python bench.py --workload llama --steps 16 --warmup 3 --no-cpu-baseline --no-e2e --logit-scale $kap --series \
     > gpurun_out/${TAG}_kappa_llama_$kap.json 2>gpurun_out/${TAG}_kappa_llama_$kap.err
done
timeout 1500 python bench.py --workload llama --beam 30 --new-tokens 1000 --requests 4 --gc-interval 15 --steps 16 --series \
   --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_fig4.json 2>gpurun_out/${TAG}_fig4.err
tail -n 3 gpurun_out/${TAG}_*.err
