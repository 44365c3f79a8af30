#!/bin/bash
# wide kernel: no mask select on full-query prompt tiles, window-free boundary path (default)
# vs HEAD (alt_src/ = git archive, not committed), 2 reps
TAG=${1:-r2e4}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
(cd alt_src && TRIE_BUILD_OUT=/tmp/alt_e2.so python -m paper_2502_00085_b200.build --force >/dev/null)
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py tests/test_gpu_graph_replay.py tests/test_gpu_fullsize.py tests/test_gpu_tree_spec.py tests/test_gpu_e2e_tiny.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
for lib in default alt; do
  if [ $lib = alt ]; then export TRIE_LIB=/tmp/alt_e2.so; else unset TRIE_LIB; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_phi_${lib}_$rep.json
  timeout 300 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_llama_${lib}_$rep.json
  timeout 300 python bench.py --workload mistral-shard --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_mis_${lib}_$rep.json
  timeout 300 python bench.py --workload sweep --beam 8 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw8_${lib}_$rep.json
done
done
unset TRIE_LIB
tail -3 gpurun_out/${TAG}_pytest.log
