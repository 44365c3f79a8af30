#!/bin/bash
# narrow kernel one-tile software pipeline (TRIE_NARROW_PIPE=1, default build) vs the plain
# loop (alt build TRIE_NARROW_PIPE=0): parity + Phi (default bench) + sweep b=2, two reps
TAG=${1:-r2p2}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
TRIE_BUILD_OUT=/tmp/alt_nnp.so TRIE_BUILD_DEFINES="TRIE_NARROW_PIPE=0" python -m paper_2502_00085_b200.build --force >/dev/null
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py tests/test_gpu_graph_replay.py tests/test_gpu_e2e_tiny.py tests/test_gpu_tree_spec.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
for lib in default alt; do
  if [ $lib = alt ]; then export TRIE_LIB=/tmp/alt_nnp.so; else unset TRIE_LIB; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_phi_${lib}_$rep.json
  timeout 300 python bench.py --workload sweep --beam 2 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw2_${lib}_$rep.json
done
done
unset TRIE_LIB
tail -3 gpurun_out/${TAG}_pytest.log
