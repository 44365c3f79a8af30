#!/bin/bash
# mbarrier try_wait with a suspend-time hint (alt builds) vs plain spin (default)
TAG=${1:-r2h1}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
TRIE_BUILD_OUT=/tmp/hint_big.so TRIE_BUILD_DEFINES="TRIE_MBAR_HINT=1000000" python -m paper_2502_00085_b200.build --force >/dev/null
TRIE_BUILD_OUT=/tmp/hint_small.so TRIE_BUILD_DEFINES="TRIE_MBAR_HINT=2000" python -m paper_2502_00085_b200.build --force >/dev/null
TRIE_LIB=/tmp/hint_big.so timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_graph_replay.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
for lib in default big small; do
  if [ $lib = default ]; then unset TRIE_LIB; else export TRIE_LIB=/tmp/hint_$lib.so; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_phi_${lib}_$rep.json
  timeout 300 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_llama_${lib}_$rep.json
  timeout 300 python bench.py --workload sweep --beam 16 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw16_${lib}_$rep.json
done
done
unset TRIE_LIB
tail -3 gpurun_out/${TAG}_pytest.log
