#!/bin/bash
# wide<D,1,4> default for 8 < Qg <= 16: full GPU tests; Qg <= 8 on it too (TRIE_WIDE1_MIN_QG=0)
# vs narrow on Phi / sweep b=2; 2-stage MT=1 build (3 CTAs / SM) on Mistral / sweep b=4
TAG=${1:-r2z4}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
TRIE_BUILD_OUT=/tmp/alt_w1s2.so TRIE_BUILD_DEFINES="TRIE_WIDE1_STAGES=2" python -m paper_2502_00085_b200.build --force >/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
  for q in 8 0; do
    TRIE_WIDE1_MIN_QG=$q timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_phi_q${q}_$rep.json
    TRIE_WIDE1_MIN_QG=$q timeout 300 python bench.py --workload sweep --beam 2 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw2_q${q}_$rep.json
  done
  for lib in default alt; do
    if [ $lib = alt ]; then export TRIE_LIB=/tmp/alt_w1s2.so; else unset TRIE_LIB; fi
    timeout 300 python bench.py --workload mistral-shard --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_mis_${lib}_$rep.json
    timeout 300 python bench.py --workload sweep --beam 4 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw4_${lib}_$rep.json
  done
  unset TRIE_LIB
done
ls gpurun_out | grep $TAG
