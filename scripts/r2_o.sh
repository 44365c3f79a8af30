#!/bin/bash
# MUFU offload A/B: every 4th (default) / 3rd / 2nd pair in software vs all on MUFU (0)
TAG=${1:-r2o}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
  for v in 4 0 3 2; do
    L=""; [ $v != 4 ] && L=$PWD/alt/lib_swexp$v.so
    for b in 4 16 32; do
      TRIE_LIB=$L timeout 300 python bench.py --workload sweep --beam $b --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_v${v}_b${b}_$rep.json
    done
    TRIE_LIB=$L timeout 300 python bench.py --workload mistral-shard --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_v${v}_mis_$rep.json
  done
done
tail -n 2 gpurun_out/${TAG}_pytest.log
