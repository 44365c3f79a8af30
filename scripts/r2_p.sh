#!/bin/bash
# dual-lane tcgen05 softmax: parity, then A/B vs the single-lane build
TAG=${1:-r2p}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 1200 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py tests/test_gpu_fullsize.py tests/test_gpu_tree_spec.py tests/test_gpu_kv_shard.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
  for v in dual nodual; do
    L=""; [ $v = nodual ] && L=$PWD/alt/lib_nodual.so
    for b in 4 8 16 32; do
      TRIE_LIB=$L timeout 300 python bench.py --workload sweep --beam $b --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_${v}_b${b}_$rep.json
    done
    TRIE_LIB=$L timeout 300 python bench.py --workload mistral-shard --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_${v}_mis_$rep.json
  done
done
tail -n 2 gpurun_out/${TAG}_pytest.log
