#!/bin/bash
# tcgen05 stream-K: parity + A/B
TAG=${1:-r2w}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 1200 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py tests/test_gpu_fullsize.py tests/test_gpu_tree_spec.py tests/test_gpu_e2e_tiny.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
  for sk in 1 0; do
    for b in 16 32; do
      TRIE_UMMA_SK=$sk timeout 300 python bench.py --workload sweep --beam $b --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sk${sk}_b${b}_$rep.json
    done
  done
done
tail -n 3 gpurun_out/${TAG}_pytest.log
