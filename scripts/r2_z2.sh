#!/bin/bash
# wide<D,1,4> for 8 < Qg <= 16 (TRIE_QG16_WIDE=1) vs narrow: parity + Mistral shard / sweep b=4
TAG=${1:-r2z2}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
TRIE_QG16_WIDE=1 timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
for w in 1 0; do
  TRIE_QG16_WIDE=$w timeout 300 python bench.py --workload mistral-shard --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_mis_w${w}_$rep.json
  TRIE_QG16_WIDE=$w timeout 300 python bench.py --workload sweep --beam 4 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw4_w${w}_$rep.json
done
done
ls gpurun_out | grep $TAG
