#!/bin/bash
# tcgen05 ring split A/B (K/V stages) and dual on/off, fused path
TAG=${1:-r2q}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 600 python -m pytest tests/test_gpu_attn.py -q -x -k "umma or b16 or b32 or evict" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
TRIE_UMMA_ST=56 timeout 600 python -m pytest tests/test_gpu_attn.py -q -x -k "umma or b16 or b32" >> gpurun_out/${TAG}_pytest.log 2>&1; echo "rc56=$?" >> gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
  for st in 46 56 38; do
    for b in 4 16 32; do
      TRIE_UMMA_ST=$st timeout 300 python bench.py --workload sweep --beam $b --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_st${st}_b${b}_$rep.json
    done
    TRIE_UMMA_ST=$st timeout 300 python bench.py --workload mistral-shard --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_st${st}_mis_$rep.json
  done
done
tail -n 4 gpurun_out/${TAG}_pytest.log
