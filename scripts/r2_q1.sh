#!/bin/bash
# query split (TRIE_QSPLIT=1): 16 < Qg <= 32 on the one-m-tile kernel, two CTAs per item, vs
# the two-m-tile kernel: parity + llama / sweep b=8, two reps
TAG=${1:-r2q1}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
TRIE_QSPLIT=1 timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py tests/test_gpu_graph_replay.py tests/test_gpu_fullsize.py tests/test_gpu_tree_spec.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
for q in 1 0; do
  TRIE_QSPLIT=$q timeout 300 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_llama_q${q}_$rep.json
  TRIE_QSPLIT=$q timeout 300 python bench.py --workload sweep --beam 8 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw8_q${q}_$rep.json
done
done
tail -3 gpurun_out/${TAG}_pytest.log
