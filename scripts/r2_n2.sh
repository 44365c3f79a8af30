#!/bin/bash
# two-m-tile wide kernel without a producer warp (4-warp CTA, no register cap; default build)
# vs the 5-warp CTA (alt build TRIE_WIDE_NP=0): parity + isolated tile rate + llama / sweep b=8
TAG=${1:-r2n2}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
TRIE_BUILD_OUT=/tmp/alt_np0.so TRIE_BUILD_DEFINES="TRIE_WIDE_NP=0" python -m paper_2502_00085_b200.build --force >/dev/null
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py tests/test_gpu_graph_replay.py tests/test_gpu_fullsize.py tests/test_gpu_tree_spec.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
O=gpurun_out/${TAG}_single.jsonl; : > $O
for lib in default alt; do
  if [ $lib = alt ]; then export TRIE_LIB=/tmp/alt_np0.so; else unset TRIE_LIB; fi
  for st in 100 400; do TRIE_ATTN_SPLITS=1 timeout 120 python scripts/attn_single.py --R 1 --hq 4 --hkv 1 --b 8 --steps $st >> $O 2>&1; done
done
for rep in 1 2; do
for lib in default alt; do
  if [ $lib = alt ]; then export TRIE_LIB=/tmp/alt_np0.so; else unset TRIE_LIB; fi
  timeout 300 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_llama_${lib}_$rep.json
  timeout 300 python bench.py --workload sweep --beam 8 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw8_${lib}_$rep.json
done
done
unset TRIE_LIB
tail -3 gpurun_out/${TAG}_pytest.log; cat $O
