#!/bin/bash
# wide<D,2,4> without a producer warp (NP, 128 regs, 2 CTAs/SM) vs wide<D,2,2>: parity + isolated
# per-CTA tile rate + llama / sweep b=8
TAG=${1:-r2s4}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
TRIE_WIDE_RS=4 timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py tests/test_gpu_fullsize.py tests/test_gpu_kv_shard.py -m gpu -q -x > gpurun_out/${TAG}_pytest_rs4.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_rs4.log
O=gpurun_out/${TAG}_single.jsonl; : > $O
for rs in 2 4; do
  TRIE_ATTN_SPLITS=1 TRIE_WIDE_RS=$rs timeout 120 python scripts/attn_single.py --R 1 --hq 4 --hkv 1 --b 8 --steps 100 >> $O 2>&1
  TRIE_ATTN_SPLITS=1 TRIE_WIDE_RS=$rs timeout 120 python scripts/attn_single.py --R 1 --hq 4 --hkv 1 --b 8 --steps 400 >> $O 2>&1
done
for rep in 1 2; do
for rs in 2 4; do
  TRIE_WIDE_RS=$rs timeout 300 python bench.py --workload llama --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_llama_rs${rs}_$rep.json
  TRIE_WIDE_RS=$rs timeout 300 python bench.py --workload sweep --beam 8 --steps 16 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw8_rs${rs}_$rep.json
done
done
tail -3 gpurun_out/${TAG}_pytest_rs4.log; cat $O
