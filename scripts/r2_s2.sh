#!/bin/bash
# (1) isolated per-CTA tile rate (one CTA per item: TRIE_ATTN_SPLITS=1); (2) beam step ring
# kernel: parity tests + microbench vs the register kernel (TRIE_BEAM_RING=0)
TAG=${1:-r2s2}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
O=gpurun_out/${TAG}_single.jsonl; : > $O
export TRIE_ATTN_SPLITS=1
for st in 100 400; do
for rs in 2 4; do
  TRIE_WIDE_RS=$rs timeout 120 python scripts/attn_single.py --R 1 --hq 4 --hkv 1 --b 8 --steps $st >> $O 2>&1
done
timeout 120 python scripts/attn_single.py --R 1 --hq 4 --hkv 1 --b 4 --steps $st >> $O 2>&1
TRIE_WIDE1_MIN_QG=16 timeout 120 python scripts/attn_single.py --R 1 --hq 4 --hkv 1 --b 4 --steps $st >> $O 2>&1
timeout 120 python scripts/attn_single.py --R 1 --hq 1 --hkv 1 --b 4 --D 96 --steps $st >> $O 2>&1
timeout 120 python scripts/attn_single.py --R 16 --hq 32 --hkv 8 --b 8 --steps $st >> $O 2>&1
done
unset TRIE_ATTN_SPLITS
timeout 600 python -m pytest tests/test_gpu_beam_step.py tests/test_gpu_integer_path.py tests/test_gpu_e2e_tiny.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python scripts/bench_beam_step.py > gpurun_out/${TAG}_beam_ring.json 2>&1
TRIE_BEAM_RING=0 timeout 300 python scripts/bench_beam_step.py > gpurun_out/${TAG}_beam_reg.json 2>&1
cat $O; tail -3 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_beam_*.json
