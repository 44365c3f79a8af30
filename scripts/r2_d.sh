#!/bin/bash
TAG=${1:-r2d}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
timeout 900 python -m pytest tests/test_gpu_kv_shard.py tests/test_gpu_attn.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 99 --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
  "tests/test_gpu_attn.py::test_attn_matches_oracle[b16-g4]" "tests/test_gpu_attn.py::test_attn_matches_oracle[b32]" \
  "tests/test_gpu_attn.py::test_fused_rope_attention_matches_oracle[umma-fused-1-16-130-8-2-128-0]" \
  "tests/test_gpu_attn.py::test_fused_rope_attention_matches_oracle[wide-fused-llama-2-8-150-32-8-128-0]" \
  "tests/test_gpu_beam_step.py::test_beam_step_matches_oracle[2-16-4097-5.0]" \
  "tests/test_gpu_integer_path.py::test_append_prune_bit_exact[3-4-12-True-30-0.0-3]" > gpurun_out/${TAG}_san_synccheck.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_san_synccheck.log
TRIE_ATTN_STREAMK=1 timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"k_attn_wide" -s 200 -c 1 \
   -o gpurun_out/${TAG}_sk_llama -f python bench.py --workload llama --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_sk.log 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"k_attn_wide" -s 200 -c 1 \
   -o gpurun_out/${TAG}_wide_llama -f python bench.py --workload llama --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_wide.log 2>&1
tail -n 3 gpurun_out/${TAG}_*.log
