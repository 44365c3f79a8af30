#!/bin/bash
# stream-K wide kernel: parity with it forced on, Llama bench A/B, stage sweep, synccheck
TAG=${1:-r2c}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
TRIE_ATTN_STREAMK=1 timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bf16_lockstep.py tests/test_gpu_fullsize.py -q -x > gpurun_out/${TAG}_pytest_sk.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_sk.log
for cfg in "0 3" "1 2" "1 3" "1 4"; do
  set -- $cfg
  TRIE_ATTN_STREAMK=$1 TRIE_SK_STAGES=$2 timeout 600 python bench.py --workload llama --steps 32 --no-cpu-baseline --no-e2e 2>gpurun_out/${TAG}_llama_sk$1_st$2.err | tail -1 > gpurun_out/${TAG}_llama_sk$1_st$2.json
done
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 99 --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
  "tests/test_gpu_attn.py::test_attn_matches_oracle[b16-g4]" "tests/test_gpu_attn.py::test_attn_matches_oracle[b32]" \
  "tests/test_gpu_attn.py::test_fused_rope_attention_matches_oracle[umma-fused-1-16-130-8-2-128-0]" \
  "tests/test_gpu_attn.py::test_fused_rope_attention_matches_oracle[wide-fused-llama-2-8-150-32-8-128-0]" \
  "tests/test_gpu_beam_step.py::test_beam_step_matches_oracle[2-16-4097-5.0]" \
  "tests/test_gpu_integer_path.py::test_append_prune_bit_exact[3-4-12-True-30-0.0-3]" > gpurun_out/${TAG}_san_synccheck.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_san_synccheck.log
tail -n 3 gpurun_out/${TAG}_*.log
