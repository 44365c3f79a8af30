#!/bin/bash
# NOTE (r2f3): compute-sanitizer has been closed on the GPU pool; kept for the record of r2l.
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over every kernel of the
# library at tiny shapes, through the GPU parity tests (SURVEY §5 / §4 tier vi).
#   bash scripts/sanitize.sh <tag>   -> gpurun_out/<tag>_san_<tool>.log
TAG=${1:-san}
mkdir -p gpurun_out
python -m paper_2502_00085_b200.build >/dev/null
T=tests
IDS=(
  "$T/test_gpu_attn.py::test_attn_matches_oracle[tiny]"            # k_attn_v1 + k_attn_combine (fp32)
  "$T/test_gpu_attn.py::test_attn_matches_oracle[tiny-walk]"       # Alg. 3 walk (k_mask_walk)
  "$T/test_gpu_attn.py::test_attn_matches_oracle[phi-like]"        # k_attn_narrow
  "$T/test_gpu_attn.py::test_attn_matches_oracle[llama-like]"      # GQA narrow
  "$T/test_gpu_attn.py::test_attn_matches_oracle[b16-g4]"          # tcgen05 / wide
  "$T/test_gpu_attn.py::test_attn_matches_oracle[b32]"
  "$T/test_gpu_attn.py::test_fused_rope_attention_matches_oracle[phi-fused-2-4-300-8-8-96-0]"
  "$T/test_gpu_attn.py::test_fused_rope_attention_matches_oracle[wide-fused-llama-2-8-150-32-8-128-0]"
  "$T/test_gpu_attn.py::test_fused_rope_attention_matches_oracle[umma-fused-1-16-130-8-2-128-0]"
  "$T/test_gpu_attn.py::test_fused_rope_attention_matches_oracle[split-fused-1-2-1500-2-2-128-0]"
  "$T/test_gpu_attn.py::test_fused_rope_attention_matches_oracle[gqa-fused-2-4-200-8-2-128-0]"          # wide<128,1,4> (Qg = 16)
  "$T/test_gpu_attn.py::test_fused_rope_attention_matches_oracle[wide1-fused-split-1-4-1500-8-2-64-0]"  # wide<64,1,4> + split-K
  "$T/test_gpu_attn.py::test_rope_kv_append_matches_oracle"
  "$T/test_gpu_beam_step.py::test_beam_step_matches_oracle[2-3-256-4.0]"
  "$T/test_gpu_beam_step.py::test_beam_step_matches_oracle[2-16-4097-5.0]"
  "$T/test_gpu_integer_path.py::test_append_prune_bit_exact[3-3-8-False-16-0.5-1-dense]"
  "$T/test_gpu_integer_path.py::test_append_prune_bit_exact[3-4-12-True-30-0.0-3-dense]"
  "$T/test_gpu_integer_path.py::test_append_prune_bit_exact[3-3-8-False-16-0.5-1-paged]"   # NEXT-2 pages
  "$T/test_gpu_integer_path.py::test_paged_pool_exhaustion_latches_and_gc_returns_pages"
  "$T/test_gpu_attn.py::test_fused_paged_pools_match_oracle[paged-wide-2-8-150-32-8-128-0]"
  "$T/test_gpu_attn.py::test_fused_paged_pools_match_oracle[paged-umma-2-16-400-8-2-128-0]"
  "$T/test_gpu_attn.py::test_swa_eviction_frees_prompt_pages_and_matches_oracle[evict-narrow-2-4-300-8-2-128-100-8]"
  "$T/test_gpu_batch_baseline.py::test_batch_reorder_matches_gather"
)
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 99 --print-limit 50 \
      python -m pytest -x -q -p no:cacheprovider "${IDS[@]}" > gpurun_out/${TAG}_san_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_san_${tool}.log
done
tail -n 4 gpurun_out/${TAG}_san_*.log
