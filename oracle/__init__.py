"""CPU oracle for trie-based parallel beam decoding (arXiv 2502.00085).

TEST INFRASTRUCTURE ONLY.  Nothing under `oracle/` is part of the product: only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it.  The CUDA path (`paper_2502_00085_b200/`) never imports it and the
oracle never imports the CUDA path; they share only the seeded input generators in
`synth/` (which hold none of the method's arithmetic).

Plain, slow, obviously-correct numpy in float64 (float32 optional), fixed
left-to-right summation, no blocking/fusion.  Each function cites the PAPER.md
(`P:<line>`) or SPEC.md (`S:<line>`) passage it follows; readings of silent or
ambiguous passages are listed in DESIGN.md "Readings".

Modules
  numerics    -- softmax_masked, log_softmax, rope (rotate-half), rms_norm, matvec
  model       -- toy pre-norm decoder: one-token forward over a caller-chosen row set
  select      -- global top-b over (beam, token) candidates (Alg. 1 l.6 / Alg. 2 l.9)
  trie        -- trie state, Alg. 3 mask, update_trie / update_mask, GC (§3.5)
  decode      -- Alg. 1 batch beam search, Alg. 2 trie beam search, greedy
  kernels_ref -- kernel-level pure functions the GPU path is compared against:
                 build_tries (teacher-forced Alg. 2 l.10-11 + §3.5 GC: the append,
                 bitset and prune/compaction reference), mask_bits / soa (Alg. 3 mask
                 packed per node), attn_ref (§3.3), beam_step_ref (Alg. 2 l.9)

Parity pins: tests/test_oracle_*.py (marker "not gpu").  Every function here is pinned;
there is no "parity unpinned" function.
"""
