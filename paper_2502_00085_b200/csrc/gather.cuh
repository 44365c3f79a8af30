// Device side of the fused KV-head-shard all-gather (trie_gather_setup
// in include/triedecode.h): peer stores from the attention epilogue + a launch-completion
// flag per rank (release / acquire at system scope: the peers are other GPUs over NVLink).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "attn_common.cuh"

namespace trie {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// The half of the gather buffers this launch writes: its sequence number - 1, mod 2.  Read
// by a writer before its own arrival, i.e. before the launch's last arrival bumps it.
__device__ __forceinline__ uint32_t gather_half(const AttnParams& p) {
  return *(volatile const uint32_t*)p.ga.epoch & 1u;
}

// Two bf16 of output row (r, beam j, local query head hl), columns d, d + 1, into every
// rank's gather buffer at head rank * Hq + hl.
__device__ __forceinline__ void gather_st32(const AttnParams& p, uint32_t half, int r, int j, int hl,
                                            int d, uint32_t v) {
  const int hq_all = p.ga.world * p.Hq;
  const size_t off =
      (size_t)half * p.ga.half_stride +
      (((size_t)r * p.b_live + j) * hq_all + (size_t)p.ga.rank * p.Hq + hl) * p.D + d;
#pragma unroll 1
  for (int q = 0; q < p.ga.world; ++q) *(uint32_t*)((__nv_bfloat16*)p.ga.out[q] + off) = v;
}

// One bf16, column d.
__device__ __forceinline__ void gather_st16(const AttnParams& p, uint32_t half, int r, int j, int hl,
                                            int d, __nv_bfloat16 v) {
  const int hq_all = p.ga.world * p.Hq;
  const size_t off =
      (size_t)half * p.ga.half_stride +
      (((size_t)r * p.b_live + j) * hq_all + (size_t)p.ga.rank * p.Hq + hl) * p.D + d;
#pragma unroll 1
  for (int q = 0; q < p.ga.world; ++q) ((__nv_bfloat16*)p.ga.out[q])[off] = v;
}

// Eight bf16 (16 bytes), columns d .. d + 7.
__device__ __forceinline__ void gather_st128(const AttnParams& p, uint32_t half, int r, int j, int hl,
                                             int d, int4 v) {
  const int hq_all = p.ga.world * p.Hq;
  const size_t off =
      (size_t)half * p.ga.half_stride +
      (((size_t)r * p.b_live + j) * hq_all + (size_t)p.ga.rank * p.Hq + hl) * p.D + d;
#pragma unroll 1
  for (int q = 0; q < p.ga.world; ++q) *(int4*)((__nv_bfloat16*)p.ga.out[q] + off) = v;
}

// One arrival per finished output unit; the caller orders the unit's stores before it (a
// barrier among the unit's writers).  The last arrival of the launch publishes the new
// sequence number to flag[rank] of every rank and re-arms the ticket.
__device__ __forceinline__ void gather_arrive(const AttnParams& p) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  const uint32_t old = atomicAdd(p.ga.ticket, 1u);
  if (old + 1 == p.ga.expected) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    const uint32_t e = *(volatile uint32_t*)p.ga.epoch + 1u;
    *(volatile uint32_t*)p.ga.ticket = 0u;
    *(volatile uint32_t*)p.ga.epoch = e;
#pragma unroll 1
    for (int q = 0; q < p.ga.world; ++q) st_release_sys(p.ga.flag[q] + p.ga.rank, e);
  }
}

}  // namespace trie
