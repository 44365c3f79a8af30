// trie_attn_decode, tcgen05 / TMEM path for wide query groups (sm_100a).
// §3.3: o = softmax(q K^T / sqrt(D)) V over each beam's root-to-leaf rows.
//
// When b_live x (Hq/Hkv) >= 33 queries share a KV head, the legacy mma.sync path becomes
// tensor-pipe bound (r05: b=16, g=4 at 8k context stalls at ~3.2 TB/s).  Here one thread
// issues 5th-generation tensor-core MMAs with the accumulators in tensor memory:
//   S[128 x 64] = Q[128 x D] . K_tile^T      (A = Q in smem, K-major SW64; B = the TMA
//                                             K tile, K-major SW64; fp32 in TMEM)
//   O[128 x D] += P[128 x 64] . V_tile        (A = P in TMEM, bf16; B = the TMA V tile,
//                                             MN-major SW64; fp32 in TMEM)
// The TMA tiles written by the producer ARE the canonical UMMA layouts (64-byte rows,
// 8-row atoms of 512 B, 32-column boxes 4096 B apart), so no re-staging is needed.
// Warp roles: 0 = TMA producer, 1 = TMEM allocator + MMA issuer, 2..5 = softmax /
// epilogue (warp w reads TMEM lanes 32*(w%4).., thread = query row).  S is double
// buffered so QK of tile i+1 overlaps the softmax of tile i; the running max is rescaled
// lazily (O is only rescaled when a row max grows by > 8 in log2 units).
// Rows >= Qg of the 128-row MMA are padding (Q rows zero, P rows zero, outputs ignored).
#include <stdio.h>
#include <stdlib.h>

#include "attn_common.cuh"
#include "common.cuh"
#include "handle.h"
#include "tc_common.cuh"

namespace trie {

// ---- tcgen05 PTX helpers ----------------------------------------------------------------
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (Blackwell)
  d |= (uint64_t)4 << 61;  // SWIZZLE_64B
  return d;
}
// kind::f16 instruction descriptor: fp32 accumulate, bf16 A and B
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                        uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
        "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
        "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
      "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {  // MUFU.EX2; ex2(-inf) = +0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

// DB: S double-buffered in TMEM.  SW: softmax warps per TMEM sub-partition (1 or 2; with 2
// the pair splits the 64 S columns and the D output columns, exchanging the row max
// through shared memory once per tile).  P (bf16, 32 columns) overwrites the first half
// of the S buffer it was computed from, so S0 | S1 | O fit in 256 TMEM columns.
template <int D, int ST, bool DB, int SW>
struct UCfg {
  using RG = Ring<D, ST>;
  static constexpr int STAGES = ST;
  static constexpr int QBYTES = 128 * D * 2;  // Q: 128 rows (padding zero), D/32 boxes
  static constexpr int OFF_Q = RG::RING_BYTES;
  static constexpr int OFF_X = OFF_Q + QBYTES;           // row-max exchange [2][4][2][32] f32
  static constexpr int OFF_BAR = OFF_X + 2 * 4 * 2 * 32 * 4;
  static constexpr int NBAR = 2 * ST + 2 + 2;  // full, empty, s_full[2], p_full, pv_done
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 64 + 1024;
  static constexpr int NSW = 4 * SW;           // softmax warps
  static constexpr int THREADS = (2 + NSW) * 32;
  static constexpr int CW = 64 / SW;           // S columns per softmax warp
  static constexpr int OW = D / SW;            // O columns per softmax warp
  static constexpr int COL_S0 = 0, COL_S1 = DB ? 64 : 0, COL_O = DB ? 128 : 64;
  static constexpr int TMEM_COLS = 256;
  static_assert(COL_O + D <= TMEM_COLS, "TMEM budget");
  static_assert(OW % 32 == 0, "O columns per warp");
};

template <int D, int ST, bool DB, int SW>
__global__ void __launch_bounds__(UCfg<D, ST, DB, SW>::THREADS) k_attn_umma(
    const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
    const AttnParams p) {
  using C = UCfg<D, ST, DB, SW>;
  using RG = typename C::RG;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  uint8_t* qsm = smem + C::OFF_Q;
  float* xch = (float*)(smem + C::OFF_X);
  uint64_t* full = (uint64_t*)(smem + C::OFF_BAR);
  uint64_t* empty = full + ST;
  uint64_t* s_full = empty + ST;
  uint64_t* p_full = s_full + 2;
  uint64_t* pv_done = p_full + 1;
  uint32_t* tmem_slot = (uint32_t*)(pv_done + 1);
  ItemInfo* info = (ItemInfo*)(tmem_slot + 4);

  const int h = blockIdx.x, r = blockIdx.y, split = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = p.Hq / p.Hkv, Qg = p.b_live * g;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(p_full, C::NSW);
    mbar_init(pv_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    item_setup(p, r, split, info);
  }
  if (warp == 1) {  // TMEM allocation (whole warp), address published through smem
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const ItemInfo it = *info;
  const uint32_t tmem = *tmem_slot;
  const int ntiles = it.ntiles;
  constexpr int QBAR_THREADS = (C::NSW + 1) * 32;

  if (warp == 0) {
    if (lane == 0) producer_loop<D, ST>(&kmap, &vmap, p, r, h, it, ring, full, empty);
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    asm volatile("bar.sync 1, %0;" ::"r"(QBAR_THREADS));  // Q staged by the softmax warps
    tc_fence_after();
    const uint32_t idesc_qk = umma_idesc(128, 64, 0);
    const uint32_t idesc_pv = umma_idesc(128, D, 1);
    const uint32_t qbase = smem_u32(qsm);
    auto issue_qk = [&](int i) {
      const int s = i % ST;
      mbar_wait(&full[s], (uint32_t)(i / ST) & 1u);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t kb = smem_u32(ring + s * RG::STAGE_BYTES);
        const uint32_t d_s = tmem + ((i & 1) ? C::COL_S1 : C::COL_S0);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          // K step ks: 32-column box ks/2 (8 KB apart for the 128-row Q, 4 KB for the 64-row
          // K tile), + 32 B inside the 64-byte swizzled row for odd steps; SBO = 8 rows = 512 B
          const uint64_t a = umma_desc_sw64(qbase + (ks >> 1) * 128 * 64 + (ks & 1) * 32, 16, 512);
          const uint64_t b = umma_desc_sw64(kb + (ks >> 1) * TC_TR * 64 + (ks & 1) * 32, 16, 512);
          umma_ss(d_s, a, b, idesc_qk, ks > 0);
        }
        umma_commit(&s_full[DB ? (i & 1) : 0]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int i) {
      mbar_wait(p_full, (uint32_t)i & 1u);
      tc_fence_after();
      if (lane == 0) {
        const int s = i % ST;
        const uint32_t vb = smem_u32(ring + s * RG::STAGE_BYTES + RG::TILE_BYTES);
        const uint32_t colp = (DB && (i & 1)) ? C::COL_S1 : C::COL_S0;  // P_i over S_i
#pragma unroll
        for (int kc = 0; kc < TC_TR / 16; ++kc) {
          // V tile as MN-major B: 16 rows per K step = two 8-row atoms (1024 B); the
          // 32-column boxes are LBO = 4096 B apart, the 8-row atoms SBO = 512 B apart
          const uint64_t b = umma_desc_sw64(vb + kc * 1024, TC_TR * 64, 512);
          umma_ts(tmem + C::COL_O, tmem + colp + kc * 8, b, idesc_pv, (i > 0 || kc > 0) ? 1u : 0u);
        }
        umma_commit(&empty[s]);
        umma_commit(pv_done);
      }
      __syncwarp();
    };
    if constexpr (DB) {
      if (ntiles > 0) issue_qk(0);
      for (int i = 0; i < ntiles; ++i) {
        if (i + 1 < ntiles) issue_qk(i + 1);  // overlaps the softmax of tile i
        issue_pv(i);
      }
    } else {
      for (int i = 0; i < ntiles; ++i) {  // S is reused: QK(i+1) waits for softmax(i)
        issue_qk(i);
        issue_pv(i);
      }
    }
  } else {
    // ===================== softmax / epilogue warps =====================
    const int sp = warp & 3;                  // TMEM sub-partition of this warp
    const int half = (warp - 2) / 4;         // column half (SW = 2) / 0
    const int row = sp * 32 + lane;           // query row (MMA M index)
    const int tid = threadIdx.x - 64;
    {  // Q -> smem, 64B-swizzled K-major boxes of [128 rows][32 cols]; padding rows zero
      const __nv_bfloat16* q = (const __nv_bfloat16*)p.q;
      const int chunks = 128 * (D / 8);
      for (int c = tid; c < chunks; c += C::NSW * 32) {
        const int m = c / (D / 8), col = (c % (D / 8)) * 8;
        int4 v = make_int4(0, 0, 0, 0);
        if (m < Qg)
          v = *(const int4*)(q + (((size_t)r * p.b_live + m / g) * p.Hq + h * g + m % g) * D + col);
        const int box = col / TC_CW;
        const uint32_t o = (uint32_t)m * 64u + (uint32_t)(col % TC_CW) * 2u;
        *(int4*)(qsm + box * 128 * 64 + (o ^ (((o >> 7) & 3u) << 4))) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"r"(QBAR_THREADS));
    }
    const bool qvalid = row < Qg;
    const bool warp_live = sp * 32 < Qg;      // warp-uniform: all 32 rows padding -> skip math
    const int beam = qvalid ? row / g : 0;
    const size_t mbase = (size_t)r * p.cap;
    const int lod = (p.window > 0 && qvalid) ? p.depth[mbase + p.leaf[r * TRIE_MAX_BEAMS + beam]] - p.window + 1 : INT_MIN;
    const float sc = p.scale_log2;
    const int fast_end = min(it.t, it.N) / TC_TR;
    const uint32_t lane_off = (uint32_t)(sp * 32) << 16;
    const int col0 = half * C::CW;            // this warp's S columns [col0, col0 + CW)
    const int ocol0 = half * C::OW;           // this warp's O columns
    float m_run = -INFINITY, l_run = 0.f;
    for (int i = 0; i < ntiles; ++i) {
      const int s = i % ST;
      const uint32_t spar = DB ? ((uint32_t)(i >> 1) & 1u) : ((uint32_t)i & 1u);
      mbar_wait(&s_full[DB ? (i & 1) : 0], spar);
      mbar_wait(&full[s], (uint32_t)(i / ST) & 1u);  // (complete) makes the mask words visible
      tc_fence_after();
      const uint32_t scol = (DB && (i & 1)) ? C::COL_S1 : C::COL_S0;
      uint32_t pk[C::CW / 2];
      float alpha = 1.f;
      bool rescale = false;
      if (warp_live) {
        float x[C::CW];
        {
          uint32_t a[32];
#pragma unroll
          for (int c = 0; c < C::CW; c += 32) {
            tmem_ld32(tmem + lane_off + scol + col0 + c, a);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 32; ++k) x[c + k] = qvalid ? __uint_as_float(a[k]) * sc : -INFINITY;
          }
        }
        const int tile = it.tile0 + i;
        const int n0 = tile * TC_TR + col0;
        if (!(tile >= it.fast_from && tile < fast_end)) {  // warp-uniform
          const uint8_t* stp = ring + s * RG::STAGE_BYTES;
          const uint32_t* tmask = (const uint32_t*)(stp + 2 * RG::TILE_BYTES) + col0;
          const int* tdep = (const int*)(stp + 2 * RG::TILE_BYTES + TC_TR * 4) + col0;
#pragma unroll
          for (int k = 0; k < C::CW; ++k) {
            const int n = n0 + k;
            const bool ok = n < it.N && (n < it.t || ((tmask[k] >> beam) & 1u)) && tdep[k] >= lod;
            x[k] = ok ? x[k] : -INFINITY;
          }
        }
        float mx[8];  // tree max
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          float v = x[u];
#pragma unroll
          for (int k = 8 + u; k < C::CW; k += 8) v = fmaxf(v, x[k]);
          mx[u] = v;
        }
        float tmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                           fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        if constexpr (SW == 2) {  // pair exchange of the row max (double-buffered by tile parity)
          float* xb = xch + (i & 1) * 256 + sp * 64;
          xb[half * 32 + lane] = tmax;
          asm volatile("bar.sync %0, 64;" ::"r"(2 + sp));
          tmax = fmaxf(tmax, xb[(1 - half) * 32 + lane]);
        }
        // lazy rescale: keep the running max unless the tile max exceeds it by > 8 (log2)
        if (tmax > m_run + 8.f || (m_run == -INFINITY && tmax > -INFINITY)) {
          alpha = (m_run == -INFINITY) ? 0.f : ex2(m_run - tmax);
          rescale = m_run != -INFINITY;
          m_run = tmax;
          l_run *= alpha;
        }
        const float mu = m_run == -INFINITY ? 0.f : m_run;  // all masked: ex2(-inf) = 0
        float ps[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) ps[u] = 0.f;
#pragma unroll
        for (int k = 0; k < C::CW / 2; ++k) {
          const float p0 = ex2(x[2 * k] - mu), p1 = ex2(x[2 * k + 1] - mu);
          ps[k & 7] += p0 + p1;
          pk[k] = pack_bf16(p0, p1);
        }
        l_run += ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
      } else {
#pragma unroll
        for (int k = 0; k < C::CW / 2; ++k) pk[k] = 0u;
      }
      if (i > 0) {  // PV of the previous tile must be done before P / O are touched
        mbar_wait(pv_done, (uint32_t)(i - 1) & 1u);
        tc_fence_after();
      }
      if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
        for (int c = 0; c < C::OW; c += 32) {
          uint32_t o[32];
          tmem_ld32(tmem + lane_off + C::COL_O + ocol0 + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
          tmem_st32(tmem + lane_off + C::COL_O + ocol0 + c, o);
        }
      }
      if constexpr (SW == 1) {
        tmem_st32(tmem + lane_off + scol, *reinterpret_cast<uint32_t(*)[32]>(pk));  // P_i over S_i
      } else {
        tmem_st16(tmem + lane_off + scol + half * 16, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // ---- epilogue: O / l ----
    if (ntiles > 0) {
      mbar_wait(pv_done, (uint32_t)(ntiles - 1) & 1u);
      tc_fence_after();
    }
    if constexpr (SW == 2) {  // total row sum = both halves
      float* xb = xch + 512 - 64 + sp * 16;  // last 64 floats of the exchange area... per sp
      (void)xb;
      float* lb = xch + sp * 64;
      asm volatile("bar.sync %0, 64;" ::"r"(2 + sp));  // both done with the exchange buffers
      lb[half * 32 + lane] = l_run;
      asm volatile("bar.sync %0, 64;" ::"r"(2 + sp));
      l_run += lb[(1 - half) * 32 + lane];
    }
    const int j = beam, ii = row % g;
    if (warp_live) {
      if (p.splits == 1) {
        __nv_bfloat16* op = (__nv_bfloat16*)p.out + (((size_t)r * p.b_live + j) * p.Hq + h * g + ii) * D + ocol0;
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll
        for (int c = 0; c < C::OW; c += 32) {
          uint32_t o[32];
          tmem_ld32(tmem + lane_off + C::COL_O + ocol0 + c, o);
          tmem_wait_ld();
          if (qvalid) {
            uint32_t w[16];
#pragma unroll
            for (int k = 0; k < 16; ++k)
              w[k] = pack_bf16(__uint_as_float(o[2 * k]) * inv, __uint_as_float(o[2 * k + 1]) * inv);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              *(int4*)(op + c + 8 * k) = make_int4((int)w[4 * k], (int)w[4 * k + 1], (int)w[4 * k + 2], (int)w[4 * k + 3]);
          }
        }
        if (qvalid && half == 0) {
          if (l_run == 0.f) latch(p.status, TRIE_ST_EMPTY_ROW);
          if (p.lse)
            p.lse[((size_t)r * p.b_live + j) * p.Hq + h * g + ii] =
                l_run > 0.f ? (m_run + log2f(l_run)) * 0.69314718055994531f : -INFINITY;
        }
      } else {
        float* pp = p.part + ((((size_t)r * p.Hkv + h) * p.splits + split) * Qg + row) * (D + 2);
#pragma unroll
        for (int c = 0; c < C::OW; c += 32) {
          uint32_t o[32];
          tmem_ld32(tmem + lane_off + C::COL_O + ocol0 + c, o);
          tmem_wait_ld();
          if (qvalid) {
#pragma unroll
            for (int k = 0; k < 32; k += 2)  // rows are (D + 2) floats: 8-byte aligned only
              *(float2*)(pp + ocol0 + c + k) = make_float2(__uint_as_float(o[k]), __uint_as_float(o[k + 1]));
          }
        }
        if (qvalid && half == 0) {
          pp[D] = m_run;
          pp[D + 1] = l_run;
        }
      }
    }
  }
  // teardown: everyone done with TMEM before the allocating warp frees it
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  }
}

// ---- host side ---------------------------------------------------------------------------
int cached_tensor_map(CUtensorMap* out, const void* base, int D, long rows);

struct UKernel {
  const void* fn;
  int smem, threads, occ;
};
template <int D, int ST, bool DB, int SW = 2>
static const UKernel& uk() {
  static const UKernel k = [] {
    using C = UCfg<D, ST, DB, SW>;
    auto kern = k_attn_umma<D, ST, DB, SW>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM);
    return UKernel{(const void*)kern, C::SMEM, C::THREADS, occ > 0 ? occ : 1};
  }();
  return k;
}

// TRIE_UMMA_DB=1 (default): double-buffered S, 4 stages, 1 CTA/SM; 0: single S, 2 stages,
// 2 CTAs/SM
static int umma_db() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TRIE_UMMA_DB");
    v = e ? atoi(e) : 1;  // r05 sweep R=16: DB=1 4.12 TB/s (b=16) vs DB=0 2.85
  }
  return v;
}
template <int D>
static const UKernel& select_ud() {
  // TRIE_UMMA_ST: ring stages (default 4; r07: 2 stages x 2 CTAs/SM starve the ring)
  static int st = -1;
  if (st < 0) {
    const char* e = getenv("TRIE_UMMA_ST");
    st = e ? atoi(e) : 4;
  }
  static int sw = -1;  // TRIE_UMMA_SW: softmax warps per TMEM sub-partition (1 or 2)
  if (sw < 0) {
    const char* e = getenv("TRIE_UMMA_SW");
    sw = e ? atoi(e) : 2;
  }
  if (sw == 1) {
    if (st >= 4) return uk<D, 4, true, 1>();
    if (st == 3) return uk<D, 3, true, 1>();
    return uk<D, 2, true, 1>();
  }
  constexpr int SW2 = (D % 64 == 0) ? 2 : 1;  // D = 96: 48 O columns per warp -> SW = 1
  if (!umma_db()) return uk<D, 2, false, SW2>();
  if (st >= 5 && UCfg<D, 5, true, SW2>::SMEM <= 227 * 1024) return uk<D, (D <= 128 ? 5 : 4), true, SW2>();
  if (st >= 4) return uk<D, 4, true, SW2>();
  if (st == 3) return uk<D, 3, true, SW2>();
  return uk<D, 2, true, SW2>();
}
static const UKernel* select_u(int D) {
  switch (D) {
    case 64: return &select_ud<64>();
    case 96: return &select_ud<96>();
    case 128: return &select_ud<128>();
  }
  return nullptr;
}

// tcgen05 path for Qg in [umma_min_qg, 128]; TRIE_UMMA_MIN_QG overrides (0 disables)
int attn_umma_min_qg() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TRIE_UMMA_MIN_QG");
    v = e ? atoi(e) : 33;
  }
  return v;
}
bool attn_umma_eligible(const AttnParams& p) {
  const int Qg = p.b_live * (p.Hq / p.Hkv);
  const int mn = attn_umma_min_qg();
  return mn > 0 && Qg >= mn && Qg <= 128 && attn_tc_shape_ok(p);
}
int attn_umma_occ(const AttnParams& p) {
  const UKernel* k = select_u(p.D);
  return k ? k->occ : 1;
}

int launch_attn_umma(const AttnParams& p, cudaStream_t s) {
  const UKernel* k = select_u(p.D);
  if (!k) return trie_set_error(TRIE_EINVAL, "tcgen05 attention: unsupported head_dim %d", p.D);
  CUtensorMap km, vm;
  const long rows = (long)p.R * p.Hkv * p.cap;
  int rc = cached_tensor_map(&km, p.k, p.D, rows);
  if (!rc) rc = cached_tensor_map(&vm, p.v, p.D, rows);
  if (rc) return rc;
  AttnParams pp = p;
  void* args[3] = {(void*)&km, (void*)&vm, (void*)&pp};
  cudaLaunchKernel(k->fn, dim3(p.Hkv, p.R, p.splits), dim3(k->threads), args, (size_t)k->smem, s);
  rc = trie_check_launch("k_attn_umma");
  if (rc) return rc;
  if (p.splits > 1) rc = launch_attn_combine_bf16(p, s);
  return rc;
}

}  // namespace trie
