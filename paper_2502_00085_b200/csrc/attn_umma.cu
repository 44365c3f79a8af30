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
// Warp roles: 0 = TMA producer, 1 = TMEM allocator + PV issuer, 2 = QK issuer, 3..10 =
// softmax / epilogue in two groups by tile parity: group e (warps 3+4e .. 6+4e) owns the
// even (e = 0) or odd (e = 1) tiles and its own accumulator O_e with its own running max
// and sum; a thread owns one query row (TMEM lane = warp % 4 quarter)
// and all 64 columns of its tiles.  The two warps on an SMSP work on consecutive tiles, so
// one's exp2 phase (MUFU) overlaps the other's TMEM load / mask / max phase (r09 trace: a
// single group ran load 200 + max 320 + exp 700 cycles per tile back to back).  O_0 and
// O_1 are merged once at the end (the in-CTA analogue of the split-K combine).  The
// running max is rescaled lazily (only when a row max grows by > 8 in log2 units).
// Rows >= Qg of the 128-row MMA are padding (Q rows zero; their warps skip the softmax).
#include <stdio.h>
#include <stdlib.h>

#include "attn_common.cuh"
#include "common.cuh"
#include "handle.h"
#include "tc_common.cuh"
#include "gather.cuh"

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

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

// S_0..S_3 | O_0 | O_1 in TMEM: tile i uses S_{i%4} (so QK(i+2) never waits for PV(i):
// r10 trace, with two S buffers each group idled ~1.1k cycles per tile on that chain);
// P (bf16, 32 columns) overwrites the first half of the S buffer it was computed from.
// K and V have separate rings with their own producers: a K tile is free as soon as QK(i)
// completes, a V tile (+ the tile's mask / depth words) only after PV(i), i.e. after the
// softmax; r10 trace: with one 33 KB stage ring the stages were held ~1.7k cycles by the
// consumers and only ~2.4 of 4 were in flight against a ~2.6k-cycle TMA latency.
template <int D, int STK, int STV>
struct UCfg {
  static_assert(STV % 2 == 0 && STV >= 4, "V stage s serves one tile parity; STV >= NSB");
  static constexpr int TILE = TC_TR * D * 2;    // one K or V tile: D/32 boxes of 64 x 64 B
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + STK * TILE;
  static constexpr int OFF_MD = OFF_V + STV * TILE;  // [STV][mask 64 x u32 | depth 64 x i32]
  static constexpr int QBYTES = 128 * D * 2;  // Q: 128 rows (padding zero), D/32 boxes
  static constexpr int OFF_Q = (OFF_MD + STV * 512 + 1023) / 1024 * 1024;
  static constexpr int OFF_X = OFF_Q + QBYTES;           // epilogue (m, l) exchange [2][4][32] f32x2
  static constexpr int OFF_BAR = OFF_X + 2 * 4 * 32 * 8;
  static constexpr int NSB = 4;                    // S buffers
  static constexpr int NBAR = 2 * STK + 2 * STV + 3 * NSB + 1;  // K/V full/empty, s_full, p_full, pv_done, app_done
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 64 + 1024;
  static constexpr int NSW = 8;                // softmax warps (2 groups x 4 sub-partitions)
  static constexpr int THREADS = (4 + NSW) * 32; // + K producer, PV, QK, V producer (last)
  static constexpr int COL_O0 = 64 * NSB, COL_O1 = 64 * NSB + D;
  static constexpr int TMEM_COLS = 512;
  static_assert(64 * NSB + 2 * D <= TMEM_COLS, "TMEM budget");
  static_assert(D % 32 == 0, "head_dim");
};

#ifndef TRIE_UMMA_TRACE
#define TRIE_UMMA_TRACE 0
#endif

// ROPE: fused a-1 (trie_attn_decode_rope), as in the narrow / wide kernels -- the softmax
// warps stage Q rotated at the beams' depths (rotate-half partners are the chunks at col
// and col + D/2) and, in the same pass, rotate and append the leaves' K/V rows of this
// CTA's tiles; both producers wait for that append before the first leaf tile.
template <int D, int STK, int STV, bool ROPE = false>
__global__ void __launch_bounds__(UCfg<D, STK, STV>::THREADS) k_attn_umma(
    const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
    const AttnParams p) {
  using C = UCfg<D, STK, STV>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* qsm = smem + C::OFF_Q;
  float2* xch = (float2*)(smem + C::OFF_X);
  uint64_t* fullK = (uint64_t*)(smem + C::OFF_BAR);
  uint64_t* emptyK = fullK + STK;
  uint64_t* fullV = emptyK + STK;
  uint64_t* emptyV = fullV + STV;
  uint64_t* s_full = emptyV + STV;
  uint64_t* p_full = s_full + C::NSB;
  uint64_t* pv_done = p_full + C::NSB;
  uint64_t* app_done = pv_done + C::NSB;
  uint32_t* tmem_slot = (uint32_t*)(app_done + 1);
  ItemInfo* info = (ItemInfo*)(tmem_slot + 4);

  const int h = blockIdx.x, r = blockIdx.y, split = blockIdx.z;
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = p.Hq / p.Hkv, Qg = p.b_live * g;
  const int n_live = min(4, (Qg + 31) / 32);  // sub-partitions holding real query rows
  if (threadIdx.x == 0) {
    for (int s = 0; s < STK; ++s) {
      mbar_init(&fullK[s], 1);
      mbar_init(&emptyK[s], 1);
    }
    for (int s = 0; s < STV; ++s) {
      mbar_init(&fullV[s], 1);
      mbar_init(&emptyV[s], 1);
    }
    // one (s_full, p_full, pv_done) triple per S buffer: a barrier's next phase always
    // needs the waiter's own progress first, so no wait can alias a later phase
    for (int e = 0; e < C::NSB; ++e) {
      mbar_init(&s_full[e], 1);
      mbar_init(&p_full[e], n_live);  // the live softmax warps of the tile's group
      mbar_init(&pv_done[e], 1);
    }
    mbar_init(app_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();  // the shared-memory setup above ran before the predecessor finished
  if (threadIdx.x < 32) item_setup(p, r, split, info);
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
#if TRIE_UMMA_TRACE
  // CTA (0,0,0) records clock() per tile into p.out (build with TRIE_UMMA_TRACE=1;
  // scripts/umma_trace.py; results are not written)
  uint32_t* trc = (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) ? (uint32_t*)p.out : nullptr;
#define TRC(i, k) do { if (trc && (i) < 400) trc[(i) * 16 + (k)] = (uint32_t)clock(); } while (0)
#else
  uint32_t* trc = nullptr;
#define TRC(i, k) do { } while (0)
#endif

  if (warp == 0 || warp == 3 + C::NSW) {
    // ============ TMA producers: warp 0 = K tiles, the last warp = V tiles + mask words ============
    const int first_leaf = ROPE ? it.N - p.b_live : INT_MAX;
    if (lane == 0) {
      const bool isv = warp != 0;
      bool appended = !ROPE;
      const size_t mbase = (size_t)r * p.cap;
      const int ns = isv ? STV : STK;
      uint64_t* fb = isv ? fullV : fullK;
      uint64_t* eb = isv ? emptyV : emptyK;
      const CUtensorMap* map = isv ? &vmap : &kmap;
      const uint32_t base = smem_u32(smem + (isv ? C::OFF_V : C::OFF_K));
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % ns;
        mbar_wait(&eb[s], ((uint32_t)(i / ns) & 1u) ^ 1u);
        TRC(i, isv ? 12 : 7);
        if (!appended && (it.tile0 + i + 1) * TC_TR > first_leaf) {
          mbar_wait(app_done, 0u);  // leaf rows written (and fenced) by warp 0's lanes 1..31
          appended = true;
        }
        const int n0 = (it.tile0 + i) * TC_TR;
        const int row = (int)attn_row(p, r, h, n0);
        // mask / depth words clamped to the [R][cap] arrays (cap % 4 == 0: 16-byte granules)
        const uint32_t mdb = isv ? (uint32_t)min(TC_TR, p.cap - n0) * 4u : 0u;
        mbar_expect_tx(&fb[s], C::TILE + 2 * mdb);
#pragma unroll
        for (int bx = 0; bx < D / TC_CW; ++bx)
          tma_load_2d(base + s * C::TILE + bx * TC_TR * 64, map, bx * TC_CW, row, &fb[s]);
        if (isv) {
          const uint32_t md = smem_u32(smem + C::OFF_MD + s * 512);
          bulk_load_1d(md, p.mask + mbase + n0, mdb, &fb[s]);
          bulk_load_1d(md + 256, p.depth + mbase + n0, mdb, &fb[s]);
        }
        TRC(i, isv ? 13 : 8);
      }
    }
  } else if (warp <= 2) {
    // ============ MMA issuers: warp 2 = QK (needs Q), warp 1 = PV ============
    // Two issuing warps so that PV(i) (which releases ring stage i) never queues behind the
    // wait for tile i+1's data that QK(i+1) needs (r08 trace: with one issuer the stage was
    // released ~1.7k cycles late).  QK(i) overwrites S_{i%4}, which holds P_{i-4}: it waits
    // for PV(i-4).  Each warp commits only its own MMAs.
    const uint32_t idesc_qk = umma_idesc(128, 64, 0);
    const uint32_t idesc_pv = umma_idesc(128, D, 1);
    if (warp == 2) {
      mbar_wait(app_done, 0u);  // Q staged (and the leaf rows appended) by the softmax warps
      tc_fence_after();
      const uint32_t qbase = smem_u32(qsm);
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % STK;
        const int sb = i % C::NSB;
        if (i >= C::NSB) mbar_wait(&pv_done[sb], (uint32_t)((i - C::NSB) / C::NSB) & 1u);
        mbar_wait(&fullK[s], (uint32_t)(i / STK) & 1u);
        tc_fence_after();
        if (lane == 0) {
          TRC(i, 5);
          const uint32_t kb = smem_u32(smem + C::OFF_K + s * C::TILE);
          const uint32_t d_s = tmem + sb * 64;
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            // K step ks: 32-column box ks/2 (8 KB apart for the 128-row Q, 4 KB for the 64-row
            // K tile), + 32 B inside the 64-byte swizzled row for odd steps; SBO = 8 rows = 512 B
            const uint64_t a = umma_desc_sw64(qbase + (ks >> 1) * 128 * 64 + (ks & 1) * 32, 16, 512);
            const uint64_t b = umma_desc_sw64(kb + (ks >> 1) * TC_TR * 64 + (ks & 1) * 32, 16, 512);
            umma_ss(d_s, a, b, idesc_qk, ks > 0);
          }
          umma_commit(&s_full[sb]);
          umma_commit(&emptyK[s]);  // K tile free once QK(i) has read it
        }
        __syncwarp();
      }
    } else {
      for (int i = 0; i < ntiles; ++i) {
        const int sb = i % C::NSB, s = i % STV;
        mbar_wait(&p_full[sb], (uint32_t)(i / C::NSB) & 1u);
        if (lane == 0) TRC(i, 6);
        mbar_wait(&fullV[s], (uint32_t)(i / STV) & 1u);
        tc_fence_after();
        if (lane == 0) {
          TRC(i, 14);
          const uint32_t vb = smem_u32(smem + C::OFF_V + s * C::TILE);
          const uint32_t colp = sb * 64;                          // P_i over S_i
          const uint32_t colo = (i & 1) ? C::COL_O1 : C::COL_O0;  // group accumulator
#pragma unroll
          for (int kc = 0; kc < TC_TR / 16; ++kc) {
            // V tile as MN-major B: 16 rows per K step = two 8-row atoms (1024 B); the
            // 32-column boxes are LBO = 4096 B apart, the 8-row atoms SBO = 512 B apart
            const uint64_t b = umma_desc_sw64(vb + kc * 1024, TC_TR * 64, 512);
            umma_ts(tmem + colo, tmem + colp + kc * 8, b, idesc_pv, (i >= 2 || kc > 0) ? 1u : 0u);
          }
          umma_commit(&emptyV[s]);
          umma_commit(&pv_done[sb]);
        }
        __syncwarp();
      }
    }
  } else {
    // ===================== softmax / epilogue warps =====================
    const int sp = warp & 3;                  // TMEM sub-partition of this warp
    const int grp = (warp - 3) / 4;           // tile parity this warp handles
    const int row = sp * 32 + lane;           // query row (MMA M index)
    const int tid = threadIdx.x - 96;
    {  // Q -> smem, 64B-swizzled K-major boxes of [128 rows][32 cols]; padding rows zero
      const __nv_bfloat16* q = (const __nv_bfloat16*)p.q;
      const int chunks = 128 * (D / 8);
      const float inv_g = 1.f / (float)g;  // exact: m < 128, g <= 128
      if constexpr (ROPE) {  // chunk pairs (col, col + D/2), rotated like trie_rope_kv_append
        constexpr int HALF = D / 2;
        for (int c = tid; c < 128 * (HALF / 8); c += C::NSW * 32) {
          const int m = c / (HALF / 8), col = (c % (HALF / 8)) * 8;
          int4 y1 = make_int4(0, 0, 0, 0), y2 = make_int4(0, 0, 0, 0);
          if (m < Qg) {
            const int j = __float2int_rz(((float)m + 0.5f) * inv_g);
            const __nv_bfloat16* src = q + (((size_t)r * p.b_live + j) * p.Hq + h * g + m - j * g) * D;
            const int4 a = *(const int4*)(src + col), b2 = *(const int4*)(src + HALF + col);
            const float4* tb = (const float4*)(p.rope_tab + ((size_t)r * p.b_live + j) * HALF + col);
            const __nv_bfloat162* a2 = (const __nv_bfloat162*)&a;
            const __nv_bfloat162* bb = (const __nv_bfloat162*)&b2;
            __nv_bfloat162* o1 = (__nv_bfloat162*)&y1;
            __nv_bfloat162* o2 = (__nv_bfloat162*)&y2;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float4 tt = __ldg(tb + u);
              const float2 x1 = __bfloat1622float2(a2[u]), x2 = __bfloat1622float2(bb[u]);
              o1[u] = __floats2bfloat162_rn(x1.x * tt.x - x2.x * tt.y, x1.y * tt.z - x2.y * tt.w);
              o2[u] = __floats2bfloat162_rn(x2.x * tt.x + x1.x * tt.y, x2.y * tt.z + x1.y * tt.w);
            }
          }
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int cc = col + hh * HALF;
            const int box = cc / TC_CW;
            const uint32_t o = (uint32_t)m * 64u + (uint32_t)(cc % TC_CW) * 2u;
            *(int4*)(qsm + box * 128 * 64 + (o ^ (((o >> 7) & 3u) << 4))) = hh ? y2 : y1;
          }
        }
      }
      for (int c = ROPE ? chunks : tid; c < chunks; c += C::NSW * 32) {
        const int m = c / (D / 8), col = (c % (D / 8)) * 8;
        int4 v = make_int4(0, 0, 0, 0);
        if (m < Qg) {
          const int j = __float2int_rz(((float)m + 0.5f) * inv_g);
          v = *(const int4*)(q + (((size_t)r * p.b_live + j) * p.Hq + h * g + m - j * g) * D + col);
        }
        const int box = col / TC_CW;
        const uint32_t o = (uint32_t)m * 64u + (uint32_t)(col % TC_CW) * 2u;
        *(int4*)(qsm + box * 128 * 64 + (o ^ (((o >> 7) & 3u) << 4))) = v;
      }
      if constexpr (ROPE)  // the leaves' K/V rows of this CTA's tiles (fused a-1), then fenced
        append_leaves_rope_work<D>(p, r, h, it.tile0 * TC_TR, (it.tile0 + ntiles) * TC_TR, tid,
                                   C::NSW * 32, it.N - p.b_live);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      // softmax warps only (one call site); then one arrival publishes Q (and, fused,
      // every softmax thread's fenced append) to the QK issuer and the producers
      __syncwarp();
      asm volatile("bar.sync 1, %0;" ::"r"(C::NSW * 32));
      if (tid == 0) mbar_arrive(app_done);
    }
    if (sp < n_live) {  // warps of padding-only sub-partitions have nothing to do
      const bool qvalid = row < Qg;
      const int beam = qvalid ? row / g : 0;
      const size_t mbase = (size_t)r * p.cap;
      const int lod = (p.window > 0 && qvalid) ? p.depth[mbase + p.leaf[r * TRIE_MAX_BEAMS + beam]] - p.window + 1 : INT_MIN;
      const float sc = p.scale_log2;
      const int fast_end = min(it.t, it.N) / TC_TR;
      const uint32_t lane_off = (uint32_t)(sp * 32) << 16;
      const uint32_t ocol = grp ? C::COL_O1 : C::COL_O0;
      const bool tr = trc && (warp == 4 || warp == 8) && lane == 0;  // sub-partition 0, both groups
      float m_run = -INFINITY, l_run = 0.f;
      for (int i = grp; i < ntiles; i += 2) {
        const int sb = i % C::NSB;
        const uint32_t scol = sb * 64;
        const int tile = it.tile0 + i;
        const bool slow = !(tile >= it.fast_from && tile < fast_end);  // warp-uniform
        if (tr) TRC(i, 0);
        mbar_wait(&s_full[sb], (uint32_t)(i / C::NSB) & 1u);
        if (tr) TRC(i, 1);
        // the V transaction carries the tile's mask / depth words.  Skipping its phase on
        // fast tiles is safe: s_full(i) implies PV(i-4), hence fullV(i-4) and every earlier
        // phase of this stage, complete (STV >= 4), so the wait below never aliases
        if (slow) mbar_wait(&fullV[i % STV], (uint32_t)(i / STV) & 1u);
        tc_fence_after();
        if (tr) TRC(i, 2);
        // raw S (the scale is folded into the exponent FFMA)
        float x[64];
        {
          uint32_t a[32];
          tmem_ld32(tmem + lane_off + scol, a);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) x[k] = __uint_as_float(a[k]);
          tmem_ld32(tmem + lane_off + scol + 32, a);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) x[32 + k] = __uint_as_float(a[k]);
        }
        if (tr) TRC(i, 9);
        const int n0 = tile * TC_TR;
        if (slow) {
          const uint32_t* tmask = (const uint32_t*)(smem + C::OFF_MD + (i % STV) * 512);
          const int* tdep = (const int*)(smem + C::OFF_MD + (i % STV) * 512 + TC_TR * 4);
#pragma unroll
          for (int k = 0; k < 64; ++k) {
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
          for (int k = 8 + u; k < 64; k += 8) v = fmaxf(v, x[k]);
          mx[u] = v;
        }
        float tmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                           fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        if (tr) TRC(i, 10);
        tmax *= sc;  // log2 units (sc > 0: the max commutes with the scaling)
        float alpha = 1.f;
        bool rescale = false;
        // lazy rescale: keep the running max unless the tile max exceeds it by > 8 (log2)
        if (tmax > m_run + 8.f || (m_run == -INFINITY && tmax > -INFINITY)) {
          alpha = (m_run == -INFINITY) ? 0.f : ex2(m_run - tmax);
          rescale = m_run != -INFINITY;
          m_run = tmax;
          l_run *= alpha;
        }
        const float nmu = m_run == -INFINITY ? 0.f : -m_run;  // all masked: ex2(-inf) = 0
        uint32_t pk[32];
        float ps[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) ps[u] = 0.f;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float p0 = ex2(fmaf(x[2 * k], sc, nmu)), p1 = ex2(fmaf(x[2 * k + 1], sc, nmu));
          ps[k & 7] += p0 + p1;
          pk[k] = pack_bf16(p0, p1);
        }
        l_run += ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
        if (tr) TRC(i, 11);
        // P_i overwrites S_i, whose previous occupant P_{i-4} was read by PV(i-4) before
        // QK(i) was issued.  Only an O_grp rescale (rare) waits for this group's last PV.
        if (__any_sync(0xffffffffu, rescale)) {
          if (i >= 2) {
            mbar_wait(&pv_done[(i - 2) % C::NSB], (uint32_t)((i - 2) / C::NSB) & 1u);
            tc_fence_after();
          }
#pragma unroll
          for (int c = 0; c < D; c += 32) {
            uint32_t o[32];
            tmem_ld32(tmem + lane_off + ocol + c, o);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
            tmem_st32(tmem + lane_off + ocol + c, o);
          }
        }
        if (tr) TRC(i, 3);
        tmem_st32(tmem + lane_off + scol, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
        if (tr) TRC(i, 4);
      }
      // ---- epilogue: merge (O_0, m_0, l_0) and (O_1, m_1, l_1); group e writes columns
      // [e*D/2, (e+1)*D/2) of every row of its sub-partition ----
      const int last = ((ntiles - 1 - grp) >> 1) * 2 + grp;  // this group's last tile
      if (last >= 0 && last < ntiles) {
        mbar_wait(&pv_done[last % C::NSB], (uint32_t)(last / C::NSB) & 1u);
        tc_fence_after();
      }
      float2* xb = xch + sp * 64;
      xb[grp * 32 + lane] = make_float2(m_run, l_run);
      __syncwarp();
      asm volatile("bar.sync %0, 64;" ::"r"(2 + sp));
      const float2 ot = xb[(1 - grp) * 32 + lane];
      // the other group's last PV must be complete too before O_{1-grp} is read
      const int olast = ((ntiles - 1 - (1 - grp)) >> 1) * 2 + (1 - grp);
      if (olast >= 0 && olast < ntiles) {
        mbar_wait(&pv_done[olast % C::NSB], (uint32_t)(olast / C::NSB) & 1u);
        tc_fence_after();
      }
      const float m0 = grp ? ot.x : m_run, l0 = grp ? ot.y : l_run;
      const float m1 = grp ? m_run : ot.x, l1 = grp ? l_run : ot.y;
      const float m = fmaxf(m0, m1);
      const float a0 = m0 == -INFINITY ? 0.f : ex2(m0 - m), a1 = m1 == -INFINITY ? 0.f : ex2(m1 - m);
      const float l = l0 * a0 + l1 * a1;
      const bool has0 = ntiles > 0, has1 = ntiles > 1;  // else O_e is uninitialised TMEM
      const int j = beam, ii = row % g;
      constexpr int HD = D / 2;
      const int c0 = grp * HD;
      const bool gat = p.ga.world > 0 && p.splits == 1;  // NEXT-4 fused all-gather
      const uint32_t ghalf = gat ? gather_half(p) : 0u;
      if (!trc && !it.done) {  // NEXT-3: a done request (all beams finished) writes nothing
        if (p.splits == 1) {
          __nv_bfloat16* op = (__nv_bfloat16*)p.out + (((size_t)r * p.b_live + j) * p.Hq + h * g + ii) * D;
          const float inv = l > 0.f ? 1.f / l : 0.f;
          const float f0 = a0 * inv, f1 = a1 * inv;
#pragma unroll
          for (int c = 0; c < HD; c += 16) {
            uint32_t o0[16], o1[16];
            tmem_ld16(tmem + lane_off + C::COL_O0 + c0 + c, o0);
            tmem_ld16(tmem + lane_off + C::COL_O1 + c0 + c, o1);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              o0[k] = has0 ? o0[k] : 0u;
              o1[k] = has1 ? o1[k] : 0u;
            }
            if (qvalid) {
              uint32_t w[8];
#pragma unroll
              for (int k = 0; k < 8; ++k)
                w[k] = pack_bf16(__uint_as_float(o0[2 * k]) * f0 + __uint_as_float(o1[2 * k]) * f1,
                                 __uint_as_float(o0[2 * k + 1]) * f0 + __uint_as_float(o1[2 * k + 1]) * f1);
              const int4 v0 = make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
              const int4 v1 = make_int4((int)w[4], (int)w[5], (int)w[6], (int)w[7]);
              *(int4*)(op + c0 + c) = v0;
              *(int4*)(op + c0 + c + 8) = v1;
              if (gat) {
                gather_st128(p, ghalf, r, j, h * g + ii, c0 + c, v0);
                gather_st128(p, ghalf, r, j, h * g + ii, c0 + c + 8, v1);
              }
            }
          }
          if (qvalid && grp == 0) {
            if (l == 0.f) latch(p.status, TRIE_ST_EMPTY_ROW);
            if (p.lse)
              p.lse[((size_t)r * p.b_live + j) * p.Hq + h * g + ii] =
                  l > 0.f ? (m + log2f(l)) * 0.69314718055994531f : -INFINITY;
          }
        } else {
          float* pp = p.part + ((((size_t)r * p.Hkv + h) * p.splits + split) * Qg + row) * (D + 2);
#pragma unroll
          for (int c = 0; c < HD; c += 16) {
            uint32_t o0[16], o1[16];
            tmem_ld16(tmem + lane_off + C::COL_O0 + c0 + c, o0);
            tmem_ld16(tmem + lane_off + C::COL_O1 + c0 + c, o1);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              o0[k] = has0 ? o0[k] : 0u;
              o1[k] = has1 ? o1[k] : 0u;
            }
            if (qvalid) {
#pragma unroll
              for (int k = 0; k < 16; k += 2)  // rows are (D + 2) floats: 8-byte aligned only
                *(float2*)(pp + c0 + c + k) =
                    make_float2(__uint_as_float(o0[k]) * a0 + __uint_as_float(o1[k]) * a1,
                                __uint_as_float(o0[k + 1]) * a0 + __uint_as_float(o1[k + 1]) * a1);
            }
          }
          if (qvalid && grp == 0) {
            pp[D] = m;
            pp[D + 1] = l;
          }
        }
      }
      if (gat) {  // the 2 * n_live writer warps meet at named barrier 6; one lane arrives
        __syncwarp();
        asm volatile("bar.sync 6, %0;" ::"r"(2 * n_live * 32) : "memory");
        if (sp == 0 && grp == 0 && lane == 0) gather_arrive(p);
      }
    }
  }
#undef TRC
  // teardown: everyone done with TMEM before the allocating warp frees it
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  }
}

// ---- host side ---------------------------------------------------------------------------

struct UKernel {
  const void* fn;
  int smem, threads, occ;
};
template <int D, int STK, int STV, bool ROPE = false>
static const UKernel& uk() {
  static const UKernel k = [] {
    using C = UCfg<D, STK, STV>;
    auto kern = k_attn_umma<D, STK, STV, ROPE>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM);
    return UKernel{(const void*)kern, C::SMEM, C::THREADS, occ > 0 ? occ : 1};
  }();
  return k;
}

template <int D>
static const UKernel& select_ud(bool rope) {
  if (rope) return uk<D, 4, 6, true>();  // fused a-1: the default stage split only
  // TRIE_UMMA_ST: V ring stages (4, 6 = default, 8; the K ring has 4, 3 with 8 V stages)
  static int st = -1;
  if (st < 0) {
    const char* e = getenv("TRIE_UMMA_ST");
    st = e ? atoi(e) : 6;
  }
  if (st >= 8 && UCfg<D, 3, 8>::SMEM <= 227 * 1024) return uk<D, 3, 8>();
  if (st >= 6) return uk<D, 4, 6>();
  return uk<D, 4, 4>();
}
static const UKernel* select_u(int D, bool rope = false) {
  switch (D) {
    case 64: return &select_ud<64>(rope);
    case 96: return &select_ud<96>(rope);
    case 128: return &select_ud<128>(rope);
  }
  return nullptr;
}

// Which query groups take the tcgen05 kernel: Qg >= 33 (mma.sync is tensor-pipe bound
// there).  Round 1 also sent Qg >= 9 with >= 1024 rows per request here (measured at job
// steps 5-35); on the mid-job window (r2r, round 2) the mma.sync kernels with split-K over
// all 148 SMs are faster per launch -- sweep b = 4 (Qg 16) 101.2 vs 104.8 us, b = 8 (Qg
// 32) 103.0 vs 114.2 us, Mistral shard (Qg 16) 60.4 vs 63.4 us -- while the tcgen05 grid
// of R x Hkv = 128 one-CTA-per-SM items leaves 20 SMs idle.
// TRIE_UMMA_MIN_QG = n overrides with the plain rule Qg >= n (0 disables).
int attn_umma_min_qg() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("TRIE_UMMA_MIN_QG");
    v = e ? atoi(e) : -1;
  }
  return v;
}
bool attn_umma_eligible(const AttnParams& p) {
  const int Qg = p.b_live * (p.Hq / p.Hkv);
  if (Qg > 128 || !attn_tc_shape_ok(p)) return false;
  const int mn = attn_umma_min_qg();
  if (mn >= 0) return mn > 0 && Qg >= mn;
  return Qg >= 33;
}
int attn_umma_occ(const AttnParams& p) {
  const UKernel* k = select_u(p.D);
  return k ? k->occ : 1;
}

int launch_attn_umma(const AttnParams& p, cudaStream_t s) {
  const UKernel* k = select_u(p.D, p.rope != 0);
  if (!k) return trie_set_error(TRIE_EINVAL, "tcgen05 attention: unsupported head_dim %d", p.D);
  CUtensorMap km, vm;
  const long rows = attn_pool_rows(p);
  int rc = cached_tensor_map(&km, p.k, p.D, rows);
  if (!rc) rc = cached_tensor_map(&vm, p.v, p.D, rows);
  if (rc) return rc;
  AttnParams pp = p;
  void* args[3] = {(void*)&km, (void*)&vm, (void*)&pp};
  launch_k_ptr(k->fn, dim3(p.Hkv, p.R, p.splits), dim3(k->threads), (size_t)k->smem, s, args);
  rc = trie_check_launch("k_attn_umma");
  if (rc) return rc;
  if (p.splits > 1) rc = launch_attn_combine_bf16(p, s);
  return rc;
}

}  // namespace trie
