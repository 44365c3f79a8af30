// trie_attn_decode, bf16 tensor-core paths (sm_100a): TMA-fed, mbarrier-pipelined
// flash-decode over the shared trie KV pool (§3.3; Alg. 3 mask P:165-186).
//
// Common structure.  One CTA per (KV head h, request r, split).  Warp 0 is the producer:
// one elected lane streams 64-slot tiles of K and V (the head-major pool makes a tile a
// contiguous 2-D box) with cp.async.bulk.tensor (TMA, 64-byte swizzle) plus the tile's
// beam_mask / depth words with 1-D bulk copies into an S-stage ring guarded by
// full/empty mbarriers.  Every unique KV row is read from HBM exactly once per
// (request, KV head) and feeds all Qg = b_live * (Hq/Hkv) queries of the head (GQA
// grouping + trie sharing).  Masked keys get -inf before the online softmax (exact
// exclusion, reading R22); tiles that lie entirely in the prompt and inside every
// beam's window skip the mask (Alg. 3 l.2: prompt columns are open to every beam).
//
// k_attn_narrow (Qg <= 16): ONE consumer warp owns the whole item.  KV rows sit on the
//   MMA M dimension and queries on N (8 per n-tile), so small beam counts waste at most
//   half an n-tile instead of 3/4 of an m-tile: S^T = K Q^T (A = K tile via ldmatrix,
//   B = Q from registers), P^T is turned into the B operand of O^T = V^T P^T with
//   movmatrix.trans, A = V^T via ldmatrix.trans.  48 ldmatrix.x4 per 64-row tile read
//   the tile exactly once.
// k_attn_wide (16 < Qg <= 128): MT = ceil(Qg/16) consumer warps, warp w owns query
//   m-tile w over the full tile rows: S = Q K^T (A = Q registers, B = K via ldmatrix),
//   P from the accumulators (FA2 layout), O += P V (B = V via ldmatrix.trans).
// No cross-warp merge in either variant; split partials go to k_attn_combine.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <float.h>
#include <stdio.h>
#include <stdlib.h>

#include "attn_common.cuh"
#include "common.cuh"
#include "handle.h"
#include "tc_common.cuh"
#include "gather.cuh"

namespace trie {

// Experiment build only (TRIE_BUILD_DEFINES="TRIE_ATTN_TRACE=1", scripts/attn_trace.py):
// %globaltimer stamps per CTA of the narrow / wide kernels -- [0] start, [1] setup done,
// [2] first tile seen by consumer warp 0, [3] last tile done, [4] epilogue done, [5] the
// producer issued its last tile, [6] smid, [7] tiles.  Results are still written.
#ifdef TRIE_ATTN_TRACE
__device__ unsigned long long g_attn_trace[8 * 65536];
__device__ __forceinline__ void attn_trc(int k, unsigned long long v = 0) {
  const size_t cta = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  if (cta >= 65536) return;
  if (k != 6 && k != 7) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  g_attn_trace[cta * 8 + k] = v;
}
#define ATTN_TRC(cond, k, ...) do { if (cond) attn_trc(k, ##__VA_ARGS__); } while (0)
#else
#define ATTN_TRC(cond, k, ...) do { } while (0)
#endif

// =========================================================================================
// narrow: Qg <= 8 * NQ (NQ in {1, 2}); CTA = producer warp + one consumer warp
// =========================================================================================
template <int D, int NQ, int ST, bool ROPE = false>
struct NarrowCfg {
  static constexpr int STAGES = ST;
  using RG = Ring<D, STAGES>;
  static constexpr int KS = D / 16;     // k-steps of S^T (over D)
  static constexpr int DM = D / 16;     // m-tiles of O^T (over D)
  // epilogue staging [8*NQ][D+4] floats aliases the ring (all tiles consumed by then)
  static_assert(NQ * 8 * (D + 4) * 4 <= RG::RING_BYTES, "staging must fit in the ring");
  static constexpr int OFF_BAR = RG::RING_BYTES;
  static constexpr int SMEM = OFF_BAR + 128 + 1024;
  static_assert(2 * ST * 8 + 8 + (int)sizeof(ItemInfo) <= 128, "barrier area");
};

template <int D, int NQ, int ST, bool ROPE = false>
__global__ void __launch_bounds__(64) k_attn_narrow(const __grid_constant__ CUtensorMap kmap,
                                                    const __grid_constant__ CUtensorMap vmap,
                                                    const AttnParams p,
                                                    const __grid_constant__ CUtensorMap kmh,
                                                    const __grid_constant__ CUtensorMap vmh) {
  using C = NarrowCfg<D, NQ, ST, ROPE>;
  using RG = typename C::RG;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  float* stage_out = (float*)smem;  // epilogue only
  uint64_t* full = (uint64_t*)(smem + C::OFF_BAR);
  uint64_t* empty = full + C::STAGES;
  uint64_t* app_done = empty + C::STAGES;
  ItemInfo* info = (ItemInfo*)(app_done + 1);

  const int h = blockIdx.x, r = blockIdx.y, split = blockIdx.z;
  pdl_trigger();
  ATTN_TRC(threadIdx.x == 0, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(app_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // prompt-only tiles loaded before the wait (see AttnParams::pre_tiles)
  const int npre = split == 0 ? min(p.pre_tiles, C::STAGES) : 0;
  if (threadIdx.x == 0 && npre > 0)
    prefetch_prompt_tiles<D, C::STAGES>(&kmap, &vmap, p, r, h, ring, full, npre);
  pdl_wait();  // the shared-memory setup above ran before the predecessor finished
  if (warp == 0) {
    // item setup, published to the consumers by a named barrier: they load (and rotate)
    // their queries meanwhile instead of waiting for it
    item_setup(p, r, split, info);
    __syncwarp();
    const ItemInfo it = *info;
    __threadfence_block();
    asm volatile("bar.arrive 2, %0;" ::"r"(64) : "memory");
#ifdef TRIE_ATTN_TRACE
    if (threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      attn_trc(1);
      attn_trc(6, smid);
      attn_trc(7, (unsigned long long)it.ntiles);
    }
#endif
    if constexpr (ROPE) {
      // lane 0 fills the ring with leaf-free tiles while lanes 1..31 append the leaves' K/V
      // rows; after the reconvergence lane 0 streams the rest, the append already done (no
      // reliance on the scheduler interleaving a spinning lane 0 with the append; r81:
      // timing-neutral vs appending after lane 0's stream)
      const int first_leaf = it.N - p.b_live;
      int fill = min(C::STAGES, it.ntiles);
      while (fill > npre && (it.tile0 + fill) * TC_TR > first_leaf) --fill;
      if (lane == 0)
        producer_loop<D, C::STAGES>(&kmap, &vmap, p, r, h, it, ring, full, empty, nullptr,
                                    INT_MAX, npre, fill, nullptr, p.half_tiles ? &kmh : nullptr, &vmh);
      else
        append_leaves_rope<D>(p, r, h, it.tile0 * TC_TR, (it.tile0 + it.ntiles) * TC_TR, lane,
                              app_done, first_leaf);
      __syncwarp();
      if (lane == 0)
        producer_loop<D, C::STAGES>(&kmap, &vmap, p, r, h, it, ring, full, empty, app_done,
                                    first_leaf, max(fill, npre), INT_MAX, nullptr, p.half_tiles ? &kmh : nullptr, &vmh);
    } else if (lane == 0) {
      producer_loop<D, C::STAGES>(&kmap, &vmap, p, r, h, it, ring, full, empty, nullptr, INT_MAX,
                                  npre, INT_MAX, nullptr, p.half_tiles ? &kmh : nullptr, &vmh);
    }
    if (it.done && lane == 0)  // no tile is consumed: let the pre-wait loads land before exit
      for (int i = 0; i < npre; ++i) mbar_wait(&full[i], 0u);
    ATTN_TRC(lane == 0, 5);
    return;
  }
  // ===== consumer warp =====
  // Waits for the item setup BEFORE loading Q: overlapping the two (as k_attn_wide does)
  // measured 4.5% slower on the Phi workload (r34 A/B, 16.01k vs 16.76k request-steps/s;
  // re-checked r72 with TRIE_NARROW_QOVERLAP builds: 16.91k vs 17.56k).
#ifndef TRIE_NARROW_QOVERLAP  // experiment builds: load Q while warp 0 runs the setup
  asm volatile("bar.sync 2, 64;" ::: "memory");  // item setup published by warp 0
#endif
  const int g = p.Hq / p.Hkv, Qg = p.b_live * g;
  const int gq = lane >> 2, cq = lane & 3;
  const size_t mbase = (size_t)r * p.cap;
  constexpr int HALF = D / 2;
  (void)HALF;
  // queries held by this thread in the S^T / O^T fragments: columns 2cq, 2cq+1 of each n-tile
  int beam[NQ][2], lod[NQ][2];
  bool qok[NQ][2];
  uint32_t bbit[NQ][2];  // this query's beam bit (0 for padding queries)
#pragma unroll
  for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int m = nq * 8 + cq * 2 + e;
      qok[nq][e] = m < Qg;
      beam[nq][e] = m < Qg ? m / g : 0;
      bbit[nq][e] = m < Qg ? 1u << beam[nq][e] : 0u;
      lod[nq][e] = INT_MIN;
      if (p.window > 0 && m < Qg)
        lod[nq][e] = p.depth[mbase + p.leaf[r * TRIE_MAX_BEAMS + beam[nq][e]]] - p.window + 1;
    }
  // Q as the B operand (B[k = d][n = query]): b0 = Q[query gq][ks*16 + 2cq..], b1 = +8
  uint32_t qb[NQ][C::KS][2];
  {
    const __nv_bfloat16* q = (const __nv_bfloat16*)p.q;
#pragma unroll
    for (int nq = 0; nq < NQ; ++nq) {
      const int m = nq * 8 + gq;
      const __nv_bfloat16* src = nullptr;
      if (m < Qg) src = q + (((size_t)r * p.b_live + m / g) * p.Hq + h * g + m % g) * D;
#pragma unroll
      for (int ks = 0; ks < C::KS; ++ks)
#pragma unroll
        for (int hi = 0; hi < 2; ++hi)
          qb[nq][ks][hi] = src ? *(const uint32_t*)(src + ks * 16 + hi * 8 + cq * 2) : 0u;
      if constexpr (ROPE) {
        // rotate-half at the beam's depth, rounded to bf16 like trie_rope_kv_append: the
        // partner of column c < D/2 is c + D/2, held by this thread in k-step ks + KS/2 (as in
        // k_attn_wide; r83: rotating with per-element partner loads cost ~3 us per Phi launch)
        static_assert(C::KS % 2 == 0, "head_dim must be a multiple of 32 for the fused RoPE");
        if (src) {
          const int j = m / g;
#pragma unroll
          for (int ks = 0; ks < C::KS / 2; ++ks)
#pragma unroll
            for (int hi = 0; hi < 2; ++hi) {
              const int col = ks * 16 + hi * 8 + cq * 2;  // < D/2
              const float4 tt = __ldg((const float4*)(p.rope_tab + ((size_t)r * p.b_live + j) * HALF + col));
              const float2 x1 = __bfloat1622float2(*(const __nv_bfloat162*)&qb[nq][ks][hi]);
              const float2 x2 = __bfloat1622float2(*(const __nv_bfloat162*)&qb[nq][ks + C::KS / 2][hi]);
              qb[nq][ks][hi] = pack_bf16(x1.x * tt.x - x2.x * tt.y, x1.y * tt.z - x2.y * tt.w);
              qb[nq][ks + C::KS / 2][hi] = pack_bf16(x2.x * tt.x + x1.x * tt.y, x2.y * tt.z + x1.y * tt.w);
            }
        }
      }
    }
  }
#ifdef TRIE_NARROW_QOVERLAP
  asm volatile("bar.sync 2, 64;" ::: "memory");
#endif
  const ItemInfo it = *info;
  float o[C::DM][NQ][4];
#pragma unroll
  for (int dm = 0; dm < C::DM; ++dm)
#pragma unroll
    for (int nq = 0; nq < NQ; ++nq) o[dm][nq][0] = o[dm][nq][1] = o[dm][nq][2] = o[dm][nq][3] = 0.f;
  float mq[NQ][2], lq[NQ][2];
#pragma unroll
  for (int nq = 0; nq < NQ; ++nq) mq[nq][0] = mq[nq][1] = -INFINITY, lq[nq][0] = lq[nq][1] = 0.f;
  const float sc = p.scale_log2;
  const int fast_end = min(it.t, it.N) / TC_TR;

  for (int i = 0; i < it.ntiles; ++i) {
    const int s = i % C::STAGES;
    mbar_wait(&full[s], (uint32_t)(i / C::STAGES) & 1u);
    ATTN_TRC(i == 0 && lane == 0, 2);
    const uint8_t* st = ring + s * RG::STAGE_BYTES;
    const uint32_t kbase = smem_u32(st), vbase = smem_u32(st + RG::TILE_BYTES);
    const int tile = it.tile0 + i;
    const int n0 = tile * TC_TR;
    const bool fast = tile >= it.fast_from && tile < fast_end;
    // ---- S^T = K Q^T : 4 row groups of 16 ----
    float sacc[4][NQ][4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
#pragma unroll
      for (int nq = 0; nq < NQ; ++nq) sacc[mt][nq][0] = sacc[mt][nq][1] = sacc[mt][nq][2] = sacc[mt][nq][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < C::KS; ++ks) {
        const int row = mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int col = ks * 16 + (lane >> 4) * 8;
        uint32_t a0, a1, a2, a3;
        ldsm_x4(kbase + tile_off(row, col), a0, a1, a2, a3);
#pragma unroll
        for (int nq = 0; nq < NQ; ++nq) mma_bf16(sacc[mt][nq], a0, a1, a2, a3, qb[nq][ks][0], qb[nq][ks][1]);
      }
    }
    // ---- scale, mask, running max per query column ----
    float tmax[NQ][2];
#pragma unroll
    for (int nq = 0; nq < NQ; ++nq) tmax[nq][0] = tmax[nq][1] = -INFINITY;
    if (fast) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float v = qok[nq][e & 1] ? sacc[mt][nq][e] : -INFINITY;
            sacc[mt][nq][e] = v;
            tmax[nq][e & 1] = fmaxf(tmax[nq][e & 1], v);
          }
    } else {
      const uint32_t* tmask = (const uint32_t*)(st + 2 * RG::TILE_BYTES);
      const int* tdep = (const int*)(st + 2 * RG::TILE_BYTES + TC_TR * 4);
      const bool win = p.window > 0;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {  // fragment rows gq (hh=0) and gq+8 (hh=1)
          const int lr = mt * 16 + gq + hh * 8;
          const int n = n0 + lr;
          // visible-beam word of the row: none past N, all on the prompt (Alg. 3 l.2)
          const uint32_t vis = n >= it.N ? 0u : (n < it.t ? ~0u : tmask[lr]);
          const int dep = win ? tdep[lr] : 0;
#pragma unroll
          for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const bool ok = (vis & bbit[nq][e]) != 0u && dep >= lod[nq][e];
              const float v = ok ? sacc[mt][nq][hh * 2 + e] : -INFINITY;
              sacc[mt][nq][hh * 2 + e] = v;
              tmax[nq][e] = fmaxf(tmax[nq][e], v);
            }
        }
    }
    float alpha[NQ][2];
#pragma unroll
    for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float v = tmax[nq][e];
        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
        const float mnew = fmaxf(mq[nq][e], v * sc);  // scores are raw until here (sc > 0)
        alpha[nq][e] = (mnew == -INFINITY) ? 1.f : ex2_ftz(mq[nq][e] - mnew);
        mq[nq][e] = mnew;
        lq[nq][e] *= alpha[nq][e];
      }
    float msafe[NQ][2];
#pragma unroll
    for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
      for (int e = 0; e < 2; ++e) msafe[nq][e] = mq[nq][e] == -INFINITY ? 0.f : mq[nq][e];
    // ---- P^T -> B fragments of O^T = V^T P^T (movmatrix.trans) ----
    uint32_t pb[4][NQ][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nq = 0; nq < NQ; ++nq) {
        float pv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float x = sacc[mt][nq][e];
          // -inf - m -> 2^-inf = 0 with one MUFU (m is finite once any key of the query was
          // visible; before that every score is -inf and msafe = 0)
          pv[e] = ex2_ftz(fmaf(x, sc, -msafe[nq][e & 1]));
          lq[nq][e & 1] += pv[e];
        }
        pb[mt][nq][0] = movm_t(pack_bf16(pv[0], pv[1]));  // rows gq      -> B rows 0..7
        pb[mt][nq][1] = movm_t(pack_bf16(pv[2], pv[3]));  // rows gq + 8  -> B rows 8..15
      }
    // the running max of a query rarely grows after the first tiles: skip the exact no-op
    // multiply by alpha = 1 warp-uniformly (bit-identical; r2e3: Phi 114.8 -> 111.5 us)
    bool grew = false;
#pragma unroll
    for (int nq = 0; nq < NQ; ++nq) grew |= alpha[nq][0] != 1.f || alpha[nq][1] != 1.f;
    if (__any_sync(0xffffffffu, grew)) {
#pragma unroll
      for (int dm = 0; dm < C::DM; ++dm)
#pragma unroll
        for (int nq = 0; nq < NQ; ++nq) {
          o[dm][nq][0] *= alpha[nq][0];
          o[dm][nq][1] *= alpha[nq][1];
          o[dm][nq][2] *= alpha[nq][0];
          o[dm][nq][3] *= alpha[nq][1];
        }
    }
    // ---- O^T += V^T P^T : A = V^T via ldmatrix.trans (16 d x 16 rows) ----
#pragma unroll
    for (int dm = 0; dm < C::DM; ++dm)
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        const int mi = lane >> 3;
        const int row = kc * 16 + (lane & 7) + (mi >> 1) * 8;
        const int col = dm * 16 + (mi & 1) * 8;
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(vbase + tile_off(row, col), a0, a1, a2, a3);
#pragma unroll
        for (int nq = 0; nq < NQ; ++nq) mma_bf16(o[dm][nq], a0, a1, a2, a3, pb[kc][nq][0], pb[kc][nq][1]);
      }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  ATTN_TRC(lane == 0, 3);
  const bool gat = p.ga.world > 0 && p.splits == 1;  // NEXT-4: fused all-gather
  if (it.done) {  // NEXT-3: finished request, output not written
    if (gat && lane == 0) gather_arrive(p);
    return;
  }
  // ---- epilogue: column sums over the 8 lanes of a column quad, transpose via smem ----
#pragma unroll
  for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      float v = lq[nq][e];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      lq[nq][e] = v;
    }
  constexpr int RW = D + 4;
#pragma unroll
  for (int dm = 0; dm < C::DM; ++dm)
#pragma unroll
    for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int d = dm * 16 + gq + (e >> 1) * 8;
        const int m = nq * 8 + cq * 2 + (e & 1);
        stage_out[m * RW + d] = o[dm][nq][e];
      }
  if (gq == 0) {
#pragma unroll
    for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = nq * 8 + cq * 2 + e;
        stage_out[m * RW + D] = mq[nq][e];
        stage_out[m * RW + D + 1] = lq[nq][e];
      }
  }
  __syncwarp();
  const int nqr = min(Qg, NQ * 8);
  const uint32_t ghalf = gat ? gather_half(p) : 0u;
  for (int m = 0; m < nqr; ++m) {
    const float M = stage_out[m * RW + D], Ls = stage_out[m * RW + D + 1];
    const int j = m / g, ii = m % g;
    if (p.splits == 1) {
      __nv_bfloat16* op = (__nv_bfloat16*)p.out + (((size_t)r * p.b_live + j) * p.Hq + h * g + ii) * D;
      const float inv = Ls > 0.f ? 1.f / Ls : 0.f;
      for (int d = lane * 2; d < D; d += 64) {
        const uint32_t v = pack_bf16(stage_out[m * RW + d] * inv, stage_out[m * RW + d + 1] * inv);
        *(uint32_t*)(op + d) = v;
        if (gat) gather_st32(p, ghalf, r, j, h * g + ii, d, v);
      }
      if (lane == 0) {
        if (Ls == 0.f) latch(p.status, TRIE_ST_EMPTY_ROW);
        if (p.lse)
          p.lse[((size_t)r * p.b_live + j) * p.Hq + h * g + ii] =
              Ls > 0.f ? (M + log2f(Ls)) * 0.69314718055994531f : -INFINITY;
      }
    } else {
      float* pp = p.part + ((((size_t)r * p.Hkv + h) * p.splits + split) * Qg + m) * (D + 2);
      for (int d = lane; d < D; d += 32) pp[d] = stage_out[m * RW + d];
      if (lane == 0) {
        pp[D] = M;
        pp[D + 1] = Ls;
      }
    }
  }
  if (gat) {  // the item's rows are stored (this warp wrote all of them)
    __syncwarp();
    if (lane == 0) gather_arrive(p);
  }
  ATTN_TRC(lane == 0, 4);
}

// =========================================================================================
// wide: 16 < Qg <= 16 * MT; CTA = producer warp + MT consumer warps (one query m-tile each)
// =========================================================================================
template <int D, int MT, int RS = 1>
struct WideCfg {
#ifdef TRIE_WIDE_STAGES  // experiment builds only
  static constexpr int STAGES = TRIE_WIDE_STAGES;
#else
#ifndef TRIE_WIDE1_STAGES  // MT = 1 (8 < Qg <= 16) experiment builds only
#define TRIE_WIDE1_STAGES 0
#endif
  static constexpr int STAGES = (MT == 1 && TRIE_WIDE1_STAGES > 0) ? TRIE_WIDE1_STAGES : (D >= 128 ? 3 : 4);
#endif
  using RG = Ring<D, STAGES>;
  static constexpr int KS = D / 16;
  static constexpr int DT = D / 8;
  static constexpr int RSZ = TC_TR / RS;  // tile rows per warp
  static constexpr int NT = RSZ / 8;      // S n-tiles per warp
  static constexpr int NC = MT * RS;      // consumer warps
  static_assert(NT % 2 == 0, "row slice must be a multiple of 16");
  static_assert((RS - 1) * MT * 16 * (D + 2) * 4 <= RG::RING_BYTES, "merge buffer must fit the ring");
  // RS >= 4: the rotated queries live in shared memory (fragment order, [MT][KS][32 lanes]
  // x 16 B) instead of 32 registers per consumer thread, which is what lets 2 CTAs of 288
  // threads share an SM under the 112-register cap below
#ifndef TRIE_WIDE_PIPE  // one-tile software pipeline of the consumer loop (A/B knob)
#define TRIE_WIDE_PIPE 1
#endif
  // one-m-tile kernel only (r2p1, one box, A/B vs the plain loop): sweep b = 4 96.0 -> 91.0
  // us per launch, Mistral shard 54.8 -> 54.0; at MT = 2 it was slower (Llama 27.5 -> 31.1
  // us, sweep b = 8 102.6 -> 107.4) -- the isolated per-CTA tile time rises there too
  static constexpr bool PIPE = TRIE_WIDE_PIPE != 0 && MT == 1;
  static constexpr bool QS = RS >= 4 || (PIPE && MT >= 2);
  static constexpr int OFF_Q = RG::RING_BYTES + 256;
  static constexpr int Q_BYTES = QS ? MT * KS * 32 * 16 : 0;
  static constexpr int SMEM = OFF_Q + Q_BYTES + 1024;
  static_assert(2 * STAGES * 8 + 8 + (int)sizeof(ItemInfo) <= 256, "barrier area");
  static constexpr int THREADS = 32 * (NC + 1);
  // Register cap: an SM sub-partition holds 16K registers and a CTA's warps are spread
  // round-robin over the 4 sub-partitions, so 2 CTAs per SM need (warps on the fullest
  // sub-partition) x 32 x regs <= 16384: 5 warps (MT = 2, RS = 4: 18 warps per SM) -> 96
  // registers (Q staged in shared memory), 3 warps (two CTAs of 5 warps) -> 168
  static constexpr int MAXREG = (MT == 2 && RS >= 4) ? 96 : 168;
};

// Warp (mt, rs) owns query m-tile mt (16 queries) and rows [rs*RSZ, (rs+1)*RSZ) of every
// tile; with RS > 1 the row slices of an m-tile are merged once, at the end, through the
// (drained) ring.  S = Q K^T with two independent n-tiles per ldmatrix.x4.
// ROPE: fused a-1 (trie_attn_decode_rope) -- Q is read un-rotated and rotated in registers
// (the rotate-half partner of column c < D/2 is column c + D/2, held by the same thread
// in k-step ks + KS/2), the leaves' K/V rows are appended by the producer warp's idle lanes.
template <int D, int MT, int RS, bool ROPE = false>
__global__ void __launch_bounds__(WideCfg<D, MT, RS>::THREADS) __maxnreg__((WideCfg<D, MT, RS>::MAXREG)) k_attn_wide(
    const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
    const AttnParams p, const __grid_constant__ CUtensorMap kmh,
    const __grid_constant__ CUtensorMap vmh) {
  using C = WideCfg<D, MT, RS>;
  using RG = typename C::RG;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  uint64_t* full = (uint64_t*)(smem + RG::RING_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* app_done = empty + C::STAGES;
  ItemInfo* info = (ItemInfo*)(app_done + 1);

  const int h = blockIdx.x, r = blockIdx.y, split = blockIdx.z;
  pdl_trigger();
  ATTN_TRC(threadIdx.x == 0, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NC);
    }
    mbar_init(app_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // prompt-only tiles loaded before the wait (see AttnParams::pre_tiles)
  const int npre = split == 0 ? min(p.pre_tiles, C::STAGES) : 0;
  if (threadIdx.x == 0 && npre > 0)
    prefetch_prompt_tiles<D, C::STAGES>(&kmap, &vmap, p, r, h, ring, full, npre);
  pdl_wait();  // the shared-memory setup above ran before the predecessor finished
  if (warp == 0) {
    // item setup, published to the consumers by a named barrier: they load (and rotate)
    // their queries meanwhile instead of waiting for it
    item_setup(p, r, split, info);
    __syncwarp();
    const ItemInfo it = *info;
    __threadfence_block();
    asm volatile("bar.arrive 2, %0;" ::"r"(C::THREADS) : "memory");
#ifdef TRIE_ATTN_TRACE
    if (threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      attn_trc(1);
      attn_trc(6, smid);
      attn_trc(7, (unsigned long long)it.ntiles);
    }
#endif
    if constexpr (ROPE) {  // as in k_attn_narrow: leaf-free tiles first, then the rest
      const int first_leaf = it.N - p.b_live;
      int fill = min(C::STAGES, it.ntiles);
      while (fill > npre && (it.tile0 + fill) * TC_TR > first_leaf) --fill;
      if (lane == 0)
        producer_loop<D, C::STAGES>(&kmap, &vmap, p, r, h, it, ring, full, empty, nullptr,
                                    INT_MAX, npre, fill, nullptr, p.half_tiles ? &kmh : nullptr, &vmh);
      else
        append_leaves_rope<D>(p, r, h, it.tile0 * TC_TR, (it.tile0 + it.ntiles) * TC_TR, lane,
                              app_done, first_leaf);
      __syncwarp();
      if (lane == 0)
        producer_loop<D, C::STAGES>(&kmap, &vmap, p, r, h, it, ring, full, empty, app_done,
                                    first_leaf, max(fill, npre), INT_MAX, nullptr, p.half_tiles ? &kmh : nullptr, &vmh);
    } else if (lane == 0) {
      producer_loop<D, C::STAGES>(&kmap, &vmap, p, r, h, it, ring, full, empty, nullptr, INT_MAX,
                                  npre, INT_MAX, nullptr, p.half_tiles ? &kmh : nullptr, &vmh);
    }
    if (it.done && lane == 0)  // no tile is consumed: let the pre-wait loads land before exit
      for (int i = 0; i < npre; ++i) mbar_wait(&full[i], 0u);
    ATTN_TRC(lane == 0, 5);
    return;
  }
  const int cw = warp - 1;
  const int mt = cw % MT, rs = cw / MT;
  const int r0 = rs * C::RSZ;
  const int g = p.Hq / p.Hkv, Qg = p.b_live * g;
  const int gq = lane >> 2, cq = lane & 3;
  const size_t mbase = (size_t)r * p.cap;
  int qm[2], beam[2], lod[2];
  uint32_t bbit[2];  // this query's beam bit (0 for padding queries)
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    qm[u] = mt * 16 + gq + 8 * u;
    beam[u] = qm[u] < Qg ? qm[u] / g : 0;
    bbit[u] = qm[u] < Qg ? 1u << beam[u] : 0u;
    lod[u] = INT_MIN;
    if (p.window > 0 && qm[u] < Qg)
      lod[u] = p.depth[mbase + p.leaf[r * TRIE_MAX_BEAMS + beam[u]]] - p.window + 1;
  }
  uint32_t qa[C::QS ? 1 : C::KS][4];
  uint4* sq = (uint4*)(smem + C::OFF_Q) + (size_t)mt * C::KS * 32 + lane;  // QS: [ks * 32]
  if (!C::QS || rs == 0) {
    uint32_t ql[C::KS][4];  // rotated query fragments (QS: staged to shared memory)
    // the two query rows' base pointers (query m = beam j * g + head i of the group)
    const __nv_bfloat16* qrow[2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
      qrow[u] = qm[u] < Qg ? (const __nv_bfloat16*)p.q +
                                 (((size_t)r * p.b_live + beam[u]) * p.Hq + h * g + qm[u] - beam[u] * g) * D
                           : nullptr;
#pragma unroll
    for (int ks = 0; ks < C::KS; ++ks)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const __nv_bfloat16* src = qrow[u & 1];
        const int col = ks * 16 + (u >> 1) * 8 + cq * 2;
        ql[ks][u] = src ? *(const uint32_t*)(src + col) : 0u;
      }
    if constexpr (ROPE) {  // rotate-half at the beam's depth, rounded to bf16 like a-1
      constexpr int HALF = D / 2;
#pragma unroll
      for (int ks = 0; ks < C::KS / 2; ++ks)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (!qrow[u & 1]) continue;
          const int col = ks * 16 + (u >> 1) * 8 + cq * 2;  // < HALF; partner col + HALF
          const float4 t = __ldg((const float4*)(p.rope_tab +
                                                 ((size_t)r * p.b_live + beam[u & 1]) * HALF + col));
          const float2 x1 = __bfloat1622float2(*(const __nv_bfloat162*)&ql[ks][u]);
          const float2 x2 = __bfloat1622float2(*(const __nv_bfloat162*)&ql[ks + C::KS / 2][u]);
          ql[ks][u] = pack_bf16(x1.x * t.x - x2.x * t.y, x1.y * t.z - x2.y * t.w);
          ql[ks + C::KS / 2][u] = pack_bf16(x2.x * t.x + x1.x * t.y, x2.y * t.z + x1.y * t.w);
        }
    }
    if constexpr (C::QS) {
#pragma unroll
      for (int ks = 0; ks < C::KS; ++ks) sq[ks * 32] = make_uint4(ql[ks][0], ql[ks][1], ql[ks][2], ql[ks][3]);
    } else {
#pragma unroll
      for (int ks = 0; ks < C::KS; ++ks)
#pragma unroll
        for (int u = 0; u < 4; ++u) qa[C::QS ? 0 : ks][u] = ql[ks][u];
    }
  }
  // item setup published by warp 0 (the queries were loaded and rotated meanwhile: r34 A/B
  // on Llama, 58.4k vs 57.4k request-steps/s)
  asm volatile("bar.sync 2, %0;" ::"r"(C::THREADS) : "memory");
  const ItemInfo it = *info;
  float o[C::DT][4];
#pragma unroll
  for (int i = 0; i < C::DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const float sc = p.scale_log2;
  const int fast_end = min(it.t, it.N) / TC_TR;

  // S = Q K^T of tile i (this warp's rows) into sacc; waits for the tile's stage
  auto qk_tile = [&](int i, float (&sacc)[C::NT][4]) {
    const int s = i % C::STAGES;
    mbar_wait(&full[s], (uint32_t)(i / C::STAGES) & 1u);
    ATTN_TRC(i == 0 && cw == 0 && lane == 0, 2);
    const uint32_t kbase = smem_u32(ring + s * RG::STAGE_BYTES);
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < C::KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < C::NT; nt += 2) {
        if constexpr (C::QS) {
          if (nt == 0) {
            const uint4 q4 = sq[ks * 32];
            qa[0][0] = q4.x; qa[0][1] = q4.y; qa[0][2] = q4.z; qa[0][3] = q4.w;
          }
        }
        const int qk = C::QS ? 0 : ks;
        // x4: (n-tile nt, k lo), (nt, k hi), (nt+1, k lo), (nt+1, k hi)
        const int row = r0 + (nt + (lane >> 4)) * 8 + (lane & 7);
        const int col = ks * 16 + ((lane >> 3) & 1) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kbase + tile_off(row, col), b0, b1, b2, b3);
        mma_bf16(sacc[nt], qa[qk][0], qa[qk][1], qa[qk][2], qa[qk][3], b0, b1);
        mma_bf16(sacc[nt + 1], qa[qk][0], qa[qk][1], qa[qk][2], qa[qk][3], b2, b3);
      }
  };
  // mask + online softmax of tile i's scores, O += P V, release the stage
  auto softmax_pv_tile = [&](int i, float (&sacc)[C::NT][4]) {
    const int s = i % C::STAGES;
    const uint8_t* st = ring + s * RG::STAGE_BYTES;
    const uint32_t vbase = smem_u32(st + RG::TILE_BYTES);
    const int tile = it.tile0 + i;
    const int n0 = tile * TC_TR;
    const bool fast = tile >= it.fast_from && tile < fast_end;
    float tmax[2] = {-INFINITY, -INFINITY};
    if (fast) {
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int u = e >> 1;
          const float v = qm[u] < Qg ? sacc[nt][e] : -INFINITY;
          sacc[nt][e] = v;
          tmax[u] = fmaxf(tmax[u], v);
        }
    } else {
      const uint32_t* tmask = (const uint32_t*)(st + 2 * RG::TILE_BYTES);
      const int* tdep = (const int*)(st + 2 * RG::TILE_BYTES + TC_TR * 4);
      const bool win = p.window > 0;
      if (!win && n0 >= it.t && n0 + TC_TR <= it.N) {
        // generated rows only, all below N, no window: the beam word alone decides
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const uint32_t vis = tmask[r0 + nt * 8 + cq * 2 + cc];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const float v = (vis & bbit[u]) != 0u ? sacc[nt][u * 2 + cc] : -INFINITY;
              sacc[nt][u * 2 + cc] = v;
              tmax[u] = fmaxf(tmax[u], v);
            }
          }
      } else {
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int lr = r0 + nt * 8 + cq * 2 + cc;
            const int n = n0 + lr;
            // visible-beam word of the row: none past N, all on the prompt (Alg. 3 l.2)
            const uint32_t vis = n >= it.N ? 0u : (n < it.t ? ~0u : tmask[lr]);
            const int dep = win ? tdep[lr] : 0;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const bool ok = (vis & bbit[u]) != 0u && dep >= lod[u];
              const float v = ok ? sacc[nt][u * 2 + cc] : -INFINITY;
              sacc[nt][u * 2 + cc] = v;
              tmax[u] = fmaxf(tmax[u], v);
            }
          }
      }
    }
    float alpha[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      tmax[u] = fmaxf(tmax[u], __shfl_xor_sync(0xffffffffu, tmax[u], 1));
      tmax[u] = fmaxf(tmax[u], __shfl_xor_sync(0xffffffffu, tmax[u], 2));
      const float mnew = fmaxf(mrow[u], tmax[u] * sc);  // scores are raw until here (sc > 0)
      alpha[u] = (mnew == -INFINITY) ? 1.f : ex2_ftz(mrow[u] - mnew);
      mrow[u] = mnew;
      lrow[u] *= alpha[u];
    }
    const float msafe[2] = {mrow[0] == -INFINITY ? 0.f : mrow[0], mrow[1] == -INFINITY ? 0.f : mrow[1]};
    uint32_t pa[C::NT][2];
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) {
      float pv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int u = e >> 1;
        pv[e] = ex2_ftz(fmaf(sacc[nt][e], sc, -msafe[u]));  // masked keys: 2^-inf = 0
        lrow[u] += pv[e];
      }
      pa[nt][0] = pack_bf16(pv[0], pv[1]);
      pa[nt][1] = pack_bf16(pv[2], pv[3]);
    }
    // (skipping the alpha = 1 rescale warp-uniformly, as k_attn_narrow does, measured ~1%
    // slower here: r2e3, Llama 23.3 -> 23.6 us)
#pragma unroll
    for (int dt = 0; dt < C::DT; ++dt) {
      o[dt][0] *= alpha[0];
      o[dt][1] *= alpha[0];
      o[dt][2] *= alpha[1];
      o[dt][3] *= alpha[1];
    }
#pragma unroll
    for (int kc = 0; kc < C::NT / 2; ++kc) {
      const uint32_t a0 = pa[2 * kc][0], a1 = pa[2 * kc][1], a2 = pa[2 * kc + 1][0],
                     a3 = pa[2 * kc + 1][1];
#pragma unroll
      for (int dt = 0; dt < C::DT; dt += 2) {
        const int row = r0 + kc * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int col = dt * 8 + (lane >> 4) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vbase + tile_off(row, col), b0, b1, b2, b3);
        mma_bf16(o[dt], a0, a1, a2, a3, b0, b1);
        mma_bf16(o[dt + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  };
  float sA[C::NT][4];
  if constexpr (C::PIPE) {
    // one-tile software pipeline: tile i+1's QK^T MMAs are issued ahead of tile i's
    // softmax, so the tensor-pipe chains overlap the ALU / MUFU work of the same warp
    float sB[C::NT][4];
    if (it.ntiles > 0) qk_tile(0, sA);
    for (int i = 0; i < it.ntiles; i += 2) {
      if (i + 1 < it.ntiles) qk_tile(i + 1, sB);
      softmax_pv_tile(i, sA);
      if (i + 1 >= it.ntiles) break;
      if (i + 2 < it.ntiles) qk_tile(i + 2, sA);
      softmax_pv_tile(i + 1, sB);
    }
  } else {
    for (int i = 0; i < it.ntiles; ++i) {
      qk_tile(i, sA);
      softmax_pv_tile(i, sA);
    }
  }
  ATTN_TRC(cw == 0 && lane == 0, 3);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    lrow[u] += __shfl_xor_sync(0xffffffffu, lrow[u], 1);
    lrow[u] += __shfl_xor_sync(0xffffffffu, lrow[u], 2);
  }
  if constexpr (RS > 1) {
    // row-slice merge: slices rs > 0 park (O, m, l) in the drained ring, slice 0 folds them
    __syncwarp();
    asm volatile("bar.sync 1, %0;" ::"r"(C::NC * 32));
    float* red = (float*)smem;  // [(RS-1) * MT][16][D + 2]
    constexpr int RW = D + 2;
    if (rs > 0) {
      float* mine = red + (size_t)((rs - 1) * MT + mt) * 16 * RW;
#pragma unroll
      for (int dt = 0; dt < C::DT; ++dt) {
        const int col = dt * 8 + cq * 2;
        mine[gq * RW + col] = o[dt][0];
        mine[gq * RW + col + 1] = o[dt][1];
        mine[(gq + 8) * RW + col] = o[dt][2];
        mine[(gq + 8) * RW + col + 1] = o[dt][3];
      }
      if (cq == 0) {
        mine[gq * RW + D] = mrow[0];
        mine[gq * RW + D + 1] = lrow[0];
        mine[(gq + 8) * RW + D] = mrow[1];
        mine[(gq + 8) * RW + D + 1] = lrow[1];
      }
    }
    __syncwarp();
    asm volatile("bar.sync 1, %0;" ::"r"(C::NC * 32));
    if (rs > 0) return;
#pragma unroll
    for (int x = 0; x < RS - 1; ++x) {
      const float* src = red + (size_t)(x * MT + mt) * 16 * RW;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int row = gq + 8 * u;
        const float m2 = src[row * RW + D], l2 = src[row * RW + D + 1];
        const float mn = fmaxf(mrow[u], m2);
        const float w1 = mrow[u] == -INFINITY ? 0.f : exp2f(mrow[u] - mn);
        const float w2 = m2 == -INFINITY ? 0.f : exp2f(m2 - mn);
#pragma unroll
        for (int dt = 0; dt < C::DT; ++dt) {
          const int col = dt * 8 + cq * 2;
          o[dt][u * 2] = o[dt][u * 2] * w1 + src[row * RW + col] * w2;
          o[dt][u * 2 + 1] = o[dt][u * 2 + 1] * w1 + src[row * RW + col + 1] * w2;
        }
        lrow[u] = lrow[u] * w1 + l2 * w2;
        mrow[u] = mn;
      }
    }
  }
  // NEXT-4 fused all-gather: the MT writer warps (row slice 0) meet at named barrier 3,
  // then one lane arrives for the item
  const bool gat = p.ga.world > 0 && p.splits == 1;
  if (it.done) {  // NEXT-3: finished request, output not written
    if (gat) {
      __syncwarp();
      asm volatile("bar.sync 3, %0;" ::"r"(MT * 32) : "memory");
      if (mt == 0 && lane == 0) gather_arrive(p);
    }
    return;
  }
  const uint32_t ghalf = gat ? gather_half(p) : 0u;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int m = qm[u];
    if (m >= Qg) continue;
    const int j = m / g, ii = m % g;
    if (p.splits == 1) {
      __nv_bfloat16* op = (__nv_bfloat16*)p.out + (((size_t)r * p.b_live + j) * p.Hq + h * g + ii) * D;
      const float inv = lrow[u] > 0.f ? 1.f / lrow[u] : 0.f;
#pragma unroll
      for (int dt = 0; dt < C::DT; ++dt) {
        const uint32_t v = pack_bf16(o[dt][u * 2] * inv, o[dt][u * 2 + 1] * inv);
        *(uint32_t*)(op + dt * 8 + cq * 2) = v;
        if (gat) gather_st32(p, ghalf, r, j, h * g + ii, dt * 8 + cq * 2, v);
      }
      if (cq == 0) {
        if (lrow[u] == 0.f) latch(p.status, TRIE_ST_EMPTY_ROW);
        if (p.lse)
          p.lse[((size_t)r * p.b_live + j) * p.Hq + h * g + ii] =
              lrow[u] > 0.f ? (mrow[u] + log2f(lrow[u])) * 0.69314718055994531f : -INFINITY;
      }
    } else {
      float* pp = p.part + ((((size_t)r * p.Hkv + h) * p.splits + split) * Qg + m) * (D + 2);
#pragma unroll
      for (int dt = 0; dt < C::DT; ++dt) {
        pp[dt * 8 + cq * 2] = o[dt][u * 2];
        pp[dt * 8 + cq * 2 + 1] = o[dt][u * 2 + 1];
      }
      if (cq == 0) {
        pp[D] = mrow[u];
        pp[D + 1] = lrow[u];
      }
    }
  }
  if (gat) {
    __syncwarp();
    asm volatile("bar.sync 3, %0;" ::"r"(MT * 32) : "memory");
    if (mt == 0 && lane == 0) gather_arrive(p);
  }
  ATTN_TRC(cw == 0 && lane == 0, 4);
}

// ---- host side ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
  }
  return fn;
}

static int make_map(CUtensorMap* map, const void* base, int D, long rows, int box_rows) {
  auto enc = get_encode();
  if (!enc) return trie_set_error(TRIE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {(cuuint32_t)TC_CW, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult rc = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS)
    return trie_set_error(TRIE_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)rc);
  return TRIE_OK;
}

// Small direct-mapped cache of encoded tensor maps (the pools of a model are a fixed set
// of per-layer base pointers), so a decode step does not re-encode 2L descriptors.
struct MapEntry {
  const void* base;
  long rows;
  int D, box_rows;
  CUtensorMap map;
};
int cached_tensor_map(CUtensorMap* out, const void* base, int D, long rows, int box_rows) {
  static MapEntry cache[1024];
  const size_t slot = ((((uintptr_t)base >> 8) ^ ((uintptr_t)base >> 20)) * 2 + (box_rows != TC_TR)) % 1024;
  MapEntry& e = cache[slot];
  if (e.base != base || e.rows != rows || e.D != D || e.box_rows != box_rows) {
    const int rc = make_map(&e.map, base, D, rows, box_rows);
    if (rc) {
      e.base = nullptr;
      return rc;
    }
    e.base = base;
    e.rows = rows;
    e.D = D;
    e.box_rows = box_rows;
  }
  *out = e.map;
  return TRIE_OK;
}

// ---- kernel table: attributes (max dynamic smem, max-shared carveout) set once, the
// occupancy queried once; the split plan uses it so a launch fills whole waves.
struct TcKernel {
  const void* fn;
  int smem, threads, occ;
};

template <typename Kern>
static TcKernel make_tc(Kern kern, int smem, int threads) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  return TcKernel{(const void*)kern, smem, threads, occ > 0 ? occ : 1};
}
template <int D, int NQ, int ST, bool ROPE = false>
static const TcKernel& narrow_k() {
  static const TcKernel k =
      make_tc(k_attn_narrow<D, NQ, ST, ROPE>, NarrowCfg<D, NQ, ST, ROPE>::SMEM, 64);
  return k;
}
template <int D, int MT, int RS, bool ROPE = false>
static const TcKernel& wide_k() {
  static const TcKernel k = make_tc(k_attn_wide<D, MT, RS, ROPE>, WideCfg<D, MT, RS>::SMEM,
                                    WideCfg<D, MT, RS>::THREADS);
  return k;
}
// row slices per wide tile (TRIE_WIDE_RS in {1, 2, 4}; default 2: two warps per query
// m-tile so each SM scheduler has more than one warp to switch to)
static int wide_rs() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TRIE_WIDE_RS");
    v = e ? atoi(e) : 2;
    if (v != 1 && v != 2 && v != 4) v = 2;
  }
  return v;
}
template <int D, int MT, bool ROPE = false>
static const TcKernel& wide_sel() {
  switch (wide_rs()) {
    case 1: return wide_k<D, MT, 1, ROPE>();
    case 4: return wide_k<D, MT, (MT <= 2 ? 4 : 2), ROPE>();
    default: return wide_k<D, MT, (MT <= 4 ? 2 : 1), ROPE>();
  }
}

// Stages per narrow CTA (tuning knob TRIE_NARROW_STAGES in {2, 3, 4}).  Default 2: at
// D = 96 a 2-stage CTA needs ~50 KB, so 3-4 CTAs (3-4 consumer warps, 6-8 tiles in
// flight) share an SM; measured r01 on the Phi workload: 2 -> 5.81 TB/s, 3 -> 5.18,
// 4 -> 5.34 (more independent streams beat deeper per-stream rings).
static int narrow_stages() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TRIE_NARROW_STAGES");
    v = e ? atoi(e) : 2;
    if (v < 2 || v > 4) v = 2;
  }
  return v;
}
template <int D, int NQ, bool ROPE>
static const TcKernel& narrow_sel() {
  switch (narrow_stages()) {
    case 3: return narrow_k<D, NQ, 3, ROPE>();
    case 4: return narrow_k<D, NQ, 4, ROPE>();
    default: return narrow_k<D, NQ, 2, ROPE>();
  }
}
// One query m-tile (Qg <= 16) over 4 row slices of the wide kernel (4 consumer warps of
// 16 queries x 16 rows) beats the one-warp narrow kernel from Qg = 9 (r2z3, one B200:
// Mistral shard Qg = 16 59.7 -> 55.3 us per launch, sweep b = 4 100.3 -> 96.1 us); knob
// TRIE_WIDE1_MIN_QG = q (experiments): the wide kernel for q < Qg <= 16 (16 = never)
static int wide1_min_qg() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TRIE_WIDE1_MIN_QG");
    v = e ? atoi(e) : 8;
    if (v < 0 || v > 16) v = 8;
  }
  return v;
}
template <int D>
static const TcKernel& select_d(int Qg, bool rope) {
  if (Qg <= 16 && Qg > wide1_min_qg()) return rope ? wide_k<D, 1, 4, true>() : wide_k<D, 1, 4, false>();
  if (Qg <= 8) return rope ? narrow_sel<D, 1, true>() : narrow_sel<D, 1, false>();
  if (Qg <= 16) return rope ? narrow_sel<D, 2, true>() : narrow_sel<D, 2, false>();
  if (Qg <= 32) return rope ? wide_sel<D, 2, true>() : wide_sel<D, 2, false>();
  if (Qg <= 64) return wide_sel<D, 4>();
  return wide_sel<D, 8>();
}
static const TcKernel* select_tc(int D, int Qg, bool rope = false) {
  switch (D) {
    case 64: return &select_d<64>(Qg, rope);
    case 96: return &select_d<96>(Qg, rope);
    case 128: return &select_d<128>(Qg, rope);
  }
  return nullptr;
}

// mma.sync kernel family for a tensor-core shape: 1 = narrow, 2 = wide (plan reporting)
int attn_tc_variant(const AttnParams& p) {
  const int Qg = p.b_live * (p.Hq / p.Hkv);
  return (Qg <= 16 && Qg > wide1_min_qg()) || Qg > 16 ? 2 : 1;
}

// The fused RoPE + append variants: narrow (Qg <= 16), wide at Qg <= 32, tcgen05.
bool attn_rope_fusable(const AttnParams& p) {
  const int Qg = p.b_live * (p.Hq / p.Hkv);
  return attn_tc_supported(p) && (attn_umma_eligible(p) || Qg <= 32);
}

bool attn_tc_shape_ok(const AttnParams& p) {
  const int Qg = p.b_live * (p.Hq / p.Hkv);
  return p.bf16 && Qg <= 128 && p.cap % 4 == 0 && (p.D == 64 || p.D == 96 || p.D == 128);
}

bool attn_tc_supported(const AttnParams& p) {
  if (!attn_tc_shape_ok(p)) return false;
  return ((((uintptr_t)p.k | (uintptr_t)p.v) & 15) == 0);  // TMA needs 16-B aligned pools
}

// Split-K plan: one CTA per (KV head, request) when that already fills the resident CTA
// slots (occupancy x SMs); otherwise split each item's tiles so the launch is close to one
// full wave, keeping >= 2 tiles (128 slots) per split.  A pure function of the shapes, so
// trie_attn_scratch_bytes and trie_attn_decode agree.
int attn_plan_splits(const AttnParams& p, int rows_est, int sms) {
  const int units = p.R * p.Hkv;
  int occ = 2;
  if (attn_umma_eligible(p)) {
    occ = attn_umma_occ(p);
  } else if (attn_tc_shape_ok(p)) {
    const TcKernel* k = select_tc(p.D, p.b_live * (p.Hq / p.Hkv), p.rope != 0);
    if (k) occ = k->occ;
  }
  const int slots = occ * sms;
  const int max_by_rows = rows_est / 128 > 0 ? rows_est / 128 : 1;
  static int forced = -1;  // TRIE_ATTN_SPLITS=n: experiments only
  if (forced < 0) {
    const char* e = getenv("TRIE_ATTN_SPLITS");
    forced = e ? atoi(e) : 0;
  }
  if (forced > 0) return std::min(std::min(forced, max_by_rows), 64);
  if (units >= slots) return 1;
  int splits = slots / units;
  if (splits > max_by_rows) splits = max_by_rows;
  if (splits > 64) splits = 64;
  return splits < 1 ? 1 : splits;
}

int launch_attn_tc(const AttnParams& p, cudaStream_t s) {
  if (attn_umma_eligible(p)) return launch_attn_umma(p, s);
  const TcKernel* k = select_tc(p.D, p.b_live * (p.Hq / p.Hkv), p.rope != 0);
  if (!k) return trie_set_error(TRIE_EINVAL, "tensor-core attention: unsupported head_dim %d", p.D);
  CUtensorMap km, vm, kmh, vmh;
  const long rows = attn_pool_rows(p);
  int rc = cached_tensor_map(&km, p.k, p.D, rows);
  if (!rc) rc = cached_tensor_map(&vm, p.v, p.D, rows);
  if (!rc) rc = cached_tensor_map(&kmh, p.k, p.D, rows, TC_TR / 2);
  if (!rc) rc = cached_tensor_map(&vmh, p.v, p.D, rows, TC_TR / 2);
  if (rc) return rc;
  AttnParams pp = p;
  static int half = -1;  // TRIE_HALF_TILE=0 disables the 32-row last tiles (A/B experiments)
  if (half < 0) {
    const char* e = getenv("TRIE_HALF_TILE");
    half = (e && e[0] == '0') ? 0 : 1;
  }
  pp.half_tiles = half;
  void* args[5] = {(void*)&km, (void*)&vm, (void*)&pp, (void*)&kmh, (void*)&vmh};
  launch_k_ptr(k->fn, dim3(p.Hkv, p.R, p.splits), dim3(k->threads), (size_t)k->smem, s, args);
  rc = trie_check_launch("k_attn_tc");
  if (rc) return rc;
  if (p.splits > 1) rc = launch_attn_combine_bf16(p, s);
  return rc;
}

}  // namespace trie

#ifdef TRIE_ATTN_TRACE
// trace build only: copy n CTA records (8 x u64 each) of the last traced launch, then clear
extern "C" int trie_debug_attn_trace(unsigned long long* host, int n) {
  if (cudaMemcpyFromSymbol(host, trie::g_attn_trace, (size_t)n * 8 * 8) != cudaSuccess) return -1;
  void* dev = nullptr;
  if (cudaGetSymbolAddress(&dev, trie::g_attn_trace) != cudaSuccess) return -1;
  return cudaMemset(dev, 0, sizeof(trie::g_attn_trace)) == cudaSuccess ? 0 : -1;
}
#endif
