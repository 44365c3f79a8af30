// trie_attn_decode, persistent bf16 tensor-core path (sm_100a).  Same math and tiles as
// attn_decode_tc.cu (§3.3; Alg. 3) with a different schedule:
//
//  * Work = chunks (request r, KV head h, split s) of consecutive 64-slot tiles; a launch
//    has occupancy x SMs CTAs that pull chunk ids from a device counter (dynamic queue)
//    until the queue is empty, so CTA start-up, pipeline fill and drain are paid once
//    per CTA instead of once per chunk, and uneven chunks balance themselves.
//  * Warp 0's elected lane (producer) runs ahead across chunk boundaries: per chunk it
//    computes the tile range / window bounds into a chunk-info slot, bulk-copies the
//    chunk's Q block (b_live segments of g*D bf16) into a Q slot (2-slot ring, qfull /
//    qempty mbarriers), then streams the tiles through the stage ring (full / empty).
//  * Consumer warps: narrow (Qg <= 16, KV rows on M, one warp) or wide (16 < Qg <= 128,
//    one warp per 16-query m-tile) exactly as in attn_decode_tc.cu.
//  * A chunk that covers its whole item writes the output; otherwise it writes its
//    (m, l, acc) partial, and the last chunk of the item to arrive (per-item counter)
//    merges all partials -- the split combine is fused, no second launch.
//  * Counters live at the start of the caller's scratch; they must be zero before the
//    first launch and every launch returns them to zero.
#include <algorithm>
#include <stdio.h>
#include <stdlib.h>

#include "attn_common.cuh"
#include "common.cuh"
#include "handle.h"
#include "tc_common.cuh"

namespace trie {

struct ChunkInfo {
  int valid, r, h, split, nsplit, tile0, ntiles, N, t, fast_from;
  int lod[TRIE_MAX_BEAMS];  // per-beam window lower depth (INT_MIN: no window)
};

struct QueueCounters {
  int next;      // next chunk id
  int done;      // CTAs finished
  int pad[30];
  int item[1];   // [R * Hkv] chunks arrived per item (flexible)
};

template <int D, int QMAX, int ST, int NCW>
struct PCfg {
  using RG = Ring<D, ST>;
  static constexpr int STAGES = ST;
  static constexpr int QSLOT = (QMAX * D * 2 + 1023) / 1024 * 1024;
  static constexpr int STAGE_OUT = (NCW == 1) ? 16 * (D + 4) * 4 : 0;  // narrow transpose
  static constexpr int OFF_Q = RG::RING_BYTES;
  static constexpr int OFF_OUT = OFF_Q + 2 * QSLOT;
  static constexpr int OFF_INFO = OFF_OUT + (STAGE_OUT + 127) / 128 * 128;
  static constexpr int OFF_BAR = OFF_INFO + 2 * (int)sizeof(ChunkInfo);
  static constexpr int SMEM = OFF_BAR + (2 * ST + 4) * 8 + 16 + 1024;
  static constexpr int THREADS = 32 * (1 + NCW);
};

// chunk id -> (item, split) ; tile range of the split, window bounds (thread 0 of producer)
__device__ __forceinline__ void chunk_setup(const AttnParams& p, int id, int nsplit, ChunkInfo* ci) {
  const int item = id / nsplit, split = id % nsplit;
  const int r = item / p.Hkv, h = item % p.Hkv;
  const size_t mbase = (size_t)r * p.cap;
  const int N = p.nn[r], t = p.tlen[r];
  int lo = 0, lo_dep_max = INT_MIN;
  if (p.window > 0) {
    int lo_dep = INT_MAX;
    for (int j = 0; j < p.b_live; ++j) {
      const int d = p.depth[mbase + p.leaf[r * TRIE_MAX_BEAMS + j]] - p.window + 1;
      ci->lod[j] = d;
      lo_dep = min(lo_dep, d);
      lo_dep_max = max(lo_dep_max, d);
    }
    int a = 0, b = N;
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (p.depth[mbase + mid] < lo_dep) a = mid + 1; else b = mid;
    }
    lo = a;
  } else {
    for (int j = 0; j < p.b_live; ++j) ci->lod[j] = INT_MIN;
  }
  const int first = lo / TC_TR;
  const int total = (N + TC_TR - 1) / TC_TR - first;
  const int per = (total + nsplit - 1) / nsplit;
  const int tb = min(total, split * per), te = min(total, (split + 1) * per);
  ci->valid = 1;
  ci->r = r;
  ci->h = h;
  ci->split = split;
  ci->nsplit = nsplit;
  ci->tile0 = first + tb;
  ci->ntiles = te - tb;
  ci->N = N;
  ci->t = t;
  ci->fast_from = p.window > 0 ? (max(lo_dep_max, 0) + TC_TR - 1) / TC_TR : 0;
}

// merge the nsplit partials of one item's query m (one warp), write bf16 output + lse
template <int D>
__device__ void combine_query(const AttnParams& p, int r, int h, int m, int nsplit, int Qg) {
  const int lane = threadIdx.x & 31;
  const int g = p.Hq / p.Hkv;
  const float* base = p.part + (((size_t)r * p.Hkv + h) * p.splits * Qg) * (D + 2);
  float ms[2], ls[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int s = lane + 32 * u;
    const float* pp = base + ((size_t)s * Qg + m) * (D + 2);
    ms[u] = s < nsplit ? __ldcg(pp + D) : -INFINITY;
    ls[u] = s < nsplit ? __ldcg(pp + D + 1) : 0.f;
  }
  const float M = warp_max(fmaxf(ms[0], ms[1]));
  float ws[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) ws[u] = ls[u] > 0.f ? exp2f(ms[u] - M) : 0.f;
  const float L = warp_sum(ls[0] * ws[0] + ls[1] * ws[1]);
  constexpr int DC = (D + 31) / 32;
  float acc[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) acc[c] = 0.f;
  for (int s = 0; s < nsplit; ++s) {
    const float w = __shfl_sync(0xffffffffu, ws[s >> 5], s & 31);
    if (w == 0.f) continue;
    const float* pp = base + ((size_t)s * Qg + m) * (D + 2);
#pragma unroll
    for (int c = 0; c < DC; ++c)
      if (lane + 32 * c < D) acc[c] += w * __ldcg(pp + lane + 32 * c);
  }
  const int j = m / g, ii = m % g;
  __nv_bfloat16* op = (__nv_bfloat16*)p.out + (((size_t)r * p.b_live + j) * p.Hq + h * g + ii) * D;
  const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
  for (int c = 0; c < DC; ++c)
    if (lane + 32 * c < D) op[lane + 32 * c] = __float2bfloat16_rn(acc[c] * inv);
  if (lane == 0) {
    if (L == 0.f) latch(p.status, TRIE_ST_EMPTY_ROW);
    if (p.lse)
      p.lse[((size_t)r * p.b_live + j) * p.Hq + h * g + ii] =
          L > 0.f ? (M + log2f(L)) * 0.69314718055994531f : -INFINITY;
  }
}

template <int D, int QMAX, int ST, int NCW, bool NARROW>
__global__ void __launch_bounds__(PCfg<D, QMAX, ST, NCW>::THREADS) k_attn_persist(
    const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
    const AttnParams p, int nsplit, int total_chunks) {
  using C = PCfg<D, QMAX, ST, NCW>;
  using RG = typename C::RG;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  uint8_t* qbuf = smem + C::OFF_Q;
  float* stage_out = (float*)(smem + C::OFF_OUT);
  ChunkInfo* info = (ChunkInfo*)(smem + C::OFF_INFO);
  uint64_t* full = (uint64_t*)(smem + C::OFF_BAR);
  uint64_t* empty = full + ST;
  uint64_t* qfull = empty + ST;
  uint64_t* qempty = qfull + 2;
  int* s_flag = (int*)(qempty + 2);
  QueueCounters* ctr = (QueueCounters*)p.aux;  // zero-initialised queue + item counters
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = p.Hq / p.Hkv, Qg = p.b_live * g;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ============================ producer ============================
    if (lane == 0) {
      uint32_t tcount = 0, ccount = 0;
      while (true) {
        const int id = atomicAdd(&ctr->next, 1);
        const int qs = ccount & 1;
        mbar_wait(&qempty[qs], ((ccount >> 1) & 1u) ^ 1u);
        ChunkInfo* ci = &info[qs];
        if (id >= total_chunks) {
          ci->valid = 0;
          mbar_arrive(&qfull[qs]);
          break;
        }
        chunk_setup(p, id, nsplit, ci);
        const int r = ci->r, h = ci->h;
        // Q block of (r, h): b_live segments of g*D bf16 (rows m = j*g + i)
        mbar_expect_tx(&qfull[qs], (uint32_t)(Qg * D * 2));
        const uint32_t qdst = smem_u32(qbuf + qs * C::QSLOT);
        const __nv_bfloat16* qsrc = (const __nv_bfloat16*)p.q;
        for (int j = 0; j < p.b_live; ++j)
          bulk_load_1d(qdst + j * g * D * 2, qsrc + (((size_t)r * p.b_live + j) * p.Hq + h * g) * D,
                       (uint32_t)(g * D * 2), &qfull[qs]);
        const int row_base = (r * p.Hkv + h) * p.cap;
        const size_t mbase = (size_t)r * p.cap;
        const int tile0 = ci->tile0, ntiles = ci->ntiles;
        for (int i = 0; i < ntiles; ++i, ++tcount) {
          const int s = tcount % ST;
          mbar_wait(&empty[s], ((tcount / ST) & 1u) ^ 1u);
          const uint32_t st = smem_u32(ring + s * RG::STAGE_BYTES);
          const int n0 = (tile0 + i) * TC_TR;
          const uint32_t mdb = (uint32_t)min(TC_TR, p.cap - n0) * 4u;
          mbar_expect_tx(&full[s], 2 * RG::TILE_BYTES + 2 * mdb);
#pragma unroll
          for (int bx = 0; bx < D / TC_CW; ++bx) {
            tma_load_2d(st + bx * TC_TR * 64, &kmap, bx * TC_CW, row_base + n0, &full[s]);
            tma_load_2d(st + RG::TILE_BYTES + bx * TC_TR * 64, &vmap, bx * TC_CW, row_base + n0, &full[s]);
          }
          bulk_load_1d(st + 2 * RG::TILE_BYTES, p.mask + mbase + n0, mdb, &full[s]);
          bulk_load_1d(st + 2 * RG::TILE_BYTES + TC_TR * 4, p.depth + mbase + n0, mdb, &full[s]);
        }
        ++ccount;
      }
    }
  } else {
    // ============================ consumers ============================
    const int cw = warp - 1;
    const int gq = lane >> 2, cq = lane & 3;
    uint32_t tcount = 0, ccount = 0;
    const float sc = p.scale_log2;
    while (true) {
      const int qs = ccount & 1;
      mbar_wait(&qfull[qs], (ccount >> 1) & 1u);
      const ChunkInfo& ci = info[qs];
      if (!ci.valid) break;
      // copy everything out of the info slot before releasing it (qempty)
      const int r = ci.r, h = ci.h, split = ci.split, ntiles = ci.ntiles, tile0 = ci.tile0;
      const int N = ci.N, t = ci.t, nsplit_c = ci.nsplit;
      const int fast_from = ci.fast_from, fast_end = min(t, N) / TC_TR;
      const __nv_bfloat16* qs_buf = (const __nv_bfloat16*)(qbuf + qs * C::QSLOT);

      if constexpr (NARROW) {
        // ---------------- narrow consumer (KV rows on M, queries on N) ----------------
        constexpr int NQ = QMAX / 8;
        constexpr int KS = D / 16, DM = D / 16;
        int beam[NQ][2], lod[NQ][2];
        bool qok[NQ][2];
#pragma unroll
        for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int m = nq * 8 + cq * 2 + e;
            qok[nq][e] = m < Qg;
            beam[nq][e] = m < Qg ? m / g : 0;
            lod[nq][e] = m < Qg ? ci.lod[beam[nq][e]] : INT_MIN;
          }
        uint32_t qb[NQ][KS][2];
#pragma unroll
        for (int nq = 0; nq < NQ; ++nq) {
          const int m = nq * 8 + gq;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            qb[nq][ks][0] = m < Qg ? *(const uint32_t*)(qs_buf + m * D + ks * 16 + cq * 2) : 0u;
            qb[nq][ks][1] = m < Qg ? *(const uint32_t*)(qs_buf + m * D + ks * 16 + 8 + cq * 2) : 0u;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&qempty[qs]);
        float o[DM][NQ][4];
#pragma unroll
        for (int dm = 0; dm < DM; ++dm)
#pragma unroll
          for (int nq = 0; nq < NQ; ++nq) o[dm][nq][0] = o[dm][nq][1] = o[dm][nq][2] = o[dm][nq][3] = 0.f;
        float mq[NQ][2], lq[NQ][2];
#pragma unroll
        for (int nq = 0; nq < NQ; ++nq) mq[nq][0] = mq[nq][1] = -INFINITY, lq[nq][0] = lq[nq][1] = 0.f;

        for (int i = 0; i < ntiles; ++i, ++tcount) {
          const int s = tcount % ST;
          mbar_wait(&full[s], (tcount / ST) & 1u);
          const uint8_t* stp = ring + s * RG::STAGE_BYTES;
          const uint32_t kbase = smem_u32(stp), vbase = smem_u32(stp + RG::TILE_BYTES);
          const int tile = tile0 + i;
          const int n0 = tile * TC_TR;
          const bool fast = tile >= fast_from && tile < fast_end;
          float sacc[4][NQ][4];
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
#pragma unroll
            for (int nq = 0; nq < NQ; ++nq) sacc[mt][nq][0] = sacc[mt][nq][1] = sacc[mt][nq][2] = sacc[mt][nq][3] = 0.f;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
              const int row = mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
              const int col = ks * 16 + (lane >> 4) * 8;
              uint32_t a0, a1, a2, a3;
              ldsm_x4(kbase + tile_off(row, col), a0, a1, a2, a3);
#pragma unroll
              for (int nq = 0; nq < NQ; ++nq) mma_bf16(sacc[mt][nq], a0, a1, a2, a3, qb[nq][ks][0], qb[nq][ks][1]);
            }
          }
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
                  const float v = qok[nq][e & 1] ? sacc[mt][nq][e] * sc : -INFINITY;
                  sacc[mt][nq][e] = v;
                  tmax[nq][e & 1] = fmaxf(tmax[nq][e & 1], v);
                }
          } else {
            const uint32_t* tmask = (const uint32_t*)(stp + 2 * RG::TILE_BYTES);
            const int* tdep = (const int*)(stp + 2 * RG::TILE_BYTES + TC_TR * 4);
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int lr = mt * 16 + gq + hh * 8;
                const int n = n0 + lr;
                const bool rowin = n < N;
                const uint32_t mw = rowin ? tmask[lr] : 0u;
                const int dep = rowin ? tdep[lr] : INT_MIN;
                const bool prompt = n < t;
#pragma unroll
                for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
                  for (int e = 0; e < 2; ++e) {
                    const bool ok = rowin && qok[nq][e] && (prompt || ((mw >> beam[nq][e]) & 1u)) &&
                                    dep >= lod[nq][e];
                    const float v = ok ? sacc[mt][nq][hh * 2 + e] * sc : -INFINITY;
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
              const float mnew = fmaxf(mq[nq][e], v);
              alpha[nq][e] = (mnew == -INFINITY) ? 1.f : exp2f(mq[nq][e] - mnew);
              mq[nq][e] = mnew;
              lq[nq][e] *= alpha[nq][e];
            }
          uint32_t pb[4][NQ][2];
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nq = 0; nq < NQ; ++nq) {
              float pv[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float x = sacc[mt][nq][e];
                pv[e] = (x == -INFINITY) ? 0.f : exp2f(x - mq[nq][e & 1]);
                lq[nq][e & 1] += pv[e];
              }
              pb[mt][nq][0] = movm_t(pack_bf16(pv[0], pv[1]));
              pb[mt][nq][1] = movm_t(pack_bf16(pv[2], pv[3]));
            }
#pragma unroll
          for (int dm = 0; dm < DM; ++dm)
#pragma unroll
            for (int nq = 0; nq < NQ; ++nq) {
              o[dm][nq][0] *= alpha[nq][0];
              o[dm][nq][1] *= alpha[nq][1];
              o[dm][nq][2] *= alpha[nq][0];
              o[dm][nq][3] *= alpha[nq][1];
            }
#pragma unroll
          for (int dm = 0; dm < DM; ++dm)
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
        // column sums, stage O^T transposed through shared memory
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
        __syncwarp();
#pragma unroll
        for (int dm = 0; dm < DM; ++dm)
#pragma unroll
          for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
            for (int e = 0; e < 4; ++e)
              stage_out[(nq * 8 + cq * 2 + (e & 1)) * RW + dm * 16 + gq + (e >> 1) * 8] = o[dm][nq][e];
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
        const int nqr = min(Qg, QMAX);
        if (nsplit_c == 1) {
          for (int m = 0; m < nqr; ++m) {
            const float M = stage_out[m * RW + D], Ls = stage_out[m * RW + D + 1];
            const int j = m / g, ii = m % g;
            __nv_bfloat16* op = (__nv_bfloat16*)p.out + (((size_t)r * p.b_live + j) * p.Hq + h * g + ii) * D;
            const float inv = Ls > 0.f ? 1.f / Ls : 0.f;
            for (int d = lane * 2; d < D; d += 64)
              *(uint32_t*)(op + d) = pack_bf16(stage_out[m * RW + d] * inv, stage_out[m * RW + d + 1] * inv);
            if (lane == 0) {
              if (Ls == 0.f) latch(p.status, TRIE_ST_EMPTY_ROW);
              if (p.lse)
                p.lse[((size_t)r * p.b_live + j) * p.Hq + h * g + ii] =
                    Ls > 0.f ? (M + log2f(Ls)) * 0.69314718055994531f : -INFINITY;
            }
          }
        } else {
          float* pbase = p.part + (((size_t)r * p.Hkv + h) * p.splits + split) * Qg * (D + 2);
          for (int m = 0; m < nqr; ++m)
            for (int d = lane; d < D + 2; d += 32) pbase[(size_t)m * (D + 2) + d] = stage_out[m * RW + d];
          __threadfence();
          __syncwarp();
          int last = 0;
          if (lane == 0) last = atomicAdd(&ctr->item[r * p.Hkv + h], 1) == nsplit_c - 1;
          last = __shfl_sync(0xffffffffu, last, 0);
          if (last) {
            __threadfence();
            for (int m = 0; m < nqr; ++m) combine_query<D>(p, r, h, m, nsplit_c, Qg);
            if (lane == 0) ctr->item[r * p.Hkv + h] = 0;
          }
        }
        __syncwarp();
      } else {
        // ---------------- wide consumer (queries on M, one warp per 16-query m-tile) ----------------
        constexpr int KS = D / 16, DT = D / 8, NT = TC_TR / 8;
        const int mt = cw;
        int qm[2], beam[2], lod[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          qm[u] = mt * 16 + gq + 8 * u;
          beam[u] = qm[u] < Qg ? qm[u] / g : 0;
          lod[u] = qm[u] < Qg ? ci.lod[beam[u]] : INT_MIN;
        }
        uint32_t qa[KS][4];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int row = (u & 1) ? qm[1] : qm[0];
            const int col = ks * 16 + (u >> 1) * 8 + cq * 2;
            qa[ks][u] = row < Qg ? *(const uint32_t*)(qs_buf + row * D + col) : 0u;
          }
        __syncwarp();
        if (lane == 0) mbar_arrive(&qempty[qs]);
        float o[DT][4];
#pragma unroll
        for (int i = 0; i < DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
        float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
        for (int i = 0; i < ntiles; ++i, ++tcount) {
          const int s = tcount % ST;
          mbar_wait(&full[s], (tcount / ST) & 1u);
          const uint8_t* stp = ring + s * RG::STAGE_BYTES;
          const uint32_t kbase = smem_u32(stp), vbase = smem_u32(stp + RG::TILE_BYTES);
          const int tile = tile0 + i;
          const int n0 = tile * TC_TR;
          const bool fast = tile >= fast_from && tile < fast_end;
          float sacc[NT][4];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
#pragma unroll
          for (int ks = 0; ks < KS; ks += 2)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const int row = nt * 8 + (lane & 7);
              const int col = ks * 16 + (lane >> 3) * 8;
              uint32_t b0, b1, b2, b3;
              ldsm_x4(kbase + tile_off(row, col), b0, b1, b2, b3);
              mma_bf16(sacc[nt], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
              mma_bf16(sacc[nt], qa[ks + 1][0], qa[ks + 1][1], qa[ks + 1][2], qa[ks + 1][3], b2, b3);
            }
          float tmax[2] = {-INFINITY, -INFINITY};
          if (fast) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int u = e >> 1;
                const float v = qm[u] < Qg ? sacc[nt][e] * sc : -INFINITY;
                sacc[nt][e] = v;
                tmax[u] = fmaxf(tmax[u], v);
              }
          } else {
            const uint32_t* tmask = (const uint32_t*)(stp + 2 * RG::TILE_BYTES);
            const int* tdep = (const int*)(stp + 2 * RG::TILE_BYTES + TC_TR * 4);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int cc = 0; cc < 2; ++cc) {
                const int lr = nt * 8 + cq * 2 + cc;
                const int n = n0 + lr;
                const bool rowin = n < N;
                const uint32_t mw = rowin ? tmask[lr] : 0u;
                const int dep = rowin ? tdep[lr] : INT_MIN;
                const bool prompt = n < t;
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  const bool ok = rowin && qm[u] < Qg && (prompt || ((mw >> beam[u]) & 1u)) && dep >= lod[u];
                  const float v = ok ? sacc[nt][u * 2 + cc] * sc : -INFINITY;
                  sacc[nt][u * 2 + cc] = v;
                  tmax[u] = fmaxf(tmax[u], v);
                }
              }
          }
          float alpha[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            tmax[u] = fmaxf(tmax[u], __shfl_xor_sync(0xffffffffu, tmax[u], 1));
            tmax[u] = fmaxf(tmax[u], __shfl_xor_sync(0xffffffffu, tmax[u], 2));
            const float mnew = fmaxf(mrow[u], tmax[u]);
            alpha[u] = (mnew == -INFINITY) ? 1.f : exp2f(mrow[u] - mnew);
            mrow[u] = mnew;
            lrow[u] *= alpha[u];
          }
          uint32_t pa[NT][2];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            float pv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int u = e >> 1;
              pv[e] = (sacc[nt][e] == -INFINITY) ? 0.f : exp2f(sacc[nt][e] - mrow[u]);
              lrow[u] += pv[e];
            }
            pa[nt][0] = pack_bf16(pv[0], pv[1]);
            pa[nt][1] = pack_bf16(pv[2], pv[3]);
          }
#pragma unroll
          for (int dt = 0; dt < DT; ++dt) {
            o[dt][0] *= alpha[0];
            o[dt][1] *= alpha[0];
            o[dt][2] *= alpha[1];
            o[dt][3] *= alpha[1];
          }
#pragma unroll
          for (int kc = 0; kc < NT / 2; ++kc) {
            const uint32_t a0 = pa[2 * kc][0], a1 = pa[2 * kc][1], a2 = pa[2 * kc + 1][0],
                           a3 = pa[2 * kc + 1][1];
#pragma unroll
            for (int dt = 0; dt < DT; dt += 2) {
              const int row = kc * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
              const int col = dt * 8 + (lane >> 4) * 8;
              uint32_t b0, b1, b2, b3;
              ldsm_x4_t(vbase + tile_off(row, col), b0, b1, b2, b3);
              mma_bf16(o[dt], a0, a1, a2, a3, b0, b1);
              mma_bf16(o[dt + 1], a0, a1, a2, a3, b2, b3);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          lrow[u] += __shfl_xor_sync(0xffffffffu, lrow[u], 1);
          lrow[u] += __shfl_xor_sync(0xffffffffu, lrow[u], 2);
        }
        if (nsplit_c == 1) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int m = qm[u];
            if (m >= Qg) continue;
            const int j = m / g, ii = m % g;
            __nv_bfloat16* op = (__nv_bfloat16*)p.out + (((size_t)r * p.b_live + j) * p.Hq + h * g + ii) * D;
            const float inv = lrow[u] > 0.f ? 1.f / lrow[u] : 0.f;
#pragma unroll
            for (int dt = 0; dt < DT; ++dt)
              *(uint32_t*)(op + dt * 8 + cq * 2) = pack_bf16(o[dt][u * 2] * inv, o[dt][u * 2 + 1] * inv);
            if (cq == 0) {
              if (lrow[u] == 0.f) latch(p.status, TRIE_ST_EMPTY_ROW);
              if (p.lse)
                p.lse[((size_t)r * p.b_live + j) * p.Hq + h * g + ii] =
                    lrow[u] > 0.f ? (mrow[u] + log2f(lrow[u])) * 0.69314718055994531f : -INFINITY;
            }
          }
        } else {
          float* pbase = p.part + (((size_t)r * p.Hkv + h) * p.splits + split) * Qg * (D + 2);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int m = qm[u];
            if (m >= Qg) continue;
            float* pp = pbase + (size_t)m * (D + 2);
#pragma unroll
            for (int dt = 0; dt < DT; ++dt) {
              pp[dt * 8 + cq * 2] = o[dt][u * 2];
              pp[dt * 8 + cq * 2 + 1] = o[dt][u * 2 + 1];
            }
            if (cq == 0) {
              pp[D] = mrow[u];
              pp[D + 1] = lrow[u];
            }
          }
          __threadfence();
          asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));  // all m-tiles of the chunk written
          if (cw == 0 && lane == 0) *s_flag = atomicAdd(&ctr->item[r * p.Hkv + h], 1) == nsplit_c - 1;
          asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));
          if (*s_flag) {
            __threadfence();
            for (int m = mt * 16; m < min(Qg, mt * 16 + 16); ++m) combine_query<D>(p, r, h, m, nsplit_c, Qg);
            asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));
            if (cw == 0 && lane == 0) ctr->item[r * p.Hkv + h] = 0;
          }
          asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));  // s_flag reuse
        }
      }
      ++ccount;
    }
  }
  // queue reset by the last CTA to finish (all producers have stopped fetching by then)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ctr->done, 1) == (int)gridDim.x - 1) {
      ctr->next = 0;
      ctr->done = 0;
      __threadfence();
    }
  }
}

// ---- host side ---------------------------------------------------------------------------

struct PKernel {
  const void* fn;
  int smem, threads, occ;
};

template <typename Kern>
static PKernel make_p(Kern kern, int smem, int threads) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  return PKernel{(const void*)kern, smem, threads, occ > 0 ? occ : 1};
}

template <int D, int QMAX, int ST, int NCW, bool NARROW>
static const PKernel& pk() {
  using C = PCfg<D, QMAX, ST, NCW>;
  static const PKernel k = make_p(k_attn_persist<D, QMAX, ST, NCW, NARROW>, C::SMEM, C::THREADS);
  return k;
}

static int p_stages_narrow() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TRIE_PNARROW_STAGES");
    v = e ? atoi(e) : 2;
    if (v < 2 || v > 4) v = 2;
  }
  return v;
}

template <int D>
static const PKernel& select_pd(int Qg) {
  if (Qg <= 8) {
    if (p_stages_narrow() == 3) return pk<D, 8, 3, 1, true>();
    return pk<D, 8, 2, 1, true>();
  }
  if (Qg <= 16) {
    if (p_stages_narrow() == 3) return pk<D, 16, 3, 1, true>();
    return pk<D, 16, 2, 1, true>();
  }
  if (Qg <= 32) return pk<D, 32, 3, 2, false>();
  if (Qg <= 64) return pk<D, 64, 2, 4, false>();
  return pk<D, 128, 2, 8, false>();
}
static const PKernel* select_p(int D, int Qg) {
  switch (D) {
    case 64: return &select_pd<64>(Qg);
    case 96: return &select_pd<96>(Qg);
    case 128: return &select_pd<128>(Qg);
  }
  return nullptr;
}

bool attn_persist_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TRIE_ATTN_PERSIST");
    v = e ? atoi(e) : 0;  // opt-in (r04: slower than the per-item path)
  }
  return v != 0;
}

// chunks per item: enough chunks for ~3 waves of resident CTAs, >= 2 tiles per chunk
int attn_persist_splits(const AttnParams& p, int rows_est, int sms) {
  const PKernel* k = select_p(p.D, p.b_live * (p.Hq / p.Hkv));
  const int occ = k ? k->occ : 2;
  const int items = p.R * p.Hkv;
  const int tiles = (rows_est + TC_TR - 1) / TC_TR;
  const char* fe = getenv("TRIE_ATTN_SPLITS");  // experiments only
  if (fe && atoi(fe) > 0) return std::min(atoi(fe), 64);
  const long target = 3L * occ * sms;
  int ct = (int)(((long)items * tiles + target - 1) / target);
  if (ct < 2) ct = 2;
  int splits = (tiles + ct - 1) / ct;
  if (splits < 1) splits = 1;
  if (splits > 64) splits = 64;
  return splits;
}

size_t attn_persist_counter_bytes(const AttnParams& p) {
  return (size_t)(32 + p.R * p.Hkv) * 4 + 256;
}

int launch_attn_persist(const AttnParams& p, cudaStream_t s) {
  const int Qg = p.b_live * (p.Hq / p.Hkv);
  const PKernel* k = select_p(p.D, Qg);
  if (!k) return trie_set_error(TRIE_EINVAL, "persistent attention: unsupported head_dim %d", p.D);
  CUtensorMap km, vm;
  const long rows = (long)p.R * p.Hkv * p.cap;
  int rc = cached_tensor_map(&km, p.k, p.D, rows);
  if (!rc) rc = cached_tensor_map(&vm, p.v, p.D, rows);
  if (rc) return rc;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (!sms) sms = 148;
  }
  const int nsplit = p.splits;
  const int total = p.R * p.Hkv * nsplit;
  int grid = k->occ * sms;
  if (grid > total) grid = total;
  AttnParams pp = p;
  int ns = nsplit, tot = total;
  void* args[5] = {(void*)&km, (void*)&vm, (void*)&pp, (void*)&ns, (void*)&tot};
  cudaLaunchKernel(k->fn, dim3(grid), dim3(k->threads), args, (size_t)k->smem, s);
  return trie_check_launch("k_attn_persist");
}

}  // namespace trie
