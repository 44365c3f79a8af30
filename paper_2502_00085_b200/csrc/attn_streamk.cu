// trie_attn_decode_rope, wide bf16 path with a stream-K work split (sm_100a).
//
// Why: the per-item wide kernel (attn_decode_tc.cu) runs one CTA per (request, KV head).
// On short, ragged tries (Llama configs[2]: 256 items of 5..15 64-row tiles, 2 CTAs per
// SM) one launch is a single partial wave whose length is set by the LONGEST item: a CTA
// keeps at most STAGES tiles in flight, so its stream is latency-bound, and the SMs that
// finished their short items idle for the rest of the launch (r08 traces: streaming CTAs
// fall from 256 to 66 over the last third of the launch).
//
// What: a grid of G = (resident CTAs per SM) x SMs CTAs.  The unique tiles of every
// (request r, KV head h) item -- the request's tiles from the window's first tile to
// ceil(N_r / 64) (§3.3: each unique row read once per KV head and shared by all b*g
// queries) -- are laid out end to end in one global tile sequence of length W (request
// major, head minor), and CTA c streams the contiguous range [c W / G, (c+1) W / G).
// A range may cover the tail of one item, several whole items and the head of another;
// the producer streams across item boundaries without draining the ring, the consumers
// restart the online softmax (§3.3 flash decode) at each boundary.  Items cut by a range
// boundary are merged exactly (online-softmax rescale of (m, l, o) partials, as k_attn_
// combine does): each participant writes its partial, the last to arrive (a per-item
// ticket, acq_rel) merges the others into its registers and writes the output; the
// ticket is left at zero for the next launch (graph-replayable).
//
// Everything else is the fused wide kernel: TMA (SWIZZLE_64B) K/V tiles + 1-D bulk copies
// of the tile's beam-mask / depth words into an S-stage mbarrier ring (warp 0, one lane),
// MT x RS consumer warps of mma.sync m16n8k16 (S = Q K^T, P V), exact exclusion of masked
// keys (reading R22), Q rotated in registers at the beams' depth, the leaves' K / V rows
// rotated and appended by warp 0's other lanes before the producer loads their tile
// (write-before-read, §3.4, Alg. 3 l.7 P:175).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <float.h>
#include <stdlib.h>

#include "attn_common.cuh"
#include "common.cuh"
#include "handle.h"
#include "tc_common.cuh"

namespace trie {

constexpr int SK_MAX_R = 256;
constexpr bool ROPE_PF = true;  // L2-prefetch the RoPE table rows of later segments too  // requests per launch held in the shared-memory table

template <int D, int MT, int RS, int ST>
struct SkCfg {
  using RG = Ring<D, ST>;
  static constexpr int STAGES = ST;
  static constexpr int KS = D / 16;
  static constexpr int DT = D / 8;
  static constexpr int RSZ = TC_TR / RS;
  static constexpr int NT = RSZ / 8;
  static constexpr int NC = MT * RS;
  static constexpr int THREADS = 32 * (NC + 1);
  static_assert(NT % 2 == 0, "row slice must be a multiple of 16");
  // row-slice merge buffer: the segment's last ring stage, held until the merge is read
  static_assert((RS - 1) * MT * 16 * (D + 2) * 4 <= RG::STAGE_BYTES, "merge buffer > stage");
  static constexpr int OFF_BAR = RG::RING_BYTES;                 // full[ST] empty[ST] app_done
  static constexpr int OFF_TAB = OFF_BAR + 256;                  // int4 rq[R] | int ff[R] | int pre[R+1]
  static constexpr int SMEM = OFF_TAB + SK_MAX_R * 20 + (SK_MAX_R + 1) * 4 + 1024;
};

// One contiguous piece of an item inside a CTA's tile range.
struct SkSeg {
  int r, h, a, e;  // request, KV head, item-relative tile range [a, e)
};

// Deterministic walk over the CTA's range; every role iterates it the same way.
struct SkIter {
  const int4* rq;
  const int* pre;
  int R, Hkv;
  int pos, end;  // global tile positions
  int r, h, a;
  __device__ void start(int b0, int b1) {
    pos = b0;
    end = b1;
    // the request whose global range holds b0: pre[r] <= b0 < pre[r + 1]
    int lo = 0, hi = R - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= b0) lo = mid; else hi = mid - 1;
    }
    r = lo;
    while (r < R && pre[r + 1] <= b0) ++r;  // zero-tile requests share the same prefix
    if (r < R) {
      const int x = b0 - pre[r], T = rq[r].y;
      h = x / T;
      a = x % T;
    }
  }
  __device__ bool next(SkSeg& s) {
    if (pos >= end || r >= R) return false;
    const int T = rq[r].y;
    const int e = min(T, a + (end - pos));
    s = SkSeg{r, h, a, e};
    pos += e - a;
    a = e;
    if (a == T) {
      a = 0;
      if (++h == Hkv) {
        h = 0;
        do { ++r; } while (r < R && rq[r].y == 0);
      }
    }
    return true;
  }
};

__device__ __forceinline__ int sk_bound(int c, int W, int G) { return (int)(((long long)c * W) / G); }
// the CTA whose range holds global tile x
__device__ __forceinline__ int sk_cta_of(int x, int W, int G) {
  return (int)((((long long)x + 1) * G - 1) / W);
}

// Warp 0: the request table (first tile, tiles, N, t), the unmasked-from tile and the
// exclusive prefix of Hkv * tiles.  The window's first slot as in item_setup (lowest
// beam's lower depth; prompt chain probe, else a binary search over the non-decreasing
// depth[] of the request).
__device__ __forceinline__ void sk_table(const AttnParams& p, int4* rq, int* ff, int* pre) {
  const int lane = threadIdx.x & 31;
  const int R = p.R;
  const int cpl = (R + 31) / 32;
  int sum = 0;
  for (int i = 0; i < cpl; ++i) {
    const int r = lane * cpl + i;
    if (r >= R) break;
    const size_t mbase = (size_t)r * p.cap;
    const int N = p.nn[r], t = p.tlen[r];
    bool done = false;
    if (p.fin) {
      done = true;
      for (int j = 0; j < p.b_live; ++j) done = done && p.fin[r * TRIE_MAX_BEAMS + j] != 0u;
    }
    int lo = 0, fast_from = 0;
    if (p.window > 0) {
      int dl = INT_MAX, dh = INT_MIN;
      for (int j = 0; j < p.b_live; ++j) {
        const int d = p.depth[mbase + p.leaf[r * TRIE_MAX_BEAMS + j]] - p.window + 1;
        dl = min(dl, d);
        dh = max(dh, d);
      }
      if (dl > 0) {
        if (dl < N && p.depth[mbase + dl - 1] < dl && p.depth[mbase + dl] >= dl) {
          lo = dl;
        } else {  // first n with depth[n] >= dl
          int a = 0, b = N;
          while (a < b) {
            const int m = (a + b) >> 1;
            if (p.depth[mbase + m] >= dl) b = m; else a = m + 1;
          }
          lo = a;
        }
      }
      fast_from = (max(dh, 0) + TC_TR - 1) / TC_TR;
    }
    const int first = lo / TC_TR;
    const int T = done ? 0 : (N + TC_TR - 1) / TC_TR - first;
    rq[r] = make_int4(first, T, N, t);
    ff[r] = fast_from;
    pre[r] = sum;  // lane-local exclusive prefix, offset below
    sum += p.Hkv * T;
  }
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int off = incl - sum;
  for (int i = 0; i < cpl; ++i) {
    const int r = lane * cpl + i;
    if (r >= R) break;
    pre[r] += off;
  }
  if (lane == 31) pre[R] = incl;
}

template <int D, int MT, int RS, int ST>
__global__ void __launch_bounds__(SkCfg<D, MT, RS, ST>::THREADS, 2) k_attn_wide_sk(
    const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
    const AttnParams p, const __grid_constant__ CUtensorMap kmh,
    const __grid_constant__ CUtensorMap vmh) {
  using C = SkCfg<D, MT, RS, ST>;
  using RG = typename C::RG;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  uint64_t* full = (uint64_t*)(smem + C::OFF_BAR);
  uint64_t* empty = full + ST;
  uint64_t* app_done = empty + ST;
  int4* rq = (int4*)(smem + C::OFF_TAB);
  int* ff = (int*)(rq + SK_MAX_R);
  int* pre = ff + SK_MAX_R;

  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NC);
    }
    mbar_init(app_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();
  if (warp == 0) {
    sk_table(p, rq, ff, pre);
    __syncwarp();
    __threadfence_block();
    asm volatile("bar.arrive 2, %0;" ::"r"(C::THREADS) : "memory");
    const int W = pre[p.R];
    // G = min(grid, W): every CTA range non-empty, so an item's participants are exactly
    // the CTAs cf..cl its tiles map to (the merge ticket counts them)
    const int G = min((int)gridDim.x, W);
    if (c >= G) return;
    SkIter it{rq, pre, p.R, p.Hkv};
    it.start(sk_bound(c, W, G), sk_bound(c + 1, W, G));
    if (lane != 0) {
      // fused a-1: rotate + append every leaf row inside this CTA's tile ranges, then
      // make the generic-proxy writes visible to the TMA reads of lane 0
      SkSeg s;
      while (it.next(s)) {
        const int4 q = rq[s.r];
        append_leaves_rope_work<D>(p, s.r, s.h, (q.x + s.a) * TC_TR, (q.x + s.e) * TC_TR, lane - 1, 31,
                                   q.z - p.b_live);
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncwarp(0xfffffffeu);
      if (lane == 1) mbar_arrive(app_done);
      return;
    }
    // ---- producer (lane 0) ----
    bool appended = false;
    int gi = 0;
    SkSeg s;
    while (it.next(s)) {
      const int4 q = rq[s.r];
      const int N = q.z, first_leaf = N - p.b_live;
      const int row_base = (s.r * p.Hkv + s.h) * p.cap;
      const size_t mbase = (size_t)s.r * p.cap;
      for (int i = s.a; i < s.e; ++i, ++gi) {
        const int st = gi % ST;
        mbar_wait(&empty[st], ((uint32_t)(gi / ST) & 1u) ^ 1u);
        const int n0 = (q.x + i) * TC_TR;
        if (!appended && n0 + TC_TR > first_leaf) {  // the tile holds leaf rows
          mbar_wait(app_done, 0u);
          appended = true;
        }
        const uint32_t sb = smem_u32(ring + st * RG::STAGE_BYTES);
        const uint32_t mdb = (uint32_t)min(TC_TR, p.cap - n0) * 4u;
        // an item's last tile with <= 32 rows below N loads 32-row boxes (stage reused:
        // its other rows hold finite K/V of an earlier tile and are masked, n >= N)
        const bool half = p.half_tiles && gi >= ST && N - n0 <= TC_TR / 2;
        mbar_expect_tx(&full[st], (half ? RG::TILE_BYTES : 2 * RG::TILE_BYTES) + 2 * mdb);
        const CUtensorMap* km = half ? &kmh : &kmap;
        const CUtensorMap* vm = half ? &vmh : &vmap;
#pragma unroll
        for (int bx = 0; bx < D / TC_CW; ++bx) {
          tma_load_2d(sb + bx * TC_TR * 64, km, bx * TC_CW, row_base + n0, &full[st]);
          tma_load_2d(sb + RG::TILE_BYTES + bx * TC_TR * 64, vm, bx * TC_CW, row_base + n0, &full[st]);
        }
        bulk_load_1d(sb + 2 * RG::TILE_BYTES, p.mask + mbase + n0, mdb, &full[st]);
        bulk_load_1d(sb + 2 * RG::TILE_BYTES + TC_TR * 4, p.depth + mbase + n0, mdb, &full[st]);
      }
    }
    return;
  }

  // ===== consumer warps =====
  const int cw = warp - 1;
  const int mt = cw % MT, rs = cw / MT;
  const int r0 = rs * C::RSZ;
  const int g = p.Hq / p.Hkv, Qg = p.b_live * g;
  const int gq = lane >> 2, cq = lane & 3;
  const float sc = p.scale_log2;
  int qm[2], beam[2];
  uint32_t bbit[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    qm[u] = mt * 16 + gq + 8 * u;
    beam[u] = qm[u] < Qg ? qm[u] / g : 0;
    bbit[u] = qm[u] < Qg ? 1u << beam[u] : 0u;
  }
  asm volatile("bar.sync 2, %0;" ::"r"(C::THREADS) : "memory");  // the table is published
  const int W = pre[p.R];
  const int G = min((int)gridDim.x, W);
  if (c >= G) return;
  SkIter it{rq, pre, p.R, p.Hkv};
  const int b0 = sk_bound(c, W, G);
  it.start(b0, sk_bound(c + 1, W, G));
  {
    // the Q rows and RoPE table of the CTA's later segments: into L2 now, so a segment
    // switch does not wait a loaded-HBM round trip (the first segment's are read at once)
    SkIter pf = it;
    SkSeg s;
    bool first = true;
    while (pf.next(s)) {
      if (first) { first = false; continue; }
      const int m = mt * 16 + (lane >> 1);
      if (m < Qg) {
        const int j = m / g;
        const char* qa = (const char*)((const __nv_bfloat16*)p.q +
                                       (((size_t)s.r * p.b_live + j) * p.Hq + s.h * g + m - j * g) * D);
        for (int off = (lane & 1) * 128; off < D * 2; off += 256)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(qa + off));
        if (ROPE_PF && rs == 0 && (m % g) == 0) {
          const char* rt = (const char*)(p.rope_tab + ((size_t)s.r * p.b_live + j) * (D / 2));
          for (int off = (lane & 1) * 128; off < D * 4; off += 256)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(rt + off));
        }
      }
    }
  }
  int gi = 0;
  SkSeg s;
  while (it.next(s)) {
    const int4 q4 = rq[s.r];
    const int r = s.r, h = s.h;
    const int N = q4.z, t = q4.w;
    const size_t mbase = (size_t)r * p.cap;
    int lod[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      lod[u] = INT_MIN;
      if (p.window > 0 && qm[u] < Qg)
        lod[u] = p.depth[mbase + p.leaf[r * TRIE_MAX_BEAMS + beam[u]]] - p.window + 1;
    }
    // Q of this item (queries m = beam * g + head of the group), rotated at the beam depth
    uint32_t qa[C::KS][4];
    {
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
          qa[ks][u] = src ? *(const uint32_t*)(src + ks * 16 + (u >> 1) * 8 + cq * 2) : 0u;
        }
      constexpr int HALF = D / 2;
#pragma unroll
      for (int ks = 0; ks < C::KS / 2; ++ks)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (!qrow[u & 1]) continue;
          const int col = ks * 16 + (u >> 1) * 8 + cq * 2;
          const float4 tt = __ldg((const float4*)(p.rope_tab + ((size_t)r * p.b_live + beam[u & 1]) * HALF + col));
          const float2 x1 = __bfloat1622float2(*(const __nv_bfloat162*)&qa[ks][u]);
          const float2 x2 = __bfloat1622float2(*(const __nv_bfloat162*)&qa[ks + C::KS / 2][u]);
          qa[ks][u] = pack_bf16(x1.x * tt.x - x2.x * tt.y, x1.y * tt.z - x2.y * tt.w);
          qa[ks + C::KS / 2][u] = pack_bf16(x2.x * tt.x + x1.x * tt.y, x2.y * tt.z + x1.y * tt.w);
        }
    }
    float o[C::DT][4];
#pragma unroll
    for (int i = 0; i < C::DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
    const int fast_end = min(t, N) / TC_TR, fast_from = ff[r];
    int st_last = 0;
    for (int i = s.a; i < s.e; ++i, ++gi) {
      const int st = gi % ST;
      mbar_wait(&full[st], (uint32_t)(gi / ST) & 1u);
      const uint8_t* stg = ring + st * RG::STAGE_BYTES;
      const uint32_t kbase = smem_u32(stg), vbase = smem_u32(stg + RG::TILE_BYTES);
      const int tile = q4.x + i;
      const int n0 = tile * TC_TR;
      const bool fast = tile >= fast_from && tile < fast_end;
      float sacc[C::NT][4];
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < C::KS; ++ks)
#pragma unroll
        for (int nt = 0; nt < C::NT; nt += 2) {
          const int row = r0 + (nt + (lane >> 4)) * 8 + (lane & 7);
          const int col = ks * 16 + ((lane >> 3) & 1) * 8;
          uint32_t b0_, b1_, b2_, b3_;
          ldsm_x4(kbase + tile_off(row, col), b0_, b1_, b2_, b3_);
          mma_bf16(sacc[nt], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0_, b1_);
          mma_bf16(sacc[nt + 1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b2_, b3_);
        }
      float tmax[2] = {-INFINITY, -INFINITY};
      if (fast) {
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int u = e >> 1;
            const float v = qm[u] < Qg ? sacc[nt][e] * sc : -INFINITY;
            sacc[nt][e] = v;
            tmax[u] = fmaxf(tmax[u], v);
          }
      } else {
        const uint32_t* tmask = (const uint32_t*)(stg + 2 * RG::TILE_BYTES);
        const int* tdep = (const int*)(stg + 2 * RG::TILE_BYTES + TC_TR * 4);
        const bool win = p.window > 0;
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int lr = r0 + nt * 8 + cq * 2 + cc;
            const int n = n0 + lr;
            const uint32_t vis = n >= N ? 0u : (n < t ? ~0u : tmask[lr]);
            const int dep = win ? tdep[lr] : 0;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const bool ok = (vis & bbit[u]) != 0u && dep >= lod[u];
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
      uint32_t pa[C::NT][2];
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) {
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
          uint32_t b0_, b1_, b2_, b3_;
          ldsm_x4_t(vbase + tile_off(row, col), b0_, b1_, b2_, b3_);
          mma_bf16(o[dt], a0, a1, a2, a3, b0_, b1_);
          mma_bf16(o[dt + 1], a0, a1, a2, a3, b2_, b3_);
        }
      }
      __syncwarp();
      st_last = st;
      // the segment's last stage is held for the row-slice merge (RS > 1)
      if (lane == 0 && (RS == 1 || i + 1 < s.e)) mbar_arrive(&empty[st]);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      lrow[u] += __shfl_xor_sync(0xffffffffu, lrow[u], 1);
      lrow[u] += __shfl_xor_sync(0xffffffffu, lrow[u], 2);
    }
    if constexpr (RS > 1) {
      // slices rs > 0 park (O, m, l) in the held stage, slice 0 folds them in
      constexpr int RW = D + 2;
      float* red = (float*)(ring + st_last * RG::STAGE_BYTES);
      __syncwarp();
      asm volatile("bar.sync 1, %0;" ::"r"(C::NC * 32) : "memory");  // the stage's K/V are consumed
      if (rs > 0) {
        float* mine = red + (size_t)((rs - 1) * MT + mt) * 16 * RW;
#pragma unroll
        for (int dt = 0; dt < C::DT; ++dt) {
          const int col = dt * 8 + cq * 2;
          *(float2*)&mine[gq * RW + col] = make_float2(o[dt][0], o[dt][1]);
          *(float2*)&mine[(gq + 8) * RW + col] = make_float2(o[dt][2], o[dt][3]);
        }
        if (cq == 0) {
          *(float2*)&mine[gq * RW + D] = make_float2(mrow[0], lrow[0]);
          *(float2*)&mine[(gq + 8) * RW + D] = make_float2(mrow[1], lrow[1]);
        }
      }
      __syncwarp();
      asm volatile("bar.sync 1, %0;" ::"r"(C::NC * 32) : "memory");
      if (rs == 0) {
#pragma unroll
        for (int x = 0; x < RS - 1; ++x) {
          const float* src = red + (size_t)(x * MT + mt) * 16 * RW;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int row = gq + 8 * u;
            const float2 ml = *(const float2*)&src[row * RW + D];
            const float mn = fmaxf(mrow[u], ml.x);
            const float w1 = mrow[u] == -INFINITY ? 0.f : exp2f(mrow[u] - mn);
            const float w2 = ml.x == -INFINITY ? 0.f : exp2f(ml.x - mn);
#pragma unroll
            for (int dt = 0; dt < C::DT; ++dt) {
              const float2 v = *(const float2*)&src[row * RW + dt * 8 + cq * 2];
              o[dt][u * 2] = o[dt][u * 2] * w1 + v.x * w2;
              o[dt][u * 2 + 1] = o[dt][u * 2 + 1] * w1 + v.y * w2;
            }
            lrow[u] = lrow[u] * w1 + ml.y * w2;
            mrow[u] = mn;
          }
        }
      }
      // generic-proxy accesses of the stage before the TMA (async proxy) refills it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st_last]);
      if (rs > 0) continue;
    }
    // ---- epilogue of the segment (row slice 0 of each m-tile) ----
    const int T = q4.y;
    if (s.a > 0 || s.e < T) {
      // the item is split over CTAs: write this partial, the last arrival merges
      const int P = pre[r] + h * T;                 // the item's first global tile
      const int cf = sk_cta_of(P, W, G), cl = sk_cta_of(P + T - 1, W, G);
      const int slot = 2 * c + ((c == cf && b0 < P) ? 1 : 0);
      constexpr int RW = D + 2;
      float* mine = p.part + ((size_t)slot * MT + mt) * 16 * RW;
#pragma unroll
      for (int dt = 0; dt < C::DT; ++dt) {
        const int col = dt * 8 + cq * 2;
        *(float2*)&mine[gq * RW + col] = make_float2(o[dt][0], o[dt][1]);
        *(float2*)&mine[(gq + 8) * RW + col] = make_float2(o[dt][2], o[dt][3]);
      }
      if (cq == 0) {
        *(float2*)&mine[gq * RW + D] = make_float2(mrow[0], lrow[0]);
        *(float2*)&mine[(gq + 8) * RW + D] = make_float2(mrow[1], lrow[1]);
      }
      __threadfence();
      __syncwarp();
      uint32_t* ticket = p.tickets + ((size_t)r * p.Hkv + h) * MT + mt;
      uint32_t old = 0;
      if (lane == 0) asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(ticket) : "memory");
      old = __shfl_sync(0xffffffffu, old, 0);
      if ((int)old != cl - cf) continue;  // another participant merges
      __threadfence();
      for (int cc = cf; cc <= cl; ++cc) {
        if (cc == c) continue;
        const int sl = 2 * cc + ((cc == cf && sk_bound(cc, W, G) < P) ? 1 : 0);
        const float* src = p.part + ((size_t)sl * MT + mt) * 16 * RW;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int row = gq + 8 * u;
          const float2 ml = __ldcg((const float2*)&src[row * RW + D]);
          const float mn = fmaxf(mrow[u], ml.x);
          const float w1 = mrow[u] == -INFINITY ? 0.f : exp2f(mrow[u] - mn);
          const float w2 = ml.x == -INFINITY ? 0.f : exp2f(ml.x - mn);
#pragma unroll
          for (int dt = 0; dt < C::DT; ++dt) {
            const float2 v = __ldcg((const float2*)&src[row * RW + dt * 8 + cq * 2]);
            o[dt][u * 2] = o[dt][u * 2] * w1 + v.x * w2;
            o[dt][u * 2 + 1] = o[dt][u * 2 + 1] * w1 + v.y * w2;
          }
          lrow[u] = lrow[u] * w1 + ml.y * w2;
          mrow[u] = mn;
        }
      }
      if (lane == 0) *ticket = 0u;  // graph-replayable: zero for the next launch
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int m = qm[u];
      if (m >= Qg) continue;
      const int j = m / g, ii = m % g;
      __nv_bfloat16* op = (__nv_bfloat16*)p.out + (((size_t)r * p.b_live + j) * p.Hq + h * g + ii) * D;
      const float inv = lrow[u] > 0.f ? 1.f / lrow[u] : 0.f;
#pragma unroll
      for (int dt = 0; dt < C::DT; ++dt)
        *(uint32_t*)(op + dt * 8 + cq * 2) = pack_bf16(o[dt][u * 2] * inv, o[dt][u * 2 + 1] * inv);
      if (cq == 0) {
        if (lrow[u] == 0.f) latch(p.status, TRIE_ST_EMPTY_ROW);
        if (p.lse)
          p.lse[((size_t)r * p.b_live + j) * p.Hq + h * g + ii] =
              lrow[u] > 0.f ? (mrow[u] + log2f(lrow[u])) * 0.69314718055994531f : -INFINITY;
      }
    }
  }
}

// ---- host side ---------------------------------------------------------------------------
struct SkKernel {
  const void* fn;
  int smem, threads, occ;
};

template <int D, int MT, int RS, int ST>
static const SkKernel& sk_kernel() {
  static const SkKernel k = [] {
    using C = SkCfg<D, MT, RS, ST>;
    auto kern = k_attn_wide_sk<D, MT, RS, ST>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM);
    return SkKernel{(const void*)kern, C::SMEM, C::THREADS, occ > 0 ? occ : 1};
  }();
  return k;
}

// stages per CTA (TRIE_SK_STAGES in {2, 3, 4}); default: 3 at D = 128, else 4
static int sk_stages(int D) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TRIE_SK_STAGES");
    v = e ? atoi(e) : 0;
    if (v != 2 && v != 3 && v != 4) v = 0;
  }
  return v ? v : (D >= 128 ? 3 : 4);
}

template <int D>
static const SkKernel* sk_select_d() {
  switch (sk_stages(D)) {
    case 2: return &sk_kernel<D, 2, 2, 2>();
    case 3: return &sk_kernel<D, 2, 2, 3>();
    default: return &sk_kernel<D, 2, 2, 4>();
  }
}

static const SkKernel* sk_select(int D) {
  switch (D) {
    case 64: return sk_select_d<64>();
    case 96: return sk_select_d<96>();
    case 128: return sk_select_d<128>();
  }
  return nullptr;
}

static bool sk_env_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TRIE_ATTN_STREAMK");  // opt-in until it beats the per-item kernel
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// The fused (handle) path of a wide shape: 16 < b_live * g <= 32, bf16, D in {64, 96, 128},
// not the tcgen05 kernel's, at most SK_MAX_R requests.
bool attn_sk_eligible(const AttnParams& p) {
  const int Qg = p.b_live * (p.Hq / p.Hkv);
  return sk_env_enabled() && p.rope && attn_tc_shape_ok(p) && !attn_umma_eligible(p) && Qg > 16 &&
         Qg <= 32 && p.R <= SK_MAX_R;
}

int attn_sk_grid(const AttnParams& p, int sms) {
  const SkKernel* k = sk_select(p.D);
  return k ? k->occ * sms : sms;
}

size_t attn_sk_part_bytes(const AttnParams& p, int sms) {
  return (size_t)2 * attn_sk_grid(p, sms) * 2 /*MT*/ * 16 * (p.D + 2) * 4;
}

int launch_attn_wide_sk(const AttnParams& p, int grid, cudaStream_t s) {
  const SkKernel* k = sk_select(p.D);
  if (!k) return trie_set_error(TRIE_EINVAL, "stream-K attention: unsupported head_dim %d", p.D);
  if (!p.tickets) return trie_set_error(TRIE_EINVAL, "stream-K attention needs the handle's tickets");
  CUtensorMap km, vm, kmh, vmh;
  const long rows = (long)p.R * p.Hkv * p.cap;
  int rc = cached_tensor_map(&km, p.k, p.D, rows);
  if (!rc) rc = cached_tensor_map(&vm, p.v, p.D, rows);
  if (!rc) rc = cached_tensor_map(&kmh, p.k, p.D, rows, TC_TR / 2);
  if (!rc) rc = cached_tensor_map(&vmh, p.v, p.D, rows, TC_TR / 2);
  if (rc) return rc;
  AttnParams pp = p;
  pp.half_tiles = 1;
  void* args[5] = {(void*)&km, (void*)&vm, (void*)&pp, (void*)&kmh, (void*)&vmh};
  launch_k_ptr(k->fn, dim3(grid), dim3(k->threads), (size_t)k->smem, s, args);
  return trie_check_launch("k_attn_wide_sk");
}

}  // namespace trie
