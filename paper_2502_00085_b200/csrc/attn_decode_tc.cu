// trie_attn_decode, bf16 tensor-core path (sm_100a): TMA-fed, mbarrier-pipelined
// split-K flash-decode over the shared trie KV pool (§3.3; Alg. 3).
//
// One CTA per (KV head h, request r, split).  Warp 0 is the producer: one elected lane
// streams 64-slot tiles of K and V (head-major pool => a tile is a contiguous 2-D box)
// with cp.async.bulk.tensor (TMA, 64-byte swizzle) plus the tile's beam_mask / depth
// words with 1-D bulk copies, into an S-stage ring guarded by full/empty mbarriers.
// Every unique KV row is read from HBM exactly once per (request, KV head) and feeds all
// Qg = b_live * (Hq/Hkv) queries of that head: GQA grouping + trie sharing.
// Consumer warps: warp w owns query m-tile (w % MT) (16 queries) and row slice
// (w / MT) of every tile; S = Q K^T and O += P V run on mma.sync.m16n8k16 (bf16 in,
// fp32 accumulate) with ldmatrix from the swizzled tiles; masked keys get -inf before
// the online softmax (exact exclusion, reading R22).  Row-slice partials (m, l, O) are
// merged in shared memory at the end; split partials go to k_attn_combine.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <float.h>
#include <stdio.h>

#include "attn_common.cuh"
#include "common.cuh"
#include "handle.h"

namespace trie {

constexpr int TC_TR = 64;      // slots per tile
constexpr int TC_CW = 32;      // elements per swizzle box column (64 bytes, SWIZZLE_64B)

// ---- PTX helpers -------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load_1d(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c,
                                        uint32_t& d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c,
                                          uint32_t& d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *(uint32_t*)&v;
}

// byte offset of (row, col) inside one tile: D/32 boxes of [TR rows][32 cols], 64B swizzle
__device__ __forceinline__ uint32_t tile_off(int row, int col) {
  const int box = col / TC_CW;
  const uint32_t o = (uint32_t)row * 64u + (uint32_t)(col % TC_CW) * 2u;
  return (uint32_t)box * (TC_TR * 64u) + (o ^ (((o >> 7) & 3u) << 4));
}

template <int D, int MT>
struct TcCfg {
  static constexpr int STAGES = D >= 128 ? 3 : 4;  // 2 CTAs per SM for D <= 128
  static constexpr int NC = MT < 4 ? 4 : MT;   // consumer warps
  static constexpr int RS = NC / MT;           // row slices per tile
  static constexpr int RSZ = TC_TR / RS;       // rows per warp per tile
  static constexpr int NT = RSZ / 8;           // S n-tiles per warp
  static constexpr int KS = D / 16;            // k-steps of Q K^T
  static constexpr int DT = D / 8;             // O n-tiles
  static constexpr int TILE_BYTES = TC_TR * D * 2;
  // stage = K tile | V tile | mask words | depth words, 1024-byte aligned (swizzle atoms)
  static constexpr int STAGE_BYTES = (2 * TILE_BYTES + 2 * TC_TR * 4 + 1023) / 1024 * 1024;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8 + 64;
  static constexpr int THREADS = 32 * (NC + 1);
};

template <int D, int MT>
__global__ void __launch_bounds__(TcCfg<D, MT>::THREADS) k_attn_tc(
    const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
    const AttnParams p) {
  using C = TcCfg<D, MT>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  int* s_info = (int*)(empty + C::STAGES);  // [0] tile0, [1] ntiles, [2] lo slot

  const int h = blockIdx.x, r = blockIdx.y, split = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = p.Hq / p.Hkv, Qg = p.b_live * g;
  const size_t mbase = (size_t)r * p.cap;
  const int N = p.nn[r], t = p.tlen[r];

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // window: slot lower bound from the smallest per-beam lower depth (depth monotone)
    int lo = 0;
    if (p.window > 0) {
      int lo_dep = INT_MAX;
      for (int j = 0; j < p.b_live; ++j)
        lo_dep = min(lo_dep, p.depth[mbase + p.leaf[r * TRIE_MAX_BEAMS + j]] - p.window + 1);
      int a = 0, b = N;
      while (a < b) {
        const int mid = (a + b) >> 1;
        if (p.depth[mbase + mid] < lo_dep) a = mid + 1; else b = mid;
      }
      lo = a;
    }
    const int first = lo / TC_TR;
    const int total = (N + TC_TR - 1) / TC_TR - first;
    const int per = (total + p.splits - 1) / p.splits;
    const int tb = min(total, split * per), te = min(total, (split + 1) * per);
    s_info[0] = first + tb;
    s_info[1] = te - tb;
    s_info[2] = lo;
  }
  __syncthreads();
  const int tile0 = s_info[0], ntiles = s_info[1];

  if (warp == 0) {
    // ===== producer =====
    if (lane == 0) {
      const int row_base = (r * p.Hkv + h) * p.cap;
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (uint32_t)(i / C::STAGES) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        uint8_t* st = smem + s * C::STAGE_BYTES;
        const int n0 = (tile0 + i) * TC_TR;
        // mask / depth words of the tile, clamped to the [R][cap] arrays (cap % 4 == 0 =>
        // 16-byte aligned, 16-byte multiple)
        const uint32_t mdb = (uint32_t)min(TC_TR, p.cap - n0) * 4u;
        mbar_expect_tx(&full[s], 2 * C::TILE_BYTES + 2 * mdb);
#pragma unroll
        for (int bx = 0; bx < D / TC_CW; ++bx) {
          tma_load_2d(st + bx * TC_TR * 64, &kmap, bx * TC_CW, row_base + n0, &full[s]);
          tma_load_2d(st + C::TILE_BYTES + bx * TC_TR * 64, &vmap, bx * TC_CW, row_base + n0,
                      &full[s]);
        }
        bulk_load_1d(st + 2 * C::TILE_BYTES, p.mask + mbase + n0, mdb, &full[s]);
        bulk_load_1d(st + 2 * C::TILE_BYTES + TC_TR * 4, p.depth + mbase + n0, mdb, &full[s]);
      }
    }
    return;
  }

  // ===== consumers =====
  const int cw = warp - 1;
  const int mt = cw % MT, rs = cw / MT;
  const int gq = lane >> 2, cq = lane & 3;  // fragment row group / column quad
  // this thread's two query rows (g, g+8) -> beam index and window lower depth
  int qm[2], beam[2], lod[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    qm[u] = mt * 16 + gq + 8 * u;
    beam[u] = qm[u] < Qg ? qm[u] / g : 0;
    lod[u] = INT_MIN;
    if (p.window > 0 && qm[u] < Qg)
      lod[u] = p.depth[mbase + p.leaf[r * TRIE_MAX_BEAMS + beam[u]]] - p.window + 1;
  }
  // Q fragments (A operand, row-major 16 x D), zero for padded queries
  uint32_t qa[C::KS][4];
  {
    const __nv_bfloat16* qb = (const __nv_bfloat16*)p.q;
#pragma unroll
    for (int ks = 0; ks < C::KS; ++ks) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int row = (u & 1) ? qm[1] : qm[0];
        const int col = ks * 16 + (u >> 1) * 8 + cq * 2;
        uint32_t v = 0u;
        if (row < Qg) {
          const int j = row / g, i = row % g;
          const __nv_bfloat16* src = qb + (((size_t)r * p.b_live + j) * p.Hq + h * g + i) * D + col;
          v = *(const uint32_t*)src;
        }
        qa[ks][u] = v;
      }
    }
  }
  float o[C::DT][4];
#pragma unroll
  for (int i = 0; i < C::DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const float sc = p.scale_log2;

  for (int i = 0; i < ntiles; ++i) {
    const int s = i % C::STAGES;
    const uint32_t ph = (uint32_t)(i / C::STAGES) & 1u;
    mbar_wait(&full[s], ph);
    const uint8_t* st = smem + s * C::STAGE_BYTES;
    const uint32_t kbase = smem_u32(st), vbase = smem_u32(st + C::TILE_BYTES);
    const uint32_t* tmask = (const uint32_t*)(st + 2 * C::TILE_BYTES);
    const int* tdep = (const int*)(st + 2 * C::TILE_BYTES + TC_TR * 4);
    const int n0 = (tile0 + i) * TC_TR;
    const int r0 = rs * C::RSZ;  // first row of this warp's slice within the tile
    // ---- S = Q K^T over the slice ----
    float sacc[C::NT][4];
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) {
#pragma unroll
      for (int ks = 0; ks < C::KS; ks += 2) {
        // x4: matrices (rows nt*8.., k ks*16+0..7), (.., +8..15), (.., (ks+1)*16+0..7), (+8..15)
        const int row = r0 + nt * 8 + (lane & 7);
        const int col = ks * 16 + (lane >> 3) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kbase + tile_off(row, col), b0, b1, b2, b3);
        mma_bf16(sacc[nt], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
        if (ks + 1 < C::KS) mma_bf16(sacc[nt], qa[ks + 1][0], qa[ks + 1][1], qa[ks + 1][2], qa[ks + 1][3], b2, b3);
      }
    }
    // ---- mask + online softmax (log2 domain) ----
    float tmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int u = e >> 1;
        const int lr = r0 + nt * 8 + cq * 2 + (e & 1);  // row within tile
        const int n = n0 + lr;
        const uint32_t mw = tmask[lr];
        const int dep = tdep[lr];
        const bool ok = n < N && (n < t || ((mw >> beam[u]) & 1u)) && dep >= lod[u] &&
                        qm[u] < Qg;  // (n < N also guards stale words past cap)
        const float v = ok ? sacc[nt][e] * sc : -INFINITY;
        sacc[nt][e] = v;
        tmax[u] = fmaxf(tmax[u], v);
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
    }
    float psum[2] = {0.f, 0.f};
    uint32_t pa[C::NT][2];
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) {
      float pv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int u = e >> 1;
        pv[e] = (sacc[nt][e] == -INFINITY) ? 0.f : exp2f(sacc[nt][e] - mrow[u]);
        psum[u] += pv[e];
      }
      pa[nt][0] = pack_bf16(pv[0], pv[1]);
      pa[nt][1] = pack_bf16(pv[2], pv[3]);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) lrow[u] = lrow[u] * alpha[u] + psum[u];
#pragma unroll
    for (int dt = 0; dt < C::DT; ++dt) {
      o[dt][0] *= alpha[0];
      o[dt][1] *= alpha[0];
      o[dt][2] *= alpha[1];
      o[dt][3] *= alpha[1];
    }
    // ---- O += P V : k = slice rows (16 per mma), n = D ----
#pragma unroll
    for (int kc = 0; kc < C::NT / 2; ++kc) {
      const uint32_t a0 = pa[2 * kc][0], a1 = pa[2 * kc][1], a2 = pa[2 * kc + 1][0],
                     a3 = pa[2 * kc + 1][1];
#pragma unroll
      for (int dt = 0; dt < C::DT; dt += 2) {
        // x4.trans: (rows k0..7, d dt*8..), (rows k8..15, d dt*8..), (k0..7, (dt+1)*8..), (k8..15, ..)
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
  }
  // quad-reduce the row sums (each thread holds partial sums of its columns)
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    lrow[u] += __shfl_xor_sync(0xffffffffu, lrow[u], 1);
    lrow[u] += __shfl_xor_sync(0xffffffffu, lrow[u], 2);
  }

  // ---- merge the RS row-slice warps of each m-tile through shared memory ----
  // all consumers must be done with the ring before it is reused
  asm volatile("bar.sync 1, %0;" ::"r"(C::NC * 32));
  float* red = (float*)smem;  // [NC][16][D + 2]
  const int RW = D + 2;
  float* mine = red + (size_t)cw * 16 * RW;
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
  asm volatile("bar.sync 1, %0;" ::"r"(C::NC * 32));
  // thread -> (query row within m-tile, column range); warps of slice 0 finalize
  if (rs == 0) {
    for (int e = lane; e < 16 * D; e += 32) {
      const int qr = e / D, d = e % D;
      const int m = mt * 16 + qr;
      if (m >= Qg) continue;
      float M = -INFINITY;
#pragma unroll
      for (int x = 0; x < C::RS; ++x) M = fmaxf(M, red[((size_t)(x * MT + mt) * 16 + qr) * RW + D]);
      float Lsum = 0.f, acc = 0.f;
#pragma unroll
      for (int x = 0; x < C::RS; ++x) {
        const float* src = red + ((size_t)(x * MT + mt) * 16 + qr) * RW;
        const float w = src[D] == -INFINITY ? 0.f : exp2f(src[D] - M);
        Lsum += src[D + 1] * w;
        acc += src[d] * w;
      }
      const int j = m / g, ii = m % g;
      if (p.splits == 1) {
        __nv_bfloat16* op = (__nv_bfloat16*)p.out + (((size_t)r * p.b_live + j) * p.Hq + h * g + ii) * D;
        op[d] = __float2bfloat16_rn(Lsum > 0.f ? acc / Lsum : 0.f);
        if (d == 0) {
          if (Lsum == 0.f) latch(p.status, TRIE_ST_EMPTY_ROW);
          if (p.lse)
            p.lse[((size_t)r * p.b_live + j) * p.Hq + h * g + ii] =
                Lsum > 0.f ? (M + log2f(Lsum)) * 0.69314718055994531f : -INFINITY;
        }
      } else {
        float* pp = p.part + ((((size_t)r * p.Hkv + h) * p.splits + split) * Qg + m) * (D + 2);
        pp[d] = acc;
        if (d == 0) {
          pp[D] = M;
          pp[D + 1] = Lsum;
        }
      }
    }
  }
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

static int make_map(CUtensorMap* map, const void* base, int D, long rows) {
  auto enc = get_encode();
  if (!enc) return trie_set_error(TRIE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {(cuuint32_t)TC_CW, (cuuint32_t)TC_TR};
  cuuint32_t estr[2] = {1, 1};
  CUresult rc = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) return trie_set_error(TRIE_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)rc);
  return TRIE_OK;
}

template <int D, int MT>
static int launch_tc_t(const AttnParams& p, cudaStream_t s) {
  using C = TcCfg<D, MT>;
  CUtensorMap km, vm;
  const long rows = (long)p.R * p.Hkv * p.cap;
  int rc = make_map(&km, p.k, D, rows);
  if (!rc) rc = make_map(&vm, p.v, D, rows);
  if (rc) return rc;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_attn_tc<D, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr_set = true;
  }
  dim3 grid(p.Hkv, p.R, p.splits);
  k_attn_tc<D, MT><<<grid, C::THREADS, C::SMEM, s>>>(km, vm, p);
  rc = trie_check_launch("k_attn_tc");
  if (rc) return rc;
  if (p.splits > 1) rc = launch_attn_combine_bf16(p, s);
  return rc;
}

template <int D>
static int launch_tc_d(const AttnParams& p, cudaStream_t s, int MT) {
  switch (MT) {
    case 1: return launch_tc_t<D, 1>(p, s);
    case 2: return launch_tc_t<D, 2>(p, s);
    case 4: return launch_tc_t<D, 4>(p, s);
    case 8: return launch_tc_t<D, 8>(p, s);
  }
  return 1;
}

bool attn_tc_supported(const AttnParams& p) {
  const int Qg = p.b_live * (p.Hq / p.Hkv);
  if (!p.bf16 || Qg > 128 || p.cap % 4) return false;
  if (p.D != 64 && p.D != 96 && p.D != 128) return false;
  // 16-byte aligned pools for TMA
  if (((uintptr_t)p.k | (uintptr_t)p.v) & 15) return false;
  return true;
}

int launch_attn_tc(const AttnParams& p, cudaStream_t s) {
  const int Qg = p.b_live * (p.Hq / p.Hkv);
  const int MT = Qg <= 16 ? 1 : Qg <= 32 ? 2 : Qg <= 64 ? 4 : 8;
  switch (p.D) {
    case 64: return launch_tc_d<64>(p, s, MT);
    case 96: return launch_tc_d<96>(p, s, MT);
    case 128: return launch_tc_d<128>(p, s, MT);
  }
  return 1;
}

}  // namespace trie
