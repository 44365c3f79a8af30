// trie_attn_decode (a-3): tree attention over the shared trie KV pool (§3.3, P:188-196;
// Alg. 3 mask), generic CUDA-core path (fp32 and bf16 pools, any D % 16 == 0,
// any b_live * g <= 256).  The bf16 tensor-core path for the shaped configs lives in
// attn_decode_tc.cu; this one is the fp32 parity path and the fallback for shapes the
// tensor-core kernel does not instantiate (never a CPU fallback).
//
// Work decomposition: one CTA per (KV head h, request r, split s).  The CTA streams the
// slots [row_lo, N) of its split ONCE from HBM (K and V rows of head h) and every one of
// the Qg = b_live * g queries that share the head consumes each tile from shared memory
// (GQA grouping + beam sharing: the unique-KV read the paper's trie enables).
// Mask: slot n is visible to beam j iff n < t or bit j of beam_mask[n]; window (reading
// R14): depth[n] >= depth[leaf_j] - W + 1, which -- depth being non-decreasing in slot
// order -- also gives a slot lower bound found by binary search.
// Online softmax in the log2 domain; split partials (m, l, acc) merged by k_attn_combine.
#include <float.h>

#include "attn_common.cuh"
#include "common.cuh"
#include "handle.h"
#include "gather.cuh"

namespace trie {

constexpr int V1_TILE = 32;

template <typename T, int DC>
__global__ void __launch_bounds__(512) k_attn_v1(const AttnParams p) {
  extern __shared__ float sm[];
  const int h = blockIdx.x, r = blockIdx.y, split = blockIdx.z;
  const int D = p.D, g = p.Hq / p.Hkv, Qg = p.b_live * g;
  const int NW = blockDim.x / 32, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Dp = D + 1;
  float* sQ = sm;                           // [Qg][D] (pre-scaled by log2e / sqrt(D))
  float* sK = sQ + Qg * D;                  // [TILE][D+1]
  float* sV = sK + V1_TILE * Dp;            // [TILE][D]
  int* sLo = (int*)(sV + V1_TILE * D);      // [b_live] window lower depth per beam
  uint32_t* sMask = (uint32_t*)(sLo + TRIE_MAX_BEAMS);  // [TILE]
  int* sDep = (int*)(sMask + V1_TILE);      // [TILE]
  __shared__ int s_range[2];

  const size_t mbase = (size_t)r * p.cap;
  const int N = p.nn[r], t = p.tlen[r];
  // queries: m = j * g + i  <->  beam j, q head h*g + i
  for (int e = threadIdx.x; e < Qg * D; e += blockDim.x) {
    const int m = e / D, d = e % D;
    const int j = m / g, i = m % g;
    const T* qp = (const T*)p.q + (((size_t)r * p.b_live + j) * p.Hq + h * g + i) * D;
    sQ[e] = to_f(qp[d]) * p.scale_log2;
  }
  if (threadIdx.x < p.b_live) {
    const int lf = p.leaf[r * TRIE_MAX_BEAMS + threadIdx.x];
    sLo[threadIdx.x] = p.window > 0 ? p.depth[mbase + lf] - p.window + 1 : INT_MIN;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int lo_dep = INT_MAX;
    for (int j = 0; j < p.b_live; ++j) lo_dep = min(lo_dep, sLo[j]);
    int lo = 0;
    if (p.window > 0) {  // first slot with depth >= lo_dep (depth non-decreasing)
      int a = 0, b = N;
      while (a < b) {
        const int mid = (a + b) >> 1;
        if (p.depth[mbase + mid] < lo_dep) a = mid + 1; else b = mid;
      }
      lo = a;
    }
    const int rows = N - lo;
    int chunk = (rows + p.splits - 1) / p.splits;
    chunk = (chunk + V1_TILE - 1) / V1_TILE * V1_TILE;
    s_range[0] = min(N, lo + split * chunk);
    s_range[1] = min(N, lo + (split + 1) * chunk);
  }
  __syncthreads();
  const int row_b = s_range[0], row_e = s_range[1];

  constexpr int QPW = 8;
  float m_i[QPW], l_i[QPW], acc[QPW][DC];
#pragma unroll
  for (int i = 0; i < QPW; ++i) {
    m_i[i] = -INFINITY;
    l_i[i] = 0.f;
#pragma unroll
    for (int c = 0; c < DC; ++c) acc[i][c] = 0.f;
  }
  const T* kb = (const T*)p.k;
  const T* vb = (const T*)p.v;

  for (int n0 = row_b; n0 < row_e; n0 += V1_TILE) {
    const int nt = min(V1_TILE, row_e - n0);
    for (int e = threadIdx.x; e < nt * D; e += blockDim.x) {
      const int n = e / D, d = e % D;
      const size_t row = (size_t)attn_row(p, r, h, n0 + n);  // dense or paged (NEXT-2)
      sK[n * Dp + d] = to_f(kb[row * D + d]);
      sV[n * D + d] = to_f(vb[row * D + d]);
    }
    if (threadIdx.x < nt) {
      sMask[threadIdx.x] = p.mask[mbase + n0 + threadIdx.x];
      sDep[threadIdx.x] = p.depth[mbase + n0 + threadIdx.x];
    }
    __syncthreads();
    const int n = lane;
    const bool in = n < nt;
    const bool prompt = (n0 + n) < t;
    const uint32_t mw = in ? sMask[n] : 0u;
    const int dep = in ? sDep[n] : 0;
#pragma unroll
    for (int i = 0; i < QPW; ++i) {
      const int m = w + i * NW;
      if (m >= Qg) break;  // warp-uniform
      const int j = m / g;
      const bool ok = in && (prompt || ((mw >> j) & 1u)) && dep >= sLo[j];
      float s = -INFINITY;
      if (ok) {
        float a = 0.f;
        const float* qr = sQ + m * D;
        const float* kr = sK + n * Dp;
        for (int d = 0; d < D; ++d) a = fmaf(qr[d], kr[d], a);
        s = a;
      }
      const float tmax = warp_max(s);
      const float m_new = fmaxf(m_i[i], tmax);
      if (m_new == -INFINITY) continue;  // nothing visible yet (warp-uniform)
      const float alpha = exp2f(m_i[i] - m_new);
      const float pr = ok ? exp2f(s - m_new) : 0.f;
      l_i[i] = l_i[i] * alpha + warp_sum(pr);
      m_i[i] = m_new;
#pragma unroll
      for (int c = 0; c < DC; ++c) acc[i][c] *= alpha;
      for (int nn = 0; nn < nt; ++nn) {
        const float pn = __shfl_sync(0xffffffffu, pr, nn);
        if (pn == 0.f) continue;  // uniform
#pragma unroll
        for (int c = 0; c < DC; ++c) {
          const int d = lane + 32 * c;
          if (d < D) acc[i][c] = fmaf(pn, sV[nn * D + d], acc[i][c]);
        }
      }
    }
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < QPW; ++i) {
    const int m = w + i * NW;
    if (m >= Qg) break;
    const int j = m / g, ii = m % g;
    if (p.splits == 1) {
      const float inv = l_i[i] > 0.f ? 1.f / l_i[i] : 0.f;
      if (l_i[i] == 0.f && lane == 0) latch(p.status, TRIE_ST_EMPTY_ROW);
      T* op = (T*)p.out + (((size_t)r * p.b_live + j) * p.Hq + h * g + ii) * D;
#pragma unroll
      for (int c = 0; c < DC; ++c) {
        const int d = lane + 32 * c;
        if (d < D) op[d] = from_f<T>(acc[i][c] * inv);
      }
      if (p.lse && lane == 0)
        p.lse[((size_t)r * p.b_live + j) * p.Hq + h * g + ii] =
            l_i[i] > 0.f ? (m_i[i] + log2f(l_i[i])) * 0.69314718055994531f : -INFINITY;
    } else {
      float* pp = p.part + ((((size_t)r * p.Hkv + h) * p.splits + split) * Qg + m) * (D + 2);
#pragma unroll
      for (int c = 0; c < DC; ++c) {
        const int d = lane + 32 * c;
        if (d < D) pp[d] = acc[i][c];
      }
      if (lane == 0) {
        pp[D] = m_i[i];
        pp[D + 1] = l_i[i];
      }
    }
  }
}

// merge split partials: one warp per (r, h, query); lane c owns columns lane + 32 c
// (c < DC = ceil(D / 32)).  The splits' (m, l) pairs are loaded lane-parallel (<= 64
// splits), then the partial rows in batches of SB splits whose loads are all issued
// before any is consumed (SB * DC <= 64 registers), so a launch costs ~ceil(splits / SB)
// L2 round trips.
template <typename T, int DC>
__global__ void __launch_bounds__(128) k_attn_combine(const AttnParams p) {
  pdl_trigger();
  pdl_wait();
  constexpr int SB = DC <= 2 ? 32 : DC <= 4 ? 16 : 8;
  const int g = p.Hq / p.Hkv, Qg = p.b_live * g;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int total = p.R * p.Hkv * Qg;
  if (gw >= total) return;
  const int m = gw % Qg, h = (gw / Qg) % p.Hkv, r = gw / (Qg * p.Hkv);
  const int D = p.D;
  // NEXT-4 fused all-gather (bf16): one arrival per combined row
  constexpr bool kBf16 = sizeof(T) == 2;
  const bool gat = kBf16 && p.ga.world > 0;
  if (p.fin != nullptr &&  // NEXT-3: a finished request's splits wrote nothing; neither do we
      __all_sync(0xffffffffu, lane >= p.b_live || p.fin[r * TRIE_MAX_BEAMS + lane] != 0u)) {
    if (gat && lane == 0) gather_arrive(p);
    return;
  }
  const float* base = p.part + (((size_t)r * p.Hkv + h) * p.splits * Qg) * (D + 2);
  // lanes own splits (<= 64): (m_s, l_s) loaded in parallel, weights w_s = 2^(m_s - M)
  float ms[2], ls[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int s = lane + 32 * u;
    const float* pp = base + ((size_t)s * Qg + m) * (D + 2);
    ms[u] = s < p.splits ? pp[D] : -INFINITY;
    ls[u] = s < p.splits ? pp[D + 1] : 0.f;
  }
  const float M = warp_max(fmaxf(ms[0], ms[1]));
  float ws[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) ws[u] = ls[u] > 0.f ? exp2f(ms[u] - M) : 0.f;
  const float L = warp_sum(ls[0] * ws[0] + ls[1] * ws[1]);
  const int j = m / g, ii = m % g;
  T* op = (T*)p.out + (((size_t)r * p.b_live + j) * p.Hq + h * g + ii) * D;
  const float inv = L > 0.f ? 1.f / L : 0.f;
  if (L == 0.f && lane == 0) latch(p.status, TRIE_ST_EMPTY_ROW);
  float acc[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) acc[c] = 0.f;
  for (int s0 = 0; s0 < p.splits; s0 += SB) {
    float v[SB][DC];
#pragma unroll
    for (int u = 0; u < SB; ++u) {
      const int s = min(s0 + u, p.splits - 1);
      const float* pp = base + ((size_t)s * Qg + m) * (D + 2);
#pragma unroll
      for (int c = 0; c < DC; ++c) v[u][c] = (lane + 32 * c < D) ? __ldcg(pp + lane + 32 * c) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < SB; ++u) {
      const int s = s0 + u;
      const float w = __shfl_sync(0xffffffffu, ws[(s >> 5) & 1], s & 31);
      if (s < p.splits) {
#pragma unroll
        for (int c = 0; c < DC; ++c) acc[c] += w * v[u][c];
      }
    }
  }
  const uint32_t ghalf = gat ? gather_half(p) : 0u;
#pragma unroll
  for (int c = 0; c < DC; ++c)
    if (lane + 32 * c < D) {
      const T v = from_f<T>(acc[c] * inv);
      op[lane + 32 * c] = v;
      if constexpr (kBf16)
        if (gat) gather_st16(p, ghalf, r, j, h * g + ii, lane + 32 * c, v);
    }
  if (p.lse && lane == 0)
    p.lse[((size_t)r * p.b_live + j) * p.Hq + h * g + ii] =
        L > 0.f ? (M + log2f(L)) * 0.69314718055994531f : -INFINITY;
  if (gat) {
    __syncwarp();
    if (lane == 0) gather_arrive(p);
  }
}

template <typename T>
static int launch_combine_t(const AttnParams& p, cudaStream_t s) {
  const int Qg = p.b_live * (p.Hq / p.Hkv);
  const int warps = p.R * p.Hkv * Qg;
  const dim3 grid((warps * 32 + 127) / 128);
  switch ((p.D + 31) / 32) {
    case 1: launch_k(k_attn_combine<T, 1>, grid, dim3(128), 0, s, p); break;
    case 2: launch_k(k_attn_combine<T, 2>, grid, dim3(128), 0, s, p); break;
    case 3: launch_k(k_attn_combine<T, 3>, grid, dim3(128), 0, s, p); break;
    case 4: launch_k(k_attn_combine<T, 4>, grid, dim3(128), 0, s, p); break;
    case 5: launch_k(k_attn_combine<T, 5>, grid, dim3(128), 0, s, p); break;
    case 6: launch_k(k_attn_combine<T, 6>, grid, dim3(128), 0, s, p); break;
    case 7: launch_k(k_attn_combine<T, 7>, grid, dim3(128), 0, s, p); break;
    default: launch_k(k_attn_combine<T, 8>, grid, dim3(128), 0, s, p); break;
  }
  return trie_check_launch("k_attn_combine");
}

template <typename T>
static int launch_v1_t(const AttnParams& p, cudaStream_t s) {
  const int g = p.Hq / p.Hkv, Qg = p.b_live * g;
  int nw = (Qg + 7) / 8;
  nw = nw < 4 ? 4 : nw;
  if (nw > 16) return trie_set_error(TRIE_EINVAL, "b_live*Hq/Hkv = %d > 128 not supported", Qg);
  const size_t smem = (size_t)(Qg * p.D + V1_TILE * (p.D + 1) + V1_TILE * p.D) * 4 +
                      TRIE_MAX_BEAMS * 4 + V1_TILE * 8;
  dim3 grid(p.Hkv, p.R, p.splits);
  const int DC = (p.D + 31) / 32;
#define V1_CASE(dc)                                                                        \
  case dc: {                                                                               \
    auto kern = k_attn_v1<T, dc>;                                                          \
    if (smem > 48 * 1024)                                                                  \
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    kern<<<grid, nw * 32, smem, s>>>(p);                                                   \
    break;                                                                                 \
  }
  switch (DC) {
    V1_CASE(1)
    V1_CASE(2)
    V1_CASE(3)
    V1_CASE(4)
    V1_CASE(5)
    V1_CASE(6)
    V1_CASE(7)
    V1_CASE(8)
    default:
      return trie_set_error(TRIE_EINVAL, "head_dim %d > 256", p.D);
  }
#undef V1_CASE
  int rc = trie_check_launch("k_attn_v1");
  if (rc) return rc;
  if (p.splits > 1) rc = launch_combine_t<T>(p, s);
  return rc;
}

int launch_attn_combine_bf16(const AttnParams& p, cudaStream_t s) {
  return launch_combine_t<__nv_bfloat16>(p, s);
}

int launch_attn_v1(const AttnParams& p, cudaStream_t s) {
  return p.bf16 ? launch_v1_t<__nv_bfloat16>(p, s) : launch_v1_t<float>(p, s);
}

}  // namespace trie
