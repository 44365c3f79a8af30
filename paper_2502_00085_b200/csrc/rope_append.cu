// trie_rope_kv_append (a-1): position-integrity RoPE at depth + write-before-read K/V append.
// §3.4: "renumbered position IDs ... assigned to match the positions in the
// original beam search" -> pos = depth[leaf].  Alg. 3 l.7 "allow attention to
// current node" + S:150-151: K/V of the new token are in the pool before it attends.
// RoPE reading R16: rotate-half pairs (i, i + D/2), theta_i = base^(-2i/D); the angle
// pos * theta_i is formed and reduced in fp64 so that positions up to 8k with base up to
// 1e8 keep ~1e-7 relative accuracy (fp32 angles would lose ~5e-4).
#include "common.cuh"
#include "handle.h"

namespace trie {

template <typename T>
__global__ void k_rope_append(T* q, T* k_new, const T* v_new, T* kpool, T* vpool,
                              const int32_t* depth, const int32_t* leaf, int b_live, int Hq,
                              int Hkv, int D, int cap, double log2_theta) {
  __shared__ float s_cos[128], s_sin[128];  // D <= 256
  const int rj = blockIdx.x;  // r * b_live + j
  const int r = rj / b_live, j = rj % b_live;
  const int slot = leaf[r * TRIE_MAX_BEAMS + j];
  const int pos = depth[(size_t)r * cap + slot];
  const int half = D / 2;
  // one fp64 angle per frequency, shared by every head of this (request, beam)
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const double inv_freq = exp2(-2.0 * (double)i / (double)D * log2_theta);
    double sn, cs;
    sincos((double)pos * inv_freq, &sn, &cs);
    s_cos[i] = (float)cs;
    s_sin[i] = (float)sn;
  }
  __syncthreads();
  const int pairs = (Hq + Hkv) * half;
  for (int p = threadIdx.x; p < pairs; p += blockDim.x) {
    const int hh = p / half, i = p % half;
    const float c = s_cos[i], s = s_sin[i];
    T* e;
    if (hh < Hq) {
      e = q + ((size_t)rj * Hq + hh) * D;
    } else {
      e = k_new + ((size_t)rj * Hkv + (hh - Hq)) * D;
    }
    const float x1 = to_f(e[i]), x2 = to_f(e[i + half]);
    const T y1 = from_f<T>(x1 * c - x2 * s);
    const T y2 = from_f<T>(x2 * c + x1 * s);
    e[i] = y1;
    e[i + half] = y2;
    if (hh >= Hq) {
      T* dst = kpool + (((size_t)r * Hkv + (hh - Hq)) * cap + slot) * D;
      dst[i] = y1;
      dst[i + half] = y2;
    }
  }
  for (int e = threadIdx.x; e < Hkv * D; e += blockDim.x) {
    const int hh = e / D, d = e % D;
    vpool[(((size_t)r * Hkv + hh) * cap + slot) * D + d] = v_new[((size_t)rj * Hkv + hh) * D + d];
  }
}

int launch_rope_append(trie_handle* h, void* q, void* k_new, const void* v_new, void* kpool,
                       void* vpool, float theta, cudaStream_t s) {
  const trie_cfg& c = h->cfg;
  const int grid = c.n_requests * h->b_live;
  const double l2 = log2((double)theta);
  if (c.kv_dtype == TRIE_BF16) {
    k_rope_append<__nv_bfloat16><<<grid, 128, 0, s>>>(
        (__nv_bfloat16*)q, (__nv_bfloat16*)k_new, (const __nv_bfloat16*)v_new,
        (__nv_bfloat16*)kpool, (__nv_bfloat16*)vpool, h->depth, h->leaf, h->b_live, c.n_q_heads,
        c.n_kv_heads, c.head_dim, c.capacity, l2);
  } else {
    k_rope_append<float><<<grid, 128, 0, s>>>((float*)q, (float*)k_new, (const float*)v_new,
                                              (float*)kpool, (float*)vpool, h->depth, h->leaf,
                                              h->b_live, c.n_q_heads, c.n_kv_heads, c.head_dim,
                                              c.capacity, l2);
  }
  return trie_check_launch("k_rope_append");
}

}  // namespace trie
