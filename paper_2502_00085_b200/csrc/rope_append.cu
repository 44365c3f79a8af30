// trie_rope_kv_append (a-1): position-integrity RoPE at depth + write-before-read K/V append.
// §3.4: "renumbered position IDs ... assigned to match the positions in the
// original beam search" -> pos = depth[leaf].  Alg. 3 l.7 "allow attention to
// current node" + S:150-151: K/V of the new token are in the pool before it attends.
// RoPE reading R16: rotate-half pairs (i, i + D/2), theta_i = base^(-2i/D); the angle
// pos * theta_i is formed and reduced in fp64 (fp32 angles lose ~5e-4 at pos 8k, base
// 1e8), once per (request, beam) and frequency, shared by all Hq + Hkv heads.
// Memory layout work: one CTA per (request, beam); every thread moves 16-byte vectors
// (8 bf16 / 4 fp32 of one half-head and the matching 8 of the other half), all loads of a
// batch issued before any store (the pointers are __restrict__: q, k_new, v_new and the
// pools never alias).
#include "common.cuh"
#include "handle.h"

namespace trie {

template <typename T>
struct Vec16 {
  static constexpr int N = 16 / sizeof(T);
};

template <typename T>
__device__ __forceinline__ void unpack(const int4& v, float* f) {
  if constexpr (sizeof(T) == 2) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 x = __bfloat1622float2(h[i]);
      f[2 * i] = x.x;
      f[2 * i + 1] = x.y;
    }
  } else {
    const float* x = reinterpret_cast<const float*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = x[i];
  }
}
template <typename T>
__device__ __forceinline__ int4 pack(const float* f) {
  int4 v;
  if constexpr (sizeof(T) == 2) {
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  } else {
    float* x = reinterpret_cast<float*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = f[i];
  }
  return v;
}

constexpr int ROPE_BS = 128;
constexpr int ROPE_BATCH = 4;

template <typename T>
__global__ void __launch_bounds__(ROPE_BS) k_rope_append(
    T* __restrict__ q, T* __restrict__ k_new, const T* __restrict__ v_new, T* __restrict__ kpool,
    T* __restrict__ vpool, const int32_t* __restrict__ leaf, const float2* __restrict__ tab,
    int b_live, int Hq, int Hkv, int D, int cap, const int32_t* __restrict__ pt) {
  constexpr int VN = Vec16<T>::N;
  __shared__ float s_cos[128], s_sin[128];  // D <= 256
  pdl_trigger();
  pdl_wait();
  const int rj = blockIdx.x;                // r * b_live + j
  const int r = rj / b_live;
  const int slot = leaf[r * TRIE_MAX_BEAMS + rj % b_live];
  const int half = D / 2;
  // pool row of (r, KV head hh, slot): dense [R][Hkv][cap][D] or paged (NEXT-2)
  auto prow = [&](int hh) -> size_t {
    return pt ? ((size_t)pt[r * (cap / 64) + (slot >> 6)] * Hkv + hh) * 64 + (slot & 63)
              : ((size_t)r * Hkv + hh) * cap + slot;
  };
  for (int i = threadIdx.x; i < half; i += ROPE_BS) {  // the step's table (k_rope_table)
    const float2 c = tab[(size_t)rj * half + i];
    s_cos[i] = c.x;
    s_sin[i] = c.y;
  }
  __syncthreads();
  const int cph = half / VN;                 // vector chunks per half-head
  const int n_rot = (Hq + Hkv) * cph;        // rotation items
  const int n_v = Hkv * (D / VN);            // V copy items
  const int total = n_rot + n_v;
  for (int base = 0; base < total; base += ROPE_BS * ROPE_BATCH) {
    int4 lo[ROPE_BATCH], hi[ROPE_BATCH];
#pragma unroll
    for (int u = 0; u < ROPE_BATCH; ++u) {  // loads
      const int it = base + u * ROPE_BS + threadIdx.x;
      if (it < n_rot) {
        const int hh = it / cph, c = it % cph;
        const T* e = hh < Hq ? q + ((size_t)rj * Hq + hh) * D : k_new + ((size_t)rj * Hkv + hh - Hq) * D;
        lo[u] = *reinterpret_cast<const int4*>(e + c * VN);
        hi[u] = *reinterpret_cast<const int4*>(e + half + c * VN);
      } else if (it < total) {
        const int e = (it - n_rot) * VN;
        lo[u] = *reinterpret_cast<const int4*>(v_new + (size_t)rj * Hkv * D + e);
      }
    }
#pragma unroll
    for (int u = 0; u < ROPE_BATCH; ++u) {  // rotate + stores
      const int it = base + u * ROPE_BS + threadIdx.x;
      if (it < n_rot) {
        const int hh = it / cph, c = it % cph;
        float x1[VN], x2[VN], y1[VN], y2[VN];
        unpack<T>(lo[u], x1);
        unpack<T>(hi[u], x2);
#pragma unroll
        for (int v = 0; v < VN; ++v) {
          const float cs = s_cos[c * VN + v], sn = s_sin[c * VN + v];
          y1[v] = x1[v] * cs - x2[v] * sn;
          y2[v] = x2[v] * cs + x1[v] * sn;
        }
        const int4 o1 = pack<T>(y1), o2 = pack<T>(y2);
        T* e = hh < Hq ? q + ((size_t)rj * Hq + hh) * D : k_new + ((size_t)rj * Hkv + hh - Hq) * D;
        *reinterpret_cast<int4*>(e + c * VN) = o1;
        *reinterpret_cast<int4*>(e + half + c * VN) = o2;
        if (hh >= Hq) {
          T* dst = kpool + prow(hh - Hq) * D;
          *reinterpret_cast<int4*>(dst + c * VN) = o1;
          *reinterpret_cast<int4*>(dst + half + c * VN) = o2;
        }
      } else if (it < total) {
        const int e = (it - n_rot) * VN;
        const int hh = e / D, d = e % D;
        *reinterpret_cast<int4*>(vpool + prow(hh) * D + d) = lo[u];
      }
    }
  }
}

// (cos, sin) of every live leaf's depth and frequency, once per step for all layers of
// the fused trie_attn_decode_rope; same fp64 angle formula as k_rope_append (bit-equal).
__global__ void k_rope_table(float2* __restrict__ tab, const int32_t* __restrict__ depth,
                             const int32_t* __restrict__ leaf, int b_live, int D, int cap,
                             double log2_theta) {
  pdl_trigger();
  pdl_wait();
  const int rj = blockIdx.x, r = rj / b_live, j = rj % b_live;
  const int pos = depth[(size_t)r * cap + leaf[r * TRIE_MAX_BEAMS + j]];
  for (int i = threadIdx.x; i < D / 2; i += blockDim.x) {
    const double inv_freq = exp2(-2.0 * (double)i / (double)D * log2_theta);
    double sn, cs;
    sincos((double)pos * inv_freq, &sn, &cs);
    tab[(size_t)rj * (D / 2) + i] = make_float2((float)cs, (float)sn);
  }
}

int launch_rope_table(trie_handle* h, float theta, cudaStream_t s) {
  const trie_cfg& c = h->cfg;
  launch_k(k_rope_table, dim3(c.n_requests * h->b_live), dim3(64), 0, s, h->rope_tab,
           (const int32_t*)h->depth, (const int32_t*)h->leaf, h->b_live, c.head_dim, c.capacity,
           log2((double)theta));
  return trie_check_launch("k_rope_table");
}

int launch_rope_append(trie_handle* h, void* q, void* k_new, const void* v_new, void* kpool,
                       void* vpool, float theta, cudaStream_t s) {
  const trie_cfg& c = h->cfg;
  const int grid = c.n_requests * h->b_live;
  if (h->rope_tab_steps != h->steps || h->rope_tab_theta != theta || h->rope_tab_blive != h->b_live) {
    const int rc = launch_rope_table(h, theta, s);  // once per step, shared by all layers
    if (rc) return rc;
    h->rope_tab_steps = h->steps;
    h->rope_tab_theta = theta;
    h->rope_tab_blive = h->b_live;
  }
  if ((((uintptr_t)q | (uintptr_t)k_new | (uintptr_t)v_new | (uintptr_t)kpool | (uintptr_t)vpool) & 15))
    return trie_set_error(TRIE_EINVAL, "rope_kv_append: buffers must be 16-byte aligned");
  if (c.kv_dtype == TRIE_BF16) {
    if ((c.head_dim / 2) % 8)
      return trie_set_error(TRIE_EINVAL, "rope_kv_append: bf16 needs head_dim % 16 == 0");
    launch_k(k_rope_append<__nv_bfloat16>, grid, dim3(ROPE_BS), 0, s,
             (__nv_bfloat16*)q, (__nv_bfloat16*)k_new, (const __nv_bfloat16*)v_new,
             (__nv_bfloat16*)kpool, (__nv_bfloat16*)vpool, (const int32_t*)h->leaf,
             (const float2*)h->rope_tab, h->b_live, c.n_q_heads, c.n_kv_heads, c.head_dim,
             c.capacity, (const int32_t*)h->page_table);
  } else {
    launch_k(k_rope_append<float>, grid, dim3(ROPE_BS), 0, s, (float*)q, (float*)k_new,
             (const float*)v_new, (float*)kpool, (float*)vpool, (const int32_t*)h->leaf,
             (const float2*)h->rope_tab, h->b_live, c.n_q_heads, c.n_kv_heads, c.head_dim,
             c.capacity, (const int32_t*)h->page_table);
  }
  return trie_check_launch("k_rope_append");
}

}  // namespace trie
