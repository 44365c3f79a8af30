// Measurement baseline for SURVEY §8(f) NEXT-2 (not on the trie path): the cache reorder of
// conventional batch beam search.  Alg. 1 keeps one sequence -- and in an
// implementation one private KV cache -- per beam; after the top-b selection the new beam r
// continues its parent beam j_r's sequence (Alg. 1 l.6-7), so its cache becomes a copy of
// the parent's (HF's _reorder_cache = index_select over the beam axis, the system the paper
// compares against, P:7).  The trie path needs no such copy: beams share rows.
//
// One CTA per (KV head, beam of a request, layer); K and V rows [t, n) of the source beam
// are contiguous in the head-major pool [R*b][Hkv][cap][D], so the copy is a flat 16-byte
// vector stream.  The prompt rows [0, t) are identical in every beam's cache and are not
// copied (this favours the baseline).
#include "common.cuh"
#include "handle.h"

namespace trie {

struct BatchPools {
  void* sk[TRIE_MAX_LAYERS];
  void* sv[TRIE_MAX_LAYERS];
  void* dk[TRIE_MAX_LAYERS];
  void* dv[TRIE_MAX_LAYERS];
};

constexpr int REORDER_BS = 256;
constexpr int REORDER_VEC = 4;  // 16-byte vectors in flight per thread

__global__ void __launch_bounds__(REORDER_BS) k_batch_reorder(const __grid_constant__ BatchPools pp,
                                                              const int32_t* sel_parent_beam,
                                                              const int32_t* prompt_len,
                                                              const int32_t* n_rows, int b,
                                                              int Hkv, int cap, int row_bytes,
                                                              uint32_t* status) {
  pdl_trigger();
  pdl_wait();
  const int h = blockIdx.x, dst_beam = blockIdx.y, layer = blockIdx.z;
  const int req = dst_beam / b;
  const int j = sel_parent_beam[dst_beam];
  if (j < 0 || j >= b) {
    if (threadIdx.x == 0) latch(status, TRIE_ST_PARENT);
    return;
  }
  const int src_beam = req * b + j;
  const int t = prompt_len[dst_beam], n = min(n_rows[src_beam], cap);
  if (n <= t) return;
  const size_t off = (((size_t)src_beam * Hkv + h) * cap + t) * row_bytes;
  const size_t doff = (((size_t)dst_beam * Hkv + h) * cap + t) * row_bytes;
  const long nvec = (long)(n - t) * row_bytes / 16;
  for (int kv = 0; kv < 2; ++kv) {
    const int4* src = (const int4*)((const char*)(kv ? pp.sv[layer] : pp.sk[layer]) + off);
    int4* dst = (int4*)((char*)(kv ? pp.dv[layer] : pp.dk[layer]) + doff);
    for (long e0 = 0; e0 < nvec; e0 += REORDER_BS * REORDER_VEC) {
      int4 v[REORDER_VEC];
#pragma unroll
      for (int u = 0; u < REORDER_VEC; ++u) {
        const long e = e0 + u * REORDER_BS + threadIdx.x;
        if (e < nvec) v[u] = __ldcs(src + e);
      }
#pragma unroll
      for (int u = 0; u < REORDER_VEC; ++u) {
        const long e = e0 + u * REORDER_BS + threadIdx.x;
        if (e < nvec) dst[e] = v[u];
      }
    }
  }
}

}  // namespace trie

extern "C" int trie_batch_reorder_kv(int32_t n_requests, int32_t beam_width, int32_t n_layers,
                                     int32_t n_kv_heads, int32_t head_dim, int32_t capacity,
                                     int32_t elem_bytes, const int32_t* sel_parent_beam,
                                     const int32_t* prompt_len, const int32_t* n_rows,
                                     void* const* src_k_host, void* const* src_v_host,
                                     void* const* dst_k_host, void* const* dst_v_host,
                                     uint32_t* status, cudaStream_t stream) {
  if (n_requests < 1 || beam_width < 1 || beam_width > TRIE_MAX_BEAMS || n_layers < 1 ||
      n_layers > TRIE_MAX_LAYERS || n_kv_heads < 1 || head_dim < 8 || capacity < 1 ||
      (elem_bytes != 2 && elem_bytes != 4) || (head_dim * elem_bytes) % 16)
    return trie_set_error(TRIE_EINVAL, "trie_batch_reorder_kv: bad shape");
  if (!sel_parent_beam || !prompt_len || !n_rows || !src_k_host || !src_v_host || !dst_k_host ||
      !dst_v_host)
    return trie_set_error(TRIE_EINVAL, "trie_batch_reorder_kv: null argument");
  trie::BatchPools pp;
  for (int l = 0; l < n_layers; ++l) {
    pp.sk[l] = src_k_host[l];
    pp.sv[l] = src_v_host[l];
    pp.dk[l] = dst_k_host[l];
    pp.dv[l] = dst_v_host[l];
    if (!pp.sk[l] || !pp.sv[l] || !pp.dk[l] || !pp.dv[l] || pp.sk[l] == pp.dk[l] || pp.sv[l] == pp.dv[l])
      return trie_set_error(TRIE_EINVAL, "trie_batch_reorder_kv: null or in-place pool");
  }
  dim3 grid(n_kv_heads, n_requests * beam_width, n_layers);
  trie::launch_k(trie::k_batch_reorder, grid, dim3(trie::REORDER_BS), 0, stream, pp, sel_parent_beam,
                 prompt_len, n_rows, beam_width, n_kv_heads, capacity, head_dim * elem_bytes, status);
  return trie_check_launch("k_batch_reorder");
}
