// the KV-head shard's per-layer all-gather fused into the attention
// epilogue (include/triedecode.h trie_gather_setup).  This file: the consumer-side wait
// (+ copy of the completed half into the caller's buffer), the handle registration and the
// CUDA IPC helpers that map every rank's gather buffer / flag array into this process.
// The producer side (peer stores + launch-completion flags) lives in the epilogues of the
// attention kernels and the split-K combine (gather.cuh).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <string.h>

#include "attn_common.cuh"
#include "common.cuh"
#include "gather.cuh"
#include "handle.h"

namespace trie {

// Every CTA: thread 0 waits until each rank's flag in the LOCAL array reaches this rank's
// own sequence number e (acquire, system scope), then the CTA copies its share of half
// (e - 1) mod 2 of the local gather buffer into dst (int4 grid-stride).
__global__ void k_gather_wait(GatherArgs ga, size_t n16, __nv_bfloat16* dst) {
  __shared__ uint32_t s_half;
  if (threadIdx.x == 0) {
    const uint32_t e = *(volatile const uint32_t*)ga.epoch;
    const uint32_t* fl = ga.flag[ga.rank];
    for (int q = 0; q < ga.world; ++q)
      while (ld_acquire_sys(fl + q) < e) __nanosleep(100);
    s_half = (e - 1u) & 1u;
  }
  __syncthreads();
  if (dst == nullptr) return;
  const int4* src = (const int4*)((const __nv_bfloat16*)ga.out[ga.rank] + (size_t)s_half * ga.half_stride);
  int4* d = (int4*)dst;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    d[i] = src[i];
}

int launch_gather_wait(const GatherArgs& ga, int R, int b_live, int Hq, int D, void* dst, cudaStream_t s) {
  const size_t n = (size_t)R * b_live * ga.world * Hq * D;  // bf16 elements of one call
  const size_t n16 = n * 2 / 16;
  int grid = (int)((n16 + 255) / 256);
  grid = grid < 1 ? 1 : (grid > 296 ? 296 : grid);
  k_gather_wait<<<grid, 256, 0, s>>>(ga, dst ? n16 : 0, (__nv_bfloat16*)dst);
  return trie_check_launch("k_gather_wait");
}

}  // namespace trie

extern "C" {

int trie_gather_setup(trie_handle* h, int32_t world, int32_t rank, void* const* peer_out_host,
                      uint32_t* const* peer_flags_host) {
  if (!h) return trie_set_error(TRIE_EINVAL, "null handle");
  if (world <= 1) {
    h->g_world = 0;
    return TRIE_OK;
  }
  if (world > 8 || rank < 0 || rank >= world || !peer_out_host || !peer_flags_host)
    return trie_set_error(TRIE_EINVAL, "gather: world %d (<= 8), rank %d", world, rank);
  if (h->cfg.kv_dtype != TRIE_BF16) return trie_set_error(TRIE_EINVAL, "gather: bf16 pools only");
  for (int q = 0; q < world; ++q) {
    if (!peer_out_host[q] || !peer_flags_host[q] || ((uintptr_t)peer_out_host[q] & 15))
      return trie_set_error(TRIE_EINVAL, "gather: rank %d buffer null or not 16-byte aligned", q);
    h->g_out[q] = peer_out_host[q];
    h->g_flags[q] = peer_flags_host[q];
  }
  h->g_world = world;
  h->g_rank = rank;
  return TRIE_OK;
}

int trie_gather_wait(trie_handle* h, void* gathered_out, cudaStream_t stream) {
  if (!h) return trie_set_error(TRIE_EINVAL, "null handle");
  if (h->g_world <= 1) return trie_set_error(TRIE_EINVAL, "gather: trie_gather_setup(world > 1) first");
  trie::GatherArgs ga = trie_gather_args(h);
  return trie::launch_gather_wait(ga, h->cfg.n_requests, h->b_live, h->cfg.n_q_heads, h->cfg.head_dim,
                                  gathered_out, stream);
}

int trie_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out || bytes == 0) return trie_set_error(TRIE_EINVAL, "ipc_alloc: bad argument");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
  cudaIpcMemHandle_t hd;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hd, p);
  if (e != cudaSuccess) {
    if (p) cudaFree(p);
    return trie_set_error(TRIE_ECUDA, "ipc_alloc: %s", cudaGetErrorString(e));
  }
  memcpy(handle_out, &hd, sizeof(hd));
  *dev_ptr = p;
  return TRIE_OK;
}

int trie_ipc_open(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return trie_set_error(TRIE_EINVAL, "ipc_open: bad argument");
  cudaIpcMemHandle_t hd;
  memcpy(&hd, handle, sizeof(hd));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return trie_set_error(TRIE_ECUDA, "ipc_open: %s", cudaGetErrorString(e));
  return TRIE_OK;
}

int trie_ipc_close(void* dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? TRIE_OK : trie_set_error(TRIE_ECUDA, "ipc_close: %s", cudaGetErrorString(e));
}

int trie_ipc_free(void* dev_ptr) {
  cudaError_t e = cudaFree(dev_ptr);
  return e == cudaSuccess ? TRIE_OK : trie_set_error(TRIE_ECUDA, "ipc_free: %s", cudaGetErrorString(e));
}

}  // extern "C"
