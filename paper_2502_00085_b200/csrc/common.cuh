// Shared device helpers of libtriedecode (sm_100a).  No method arithmetic lives here
// beyond type conversion and warp/block reductions.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/triedecode.h"

#define TRIE_MAX_BEAMS 32
#define TRIE_MAX_LAYERS 128

namespace trie {

// ---- element conversion ----------------------------------------------------------------
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// ---- reductions ------------------------------------------------------------------------
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// order-preserving map float -> uint32 (larger float -> larger uint); -0 < +0, NaN largest
__device__ __forceinline__ uint32_t f2ord(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__device__ __forceinline__ void latch(uint32_t* status, uint32_t bit) {
  if (status) atomicOr(status, bit);
}

// ---- programmatic dependent launch (PDL) ---------------------------------------------------
// Hot-path kernels are launched with programmatic stream serialization (launch_k below):
// a kernel may be scheduled while its predecessor drains.  pdl_trigger() lets the NEXT
// kernel's CTAs launch once every CTA of this grid has started; pdl_wait() blocks until the
// predecessor grid has completed and its memory is visible -- every kernel calls it before
// its first global-memory access (setup that touches only shared memory / TMEM / tensor
// maps may run before it).  Both are no-ops for a plain launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

bool pdl_enabled();  // TRIE_PDL=0 disables (api.cu)

inline void pdl_config(cudaLaunchConfig_t* cfg, cudaLaunchAttribute* attr, dim3 grid, dim3 block,
                       size_t smem, cudaStream_t s) {
  cfg->gridDim = grid;
  cfg->blockDim = block;
  cfg->dynamicSmemBytes = smem;
  cfg->stream = s;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg->attrs = attr;
  cfg->numAttrs = pdl_enabled() ? 1 : 0;
}

// kernel<<<grid, block, smem, s>>>(args...) with the PDL attribute
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  pdl_config(&cfg, attr, grid, block, smem, s);
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
// the same for a kernel held as a void pointer with a packed argument array
inline cudaError_t launch_k_ptr(const void* kern, dim3 grid, dim3 block, size_t smem,
                                cudaStream_t s, void** args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  pdl_config(&cfg, attr, grid, block, smem, s);
  return cudaLaunchKernelExC(&cfg, kern, args);
}

}  // namespace trie

// ---- host-side error plumbing (api.cu) --------------------------------------------------
int trie_set_error(int code, const char* fmt, ...);
int trie_check_launch(const char* what);
