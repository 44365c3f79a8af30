// Microbenchmark: MUFU.EX2 vs FFMA throughput per SM on this GPU (clock64 per CTA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu scripts/mufu_bench.cu && /tmp/mufu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, long long* clk, int iters) {
  float a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = -0.001f * (threadIdx.x + u);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[u]));
      else if (MODE == 1) a[u] = fmaf(a[u], 0.999f, -0.001f);
      else {  // MUFU + 3 FFMA mix (one ex2 per 4 ops)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[u]));
        a[u] = fmaf(a[u], 0.999f, -0.5f);
        a[u] = fmaf(a[u], 0.999f, -0.001f);
        a[u] = fmaf(a[u], 0.999f, -0.001f);
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += a[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps) {
  const int blocks = 148, threads = warps * 32, iters = 2048;
  float* out; long long* clk;
  cudaMalloc(&out, blocks * threads * 4);
  cudaMalloc(&clk, blocks * 8);
  k<MODE><<<blocks, threads>>>(out, clk, iters);
  k<MODE><<<blocks, threads>>>(out, clk, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double ops = (double)threads * iters * 8;
  printf("%-10s warps=%2d  ops/clk/SM = %.1f (cycles %lld)\n", name, warps, ops / h[0], h[0]);
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("ex2", w);
    run<1>("ffma", w);
    run<2>("ex2+3ffma", w);
  }
  return 0;
}
