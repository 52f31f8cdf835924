// MUFU.EX2 / FMA-pipe throughput on one SM (clock64 per warp), to ground the
// attention softmax budget: cycles per warp-instruction of ex2.approx.ftz.f32
// with 1..8 warps per SM sub-partition, alone and interleaved with FFMA2 work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_mufu_bench tools/mufu_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[8], b[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i), b[i] = 0.5f + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (MODE == 1 || MODE == 2) {
        asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f00000001;" : "+f"(b[i]));
        asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f00000001;" : "+f"(b[i]));
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + b[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1 << 16);
  const int iters = 4096;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<1, warps * 32>>>(out, cyc, iters);
        if (mode == 1) k<1><<<1, warps * 32>>>(out, cyc, iters);
        if (mode == 2) k<2><<<1, warps * 32>>>(out, cyc, iters);
        cudaDeviceSynchronize();
      }
      long long h[32];
      cudaMemcpy(h, cyc, warps * sizeof(long long), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
      const double per_smsp = warps / 4.0;
      const double n_mufu = mode == 1 ? 0 : 8.0 * iters * per_smsp;
      const double n_fma = mode == 0 ? 0 : 16.0 * iters * per_smsp;
      printf("mode %s warps/SM %2d: %lld cycles; per SMSP: %.2f cyc/MUFU-instr, %.2f cyc/FFMA-instr\n",
             mode == 0 ? "ex2 " : mode == 1 ? "ffma" : "both", warps, mx, n_mufu ? mx / n_mufu : 0.0,
             n_fma ? mx / n_fma : 0.0);
    }
  return 0;
}
