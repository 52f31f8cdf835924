// The attention softmax's exponential loop in isolation (one thread = one row
// of 128 scores, as attention_fa4.cuh; or 64 scores, as attention_tc.cuh's
// column groups), on 1 or 2 warps per SM sub-partition, timed with clock64:
// what the MUFU / FMA budget allows without TMEM traffic or other warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2410_03065_b200/csrc/cuda -o tools/_softmax_bench tools/softmax_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "attention_tc.cuh"

using namespace cake_dev;

__device__ __forceinline__ float2 ex2_f16x2(float2 x) {
  unsigned h, e;
  asm("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(x.x), "f"(x.y));
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(e) : "r"(h));
  float2 p;
  asm("{.reg .f16 l, h; mov.b32 {l, h}, %2; cvt.f32.f16 %0, l; cvt.f32.f16 %1, h;}" : "=f"(p.x), "=f"(p.y) : "r"(e));
  return p;
}

template <int N, int POLY, int MODE = 0>
__global__ void k(const float* in, unsigned* out, long long* cyc, int iters) {
  float s[N];
  for (int i = 0; i < N; ++i) s[i] = in[(threadIdx.x * N + i) % 4096];
  const float sc = 0.0883883f * 1.442695f;
  const float2 sc2 = make_float2(sc, sc);
  float l = 0.f;
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float mc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) mc[c] = s[c];
#pragma unroll
    for (int i = 8; i < N; ++i) mc[i & 7] = fmaxf(mc[i & 7], s[i]);
    const float m = fmaxf(fmaxf(fmaxf(mc[0], mc[1]), fmaxf(mc[2], mc[3])), fmaxf(fmaxf(mc[4], mc[5]), fmaxf(mc[6], mc[7]))) * sc;
    const float2 nb2 = make_float2(-m, -m);
    float2 rs[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    unsigned pk[N / 2];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      const float2 x = ffma2(make_float2(s[2 * i], s[2 * i + 1]), sc2, nb2);
      float2 p;
      if ((i & 7) >= 8 - POLY) {
        p = ex2_poly2(x);
      } else if (MODE == 1) {
        p = ex2_f16x2(x);
      } else {
        p.x = ex2_approx(x.x);
        p.y = ex2_approx(x.y);
      }
      rs[i & 3] = fadd2(rs[i & 3], p);
      pk[i] = pack_bf16(p.x, p.y);
    }
    const float2 r01 = fadd2(rs[0], rs[1]), r23 = fadd2(rs[2], rs[3]);
    l += (r01.x + r23.x) + (r01.y + r23.y);
#pragma unroll
    for (int i = 0; i < N / 2; ++i) acc ^= pk[i];
    // perturb the scores so the loop is not hoisted
#pragma unroll
    for (int i = 0; i < N; ++i) s[i] = __uint_as_float(__float_as_uint(s[i]) ^ (acc & 1));
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(l);
  if ((threadIdx.x & 31) == 0) cyc[threadIdx.x / 32] = t1 - t0;
}

template <int N, int POLY, int MODE = 0>
void run(float* in, unsigned* out, long long* cyc, int warps) {
  const int iters = 256;
  for (int r = 0; r < 2; ++r) k<N, POLY, MODE><<<1, warps * 32>>>(in, out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[32];
  cudaMemcpy(h, cyc, warps * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
  const double per_block = double(mx) / iters;
  const double mufu = (warps / 4.0) * 32.0 * (N - 2.0 * POLY * N / 16) / 4.0;  // MUFU cycles per SMSP per iteration
  printf("%s scores/thread %3d poly %d/8 warps/SMSP %d: %.0f cycles per row-block (f32 MUFU floor %.0f)\n",
         MODE ? "f16-mufu" : "f32-mufu", N, POLY, warps / 4, per_block, mufu);
}

int main() {
  float* in;
  unsigned* out;
  long long* cyc;
  cudaMalloc(&in, 4096 * 4);
  float h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = (float)((i * 37) % 97) * 0.1f - 4.0f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&out, 1 << 16);
  cudaMalloc(&cyc, 1024);
  for (int warps : {4, 8}) {
    run<64, 0>(in, out, cyc, warps);
    run<64, 2>(in, out, cyc, warps);
    run<64, 8>(in, out, cyc, warps);
    run<64, 0, 1>(in, out, cyc, warps);
    run<64, 2, 1>(in, out, cyc, warps);
    run<128, 2>(in, out, cyc, warps);
    run<128, 0, 1>(in, out, cyc, warps);
  }
  for (int warps : {16}) {
    run<32, 0>(in, out, cyc, warps);
    run<32, 2>(in, out, cyc, warps);
    run<32, 0, 1>(in, out, cyc, warps);
  }
  return 0;
}
