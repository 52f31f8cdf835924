// tcgen05.mma issue microbenchmark (one CTA, M=128 N=128 K=16 bf16, 8 MMAs per
// group, 2 commits per group). Prints cycles per MMA; the floor is 64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Ipaper_2410_03065_b200/csrc/cuda \
//        -o tools/_mma_issue_bench tools/mma_issue_bench.cu && ./tools/_mma_issue_bench
// Findings on B200 (profiles/r01_ncu_summary.md, "MMA issue"):
//  * SS / TS (A from TMEM), K- or MN-major B: all 64 cycles; concurrent TMEM
//    loads or shared-memory stores from other warps do not slow the pipe.
//  * Issued from a divergent single lane, any pause between groups costs the
//    pause plus ~100 cycles (the pipe drains): an mbarrier test on an
//    already-complete barrier costs ~160 cycles per group (83.9 cycles/MMA).
//  * Issued by a converged warp (elect.sync lane), the same wait costs ~70
//    (73.0/MMA), and a named-barrier handoff from a helper warp that does the
//    mbarrier wait costs nothing (64.0/MMA).
#include <cstdio>

#include "ptx.cuh"
using namespace cake_dev;

__device__ __forceinline__ void bsync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ bool test_done(uint64_t* bar) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(0u)
      : "memory");
  return ok != 0;
}

// MODE 0: single lane, no pause      1: single lane, test_wait(done) per group
//      2: converged warp, no pause   3: converged warp, lane-0 mbar_wait(done) + syncwarp
//      4: converged warp, bar.sync handoff from a helper warp that waits on the mbarrier
template <int MODE>
__global__ void issue_kernel(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done, commit_bar[2], ready;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    mbar_init(&commit_bar[0], 1);
    mbar_init(&commit_bar[1], 1);
    mbar_init(&ready, 1);
    mbar_arrive(&ready);  // phase 0 complete: every wait below finds it done
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = umma_idesc_bf16(128, 128, false, false);
  const uint32_t b = smem_u32(smem);
  auto group = [&](int i) {
    const uint64_t base = umma_desc_sw128(b + (i % 3) * 32768);
    const uint32_t d = tmem + (i & 1) * 128;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
      umma_bf16_ts(d, tmem + 384 + kk * 8, base + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4), idesc, kk > 0);
    umma_commit(&commit_bar[0]);
    umma_commit(&commit_bar[1]);
  };
  if (MODE <= 1 && threadIdx.x == 32) {
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (MODE == 1)
        while (!test_done(&ready)) {
        }
      tc_fence_after();
      group(i);
    }
    umma_commit(&done);
    mbar_wait(&done, 0);
    out[MODE] = clock64() - t0;
  } else if (MODE >= 2 && warp == 1) {
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (MODE == 3) {
        if (lane == 0) mbar_wait(&ready, 0);
        __syncwarp();
      }
      if (MODE == 4) bsync(1 + (i & 1), 64);
      tc_fence_after();
      if (elect_one()) group(i);
      __syncwarp();
    }
    if (elect_one()) umma_commit(&done);
    mbar_wait(&done, 0);
    if (lane == 0) out[MODE] = clock64() - t0;
  } else if (MODE == 4 && warp == 2) {
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&ready, 0);
      bsync(1 + (i & 1), 64);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  long long h[8];
  const int iters = 999;
  const char* names[5] = {"single lane, no pause", "single lane, test_wait(done)", "converged warp, no pause",
                          "converged warp, mbar_wait(done)", "converged warp, bar.sync handoff"};
  void (*k[5])(long long*, int) = {issue_kernel<0>, issue_kernel<1>, issue_kernel<2>, issue_kernel<3>,
                                   issue_kernel<4>};
  for (int m = 0; m < 5; ++m) {
    cudaFuncSetAttribute(k[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 110000);
    k[m]<<<1, 128, 110000>>>(d, iters);
    const cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-34s %s  %.1f cycles per MMA (floor 64)\n", names[m], cudaGetErrorString(e),
           static_cast<double>(h[m]) / (iters * 8));
  }
  return 0;
}
