// Head-sharded TP over peer memory (one process per GPU, CUDA IPC mappings of
// every rank's exchange buffers; NVLink / NVSwitch loads and stores between
// B200s, plain device memory when two ranks share one GPU in the tests).
//
// Replaces ncclAllReduce + add + RMSNorm after each row-parallel projection
// (O and MLP-down) with ONE kernel per reduction:
//
//   slice mode (prefill chunks, M > 1): the residual stream h stays sharded by
//   rows (row r lives on rank r % N). Each rank pulls the bf16 partials of its
//   rows from every rank, sums them in rank order (fp32; every rank computes
//   its rows the same way, so the result does not depend on who reduces),
//   adds them into h, applies the RMSNorm of the next projection and stores
//   the normalized bf16 row into EVERY rank's xn (the A operand of the next
//   column-parallel GEMM). Wire bytes per rank and reduction:
//   (N-1)/N * M * H * (2 pulled + 2 pushed), half of a fp32 ring all-reduce.
//
//   replicated mode (the 1-token first-token pass, M = 1): every rank pulls
//   every rank's fp32 partial of the row and adds the rank-ordered sum into its
//   own full h (the folded-norm GEMVs that follow read h).
//
// Synchronisation: monotonically increasing 64-bit epochs, one per reduction
// call (every rank makes the same calls in the same order: the TP
// coordinator mirrors the leader's launch sequence). Flag A[src] = "src's
// partial of this epoch is complete"; flag B[src] = "src finished pulling
// from everyone (and pushing its rows)". A rank's kernel completes only after
// every B of the epoch arrived, so its next GEMM may overwrite its partial
// and its next column-parallel GEMM sees every pushed row.
#pragma once

#include "ptx.cuh"

namespace cake_dev {

constexpr int kTpMaxRanks = 8;
constexpr int kTpThreads = 256;
// flag block per rank (device memory, IPC-mapped by every peer):
//   [0, 8)   A[src]   [8, 16)  B[src]   [16] CTA arrival counter (own)
constexpr int kTpFlagA = 0, kTpFlagB = 8, kTpFlagCount = 16, kTpFlagWords = 32;

struct TpReduceArgs {
  const void* part[kTpMaxRanks];            // each rank's partial buffer [rows][H] (bf16 slice mode, fp32 replicated)
  __nv_bfloat16* xn[kTpMaxRanks];           // slice mode: every rank's xn (push targets)
  unsigned long long* flags[kTpMaxRanks];   // every rank's flag block
  float* h;                                 // own residual [rows][H]
  const __nv_bfloat16* gamma;               // slice mode: norm weight of the next projection
  float eps;
  int rank, nranks, M, H;
  int replicated;
  unsigned long long epoch;
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void tp_wait_flags(const unsigned long long* mine, int base, int rank, int nranks,
                                              unsigned long long epoch) {
  for (int src = 0; src < nranks; ++src) {
    if (src == rank) continue;
    while (ld_acquire_sys(mine + base + src) < epoch) __nanosleep(64);
  }
}

// grid <= one wave of small CTAs (all resident: CTA 0 signals, every CTA waits)
__global__ void __launch_bounds__(kTpThreads) tp_reduce_kernel(const TpReduceArgs a) {
  unsigned long long* mine = a.flags[a.rank];
  // A: this rank's partial (the preceding kernel in stream order) is complete
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < a.nranks; ++p)
      if (p != a.rank) st_release_sys(a.flags[p] + kTpFlagA + a.rank, a.epoch);
  }
  if (threadIdx.x == 0) tp_wait_flags(mine, kTpFlagA, a.rank, a.nranks, a.epoch);
  __syncthreads();
  __threadfence();

  const int H = a.H;
  const int nvec = H / 8;  // 8 elements per thread-step (one 16-B bf16 vector, two fp32 float4)
  __shared__ float red[kTpThreads / 32];
  __shared__ float s_scale;
  const int stride = a.replicated ? 1 : a.nranks;
  const int first = a.replicated ? 0 : a.rank;
  const int my_rows = a.M > first ? (a.M - first + stride - 1) / stride : 0;
  for (int i = blockIdx.x; i < my_rows; i += gridDim.x) {
    const long long row = first + static_cast<long long>(i) * stride;
    float* hrow = a.h + row * H;
    float ss = 0.f;
    // H <= 8192: at most 4 vectors of 8 per thread
    float acc[4][8];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int idx = threadIdx.x + v * kTpThreads;
      if (idx >= nvec) break;
      const float4 h0 = reinterpret_cast<const float4*>(hrow)[2 * idx];
      const float4 h1 = reinterpret_cast<const float4*>(hrow)[2 * idx + 1];
      float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int r = 0; r < a.nranks; ++r) {  // rank order: identical sums on every rank
        if (a.replicated) {
          const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(a.part[r]) + row * H);
          const float4 p0 = __ldcg(p + 2 * idx), p1 = __ldcg(p + 2 * idx + 1);
          s[0] += p0.x, s[1] += p0.y, s[2] += p0.z, s[3] += p0.w;
          s[4] += p1.x, s[5] += p1.y, s[6] += p1.z, s[7] += p1.w;
        } else {
          const uint4 q = __ldcg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.part[r]) + row * H) + idx);
          const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
            s[2 * k] += f.x;
            s[2 * k + 1] += f.y;
          }
        }
      }
      acc[v][0] = h0.x + s[0], acc[v][1] = h0.y + s[1], acc[v][2] = h0.z + s[2], acc[v][3] = h0.w + s[3];
      acc[v][4] = h1.x + s[4], acc[v][5] = h1.y + s[5], acc[v][6] = h1.z + s[6], acc[v][7] = h1.w + s[7];
      reinterpret_cast<float4*>(hrow)[2 * idx] = make_float4(acc[v][0], acc[v][1], acc[v][2], acc[v][3]);
      reinterpret_cast<float4*>(hrow)[2 * idx + 1] = make_float4(acc[v][4], acc[v][5], acc[v][6], acc[v][7]);
#pragma unroll
      for (int k = 0; k < 8; ++k) ss += acc[v][k] * acc[v][k];
    }
    if (a.replicated) continue;
    // RMSNorm of the updated row (fixed-order: thread-sequential, shuffle tree, warps in index order)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int w = 0; w < kTpThreads / 32; ++w) t += red[w];
      s_scale = rsqrtf(t / static_cast<float>(H) + a.eps);
    }
    __syncthreads();
    const float rr = s_scale;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int idx = threadIdx.x + v * kTpThreads;
      if (idx >= nvec) break;
      const uint4 g = reinterpret_cast<const uint4*>(a.gamma)[idx];
      const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 gf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gw[k]));
        o[k] = pack_bf16(acc[v][2 * k] * rr * gf.x, acc[v][2 * k + 1] * rr * gf.y);
      }
      const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
      for (int p = 0; p < a.nranks; ++p)  // push: own xn and every peer's
        reinterpret_cast<uint4*>(a.xn[p] + row * H)[idx] = ov;
    }
    __syncthreads();  // red / s_scale reuse by the next row
  }

  // B: this CTA's pulls (and pushes) are done; the last CTA tells the peers
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long old = atomicAdd(mine + kTpFlagCount, 1ull);
    if (old == gridDim.x - 1) {
      mine[kTpFlagCount] = 0;
      __threadfence_system();
      for (int p = 0; p < a.nranks; ++p)
        if (p != a.rank) st_release_sys(a.flags[p] + kTpFlagB + a.rank, a.epoch);
    }
  }
  // the kernel (and so the stream) completes only when every peer is done with this epoch
  if (blockIdx.x == 0 && threadIdx.x == 0) tp_wait_flags(mine, kTpFlagB, a.rank, a.nranks, a.epoch);
}

// Flag-only barrier of the TP group (same epochs and flag block as the
// reductions): A = "my stores of this epoch are issued and fenced", then wait
// for every peer's A. One thread.
__global__ void tp_barrier_kernel(const TpReduceArgs a) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int p = 0; p < a.nranks; ++p)
    if (p != a.rank) st_release_sys(a.flags[p] + kTpFlagA + a.rank, a.epoch);
  tp_wait_flags(a.flags[a.rank], kTpFlagA, a.rank, a.nranks, a.epoch);
}

// Vocab-sharded LM head of the first token: logits rows [n0, n1) of the
// replicated weight, each stored into EVERY rank's logits buffer (one warp per
// row, 16-B loads, x staged in shared memory as fp32; gemv_kernel's loop).
struct TpGemvArgs {
  const __nv_bfloat16* W;
  const __nv_bfloat16* x;
  float* out[kTpMaxRanks];
  int nranks, n0, n1, K;
};

__global__ void tp_gemv_kernel(const TpGemvArgs a) {
  extern __shared__ float xs_tp[];
  for (int i = threadIdx.x; i < a.K; i += blockDim.x) xs_tp[i] = __bfloat162float(a.x[i]);
  __syncthreads();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int n = a.n0 + blockIdx.x * warps + (threadIdx.x >> 5); n < a.n1; n += gridDim.x * warps) {
    const __nv_bfloat16* w = a.W + static_cast<size_t>(n) * a.K;
    float acc = 0.f;
#pragma unroll 4
    for (int k = lane * 8; k < a.K; k += 256) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(w + k));
      const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(p[e]);
        acc += f.x * xs_tp[k + 2 * e] + f.y * xs_tp[k + 2 * e + 1];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, o);
    if (lane == 0)
      for (int r = 0; r < a.nranks; ++r) a.out[r][n] = acc;
  }
  __threadfence_system();  // the remote stores, before the barrier kernel that follows
}

}  // namespace cake_dev
