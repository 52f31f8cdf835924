// Weight-streaming projections for the first-token step (M <= 4 rows).
//
// With one query row a projection is a pure weight read (HBM-bound: 416 MB
// per Llama-3-8B layer for q/o/gate-up/down). The tcgen05 tile kernel would
// run it on N/BLOCK_N CTAs only (16..112), far below the SM count; here
// every warp owns one output unit and streams its weight row(s) with 16-B
// loads, so thousands of warps keep the HBM pipes full. The unit epilogues
// mirror the tile kernel's: q rows pair (d, d + hd/2) for RoPE, gate/up rows
// pair through the 128-row interleave, o/down rows add into the fp32
// residual stream.
#pragma once

#include "ptx.cuh"

namespace cake_dev {

enum SkinnyEpi : int { kSkF32 = 0, kSkResid = 1, kSkQRope = 2, kSkSwiglu = 3 };

struct SkinnyArgs {
  const __nv_bfloat16* W;  // [rows, K]
  const __nv_bfloat16* x;  // [M, K]
  int M, K;
  int units;               // output units (rows, or row pairs)
  float* out;              // kSkF32: [M, rows]
  int ldo;
  float* resid;            // kSkResid: [M, ldr]
  int ldr;
  __nv_bfloat16* q_out;    // kSkQRope: [M, n_q * hd]
  const float2* rope;      // [pos][hd/2]
  long long pos0;
  int head_dim;
  __nv_bfloat16* act;      // kSkSwiglu: [M, F]
  int ld_act;
  // RMSNorm folded in (nullptr: x is already normalised): every CTA normalises
  // the M fp32 residual rows itself into its shared copy of x, so the step
  // needs no separate norm launch.
  const float* norm_h;     // [M, K]
  const __nv_bfloat16* norm_gamma;
  float norm_eps;
};

constexpr int kSkinnyWarps = 8;
// dot-loop unroll (16-B loads in flight per row and lane). A/B on the
// first-token step: 2 / 4 / 8 -> 5.42 / 5.44 / 5.38 ms; 16 (with 8 CTAs per SM)
// 5.29 ms. Touching the weights before the PDL wait measured slower: an L2
// prefetch of each warp's first rows 5.76 ms, a register preload of its first
// 4 / 8 batches 6.99 / 8.72 ms (the early loads compete with the still-running
// memory-bound predecessor). Two warps per row of the long-K down projection
// (K halves summed in order) measured within noise (5.23 vs 5.27 ms).
constexpr int kSkinnyUnroll = 16;

template <int NR>
__device__ __forceinline__ void skinny_dot(const __nv_bfloat16* const (&w)[NR], const __nv_bfloat16* xs, int M,
                                           int K, float (&acc)[NR][4]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int m = 0; m < 4; ++m) acc[r][m] = 0.f;
#pragma unroll kSkinnyUnroll
  for (int k = lane * 8; k < K; k += 256) {
    uint4 wv[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) wv[r] = __ldg(reinterpret_cast<const uint4*>(w[r] + k));
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      if (m >= M) break;
      const uint4 xv = *reinterpret_cast<const uint4*>(xs + static_cast<size_t>(m) * K + k);
      const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&xv);
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const __nv_bfloat162* wp = reinterpret_cast<const __nv_bfloat162*>(&wv[r]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 a = __bfloat1622float2(wp[e]);
          const float2 b = __bfloat1622float2(xp[e]);
          acc[r][m] = fmaf(a.x, b.x, acc[r][m]);
          acc[r][m] = fmaf(a.y, b.y, acc[r][m]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[r][m] += __shfl_xor_sync(0xffffffff, acc[r][m], o);
}

template <int EPI>
__global__ void __launch_bounds__(kSkinnyWarps * 32) skinny_kernel(const SkinnyArgs a) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t sm[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sm);
  const int total = a.M * a.K;
  if (a.norm_h == nullptr) {
    for (int i = threadIdx.x * 8; i < total; i += blockDim.x * 8)
      *reinterpret_cast<uint4*>(xs + i) = *reinterpret_cast<const uint4*>(a.x + i);
  } else {
    __shared__ float red[kSkinnyWarps];
    for (int mrow = 0; mrow < a.M; ++mrow) {
      const float4* hr = reinterpret_cast<const float4*>(a.norm_h + static_cast<size_t>(mrow) * a.K);
      float ss = 0.f;
      for (int i = threadIdx.x; i < a.K / 4; i += blockDim.x) {
        const float4 v = hr[i];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
      __syncthreads();
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < kSkinnyWarps; ++w) tot += red[w];  // fixed order: every CTA gets the same scale
      const float r = rsqrtf(tot / static_cast<float>(a.K) + a.norm_eps);
      for (int i = threadIdx.x; i < a.K / 4; i += blockDim.x) {
        const float4 v = hr[i];
        const uint2 gg = *reinterpret_cast<const uint2*>(a.norm_gamma + 4 * i);
        const float2 ga = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gg.x));
        const float2 gb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gg.y));
        uint2 o;
        o.x = pack_bf16(v.x * r * ga.x, v.y * r * ga.y);
        o.y = pack_bf16(v.z * r * gb.x, v.w * r * gb.y);
        *reinterpret_cast<uint2*>(xs + static_cast<size_t>(mrow) * a.K + 4 * i) = o;
      }
      __syncthreads();  // red[] is reused by the next row
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int u = blockIdx.x * kSkinnyWarps + (threadIdx.x >> 5); u < a.units; u += gridDim.x * kSkinnyWarps) {
    if constexpr (EPI == kSkF32 || EPI == kSkResid) {
      const __nv_bfloat16* w[1] = {a.W + static_cast<size_t>(u) * a.K};
      float acc[1][4];
      skinny_dot<1>(w, xs, a.M, a.K, acc);
      if (lane == 0)
        for (int m = 0; m < a.M; ++m) {
          if constexpr (EPI == kSkF32)
            a.out[static_cast<size_t>(m) * a.ldo + u] = acc[0][m];
          else
            a.resid[static_cast<size_t>(m) * a.ldr + u] += acc[0][m];
        }
    } else if constexpr (EPI == kSkQRope) {
      const int half = a.head_dim >> 1;
      const int head = u / half, i = u % half;
      const int r0 = head * a.head_dim + i;  // canonical q column
      // physical weight rows: rope-unit order (qkv_row_of): i -> 64 (i / 32) + i % 32, its partner 32 later
      const int p0 = head * a.head_dim + (i >> 5) * 64 + (i & 31);
      const __nv_bfloat16* w[2] = {a.W + static_cast<size_t>(p0) * a.K, a.W + static_cast<size_t>(p0 + 32) * a.K};
      float acc[2][4];
      skinny_dot<2>(w, xs, a.M, a.K, acc);
      if (lane == 0)
        for (int m = 0; m < a.M; ++m) {
          const float2 cs = a.rope[(a.pos0 + m) * half + i];
          const float x0 = acc[0][m], x1 = acc[1][m];
          __nv_bfloat16* q = a.q_out + static_cast<size_t>(m) * a.ldo + r0;
          q[0] = __float2bfloat16_rn(x0 * cs.x - x1 * cs.y);
          q[half] = __float2bfloat16_rn(x1 * cs.x + x0 * cs.y);
        }
    } else if constexpr (EPI == kSkSwiglu) {
      const int g = (u / 128) * 256 + (u % 128);
      const __nv_bfloat16* w[2] = {a.W + static_cast<size_t>(g) * a.K, a.W + static_cast<size_t>(g + 128) * a.K};
      float acc[2][4];
      skinny_dot<2>(w, xs, a.M, a.K, acc);
      if (lane == 0)
        for (int m = 0; m < a.M; ++m) {
          const float gt = acc[0][m];
          a.act[static_cast<size_t>(m) * a.ld_act + u] = __float2bfloat16_rn(gt / (1.0f + __expf(-gt)) * acc[1][m]);
        }
    }
  }
}

}  // namespace cake_dev
