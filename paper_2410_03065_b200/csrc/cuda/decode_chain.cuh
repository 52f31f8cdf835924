// First-token step projections as ONE persistent weight-streaming kernel per
// layer boundary (the q-only 1-token pass over the assembled cache, the
// reference's "first token" that its simulator never models).
//
// With one query row every projection is a pure weight read: 416 MB per
// Llama-3-8B layer, ~65 us at HBM speed. As separate GEMV launches (q, o,
// gate/up, down; skinny.cuh) each kernel pays its launch, its x-prologue
// (RMSNorm of h per CTA) and a ragged tail before the next one can start —
// the 32-MB projections ran at 2 TB/s. Here one launch runs a CHAIN of phases
//     o(l) -> [norm2] gate/up(l) + SwiGLU -> down(l) -> [norm1] q(l+1) + RoPE
// (the attention of layer l+1 needs q(l+1), so it ends the chain), one CTA
// per SM, phases separated by a grid barrier. Before a CTA waits in a
// barrier (and before the PDL wait at launch) it asks L2 for the first rows
// it will stream in the next phase (cp.async.bulk.prefetch.L2), so HBM keeps
// working while the grid synchronises.
//
// Rows are streamed with 16-B LDGs by 32 warps per SM (a TMA ring with one
// bulk copy in flight per row measured 2.2 TB/s: too few bytes in flight per
// SM); x of the phase sits in shared memory as bf16. Row sums are reduced per
// warp, in a fixed order, so the result is deterministic. Epilogues are the
// skinny kernel's: RoPE pairs for q, SwiGLU for gate/up, residual adds for
// o / down.
#pragma once

#include "ptx.cuh"

namespace cake_dev {

enum DecKind : int { kDecQ = 0, kDecO = 1, kDecGU = 2, kDecD = 3 };

struct DecPhase {
  int kind;
  const __nv_bfloat16* W;      // weight rows [rows, K] (q: rope-unit row order; gate/up: 128-row interleave)
  const __nv_bfloat16* gamma;  // RMSNorm weight of the phase's input (q, gate/up), else nullptr
  int K;                       // row length
  int units;                   // output units (q: rope pairs, gate/up: SwiGLU outputs, o/down: rows)
};

constexpr int kDecMaxPhases = 4;
#ifndef DEC_WARPS
#define DEC_WARPS 32
#endif
#ifndef DEC_UNROLL
#define DEC_UNROLL 8
#endif
constexpr int kDecWarps = DEC_WARPS;
constexpr int kDecThreads = kDecWarps * 32;
constexpr int kDecUnroll = DEC_UNROLL;  // 16-B loads in flight per lane and row batch (4 KB per warp)

struct DecArgs {
  DecPhase ph[kDecMaxPhases];
  int n_phases;
  int max_k;           // x buffer (bf16) in shared memory
  int red_rows;        // row sums in shared memory: >= this CTA's rows of any phase
  int prefetch_bytes;  // L2 prefetch per CTA ahead of each phase
  float* h;            // [H] fp32 residual stream (row 0)
  int H;
  float eps;
  const __nv_bfloat16* attn;  // o input [nq * hd]
  __nv_bfloat16* act;         // gate/up output, down input [F]
  __nv_bfloat16* q_out;       // [nq * hd]
  const float2* rope;         // [pos][hd / 2]
  long long pos;
  int head_dim;
  unsigned long long* gbar;   // grid barrier: monotone arrival counter
  long long* trace;           // debug (cake_dec_debug_trace): %globaltimer per CTA [cta][16]
};

__device__ __forceinline__ void dec_stamp(const DecArgs& a, int slot) {
  if (a.trace != nullptr && threadIdx.x == 0) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[blockIdx.x * 16 + slot] = t;
  }
}

__device__ __forceinline__ int dec_rows_per_unit(int kind) { return (kind == kDecQ || kind == kDecGU) ? 2 : 1; }

// Weight row of phase-row index ri = unit * rows_per_unit + r.
__device__ __forceinline__ const __nv_bfloat16* dec_row(const DecPhase& p, int ri, int head_dim) {
  size_t row;
  if (p.kind == kDecQ) {
    const int u = ri >> 1, r = ri & 1;
    const int half = head_dim >> 1;
    const int head = u / half, i = u % half;
    row = static_cast<size_t>(head) * head_dim + (i >> 5) * 64 + (i & 31) + r * 32;  // qkv_row_of pairs
  } else if (p.kind == kDecGU) {
    const int u = ri >> 1, r = ri & 1;
    row = static_cast<size_t>(u / 128) * 256 + (u % 128) + r * 128;
  } else {
    row = static_cast<size_t>(ri);
  }
  return p.W + row * p.K;
}

__device__ __forceinline__ void dec_range(int units, int cta, int ctas, int& u0, int& u1) {
  u0 = static_cast<int>((static_cast<long long>(units) * cta) / ctas);
  u1 = static_cast<int>((static_cast<long long>(units) * (cta + 1)) / ctas);
}

__device__ __forceinline__ DecPhase dec_phase(const DecArgs& a, int p) {
  // (static indices into the parameter array: a dynamic one copies it to local memory)
  return p == 0 ? a.ph[0] : p == 1 ? a.ph[1] : p == 2 ? a.ph[2] : a.ph[3];
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(p)), "r"(bytes)
               : "memory");
}

// Ask L2 for the first `budget` bytes of this CTA's rows of phase p; lane l
// of the calling warp issues rows l, l+32, ... (one bulk prefetch per row),
// so the issue takes one round instead of a serial loop.
__device__ __forceinline__ void dec_prefetch(const DecArgs& a, int p, int cta, int ctas, int lane) {
  if (p >= a.n_phases) return;
  const DecPhase ph = dec_phase(a, p);
  const int rpu = dec_rows_per_unit(ph.kind);
  int u0, u1;
  dec_range(ph.units, cta, ctas, u0, u1);
  const uint32_t row_bytes = static_cast<uint32_t>(ph.K) * 2u;
  const int n = min((u1 - u0) * rpu, static_cast<int>((static_cast<uint32_t>(a.prefetch_bytes) + row_bytes - 1) / row_bytes));
  for (int i = lane; i < n; i += 32) prefetch_l2_bulk(dec_row(ph, u0 * rpu + i, a.head_dim), row_bytes);
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// All CTAs of the grid (one per SM, all resident: cooperative launch) meet
// here; the phase's global writes are visible to every CTA after it. One
// monotone 64-bit arrival counter (never reset): barrier k completes when it
// reaches (k+1) * ctas, which each CTA derives from its own atomicAdd — one
// L2 round trip for the last arrival instead of reset + generation bump.
// `between` runs after this CTA arrived and before it waits (the L2 prefetch
// of the next phase's rows), so it costs no barrier time.
template <typename F>
__device__ __forceinline__ void dec_grid_barrier(unsigned long long* ctr, int ctas, F&& between) {
  __syncthreads();
  if (threadIdx.x < 32) {  // warp 0: lane 0 arrives, then the warp issues the prefetches, then lane 0 waits
    unsigned long long target = 0;
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned long long old = atomicAdd(ctr, 1ull);
      target = (old / static_cast<unsigned long long>(ctas) + 1ull) * ctas;
    }
    __syncwarp();
    between(static_cast<int>(threadIdx.x));
    if (threadIdx.x == 0) {
      while (ld_acquire_gpu_u64(ctr) < target) __nanosleep(32);  // (a tight spin floods the counter's L2 line)
      __threadfence();
    }
  }
  __syncthreads();
}

__device__ __forceinline__ float2 bf2_to_f2(uint32_t v) {
  return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xFFFF0000u));
}

__device__ __forceinline__ float2 dot8(const uint4 w, const uint4 x, float2 s) {
  s = ffma2(bf2_to_f2(w.x), bf2_to_f2(x.x), s);
  s = ffma2(bf2_to_f2(w.y), bf2_to_f2(x.y), s);
  s = ffma2(bf2_to_f2(w.z), bf2_to_f2(x.z), s);
  return ffma2(bf2_to_f2(w.w), bf2_to_f2(x.w), s);
}

__global__ void __launch_bounds__(kDecThreads, 1) dec_chain_kernel(const DecArgs a) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(dsm);                      // [max_k]
  float* rsum = reinterpret_cast<float*>(dsm + static_cast<size_t>(a.max_k) * 2);  // [red_rows]
  __shared__ float s_norm[kDecWarps];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int ctas = gridDim.x;
  const int cta = blockIdx.x;

  dec_stamp(a, 0);
  if (tid < 32) dec_prefetch(a, 0, cta, ctas, tid);  // weights do not depend on the predecessor
  pdl_wait();  // the first phase's input (attn / h) is the predecessor's output
  pdl_trigger();
  dec_stamp(a, 1);
#pragma unroll 1
  for (int p = 0; p < a.n_phases; ++p) {
    const DecPhase ph = dec_phase(a, p);
    if (p > 0) dec_grid_barrier(a.gbar, ctas, [&](int ln) { dec_prefetch(a, p, cta, ctas, ln); });
    dec_stamp(a, 2 + 3 * p);
    const int K = ph.K;
    // ---- x of the phase into shared memory (bf16)
    if (ph.kind == kDecQ || ph.kind == kDecGU) {
      // RMSNorm of the residual row, identical on every CTA (fixed-order sum)
      float ss = 0.f;
      for (int i = tid; i < (a.H >> 2); i += kDecThreads) {
        const float4 v = reinterpret_cast<const float4*>(a.h)[i];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) s_norm[warp] = ss;
      __syncthreads();
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < kDecWarps; ++w) tot += s_norm[w];
      const float rn = rsqrtf(tot / static_cast<float>(a.H) + a.eps);
      for (int c = tid; c < (K >> 3); c += kDecThreads) {
        const float4 h0 = reinterpret_cast<const float4*>(a.h)[2 * c];
        const float4 h1 = reinterpret_cast<const float4*>(a.h)[2 * c + 1];
        const uint4 gg = reinterpret_cast<const uint4*>(ph.gamma)[c];
        const float2 g0 = bf2_to_f2(gg.x), g1 = bf2_to_f2(gg.y), g2 = bf2_to_f2(gg.z), g3 = bf2_to_f2(gg.w);
        uint4 o;
        o.x = pack_bf16(h0.x * rn * g0.x, h0.y * rn * g0.y);
        o.y = pack_bf16(h0.z * rn * g1.x, h0.w * rn * g1.y);
        o.z = pack_bf16(h1.x * rn * g2.x, h1.y * rn * g2.y);
        o.w = pack_bf16(h1.z * rn * g3.x, h1.w * rn * g3.y);
        reinterpret_cast<uint4*>(xs)[c] = o;
      }
    } else {
      const uint4* x = reinterpret_cast<const uint4*>(ph.kind == kDecO ? a.attn : a.act);
      for (int c = tid; c < (K >> 3); c += kDecThreads) reinterpret_cast<uint4*>(xs)[c] = x[c];
    }
    __syncthreads();
    dec_stamp(a, 3 + 3 * p);
    // ---- this CTA's rows, one warp per row at a time
    const int rpu = dec_rows_per_unit(ph.kind);
    int u0, u1;
    dec_range(ph.units, cta, ctas, u0, u1);
    const int r0 = u0 * rpu, nrows = (u1 - u0) * rpu;
    const int chunks = K >> 3;
    const uint4* xv = reinterpret_cast<const uint4*>(xs);
    for (int i = warp; i < nrows; i += kDecWarps) {
      const uint4* w = reinterpret_cast<const uint4*>(dec_row(ph, r0 + i, a.head_dim));
      float2 s2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      for (int c0 = lane; c0 < chunks; c0 += 32 * kDecUnroll) {
        uint4 wv[kDecUnroll];
#pragma unroll
        for (int u = 0; u < kDecUnroll; ++u) {
          const int c = c0 + 32 * u;
          wv[u] = c < chunks ? __ldg(w + c) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < kDecUnroll; ++u) {
          const int c = c0 + 32 * u;
          if (c < chunks) s2[u & 1] = dot8(wv[u], xv[c], s2[u & 1]);
        }
      }
      float s = (s2[0].x + s2[0].y) + (s2[1].x + s2[1].y);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) rsum[i] = s;
    }
    __syncthreads();
    dec_stamp(a, 4 + 3 * p);
    // ---- epilogue: one thread per unit
    for (int i = tid; i < u1 - u0; i += kDecThreads) {
      const int uu = u0 + i;
      const float v0 = rsum[i * rpu];
      const float v1 = rpu == 2 ? rsum[i * rpu + 1] : 0.f;
      if (ph.kind == kDecQ) {
        const int half = a.head_dim >> 1;
        const int head = uu / half, k = uu % half;
        const float2 cs = a.rope[a.pos * half + k];
        __nv_bfloat16* q = a.q_out + static_cast<size_t>(head) * a.head_dim + k;
        q[0] = __float2bfloat16_rn(v0 * cs.x - v1 * cs.y);
        q[half] = __float2bfloat16_rn(v1 * cs.x + v0 * cs.y);
      } else if (ph.kind == kDecGU) {
        a.act[uu] = __float2bfloat16_rn(v0 / (1.0f + __expf(-v0)) * v1);
      } else {
        a.h[uu] += v0;
      }
    }
    // (xs / rsum are rewritten only after the next phase's grid barrier)
  }
}

}  // namespace cake_dev
