// Prefix-causal attention of one chunk's queries over the paged KV cache.
//
// Query rows of a CTA are (token, q-head-in-group) pairs for one KV head, so
// the 4 query heads of a Llama-3 GQA group share every K/V page load. Keys
// are visited one 64-token page at a time through the block table; tokens
// before the chunk are all visible, tokens inside the chunk causally.
// Long prefixes are split across CTAs (split-KV) and merged by a fixed-order
// log-sum-exp combine, so results are bit-deterministic.
//
// v1 math path: mma.sync m16n8k16 bf16 (fp32 accumulate) with online softmax
// in registers; K/V pages stream through a double-buffered, XOR-swizzled smem
// ring with cp.async.
#pragma once

#include "ptx.cuh"

namespace cake_dev {

constexpr int kAttnPage = 64;       // tokens per KV page (== model page_tokens)
constexpr int kAttnRows = 64;       // query rows per CTA (4 warps x 16)
constexpr int kAttnThreads = 128;

struct AttnArgs {
  const __nv_bfloat16* q;      // [C, n_q, hd]
  const __nv_bfloat16* pool;   // paged KV
  const int* block_table;
  __nv_bfloat16* out;          // [C, n_q, hd]   (num_splits == 1)
  float* part_o;               // [splits, C, n_q, hd]
  float* part_lse;             // [splits, C, n_q]
  long long chunk_start;       // absolute position of query token 0
  int chunk_len;
  int n_q_heads, n_kv_heads, layer, n_layers;
  int num_splits;
  float scale_log2;            // log2(e) / sqrt(hd)
  const int* abort_flag;
};

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t saddr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(saddr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t saddr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(saddr));
}

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Byte offset of 16-B chunk `c` of row `r` in a swizzled tile with HD columns.
template <int HD>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return static_cast<uint32_t>(r * (HD * 2) + ((c ^ (r & 7)) << 4));
}

template <int HD>
__global__ void __launch_bounds__(kAttnThreads, 2) attn_prefill_kernel(const AttnArgs args) {
  constexpr int kChunks = HD / 8;                 // 16-B chunks per row
  constexpr int kTileBytes = kAttnPage * HD * 2;  // one K or V page
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;                        // [64][HD]
  uint8_t* sK = smem + kAttnRows * HD * 2;   // [2][64][HD]
  uint8_t* sV = sK + 2 * kTileBytes;         // [2][64][HD]

  if (args.abort_flag != nullptr && *(volatile const int*)args.abort_flag) return;

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int kvh = blockIdx.y;
  const int split = blockIdx.z;
  const int G = args.n_q_heads / args.n_kv_heads;
  const int tok_per_tile = kAttnRows / G;
  const int tok0 = blockIdx.x * tok_per_tile;
  if (tok0 >= args.chunk_len) return;
  const int tok_last = min(tok0 + tok_per_tile, args.chunk_len) - 1;

  // KV range this CTA must cover and this split's share (whole pages).
  const long long kv_end = args.chunk_start + tok_last + 1;
  const int n_pages = static_cast<int>((kv_end + kAttnPage - 1) / kAttnPage);
  const int per_split = (n_pages + args.num_splits - 1) / args.num_splits;
  const int p_begin = split * per_split;
  const int p_end = min(n_pages, p_begin + per_split);

  const size_t head_stride = static_cast<size_t>(kAttnPage) * HD;  // elements
  const size_t kv_plane = head_stride * args.n_kv_heads;
  auto page_ptr = [&](int lpage, int kv) -> const __nv_bfloat16* {
    const size_t phys = static_cast<size_t>(args.block_table[lpage]);
    return args.pool + ((phys * args.n_layers + args.layer) * 2 + kv) * kv_plane + kvh * head_stride;
  };
  auto load_page = [&](int lpage, int buf) {
    const __nv_bfloat16* gk = page_ptr(lpage, 0);
    const __nv_bfloat16* gv = page_ptr(lpage, 1);
    const uint32_t sk = smem_u32(sK + buf * kTileBytes);
    const uint32_t sv = smem_u32(sV + buf * kTileBytes);
#pragma unroll
    for (int i = tid; i < kAttnPage * kChunks; i += kAttnThreads) {
      const int r = i / kChunks, c = i % kChunks;
      cp_async16(sk + swz<HD>(r, c), gk + r * HD + c * 8);
      cp_async16(sv + swz<HD>(r, c), gv + r * HD + c * 8);
    }
  };

  // Q tile: row r = (token tok0 + r / G, head kvh*G + r % G).
  {
    const uint32_t sq = smem_u32(sQ);
    for (int i = tid; i < kAttnRows * kChunks; i += kAttnThreads) {
      const int r = i / kChunks, c = i % kChunks;
      const int t = tok0 + r / G;
      const int h = kvh * G + r % G;
      if (t < args.chunk_len) {
        cp_async16(sq + swz<HD>(r, c), args.q + (static_cast<size_t>(t) * args.n_q_heads + h) * HD + c * 8);
      } else {
        *reinterpret_cast<uint4*>(sQ + swz<HD>(r, c)) = make_uint4(0, 0, 0, 0);
      }
    }
  }
  if (p_begin < p_end) load_page(p_begin, 0);
  cp_async_commit();

  // Per-thread rows (within the warp's 16): lane/4 and lane/4 + 8.
  const int rw0 = warp * 16 + (lane >> 2);
  const int rw1 = rw0 + 8;
  const long long qpos0 = args.chunk_start + tok0 + rw0 / G;
  const long long qpos1 = args.chunk_start + tok0 + rw1 / G;

  float o[HD / 8][4];
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  uint32_t qa[HD / 16][4];

  for (int p = p_begin; p < p_end; ++p) {
    const int buf = (p - p_begin) & 1;
    if (p + 1 < p_end) load_page(p + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (p == p_begin) {
      const uint32_t sq = smem_u32(sQ);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int r = warp * 16 + (lane & 15);
        const int c = kk * 2 + (lane >> 4);
        ldsm_x4(sq + swz<HD>(r, c), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
      }
    }
    const uint32_t sk = smem_u32(sK + buf * kTileBytes);
    const uint32_t sv = smem_u32(sV + buf * kTileBytes);

    // S = Q K^T  (16 x 64 per warp)
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const int mi = lane >> 3;
        const int r = (j + (mi >> 1)) * 8 + (lane & 7);
        const int c = kk * 2 + (mi & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sk + swz<HD>(r, c), b0, b1, b2, b3);
        mma_bf16_16816(s[j], qa[kk], b0, b1);
        mma_bf16_16816(s[j + 1], qa[kk], b2, b3);
      }
    }

    // Scale, causal mask (only pages that reach into the chunk), online softmax.
    const long long kbase = static_cast<long long>(p) * kAttnPage;
    const bool need_mask = kbase + kAttnPage - 1 > args.chunk_start + tok0;
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = s[j][e] * args.scale_log2;
        if (need_mask) {
          const long long kpos = kbase + j * 8 + 2 * (lane & 3) + (e & 1);
          const long long qp = (e < 2) ? qpos0 : qpos1;
          if (kpos > qp) v = -INFINITY;
        }
        s[j][e] = v;
      }
      mx0 = fmaxf(mx0, fmaxf(s[j][0], s[j][1]));
      mx1 = fmaxf(mx1, fmaxf(s[j][2], s[j][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, 2));
    const float base0 = (mx0 == -INFINITY) ? 0.f : mx0;
    const float base1 = (mx1 == -INFINITY) ? 0.f : mx1;
    const float corr0 = exp2f(m0 - base0);
    const float corr1 = exp2f(m1 - base1);
    m0 = mx0;
    m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
    uint32_t pa[4][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float p0 = exp2f(s[j][0] - base0);
      const float p1 = exp2f(s[j][1] - base0);
      const float p2 = exp2f(s[j][2] - base1);
      const float p3 = exp2f(s[j][3] - base1);
      rs0 += p0 + p1;
      rs1 += p2 + p3;
      const int kk = j >> 1;
      if ((j & 1) == 0) {
        pa[kk][0] = pack_bf16(p0, p1);
        pa[kk][1] = pack_bf16(p2, p3);
      } else {
        pa[kk][2] = pack_bf16(p0, p1);
        pa[kk][3] = pack_bf16(p2, p3);
      }
    }
    l0 = l0 * corr0 + rs0;
    l1 = l1 * corr1 + rs1;
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
      o[j][0] *= corr0;
      o[j][1] *= corr0;
      o[j][2] *= corr1;
      o[j][3] *= corr1;
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int j = 0; j < HD / 8; j += 2) {
        const int mi = lane >> 3;
        const int r = kk * 16 + (mi & 1) * 8 + (lane & 7);
        const int c = j + (mi >> 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(sv + swz<HD>(r, c), b0, b1, b2, b3);
        mma_bf16_16816(o[j], pa[kk], b0, b1);
        mma_bf16_16816(o[j + 1], pa[kk], b2, b3);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  // Row sums across the quad.
  l0 += __shfl_xor_sync(0xffffffff, l0, 1);
  l0 += __shfl_xor_sync(0xffffffff, l0, 2);
  l1 += __shfl_xor_sync(0xffffffff, l1, 1);
  l1 += __shfl_xor_sync(0xffffffff, l1, 2);

  const int t0 = tok0 + rw0 / G, h0 = kvh * G + rw0 % G;
  const int t1 = tok0 + rw1 / G, h1 = kvh * G + rw1 % G;
  const int col = 2 * (lane & 3);
  if (args.num_splits == 1) {
    const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f;
    const float inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
      if (t0 < args.chunk_len)
        *reinterpret_cast<uint32_t*>(args.out + (static_cast<size_t>(t0) * args.n_q_heads + h0) * HD + j * 8 + col) =
            pack_bf16(o[j][0] * inv0, o[j][1] * inv0);
      if (t1 < args.chunk_len)
        *reinterpret_cast<uint32_t*>(args.out + (static_cast<size_t>(t1) * args.n_q_heads + h1) * HD + j * 8 + col) =
            pack_bf16(o[j][2] * inv1, o[j][3] * inv1);
    }
  } else {
    // Partial: normalised O of this split + its log2-sum-exp.
    const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f;
    const float inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
    const size_t rows = static_cast<size_t>(args.chunk_len) * args.n_q_heads;
    float* po = args.part_o + static_cast<size_t>(split) * rows * HD;
    float* pl = args.part_lse + static_cast<size_t>(split) * rows;
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
      if (t0 < args.chunk_len)
        *reinterpret_cast<float2*>(po + (static_cast<size_t>(t0) * args.n_q_heads + h0) * HD + j * 8 + col) =
            make_float2(o[j][0] * inv0, o[j][1] * inv0);
      if (t1 < args.chunk_len)
        *reinterpret_cast<float2*>(po + (static_cast<size_t>(t1) * args.n_q_heads + h1) * HD + j * 8 + col) =
            make_float2(o[j][2] * inv1, o[j][3] * inv1);
    }
    if ((lane & 3) == 0) {
      if (t0 < args.chunk_len)
        pl[static_cast<size_t>(t0) * args.n_q_heads + h0] = l0 > 0.f ? m0 + log2f(l0) : -INFINITY;
      if (t1 < args.chunk_len)
        pl[static_cast<size_t>(t1) * args.n_q_heads + h1] = l1 > 0.f ? m1 + log2f(l1) : -INFINITY;
    }
  }
}

// out[row, :] = sum_s 2^(lse_s - lse) * O_s[row, :], fixed split order.
// One CTA of HD threads per row: warp 0 turns the split LSEs into weights in
// shared memory (lane-parallel over splits), then thread t sums column t over
// the splits with 8 independent loads in flight (a warp per row walking the
// splits one dependent L2 round trip at a time took 17 us for 32 rows x 37
// splits in the first-token step).
constexpr int kCombineMaxSplits = 128;
template <int HD>
__global__ void __launch_bounds__(HD) attn_combine_kernel(const float* __restrict__ part_o,
                                                          const float* __restrict__ part_lse,
                                                          __nv_bfloat16* __restrict__ out, int rows, int num_splits,
                                                          const int* abort_flag) {
  __shared__ float w[kCombineMaxSplits];
  __shared__ float s_inv;
  pdl_wait();
  pdl_trigger();
  if (abort_flag != nullptr && *(volatile const int*)abort_flag) return;
  const int row = blockIdx.x;
  const int t = threadIdx.x;
  if (t < 32) {
    float mx = -INFINITY;
    for (int s = t; s < num_splits; s += 32) mx = fmaxf(mx, __ldcg(part_lse + static_cast<size_t>(s) * rows + row));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    for (int s = t; s < num_splits; s += 32) {
      const float l = __ldcg(part_lse + static_cast<size_t>(s) * rows + row);
      w[s] = (l == -INFINITY) ? 0.f : exp2f(l - mx);
    }
    __syncwarp();
    if (t == 0) {
      float wsum = 0.f;
      for (int s = 0; s < num_splits; ++s) wsum += w[s];  // fixed order
      s_inv = wsum > 0.f ? 1.f / wsum : 0.f;
    }
  }
  __syncthreads();
  const float* po = part_o + static_cast<size_t>(row) * HD + t;
  const size_t split_stride = static_cast<size_t>(rows) * HD;
  float acc = 0.f;
  int s = 0;
  for (; s + 8 <= num_splits; s += 8) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldcg(po + (s + i) * split_stride);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += w[s + i] * v[i];
  }
  for (; s < num_splits; ++s) acc += w[s] * __ldcg(po + s * split_stride);
  out[static_cast<size_t>(row) * HD + t] = __float2bfloat16_rn(acc * s_inv);
}

}  // namespace cake_dev
