// Persistent warp-specialised stream-K tcgen05 GEMM for the chunk projections.
//
//   C[M, N] = A[M, K] · B[N, K]^T     (both operands K-major bf16, fp32 accumulate in TMEM)
//
// A is the chunk's activations (M = chunk tokens), B a weight matrix stored
// [out_features, in_features]. The work is the list of (tile, k-block) units,
// tiles ordered m-fastest so CTAs that share a weight tile run together and
// the weight is read from HBM once per chunk. Each of the grid's CTAs (one
// per SM) takes an equal, contiguous run of units ("stream-K"): with M = 512
// the per-projection tile counts (96 / 128 / 448) are not multiples of 148,
// and whole-tile scheduling leaves up to a third of the SMs idle in the last
// wave. A tile split across CTAs is reduced deterministically: a CTA's first
// segment, if it starts inside a tile, is a partial (written to that CTA's
// fp32 workspace slot, then flagged); the CTA that holds the tile's k = 0
// segment (processed last by it) waits for those flags and adds the partials
// in k order before the fused epilogue.
//
// Clusters: the cs (<= 4) m-blocks of a chunk (M <= 512) form one thread-
// block cluster that walks the (n-block, k-block) units in lockstep. Each CTA
// TMA-loads 1/cs of the weight k-block and multicasts it to the whole
// cluster, and each CTA's MMA completion is multicast to every CTA's
// empty barrier, so a weight byte leaves HBM once and crosses L2->SM once
// per cluster (not once per m-block). Stream-K then splits the unit list
// across clusters (partials/owners per CTA as below).
//
// Roles (192 threads):
//   warp 0      TMA producer: A/B k-blocks into a kStages smem ring (SW128)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld -> (+partials) -> fused op -> global
// Accumulators are double-buffered in TMEM so segment s's epilogue overlaps
// segment s+1's MMAs.
//
// Fused epilogues (the ops that follow each projection in a Llama block):
//   kEpiBf16    plain bf16 store (tests / generic)
//   kEpiF32     fp32 store (tensor-parallel partial sums)
//   kEpiResid   h[m, n] += acc (fp32 residual stream; O-proj and down-proj)
//   kEpiSwiglu  out[m, j] = silu(gate) * up, gate/up interleaved per 128 cols
//   kEpiQkv     RoPE on q/k, q -> Q buffer, k/v -> paged KV cache
#pragma once

#include "ptx.cuh"

#ifndef GEMM_ISSUE_LANE0
#define GEMM_ISSUE_LANE0 1  // 1-SM kernel: single-lane issuer measured faster (O 21.0 vs 23.8 us)
#endif

namespace cake_dev {

enum GemmEpi : int { kEpiBf16 = 0, kEpiF32 = 1, kEpiResid = 2, kEpiSwiglu = 3, kEpiQkv = 4 };

struct GemmArgs {
  int M, N, K;
  int num_m_blocks, num_n_blocks, num_k_blocks;
  // plain epilogues
  void* out;  // bf16 or f32
  int ldo;
  float* resid;
  int ldr;
  // QKV epilogue
  __nv_bfloat16* q_out;     // [M, n_q * hd]
  __nv_bfloat16* kv_pool;   // [phys_page][layer][2][n_kv][page_tokens][hd]
  const int* block_table;   // logical page -> physical page
  const float2* rope;       // [pos][hd/2] (cos, sin)
  long long pos0;           // absolute position of row 0
  int n_q_heads, n_kv_heads, head_dim, page_tokens, layer, n_layers;
  const int* abort_flag;    // optional: non-zero => skip (lost race / cancelled chunk)
  // stream-K
  float* sk_ws;             // [gridDim.x][128][BLOCK_N] partial tiles
  int* sk_flags;            // [gridDim.x] = epoch when the CTA's partial is published
  int epoch;
  int whole_tiles;          // 1: classic persistent schedule (tile t -> CTA t % grid), no splits;
                            // 2: the same for the full rounds; the short last round is split along K,
                            //    its parts land in tail_ws and a separate kernel sums them + epilogue
  float* tail_ws;           // [tail tile][part][256 rows][256 cols] fp32 (whole_tiles == 2)
  int cs;                   // cluster size = CTAs sharing (multicasting) each weight k-block, one m-block each
  // RMSNorm folded into the projections. Producer side (kEpiResid): besides
  // h += acc, write bf16(h) (the next projection's A operand) and this tile's
  // per-row partial sum of squares. Consumer side (any other epilogue): the
  // row scale rsqrt(sum(partials) / rms_dim + eps) multiplies the accumulator
  // (norm(x) W^T = rsqrt(ms(x)) * (x W^T) row-wise; gamma = 1 in this model).
  __nv_bfloat16* xb_out;    // producer: [M, N] bf16 copy of the updated residual (nullptr: off)
  float* ss_out;            // producer: [num_n_blocks][ss_ld] partial sums of squares
  const float* ss_in;       // consumer: partials to reduce (nullptr: A is already normalised)
  int ss_parts, ss_ld, rms_dim;
  float rms_eps;
  int l2_hints;             // experiment: bit 0 A evict_last, bit 1 B evict_last (else evict_normal)
  long long* trace;         // debug (cake_gemm_debug_trace): %globaltimer stamps of the first and last CTA
  int staged;               // gemm2c kEpiResid: stage h / bf16(h) in shared memory, TMA-store them (1 tile per CTA)
  int prefetch;             // gemm2c: weight k-blocks requested before the PDL wait (-1: the whole ring)
};

__device__ __forceinline__ long long globaltimer_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Stamp slot i of the launch's trace (first CTA: slots 0..15, last CTA: 16..31).
__device__ __forceinline__ void gemm_stamp(const GemmArgs& a, int i) {
  if (a.trace == nullptr) return;
  if (blockIdx.x == 0) a.trace[i] = globaltimer_ns();
  else if (blockIdx.x == gridDim.x - 1) a.trace[16 + i] = globaltimer_ns();
}

__device__ __forceinline__ uint64_t gemm_policy(int hints, int bit) {
  return (hints >> bit) & 1 ? policy_evict_last() : policy_evict_normal();
}

constexpr int kGemmBlockM = 128;
constexpr int kGemmBlockK = 64;  // 64 bf16 = one 128-B swizzle row
constexpr int kGemmThreads = 192;

template <int BLOCK_N>
struct GemmCfg {
  static constexpr int kABytes = kGemmBlockM * kGemmBlockK * 2;
  static constexpr int kBBytes = BLOCK_N * kGemmBlockK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (200 * 1024) / kStageBytes;
  static constexpr int kTmemCols = (2 * BLOCK_N <= 256) ? 256 : 512;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + __expf(-x)); }

// Contiguous unit range of one CTA and its walk over (tile, [kb0, kb1)) segments.
// Mode 2 (tail split): whole tiles round-robin while every CTA gets one; each
// of the r < grid leftover tiles is then cut along K into S = tail_parts(r, g)
// parts on CTAs [t*S, t*S+S). The kernel ends after floor(tiles/grid) whole
// tiles plus 1/S of one, instead of one more whole round (gate/up at M = 512:
// 224 tiles on 74 pairs = 3 rounds + 2 tiles).
constexpr int kTailSplit = 8;
__host__ __device__ inline int tail_parts(int r, int g) { return r > 0 ? (g / r < kTailSplit ? g / r : kTailSplit) : 1; }
struct StreamK {
  long long total, u, u_end;
  int nk, grid;
  int tile_mode = 0, next_tile = 0, n_tiles = 0;
  int n_full = 0, tail_s = 1, cta_id = 0;
  bool tail_done = false;
  __device__ StreamK(long long units, int num_k, int cta, int g, int whole_tiles = 0)
      : total(units), nk(num_k), grid(g), cta_id(cta) {
    u = units * cta / g;
    u_end = units * (cta + 1) / g;
    if (whole_tiles) {
      tile_mode = whole_tiles;
      next_tile = cta;
      n_tiles = static_cast<int>(units / num_k);
      n_full = whole_tiles == 2 ? n_tiles / g * g : n_tiles;
      tail_s = tail_parts(n_tiles - n_full, g);
    }
  }
  // CTA that owns unit v under the balanced split
  __device__ int cta_of(long long v) const { return static_cast<int>(((v + 1) * grid + total - 1) / total - 1); }
  __device__ bool next(int& tile, int& kb0, int& kb1) {
    if (tile_mode) {
      if (next_tile < n_full) {
        tile = next_tile;
        next_tile += grid;
        kb0 = 0;
        kb1 = nk;
        return true;
      }
      if (tile_mode == 2 && !tail_done) {
        tail_done = true;
        const int r = n_tiles - n_full;
        if (cta_id < r * tail_s) {
          const int part = cta_id % tail_s;
          tile = n_full + cta_id / tail_s;
          kb0 = nk * part / tail_s;
          kb1 = nk * (part + 1) / tail_s;
          return true;
        }
      }
      return false;
    }
    if (u >= u_end) return false;
    tile = static_cast<int>(u / nk);
    kb0 = static_cast<int>(u - static_cast<long long>(tile) * nk);
    const long long rest = u_end - u;
    kb1 = static_cast<int>(rest < static_cast<long long>(nk - kb0) ? kb0 + rest : nk);
    u += kb1 - kb0;
    return true;
  }
};

// Epilogue inputs that do not depend on the accumulator, loaded by the
// epilogue warps BEFORE they wait for it (they are idle during the tile's
// mainloop, and at M = 512 most CTAs own a single tile, so anything loaded
// after the wait is exposed): the residual rows this thread will update
// (kEpiResid, <= 128 columns: 128 registers) and the fused-RMSNorm row scale.
template <int BLOCK_N, int EPI>
struct EpiPre {
  static constexpr bool kH = (EPI == kEpiResid) && BLOCK_N <= 128;
  // QKV: the row's RoPE (cos, sin) pairs for both rope units of a head (hd 128: j = 0, 1;
  // hd 64: j = 0) and the physical page of its position — loaded while the mainloop runs, so
  // the epilogue after the accumulator is ready does no dependent global loads
  static constexpr bool kQ = EPI == kEpiQkv;
  float4 h[kH ? BLOCK_N / 4 : 1];
  float4 cs[kQ ? 2 : 1][kQ ? 16 : 1];
  long long phys = 0;
  float rs = 1.f;
  __device__ __forceinline__ void load(const GemmArgs& a, int m, int n_blk, bool partial) {
    if (partial || m >= a.M) return;
    if (a.ss_in != nullptr) {
      float t = 0.f;
      for (int p = 0; p < a.ss_parts; ++p) t += __ldcg(a.ss_in + static_cast<size_t>(p) * a.ss_ld + m);
      rs = rsqrtf(t / static_cast<float>(a.rms_dim) + a.rms_eps);
    }
    if constexpr (kH) {
      const float4* src = reinterpret_cast<const float4*>(a.resid + static_cast<size_t>(m) * a.ldr + n_blk * BLOCK_N);
#pragma unroll
      for (int q = 0; q < BLOCK_N / 4; ++q) h[q] = src[q];
    }
    if constexpr (kQ) {
      const long long pos = a.pos0 + m;
      const int half = a.head_dim >> 1;
      const float4* c0 = reinterpret_cast<const float4*>(a.rope + pos * half);
#pragma unroll
      for (int i = 0; i < 16; ++i) cs[0][i] = __ldg(c0 + i);
      if (a.head_dim >= 128) {
#pragma unroll
        for (int i = 0; i < 16; ++i) cs[1][i] = __ldg(c0 + 16 + i);
      }
      if (a.n_kv_heads > 0) phys = a.block_table[pos / a.page_tokens];
    }
  }
};

// Fused epilogue of one accumulator tile: this thread owns TMEM lane `row`
// (output row m). partial: publish the fp32 tile into workspace slot my_slot
// and raise its flag; otherwise wait for n_parts partial slots (first_slot +
// p * slot_stride, k order), add them, and apply the fused op.
template <int BLOCK_N, int EPI>
__device__ __forceinline__ void gemm_epilogue(const GemmArgs& args, uint32_t tbase, int row, int m, int n_blk,
                                              bool partial, int my_slot, int first_slot, int n_parts,
                                              int slot_stride, int ep_tid, const EpiPre<BLOCK_N, EPI>& pre) {
  const bool valid = m < args.M;
  if (partial) {
    // ---- partial segment: publish the fp32 tile in this CTA's slot
    // column-major slot [BLOCK_N][128]: for each column the warp's 32 rows are
    // one coalesced 128-B line
    float* slot = args.sk_ws + static_cast<size_t>(my_slot) * kGemmBlockM * BLOCK_N + row;
#pragma unroll 1
    for (int c = 0; c < BLOCK_N / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(tbase + c * 32, r);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) __stcg(slot + (c * 32 + i) * kGemmBlockM, __uint_as_float(r[i]));
    }
    __threadfence();
    named_bar_sync(1, 128);
    if (ep_tid == 0) atomicExch(args.sk_flags + my_slot, args.epoch);
  } else {
    // ---- full tile, or the k = 0 owner of a split tile: wait for the other parts
    const float rs = pre.rs;  // fused RMSNorm row scale (consumer side)
    if (n_parts > 0) {
      if (ep_tid == 0) {
        for (int p = 0; p < n_parts; ++p)
          while (*(volatile int*)(args.sk_flags + first_slot + p * slot_stride) != args.epoch) __nanosleep(64);
        __threadfence();
      }
      named_bar_sync(1, 128);
    }
    // accumulator chunk c (32 columns) of this thread's row, partials added in k order
    auto load_acc = [&](int col, uint32_t (&r)[32]) {
      tmem_ld32(tbase + col, r);
      tmem_ld_wait();
      for (int p = 0; p < n_parts; ++p) {
        const float* part = args.sk_ws + static_cast<size_t>(first_slot + p * slot_stride) * kGemmBlockM * BLOCK_N +
                            static_cast<size_t>(col) * kGemmBlockM + row;
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) + __ldcg(part + i * kGemmBlockM));
      }
      if (args.ss_in != nullptr) {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * rs);
      }
    };

    if constexpr (EPI == kEpiBf16 || EPI == kEpiF32 || EPI == kEpiResid) {
      float ss = 0.f;  // kEpiResid: this row's sum of squares over the tile's columns
#pragma unroll
      for (int c = 0; c < BLOCK_N / 32; ++c) {
        uint32_t r[32];
        load_acc(c * 32, r);
        const int n0 = n_blk * BLOCK_N + c * 32;
        if (valid && n0 < args.N) {
          if constexpr (EPI == kEpiBf16) {
            __nv_bfloat16* dst =
                reinterpret_cast<__nv_bfloat16*>(args.out) + static_cast<size_t>(m) * args.ldo + n0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              st_global_v4(dst + q * 8,
                           pack_bf16(__uint_as_float(r[q * 8 + 0]), __uint_as_float(r[q * 8 + 1])),
                           pack_bf16(__uint_as_float(r[q * 8 + 2]), __uint_as_float(r[q * 8 + 3])),
                           pack_bf16(__uint_as_float(r[q * 8 + 4]), __uint_as_float(r[q * 8 + 5])),
                           pack_bf16(__uint_as_float(r[q * 8 + 6]), __uint_as_float(r[q * 8 + 7])));
            }
          } else if constexpr (EPI == kEpiF32) {
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(args.out) +
                                                    static_cast<size_t>(m) * args.ldo + n0);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              dst[q] = make_float4(__uint_as_float(r[q * 4]), __uint_as_float(r[q * 4 + 1]),
                                   __uint_as_float(r[q * 4 + 2]), __uint_as_float(r[q * 4 + 3]));
          } else {
            float4* dst =
                reinterpret_cast<float4*>(args.resid + static_cast<size_t>(m) * args.ldr + n0);
            float4 hv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if constexpr (EpiPre<BLOCK_N, EPI>::kH)
                hv[q] = pre.h[c * 8 + q];
              else
                hv[q] = dst[q];
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float4 h = hv[q];
              h.x += __uint_as_float(r[q * 4]);
              h.y += __uint_as_float(r[q * 4 + 1]);
              h.z += __uint_as_float(r[q * 4 + 2]);
              h.w += __uint_as_float(r[q * 4 + 3]);
              dst[q] = h;
              hv[q] = h;
              ss += h.x * h.x + h.y * h.y + h.z * h.z + h.w * h.w;
            }
            if (args.xb_out != nullptr) {
              __nv_bfloat16* xb = args.xb_out + static_cast<size_t>(m) * args.ldr + n0;
#pragma unroll
              for (int q = 0; q < 4; ++q)
                st_global_v4(xb + q * 8, pack_bf16(hv[2 * q].x, hv[2 * q].y), pack_bf16(hv[2 * q].z, hv[2 * q].w),
                             pack_bf16(hv[2 * q + 1].x, hv[2 * q + 1].y),
                             pack_bf16(hv[2 * q + 1].z, hv[2 * q + 1].w));
            }
          }
        }
      }
      if constexpr (EPI == kEpiResid) {
        if (args.ss_out != nullptr && valid) args.ss_out[static_cast<size_t>(n_blk) * args.ss_ld + m] = ss;
      }
    } else if constexpr (EPI == kEpiSwiglu) {
      static_assert(BLOCK_N == 256, "gate/up interleave is 128 columns");
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t g[32], u[32];
        load_acc(c * 32, g);
        load_acc(128 + c * 32, u);
        if (valid) {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.out) +
                               static_cast<size_t>(m) * args.ldo + n_blk * 128 + c * 32;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i = q * 8 + e * 2;
              float a0 = silu_f(__uint_as_float(g[i])) * __uint_as_float(u[i]);
              float a1 = silu_f(__uint_as_float(g[i + 1])) * __uint_as_float(u[i + 1]);
              w[e] = pack_bf16(a0, a1);
            }
            st_global_v4(dst + q * 8, w[0], w[1], w[2], w[3]);
          }
        }
      }
    } else if constexpr (EPI == kEpiQkv) {
      // rows of the QKV weight are in rope-unit order (qkv_row_of): tile column
      // block [64u, 64u + 64) holds a head's canonical columns [32j, 32j + 32) and
      // their rotation partners [hd/2 + 32j, ...), with j = unit % (hd / 64)
      static_assert(BLOCK_N % 64 == 0, "QKV tiles hold whole rope units");
      const int hd = args.head_dim;
      const int half = hd >> 1;
      const int units_per_head = hd >> 6;
      const long long pos = args.pos0 + m;
#pragma unroll
      for (int k = 0; k < BLOCK_N / 64; ++k) {
        const int unit = n_blk * (BLOCK_N / 64) + k;
        const int head = unit / units_per_head;
        const int j = unit % units_per_head;
        const int region =
            head < args.n_q_heads ? 0 : (head < args.n_q_heads + args.n_kv_heads ? 1 : 2);
        {
          uint32_t x0[32], x1[32];
          load_acc(k * 64, x0);
          load_acc(k * 64 + 32, x1);
          if (!valid) continue;
          float o0[32], o1[32];
          if (region < 2) {
            // (cos, sin) of dims i, i+1 (loaded with the epilogue inputs during the mainloop)
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float4 t = j == 0 ? pre.cs[0][i / 2] : pre.cs[1][i / 2];
              const float a0 = __uint_as_float(x0[i]), b0 = __uint_as_float(x1[i]);
              const float a1 = __uint_as_float(x0[i + 1]), b1 = __uint_as_float(x1[i + 1]);
              o0[i] = a0 * t.x - b0 * t.y;
              o1[i] = b0 * t.x + a0 * t.y;
              o0[i + 1] = a1 * t.z - b1 * t.w;
              o1[i + 1] = b1 * t.z + a1 * t.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              o0[i] = __uint_as_float(x0[i]);
              o1[i] = __uint_as_float(x1[i]);
            }
          }
          __nv_bfloat16* dst;
          if (region == 0) {
            dst = args.q_out + static_cast<size_t>(m) * (args.n_q_heads * hd) + head * hd;
          } else {
            const int kvh = region == 1 ? head - args.n_q_heads : head - args.n_q_heads - args.n_kv_heads;
            const long long lpage = pos / args.page_tokens;
            const int slot = static_cast<int>(pos - lpage * args.page_tokens);
            const long long phys = pre.phys;
            const size_t off =
                ((((static_cast<size_t>(phys) * args.n_layers + args.layer) * 2 + (region - 1)) *
                      args.n_kv_heads + kvh) * args.page_tokens + slot) * static_cast<size_t>(hd);
            dst = args.kv_pool + off;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            st_global_v4(dst + j * 32 + q * 8, pack_bf16(o0[q * 8 + 0], o0[q * 8 + 1]),
                         pack_bf16(o0[q * 8 + 2], o0[q * 8 + 3]), pack_bf16(o0[q * 8 + 4], o0[q * 8 + 5]),
                         pack_bf16(o0[q * 8 + 6], o0[q * 8 + 7]));
            st_global_v4(dst + half + j * 32 + q * 8, pack_bf16(o1[q * 8 + 0], o1[q * 8 + 1]),
                         pack_bf16(o1[q * 8 + 2], o1[q * 8 + 3]), pack_bf16(o1[q * 8 + 4], o1[q * 8 + 5]),
                         pack_bf16(o1[q * 8 + 6], o1[q * 8 + 7]));
          }
        }
      }
    }
  }
}

template <int BLOCK_N, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_b, const GemmArgs args) {
  using Cfg = GemmCfg<BLOCK_N>;
  constexpr int kStages = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];

  __shared__ int s_abort;
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t pad = ((raw_base + 1023u) & ~1023u) - raw_base;
  uint8_t* smem = smem_raw + pad;
  uint8_t* smem_a = smem;                                   // [stages][A]
  uint8_t* smem_b = smem + kStages * Cfg::kABytes;          // [stages][B]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], args.cs);  // every CTA of the cluster must release the stage
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  // (PDL) everything above overlaps the predecessor's tail; its outputs are read below
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) s_abort = (args.abort_flag != nullptr) ? *(volatile const int*)args.abort_flag : 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (args.cs > 1) {
    // one abort decision per cluster (rank 0's): a lone CTA leaving would strand its peers' multicasts
    cluster_sync();
    const int ab = ld_shared_cluster_s32(mapa_shared(smem_u32(&s_abort), 0));
    __syncthreads();
    if (ab) {
      cluster_sync();
      if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(tmem_base);
      return;
    }
  } else if (s_abort) {
    if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(tmem_base);
    return;
  }

  const int nk = args.num_k_blocks;
  const int cs = args.cs;
  const int rank = cs > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const int cluster = blockIdx.x / cs;
  const int n_clusters = gridDim.x / cs;
  const uint16_t mc_mask = static_cast<uint16_t>((1u << cs) - 1u);
  // unit space: (tile, k) with tile = n-block x (m-group of cs m-blocks); this CTA takes m-block rank
  const int m_groups = (args.num_m_blocks + cs - 1) / cs;
  const long long units = static_cast<long long>(m_groups) * args.num_n_blocks * nk;
  int tile, kb0, kb1;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      const uint64_t pol_w = gemm_policy(args.l2_hints, 1);  // weights: reused by the other m-blocks
      const uint64_t pol_a = gemm_policy(args.l2_hints, 0);
      StreamK sk(units, nk, cluster, n_clusters, args.whole_tiles);
      int stage = 0;
      uint32_t phase = 0;
      const int b_rows = BLOCK_N / cs;  // this CTA's share of the weight k-block
      while (sk.next(tile, kb0, kb1)) {
        const int m_blk = (tile % m_groups) * cs + rank;
        const int n_blk = tile / m_groups;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1u);
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          tma_load_2d_hint(smem_a + stage * Cfg::kABytes, &tmap_a, &full_bar[stage], kb * kGemmBlockK,
                           m_blk * kGemmBlockM, pol_a);
          if (cs > 1)
            tma_load_2d_mc(smem_b + stage * Cfg::kBBytes + rank * b_rows * 128, &tmap_b, &full_bar[stage],
                           kb * kGemmBlockK, n_blk * BLOCK_N + rank * b_rows, mc_mask, pol_w);
          else
            tma_load_2d_hint(smem_b + stage * Cfg::kBBytes, &tmap_b, &full_bar[stage], kb * kGemmBlockK,
                             n_blk * BLOCK_N, pol_w);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (!GEMM_ISSUE_LANE0 || lane == 0) {
      // ------------------------------------------------ MMA issuer
      // GEMM_ISSUE_LANE0 = 1 (default): lane 0 alone runs the schedule and
      // issues. 0: the whole warp waits and an elected lane issues. A/B on the
      // box: O 21.0 vs 23.8 us, down 59.1 vs 63.8 us, so lane 0 it is.
      constexpr uint32_t idesc = umma_idesc_bf16(kGemmBlockM, BLOCK_N);
      StreamK sk(units, nk, cluster, n_clusters, args.whole_tiles);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      while (sk.next(tile, kb0, kb1)) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BLOCK_N);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem_a + stage * Cfg::kABytes);
          const uint32_t b_addr = smem_u32(smem_b + stage * Cfg::kBBytes);
          if (GEMM_ISSUE_LANE0 ? lane == 0 : elect_one()) {
#pragma unroll
            for (int k = 0; k < kGemmBlockK / 16; ++k) {
              umma_bf16_ss(d_tmem, umma_desc_sw128(a_addr + k * 32), umma_desc_sw128(b_addr + k * 32),
                           idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            }
            if (cs > 1)
              umma_commit_mc(&empty_bar[stage], mc_mask);
            else
              umma_commit(&empty_bar[stage]);
          }
          if (!GEMM_ISSUE_LANE0) __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (GEMM_ISSUE_LANE0 ? lane == 0 : elect_one()) umma_commit(&tfull_bar[acc]);
        if (!GEMM_ISSUE_LANE0) __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..5)
    const int ew = warp & 3;  // TMEM lane quarter this warp may access
    const int row = ew * 32 + static_cast<int>(lane);
    const int ep_tid = threadIdx.x - 64;  // 0..127
    StreamK sk(units, nk, cluster, n_clusters, args.whole_tiles);
    int acc = 0;
    uint32_t acc_phase = 0;
    while (sk.next(tile, kb0, kb1)) {
      const int m_blk = (tile % m_groups) * cs + rank;
      const int n_blk = tile / m_groups;
      const int m = m_blk * kGemmBlockM + row;
      EpiPre<BLOCK_N, EPI> pre;
      pre.load(args, m, n_blk, kb0 > 0);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase =
          tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * BLOCK_N);

      {
        const bool partial = kb0 > 0;
        int first_part = 0, n_parts = 0;
        if (!partial && kb1 < nk) {
          const long long u_tile = static_cast<long long>(tile) * nk;
          first_part = sk.cta_of(u_tile) + 1;
          n_parts = sk.cta_of(u_tile + nk - 1) - first_part + 1;
        }
        gemm_epilogue<BLOCK_N, EPI>(args, tbase, row, m, n_blk, partial, blockIdx.x, first_part * cs + rank, n_parts,
                                    cs, ep_tid, pre);
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  }

  __syncthreads();
  if (cs > 1) cluster_sync();  // no peer may still multicast into this CTA's smem / barriers
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

}  // namespace cake_dev
