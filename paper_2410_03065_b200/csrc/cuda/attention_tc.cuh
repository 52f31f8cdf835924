// Prefix-causal attention on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// One CTA = 128 query rows of one KV head (rows are (token, q-head) pairs of
// the GQA group, so K/V pages are fetched once for all heads of the group),
// over the keys of one split of the prefix. Per 128-key block (two 64-token
// KV pages, TMA-loaded straight out of the paged pool through the block
// table):
//   S   = Q K^T      tcgen05.mma, A = Q (smem, K-major SW128), B = K page
//                    (smem, K-major SW128), fp32 accumulator in TMEM;
//                    double-buffered so softmax(j) overlaps QK(j+1)
//   P   = exp2(S*scale - m)  4 softmax warps, thread = row, S read with
//                    tcgen05.ld, P written back over S as packed bf16
//                    (tcgen05.st) — P never touches shared memory
//   O  += P V        tcgen05.mma with A = P from TMEM, B = V page (smem,
//                    MN-major SW128), O accumulator in TMEM
// The running max is only moved (and O rescaled in TMEM) when it grows by
// more than 2^8, so the common block costs no O round trip.
// Roles (256 threads): warp 0 TMA producer, warp 1 TMEM owner + MMA issuer,
// warps 4-7 softmax + epilogue (warp w%4 owns TMEM lanes 32*(w%4)..).
#pragma once

#include "attention.cuh"
#include "ptx.cuh"

namespace cake_dev {

constexpr int kFaRows = 128;
constexpr int kFaKeys = 128;  // two pages
constexpr int kFaThreads = 256;

template <int HD>
struct FaCfg {
  static constexpr int kHalves = HD / 64;                    // 64-element (128 B) K slices
  static constexpr int kTileBytes = kFaRows * HD * 2;        // Q / K / V tile (128 rows)
  static constexpr int kHalfBytes = kFaRows * 128;           // one 64-wide slice of a tile
  static constexpr int kPageHalfBytes = 64 * 128;            // one page x 64 elements
  static constexpr int kSmem = 5 * kTileBytes + 1024 + 256;  // Q + 2 K + 2 V + align + barriers
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO = 256;
};

struct FaArgs {
  const int* block_table;
  __nv_bfloat16* out;     // [C, n_q, hd] (splits == 1)
  float* part_o;          // [splits, C*n_q, hd]
  float* part_lse;        // [splits, C*n_q]
  long long chunk_start;
  int chunk_len;
  int n_q_heads, n_kv_heads, layer, n_layers;
  int num_splits;
  float scale_log2;
  const int* abort_flag;
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int HD>
__global__ void __launch_bounds__(kFaThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                   const FaArgs a) {
  using Cfg = FaCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_abort;
  if (threadIdx.x == 0) s_abort = a.abort_flag != nullptr ? *(volatile const int*)a.abort_flag : 0;
  __syncthreads();
  if (s_abort) return;

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  const int kvh = blockIdx.y;
  const int split = blockIdx.z;
  const int G = a.n_q_heads / a.n_kv_heads;
  const int tok_per_tile = kFaRows / G;
  const int tok0 = blockIdx.x * tok_per_tile;
  if (tok0 >= a.chunk_len) return;
  const int tok_last = min(tok0 + tok_per_tile, a.chunk_len) - 1;
  const long long kv_end = a.chunk_start + tok_last + 1;
  const int n_pages = static_cast<int>((kv_end + kAttnPage - 1) / kAttnPage);
  const int per_split = (n_pages + a.num_splits - 1) / a.num_splits;
  const int p_begin = split * per_split;
  const int p_end = min(n_pages, p_begin + per_split);
  const int nb = p_end > p_begin ? (p_end - p_begin + 1) / 2 : 0;  // 128-key blocks

  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sQ = smem;
  uint8_t* sK = smem + Cfg::kTileBytes;        // [2][tile]
  uint8_t* sV = sK + 2 * Cfg::kTileBytes;      // [2][tile]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + 2 * Cfg::kTileBytes);
  uint64_t* q_full = bar;
  uint64_t* k_full = bar + 1;     // [2]
  uint64_t* v_full = bar + 3;     // [2]
  uint64_t* kv_empty = bar + 5;   // [2]
  uint64_t* s_full = bar + 7;     // [2]
  uint64_t* p_ready = bar + 9;    // [2]
  uint64_t* pv_done = bar + 11;
  uint64_t* o_final = bar + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 13);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kv);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_ready[s], 128);
    }
    mbar_init(pv_done, 1);
    mbar_init(o_final, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && nb > 0) {
      // ------------------------------------------------ TMA producer
      mbar_arrive_expect_tx(q_full, Cfg::kTileBytes);
#pragma unroll
      for (int h = 0; h < Cfg::kHalves; ++h) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(sQ + h * Cfg::kHalfBytes)),
            "l"(reinterpret_cast<uint64_t>(&tm_q)), "r"(smem_u32(q_full)), "r"(h * 64), "r"(kvh * G), "r"(tok0)
            : "memory");
      }
      const long long planes = static_cast<long long>(a.n_layers) * 2 * a.n_kv_heads;
      for (int j = 0; j < nb; ++j) {
        const int s = j & 1;
        mbar_wait(&kv_empty[s], ((j >> 1) & 1) ^ 1u);
        const int lp0 = p_begin + 2 * j;
        const int lp1 = (lp0 + 1 < p_end) ? lp0 + 1 : lp0;  // odd tail: reload page 0 (its keys are masked)
        const long long ph0 = a.block_table[lp0], ph1 = a.block_table[lp1];
        const long long base_k0 = ((ph0 * planes) + (static_cast<long long>(a.layer) * 2 + 0) * a.n_kv_heads + kvh) * 64;
        const long long base_k1 = ((ph1 * planes) + (static_cast<long long>(a.layer) * 2 + 0) * a.n_kv_heads + kvh) * 64;
        const long long vstep = static_cast<long long>(a.n_kv_heads) * 64;  // K plane -> V plane
        mbar_arrive_expect_tx(&k_full[s], Cfg::kTileBytes);
#pragma unroll
        for (int h = 0; h < Cfg::kHalves; ++h) {
          tma_load_2d(sK + s * Cfg::kTileBytes + h * Cfg::kHalfBytes, &tm_kv, &k_full[s], h * 64,
                      static_cast<int32_t>(base_k0));
          tma_load_2d(sK + s * Cfg::kTileBytes + h * Cfg::kHalfBytes + Cfg::kPageHalfBytes, &tm_kv, &k_full[s],
                      h * 64, static_cast<int32_t>(base_k1));
        }
        mbar_arrive_expect_tx(&v_full[s], Cfg::kTileBytes);
#pragma unroll
        for (int h = 0; h < Cfg::kHalves; ++h) {
          tma_load_2d(sV + s * Cfg::kTileBytes + h * Cfg::kHalfBytes, &tm_kv, &v_full[s], h * 64,
                      static_cast<int32_t>(base_k0 + vstep));
          tma_load_2d(sV + s * Cfg::kTileBytes + h * Cfg::kHalfBytes + Cfg::kPageHalfBytes, &tm_kv, &v_full[s],
                      h * 64, static_cast<int32_t>(base_k1 + vstep));
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nb > 0) {
      // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = umma_idesc_bf16(kFaRows, kFaKeys, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(kFaRows, HD, false, true);
      const uint32_t q_addr = smem_u32(sQ);
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int jj) {
        const int s = jj & 1;
        mbar_wait(&p_ready[s], (jj >> 1) & 1);
        mbar_wait(&v_full[s], (jj >> 1) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + s * Cfg::kTileBytes);
        const uint32_t p_col = tmem + (s ? Cfg::kColS1 : Cfg::kColS0);
#pragma unroll
        for (int kk = 0; kk < kFaKeys / 16; ++kk) {
          const uint64_t bdesc = umma_desc_sw128_mn(v_addr + kk * 16 * 128, Cfg::kHalfBytes, 1024);
          umma_bf16_ts(tmem + Cfg::kColO, p_col + kk * 8, bdesc, idesc_o, (jj > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&kv_empty[s]);
        umma_commit(pv_done);
      };
      for (int j = 0; j < nb; ++j) {
        const int s = j & 1;
        mbar_wait(&k_full[s], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + s * Cfg::kTileBytes);
        const uint32_t d = tmem + (s ? Cfg::kColS1 : Cfg::kColS0);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * Cfg::kHalfBytes + (kk & 3) * 32;
          umma_bf16_ss(d, umma_desc_sw128(q_addr + off), umma_desc_sw128(k_addr + off), idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[s]);
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(nb - 1);
      umma_commit(o_final);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax + epilogue
    const int q4 = warp & 3;
    const int row = q4 * 32 + static_cast<int>(lane);
    const int t = tok0 + row / G;
    const int head = kvh * G + row % G;
    const long long qpos = a.chunk_start + t;
    const long long kmax_valid = static_cast<long long>(p_end) * kAttnPage;  // keys past the split are absent
    const long long qpos_min = a.chunk_start + tok0;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nb; ++j) {
      const int s = j & 1;
      mbar_wait(&s_full[s], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t tS = tmem + lane_off + (s ? Cfg::kColS1 : Cfg::kColS0);
      float sv[kFaKeys];
#pragma unroll
      for (int c = 0; c < kFaKeys / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tS + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(r[i]) * a.scale_log2;
      }
      const long long kbase = static_cast<long long>(p_begin + 2 * j) * kAttnPage;
      if (kbase + kFaKeys - 1 > qpos_min || kbase + kFaKeys > kmax_valid) {
#pragma unroll
        for (int i = 0; i < kFaKeys; ++i) {
          const long long key = kbase + i;
          if (key > qpos || key >= kmax_valid) sv[i] = -INFINITY;
        }
      }
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < kFaKeys; ++i) mx = fmaxf(mx, sv[i]);
      if (mx > m + 8.0f) {  // (also true on the first block with a visible key)
        if (m != -INFINITY) {
          // move the reference max: O (all blocks < j, i.e. after PV(j-1)) and l scale by 2^(m - mx)
          mbar_wait(pv_done, (j - 1) & 1);
          tc_fence_after();
          const float f = ex2_approx(m - mx);
          const uint32_t tO = tmem + lane_off + Cfg::kColO;
#pragma unroll
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tO + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
            tmem_st32(tO + c * 32, r);
          }
          tmem_st_wait();
          l *= f;
        }
        m = mx;
      }
      const float base = (m == -INFINITY) ? 0.f : m;
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < kFaKeys / 64; ++c) {
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float p0 = ex2_approx(sv[c * 64 + 2 * i] - base);
          const float p1 = ex2_approx(sv[c * 64 + 2 * i + 1] - base);
          rs += p0 + p1;
          pk[i] = pack_bf16(p0, p1);
        }
        tmem_st32(tS + c * 32, pk);
      }
      l += rs;
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_ready[s]);
    }
    // epilogue
    const bool valid = t < a.chunk_len;
    const size_t orow = static_cast<size_t>(t) * a.n_q_heads + head;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    if (nb > 0) {
      mbar_wait(o_final, 0);
      tc_fence_after();
    }
    const uint32_t tO = tmem + lane_off + Cfg::kColO;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t r[32];
      if (nb > 0) {
        tmem_ld32(tO + c * 32, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = 0u;
      }
      if (!valid) continue;
      if (a.num_splits == 1) {
        __nv_bfloat16* dst = a.out + orow * HD + c * 32;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_global_v4(dst + q * 8, pack_bf16(__uint_as_float(r[q * 8]) * inv, __uint_as_float(r[q * 8 + 1]) * inv),
                       pack_bf16(__uint_as_float(r[q * 8 + 2]) * inv, __uint_as_float(r[q * 8 + 3]) * inv),
                       pack_bf16(__uint_as_float(r[q * 8 + 4]) * inv, __uint_as_float(r[q * 8 + 5]) * inv),
                       pack_bf16(__uint_as_float(r[q * 8 + 6]) * inv, __uint_as_float(r[q * 8 + 7]) * inv));
      } else {
        const size_t rows = static_cast<size_t>(a.chunk_len) * a.n_q_heads;
        float4* dst = reinterpret_cast<float4*>(a.part_o + (static_cast<size_t>(split) * rows + orow) * HD + c * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          dst[q] = make_float4(__uint_as_float(r[q * 4]) * inv, __uint_as_float(r[q * 4 + 1]) * inv,
                               __uint_as_float(r[q * 4 + 2]) * inv, __uint_as_float(r[q * 4 + 3]) * inv);
      }
    }
    if (valid && a.num_splits > 1) {
      const size_t rows = static_cast<size_t>(a.chunk_len) * a.n_q_heads;
      a.part_lse[static_cast<size_t>(split) * rows + orow] = l > 0.f ? m + __log2f(l) : -INFINITY;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem);
  }
}

}  // namespace cake_dev
