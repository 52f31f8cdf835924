// Prefix-causal attention, one 128-row Q tile per CTA, with the two softmax
// groups DECOUPLED (impl 4; cake_model_set_attention_impl).
//
// The one-tile kernel (attention_tc.cuh) splits each 128-key block between two
// softmax warpgroups by columns and exchanges the row max through shared
// memory every block (a named barrier), so the two warps on each SM
// sub-partition run the same phase at the same time: both on MUFU, then both on
// the FMA pipe. Here each group keeps its own running max m_g, row sum l_g and
// its own O accumulator in TMEM:
//   S(j)    = Q K(j)^T       Q in shared memory (SS MMA), S double-buffered (cols 0/128)
//   P_g(j)  = exp2(S_g*scale - m_g)   group g: keys [64g, 64g+64) of the block
//   O_g    += P_g(j) V_g(j)  O_0 at cols 256..383, O_1 at 384..511
// No per-block barrier between the groups; the MMA warp issues PV_g as soon as
// group g's P is in TMEM. The epilogue merges O_0 and O_1 once (the same LSE
// merge as split-KV, fixed order, deterministic).
// TMEM is full (S0, S1, O_0, O_1), so Q moves to shared memory (written by the
// softmax threads in the SW128 K-major layout), and V keeps two stages.
#pragma once

#include "attention_tc.cuh"

namespace cake_dev {

// DEC_SPLIT_S = 1 measured slower (block period 1973 vs 1621 cycles at 32K):
// with Q in shared memory an N = 64 SS MMA reads 6 KB per 32 cycles, above the
// 128 B/clk shared-memory port, and the split serialises the groups' S.
#ifndef DEC_SPLIT_S
#define DEC_SPLIT_S 0
#endif

template <int HD>
struct FdCfg {
  static constexpr int kHalves = HD / 64;
  static constexpr int kTileBytes = kFaRows * HD * 2;
  static constexpr int kHalfBytes = kFaRows * 128;
  static constexpr int kPageHalfBytes = 64 * 128;
  static constexpr int kKStages = 3;
  static constexpr int kVStages = 2;
  static constexpr int kSmem = (1 + kKStages + kVStages) * kTileBytes + 1024 + 256;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO = 256;  // O_g at kColO + 128 g
};

template <int HD>
__global__ void __launch_bounds__(fa_threads<2>(), 1)
    attn_dec_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                    const FaArgs a) {
  using Cfg = FdCfg<HD>;
  constexpr int NG = 2;
  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_abort;

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  const int kvh = blockIdx.y;
  const int split = blockIdx.z;
  const int G = a.n_q_heads / a.n_kv_heads;
  const int tok_per_tile = kFaRows / G;
  const int tok0 = blockIdx.x * tok_per_tile;
  const int tok_last = min(tok0 + tok_per_tile, a.chunk_len) - 1;
  const long long kv_end = a.chunk_start + tok_last + 1;
  const int n_pages = static_cast<int>((kv_end + kAttnPage - 1) / kAttnPage);
  const int per_split = (n_pages + a.num_splits - 1) / a.num_splits;
  const int p_begin = split * per_split;
  const int p_end = min(n_pages, p_begin + per_split);
  const int nb = p_end > p_begin ? (p_end - p_begin + 1) / 2 : 0;  // 128-key blocks

  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sQ = smem;                                       // [tile], SW128 K-major
  uint8_t* sK = sQ + Cfg::kTileBytes;                       // [kKStages][tile]
  uint8_t* sV = sK + Cfg::kKStages * Cfg::kTileBytes;      // [kVStages][tile]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + Cfg::kVStages * Cfg::kTileBytes);
  uint64_t* q_ready = bar;        // Q rows stored by the softmax threads
  uint64_t* k_full = bar + 1;     // [3]
  uint64_t* k_empty = bar + 4;    // [3]
  uint64_t* v_full = bar + 7;     // [2]
  uint64_t* v_empty = bar + 9;    // [2]
  uint64_t* s_full = bar + 11;    // [2 buffers][2 groups]
  uint64_t* p_ready = bar + 15;   // [2 buffers][2 groups]
  uint64_t* pv_done = bar + 19;   // [2 groups]
  uint64_t* o_final = bar + 21;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 22);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_kv);
    mbar_init(q_ready, 128 * NG);
    for (int s = 0; s < Cfg::kKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < Cfg::kVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&s_full[i], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&p_ready[i], 128);
    mbar_init(&pv_done[0], 1);
    mbar_init(&pv_done[1], 1);
    mbar_init(o_final, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) s_abort = a.abort_flag != nullptr ? *(volatile const int*)a.abort_flag : 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (s_abort || tok0 >= a.chunk_len) {
    if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(tmem);
    return;
  }

  const long long planes = static_cast<long long>(a.n_layers) * 2 * a.n_kv_heads;
  auto page_row = [&](int lp, int kv) -> int32_t {
    const long long ph = a.block_table[lp];
    return static_cast<int32_t>(((ph * planes) + (static_cast<long long>(a.layer) * 2 + kv) * a.n_kv_heads + kvh) * 64);
  };
  if (warp == 0) {
    if (lane == 0 && nb > 0) {
      // ------------------------------------------------ TMA producer: K blocks
      for (int j = 0; j < nb; ++j) {
        const int s = j % Cfg::kKStages;
        mbar_wait(&k_empty[s], ((j / Cfg::kKStages) & 1) ^ 1u);
        const int lp0 = p_begin + 2 * j;
        const int lp1 = (lp0 + 1 < p_end) ? lp0 + 1 : lp0;  // odd tail: reload page 0 (its keys are masked)
        const int32_t r0 = page_row(lp0, 0), r1 = page_row(lp1, 0);
        mbar_arrive_expect_tx(&k_full[s], Cfg::kTileBytes);
#pragma unroll
        for (int h = 0; h < Cfg::kHalves; ++h) {
          tma_load_2d(sK + s * Cfg::kTileBytes + h * Cfg::kHalfBytes, &tm_kv, &k_full[s], h * 64, r0);
          tma_load_2d(sK + s * Cfg::kTileBytes + h * Cfg::kHalfBytes + Cfg::kPageHalfBytes, &tm_kv, &k_full[s],
                      h * 64, r1);
        }
      }
    }
  } else if (warp == 2) {
    if (lane == 0 && nb > 0) {
      // ------------------------------------------------ TMA producer: V blocks
      for (int j = 0; j < nb; ++j) {
        const int s = j % Cfg::kVStages;
        mbar_wait(&v_empty[s], ((j / Cfg::kVStages) & 1) ^ 1u);
        const int lp0 = p_begin + 2 * j;
        const int lp1 = (lp0 + 1 < p_end) ? lp0 + 1 : lp0;
        const int32_t r0 = page_row(lp0, 1), r1 = page_row(lp1, 1);
        mbar_arrive_expect_tx(&v_full[s], Cfg::kTileBytes);
#pragma unroll
        for (int h = 0; h < Cfg::kHalves; ++h) {
          tma_load_2d(sV + s * Cfg::kTileBytes + h * Cfg::kHalfBytes, &tm_kv, &v_full[s], h * 64, r0);
          tma_load_2d(sV + s * Cfg::kTileBytes + h * Cfg::kHalfBytes + Cfg::kPageHalfBytes, &tm_kv, &v_full[s],
                      h * 64, r1);
        }
      }
    }
  } else if (warp == 1) {
    if (nb > 0) {
      // ------------------------------------------------ MMA issuer (converged warp, elected lane)
      constexpr uint32_t idesc_s = umma_idesc_bf16(kFaRows, kFaKeys, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(kFaRows, HD, false, true);
      mbar_wait(q_ready, 0);
      tc_fence_after();
      const uint32_t q_addr = smem_u32(sQ);
      const bool trm = a.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0;
      if (trm) a.trace[0] = clock64(), a.trace[1] = nb;
      // DEC_SPLIT_S: S(j) as two N = 64 MMAs, one per group's keys, issued
      // between the PVs so the two groups start their blocks at different times
      // (their phases then overlap on each sub-partition); else one N = 128 MMA.
      constexpr uint32_t idesc_s64 = umma_idesc_bf16(kFaRows, kFaKeys / 2, false, false);
      auto issue_s = [&](int jj, int g) {  // g < 0: both halves as one N = 128 MMA
        const int s = jj & 1;
        const int ks = jj % Cfg::kKStages;
        if (g <= 0) mbar_wait(&k_full[ks], (jj / Cfg::kKStages) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + ks * Cfg::kTileBytes) + (g > 0 ? Cfg::kPageHalfBytes : 0);
        const uint32_t d = tmem + (s ? Cfg::kColS1 : Cfg::kColS0) + (g > 0 ? kFaKeys / 2 : 0);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk >> 2) * Cfg::kHalfBytes + (kk & 3) * 32;
            umma_bf16_ss(d, umma_desc_sw128(q_addr + off), umma_desc_sw128(k_addr + off), g < 0 ? idesc_s : idesc_s64,
                         kk > 0 ? 1u : 0u);
          }
          if (g <= 0) umma_commit(&s_full[s * 2]);
          if (g != 0) umma_commit(&s_full[s * 2 + 1]);
          if (g != 0) umma_commit(&k_empty[ks]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int jj, int g) {
        const int s = jj & 1;
        const int vs = jj % Cfg::kVStages;
        if (trm && jj < 64) a.trace[64 + jj * 8 + 6 + g] = clock64();
        mbar_wait(&p_ready[s * 2 + g], (jj >> 1) & 1);
        if (g == 0) mbar_wait(&v_full[vs], (jj / Cfg::kVStages) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + vs * Cfg::kTileBytes);
        const uint32_t p_col = tmem + (s ? Cfg::kColS1 : Cfg::kColS0) + g * 32;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kFaKeys / 32; ++kk) {
            const uint64_t bdesc = umma_desc_sw128_mn(v_addr + (g * 4 + kk) * 16 * 128, Cfg::kHalfBytes, 1024);
            umma_bf16_ts(tmem + Cfg::kColO + g * 128, p_col + kk * 8, bdesc, idesc_o, (jj > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&pv_done[g]);
          if (g == 1) umma_commit(&v_empty[vs]);
        }
        __syncwarp();
      };
      // S(j+1) before PV(j): the pipe computes the next scores while the groups
      // finish P(j). S(j+1) overwrites P(j-1), whose PVs were issued before it.
      if (DEC_SPLIT_S) {
        issue_s(0, 0);
        issue_s(0, 1);
        for (int j = 0; j < nb; ++j) {
          if (j + 1 < nb) issue_s(j + 1, 0);
          issue_pv(j, 0);
          if (j + 1 < nb) issue_s(j + 1, 1);
          issue_pv(j, 1);
        }
      } else {
        issue_s(0, -1);
        for (int j = 0; j < nb; ++j) {
          if (j + 1 < nb) issue_s(j + 1, -1);
          issue_pv(j, 0);
          issue_pv(j, 1);
        }
      }
      if (elect_one()) umma_commit(o_final);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax + epilogue
    constexpr int kKeysPerG = kFaKeys / NG;  // 64
    constexpr int kOCols = HD / NG;          // output columns this group writes
    __shared__ float xm[NG][kFaRows];
    __shared__ float xl[NG][kFaRows];
    const int g = (warp - 4) >> 2;
    const int q4 = warp & 3;
    const int row = q4 * 32 + static_cast<int>(lane);
    const int t = tok0 + row / G;
    const int head = kvh * G + row % G;
    const long long qpos = a.chunk_start + t;
    const long long kmax_valid = static_cast<long long>(p_end) * kAttnPage;
    const long long qpos_min = a.chunk_start + tok0;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const float sc = a.scale_log2;
    {
      // this thread's Q row, half g (64 bf16 = 8 x 16 B), into the SW128 K-major tile
      static_assert(HD / NG == 64 || HD / NG == 32, "Q slice per group");
      const bool live = t < a.chunk_len && nb > 0;
      const uint4* src = reinterpret_cast<const uint4*>(a.q + (static_cast<size_t>(t) * a.n_q_heads + head) * HD +
                                                        g * (HD / NG));
      if constexpr (HD / NG == 64) {
        uint8_t* dst_row = sQ + g * Cfg::kHalfBytes + row * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 v = live ? __ldg(src + c) : make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(dst_row + ((c ^ (row & 7)) << 4)) = v;
        }
      } else {
        // HD = 64: one 128-B row per Q row; group g holds chunks [4g, 4g+4)
        uint8_t* dst_row = sQ + row * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint4 v = live ? __ldg(src + c) : make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(dst_row + (((g * 4 + c) ^ (row & 7)) << 4)) = v;
        }
      }
      fence_proxy_async();
      mbar_arrive(q_ready);
    }
    float m = -INFINITY, l = 0.f;
    const bool tr = a.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && q4 == 0 &&
                    lane == 0;
    long long* trp = tr ? a.trace + 64 + g * 8 * 64 : nullptr;
    const uint32_t tO = tmem + lane_off + Cfg::kColO + g * 128;
    for (int j = 0; j < nb; ++j) {
      const int s = j & 1;
      if (tr && j < 64) trp[j * 8] = clock64();
      mbar_wait(&s_full[s * 2 + g], (j >> 1) & 1);
      tc_fence_after();
      if (tr && j < 64) trp[j * 8 + 1] = clock64();
      const uint32_t tS = tmem + lane_off + (s ? Cfg::kColS1 : Cfg::kColS0);
      float sv[kKeysPerG];
#pragma unroll
      for (int c = 0; c < kKeysPerG / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tS + g * kKeysPerG + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(r[i]);
      }
      const long long kbase = static_cast<long long>(p_begin + 2 * j) * kAttnPage + g * kKeysPerG;
      if (kbase + kKeysPerG - 1 > qpos_min || kbase + kKeysPerG > kmax_valid) {
#pragma unroll
        for (int i = 0; i < kKeysPerG; ++i) {
          const long long key = kbase + i;
          if (key > qpos || key >= kmax_valid) sv[i] = -INFINITY;
        }
      }
      if (tr && j < 64) trp[j * 8 + 2] = clock64();
      // row max over 8 independent chains (a single chain is kKeysPerG dependent FMNMX)
      float mc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) mc[c] = sv[c];
#pragma unroll
      for (int i = 8; i < kKeysPerG; ++i) mc[i & 7] = fmaxf(mc[i & 7], sv[i]);
      float mx = fmaxf(fmaxf(fmaxf(mc[0], mc[1]), fmaxf(mc[2], mc[3])), fmaxf(fmaxf(mc[4], mc[5]), fmaxf(mc[6], mc[7])));
      mx *= sc;
      if (tr && j < 64) trp[j * 8 + 3] = clock64();
      // tcgen05.ld/st are warp-collective (.sync.aligned): when any row of the warp moves its
      // reference max the whole warp runs the rescale pass (factor 1 for the other rows)
      const bool up = mx > m + 8.0f;  // (also true on the first block with a visible key)
      const bool resc = up && m != -INFINITY;
      if (__any_sync(0xffffffffu, resc)) {
        // move this group's reference max: O_g (blocks < j, i.e. after PV_g(j-1)) and l scale by 2^(m - mx)
        mbar_wait(&pv_done[g], (j - 1) & 1);
        tc_fence_after();
        const float f = resc ? ex2_approx(m - mx) : 1.f;
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
      if (up) m = mx;
      const float nbase = (m == -INFINITY) ? 0.f : -m;
      const float2 sc2 = make_float2(sc, sc), nb2 = make_float2(nbase, nbase);
      float2 rs[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      uint32_t pk[kKeysPerG / 2];
#pragma unroll
      for (int i = 0; i < kKeysPerG / 2; ++i) {
        const float2 x = ffma2(make_float2(sv[2 * i], sv[2 * i + 1]), sc2, nb2);
        float2 p;
        if ((i & 7) >= 8 - FA_POLY) {
          p = ex2_poly2(x);
        } else {
          p.x = ex2_approx(x.x);
          p.y = ex2_approx(x.y);
        }
        rs[i & 3] = fadd2(rs[i & 3], p);
        pk[i] = pack_bf16(p.x, p.y);
      }
      if (tr && j < 64) trp[j * 8 + 4] = clock64();
      tmem_st32(tS + g * 32, pk);
      const float2 rs01 = fadd2(rs[0], rs[1]), rs23 = fadd2(rs[2], rs[3]);
      l += (rs01.x + rs23.x) + (rs01.y + rs23.y);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_ready[s * 2 + g]);
      if (tr && j < 64) trp[j * 8 + 5] = clock64();
    }
    // epilogue: merge (m_0, l_0, O_0) and (m_1, l_1, O_1) per row, fixed order
    xm[g][row] = m;
    xl[g][row] = l;
    named_bar_sync(2, 128 * NG);
    const float m0 = xm[0][row], m1 = xm[1][row];
    const float mt = fmaxf(m0, m1);
    const float f0 = m0 == -INFINITY ? 0.f : ex2_approx(m0 - mt);
    const float f1 = m1 == -INFINITY ? 0.f : ex2_approx(m1 - mt);
    const float lt = xl[0][row] * f0 + xl[1][row] * f1;
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    const bool valid = t < a.chunk_len;
    const size_t orow = static_cast<size_t>(t) * a.n_q_heads + head;
    if (nb > 0) {
      mbar_wait(o_final, 0);
      tc_fence_after();
    }
    const float w0 = f0 * inv, w1 = f1 * inv;
    const uint32_t tO0 = tmem + lane_off + Cfg::kColO, tO1 = tO0 + 128;
#pragma unroll
    for (int c = 0; c < kOCols / 32; ++c) {
      const int col = g * kOCols + c * 32;
      uint32_t r0[32], r1[32];
      if (nb > 0) {
        tmem_ld32(tO0 + col, r0);
        tmem_ld32(tO1 + col, r1);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) r0[i] = r1[i] = 0u;
      }
      if (!valid) continue;
      float o[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(r0[i]) * w0 + __uint_as_float(r1[i]) * w1;
      if (a.num_splits == 1) {
        __nv_bfloat16* dst = a.out + orow * HD + col;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_global_v4(dst + q * 8, pack_bf16(o[q * 8], o[q * 8 + 1]), pack_bf16(o[q * 8 + 2], o[q * 8 + 3]),
                       pack_bf16(o[q * 8 + 4], o[q * 8 + 5]), pack_bf16(o[q * 8 + 6], o[q * 8 + 7]));
      } else {
        const size_t rows = static_cast<size_t>(a.chunk_len) * a.n_q_heads;
        float4* dst = reinterpret_cast<float4*>(a.part_o + (static_cast<size_t>(split) * rows + orow) * HD + col);
#pragma unroll
        for (int q = 0; q < 8; ++q) dst[q] = make_float4(o[q * 4], o[q * 4 + 1], o[q * 4 + 2], o[q * 4 + 3]);
      }
    }
    if (valid && a.num_splits > 1 && g == 0) {
      const size_t rows = static_cast<size_t>(a.chunk_len) * a.n_q_heads;
      a.part_lse[static_cast<size_t>(split) * rows + orow] = lt > 0.f ? mt + __log2f(lt) : -INFINITY;
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
