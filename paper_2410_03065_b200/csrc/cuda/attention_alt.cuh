// Prefix-causal attention, one 128-row Q tile per CTA, with the two softmax
// warpgroups on ALTERNATE key blocks: the product kernel (cake_cuda.cu
// attention(), impl 0; the column-split one-tile kernel of attention_tc.cuh
// stays as impl 2).
//
// In the one-tile kernel (attention_tc.cuh) both softmax warpgroups work on
// the same 128-key block (column halves) and wait for the same S(j), so the
// two warps of every SM sub-partition run the same phase at the same time and
// the block's softmax (~1.5K cycles) bounds the block against the 1024-cycle
// MMA floor. Here warpgroup g owns blocks j = g, g+2, ... whole (one thread =
// one row, 128 scores), with its own running max, row sum and O accumulator:
//
//   TMEM  S0 [0,128) (even blocks)  S1 [128,256) (odd blocks)  O_0 [256,384)  O_1 [384,512)
//   pipe  S(0) S(1) | PV(0) S(2) | PV(1) S(3) | ...   (S(j+2) into the buffer PV(j) just read)
//
// so a warpgroup has the other group's PV + S (1024 tensor cycles) in which to
// turn its block into P, and the two warps of a sub-partition are half a block
// apart (one on MUFU while the other loads / reduces / stores). Q lives in
// shared memory (TMEM is full), written by the softmax threads; the epilogue
// merges (m_0, l_0, O_0) and (m_1, l_1, O_1) once, in a fixed order.
#pragma once

#include "attention_tc.cuh"

namespace cake_dev {

template <int HD>
struct FaltCfg {
  static constexpr int kHalves = HD / 64;
  static constexpr int kTileBytes = kFaRows * HD * 2;
  static constexpr int kHalfBytes = kFaRows * 128;
  static constexpr int kPageHalfBytes = 64 * 128;
  static constexpr int kKStages = 3;
  static constexpr int kVStages = 2;
  static constexpr int kSmem = (1 + kKStages + kVStages) * kTileBytes + 1024 + 256;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColO = 256;  // O_g at kColO + 128 g
};

template <int HD>
__global__ void __launch_bounds__(fa_threads<2>(), 1)
    attn_alt_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                    const FaArgs a) {
  using Cfg = FaltCfg<HD>;
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
  const int nb = p_end > p_begin ? (p_end - p_begin + 1) / 2 : 0;

  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Cfg::kTileBytes;
  uint8_t* sV = sK + Cfg::kKStages * Cfg::kTileBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + Cfg::kVStages * Cfg::kTileBytes);
  uint64_t* q_ready = bar;       // Q rows stored by the softmax threads
  uint64_t* k_full = bar + 1;    // [3]
  uint64_t* k_empty = bar + 4;   // [3]
  uint64_t* v_full = bar + 7;    // [2]
  uint64_t* v_empty = bar + 9;   // [2]
  uint64_t* s_full = bar + 11;   // [2] per buffer = per group
  uint64_t* p_ready = bar + 13;  // [2]
  uint64_t* pv_done = bar + 15;  // [2]
  uint64_t* o_final = bar + 17;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 18);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_kv);
    mbar_init(q_ready, 256);
    for (int s = 0; s < Cfg::kKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < Cfg::kVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&s_full[g], 1);
      mbar_init(&p_ready[g], 128);
      mbar_init(&pv_done[g], 1);
    }
    mbar_init(o_final, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  // K/V blocks over stable pages (FaArgs::stable_pages: the prefix before the chunk, or the
  // whole cache in the q-only first-token pass) are requested before the PDL wait
  __shared__ int s_npre;
  if (warp == 0 && lane == 0) {
    int n_pre = 0;
    if (tok0 < a.chunk_len) {
      const long long planes0 = static_cast<long long>(a.n_layers) * 2 * a.n_kv_heads;
      for (int j = 0; j < nb && j < Cfg::kKStages && j < Cfg::kVStages; ++j) {
        const int lp0 = p_begin + 2 * j;
        const int lp1 = (lp0 + 1 < p_end) ? lp0 + 1 : lp0;
        if (lp1 >= a.stable_pages) break;
        int32_t r[2][2];
        for (int kv = 0; kv < 2; ++kv)
          for (int q = 0; q < 2; ++q) {
            const long long ph = a.block_table[q ? lp1 : lp0];
            r[kv][q] = static_cast<int32_t>(
                ((ph * planes0) + (static_cast<long long>(a.layer) * 2 + kv) * a.n_kv_heads + kvh) * 64);
          }
        mbar_arrive_expect_tx(&k_full[j], Cfg::kTileBytes);
        mbar_arrive_expect_tx(&v_full[j], Cfg::kTileBytes);
#pragma unroll
        for (int h = 0; h < Cfg::kHalves; ++h) {
          tma_load_2d(sK + j * Cfg::kTileBytes + h * Cfg::kHalfBytes, &tm_kv, &k_full[j], h * 64, r[0][0]);
          tma_load_2d(sK + j * Cfg::kTileBytes + h * Cfg::kHalfBytes + Cfg::kPageHalfBytes, &tm_kv, &k_full[j],
                      h * 64, r[0][1]);
          tma_load_2d(sV + j * Cfg::kTileBytes + h * Cfg::kHalfBytes, &tm_kv, &v_full[j], h * 64, r[1][0]);
          tma_load_2d(sV + j * Cfg::kTileBytes + h * Cfg::kHalfBytes + Cfg::kPageHalfBytes, &tm_kv, &v_full[j],
                      h * 64, r[1][1]);
        }
        ++n_pre;
      }
    }
    s_npre = n_pre;
  }
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) s_abort = a.abort_flag != nullptr ? *(volatile const int*)a.abort_flag : 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_pre = s_npre;
  if (s_abort || tok0 >= a.chunk_len) {
    if (warp == 0 && lane == 0)  // requested blocks must land before the shared memory goes away
      for (int j = 0; j < n_pre; ++j) {
        mbar_wait(&k_full[j], 0);
        mbar_wait(&v_full[j], 0);
      }
    if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(tmem);
    return;
  }

  const long long planes = static_cast<long long>(a.n_layers) * 2 * a.n_kv_heads;
  auto page_row = [&](int lp, int kv) -> int32_t {
    const long long ph = a.block_table[lp];
    return static_cast<int32_t>(((ph * planes) + (static_cast<long long>(a.layer) * 2 + kv) * a.n_kv_heads + kvh) * 64);
  };
  if (warp < 4) {
    setmaxnreg_dec<56>();  // one instruction for the whole role warpgroup (.aligned)
    if (warp == 0) {
      if (lane == 0 && nb > 0) {
        for (int j = n_pre; j < nb; ++j) {  // K blocks
          const int s = j % Cfg::kKStages;
          mbar_wait(&k_empty[s], ((j / Cfg::kKStages) & 1) ^ 1u);
          const int lp0 = p_begin + 2 * j;
          const int lp1 = (lp0 + 1 < p_end) ? lp0 + 1 : lp0;
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
        for (int j = n_pre; j < nb; ++j) {  // V blocks
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
    } else if (warp == 1 && nb > 0) {
      // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = umma_idesc_bf16(kFaRows, kFaKeys, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(kFaRows, HD, false, true);
      mbar_wait(q_ready, 0);
      tc_fence_after();
      const uint32_t q_addr = smem_u32(sQ);
      auto issue_s = [&](int jj) {  // S(jj) into buffer jj & 1 (its previous P was read by PV(jj - 2))
        const int ks = jj % Cfg::kKStages;
        mbar_wait(&k_full[ks], (jj / Cfg::kKStages) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + ks * Cfg::kTileBytes);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk >> 2) * Cfg::kHalfBytes + (kk & 3) * 32;
            umma_bf16_ss(tmem + (jj & 1) * 128, umma_desc_sw128(q_addr + off), umma_desc_sw128(k_addr + off),
                         idesc_s, kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[jj & 1]);
          umma_commit(&k_empty[ks]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int jj) {  // O_g += P(jj) V(jj), g = jj & 1 (the group's first block initialises O_g)
        const int g = jj & 1;
        const int vs = jj % Cfg::kVStages;
        mbar_wait(&p_ready[g], (jj >> 1) & 1);
        mbar_wait(&v_full[vs], (jj / Cfg::kVStages) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + vs * Cfg::kTileBytes);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kFaKeys / 16; ++kk) {
            const uint64_t bdesc = umma_desc_sw128_mn(v_addr + kk * 16 * 128, Cfg::kHalfBytes, 1024);
            umma_bf16_ts(tmem + Cfg::kColO + g * 128, tmem + g * 128 + kk * 8, bdesc, idesc_o,
                         (jj >= 2 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&pv_done[g]);
          umma_commit(&v_empty[vs]);
        }
        __syncwarp();
      };
      issue_s(0);
      if (nb > 1) issue_s(1);
      for (int j = 0; j < nb; ++j) {
        issue_pv(j);
        if (j + 2 < nb) issue_s(j + 2);
      }
      if (elect_one()) umma_commit(o_final);
      __syncwarp();
    }
  } else {
    setmaxnreg_inc<224>();
    // ------------------------------------------------ softmax + epilogue: group g = blocks j = g (mod 2)
    __shared__ float xm[2][kFaRows];
    __shared__ float xl[2][kFaRows];
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
      // this thread's Q row, half g, into the SW128 K-major tile (attention_dec.cuh's layout)
      const bool live = t < a.chunk_len && nb > 0;
      const uint4* src = reinterpret_cast<const uint4*>(a.q + (static_cast<size_t>(t) * a.n_q_heads + head) * HD +
                                                        g * (HD / 2));
      if constexpr (HD / 2 == 64) {
        uint8_t* dst_row = sQ + g * Cfg::kHalfBytes + row * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 v = live ? __ldg(src + c) : make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(dst_row + ((c ^ (row & 7)) << 4)) = v;
        }
      } else {
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
    const uint32_t tS = tmem + lane_off + g * 128;
    const uint32_t tO = tmem + lane_off + Cfg::kColO + g * 128;
    for (int j = g; j < nb; j += 2) {
      const int n = j >> 1;  // this group's block count so far
      mbar_wait(&s_full[g], n & 1);
      tc_fence_after();
      uint32_t su[kFaKeys];
#pragma unroll
      for (int c = 0; c < kFaKeys / 32; ++c) tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&su[c * 32]));
      tmem_ld_wait();
      const long long kbase = static_cast<long long>(p_begin + 2 * j) * kAttnPage;
      if (kbase + kFaKeys - 1 > qpos_min || kbase + kFaKeys > kmax_valid) {
        const long long lim64 = min(qpos, kmax_valid - 1) - kbase;  // last visible key, relative
        const int lim = static_cast<int>(max(lim64, -1LL));
#pragma unroll
        for (int e = 0; e < kFaKeys; ++e)
          if (e > lim) su[e] = __float_as_uint(-INFINITY);
      }
      float mc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) mc[c] = __uint_as_float(su[c]);
#pragma unroll
      for (int e = 8; e < kFaKeys; ++e) mc[e & 7] = fmaxf(mc[e & 7], __uint_as_float(su[e]));
      const float mx =
          fmaxf(fmaxf(fmaxf(mc[0], mc[1]), fmaxf(mc[2], mc[3])), fmaxf(fmaxf(mc[4], mc[5]), fmaxf(mc[6], mc[7]))) * sc;
      // tcgen05.ld/st are warp-collective (.sync.aligned): when any row of the warp moves its
      // reference max the whole warp runs the rescale pass (factor 1 for the other rows)
      const bool up = mx > m + 8.0f;  // (also true on the first block with a visible key)
      const bool resc = up && m != -INFINITY;
      if (__any_sync(0xffffffffu, resc)) {
        // O_g holds this group's blocks < j: wait for the PV of its previous block, then rescale
        mbar_wait(&pv_done[g], (n - 1) & 1);
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
      // P packed in place: word w (keys 2w, 2w+1) lands in su[w], never ahead of a read
#pragma unroll
      for (int w = 0; w < kFaKeys / 2; ++w) {
        const float2 x = ffma2(make_float2(__uint_as_float(su[2 * w]), __uint_as_float(su[2 * w + 1])), sc2, nb2);
        float2 p;
        if ((w & 7) >= 8 - FA_POLY) {
          p = ex2_poly2(x);
        } else {
          p.x = ex2_approx(x.x);
          p.y = ex2_approx(x.y);
        }
        rs[w & 3] = fadd2(rs[w & 3], p);
        su[w] = pack_bf16(p.x, p.y);
      }
      tmem_st32(tS, *reinterpret_cast<uint32_t(*)[32]>(&su[0]));
      tmem_st32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&su[32]));
      const float2 rs01 = fadd2(rs[0], rs[1]), rs23 = fadd2(rs[2], rs[3]);
      l += (rs01.x + rs23.x) + (rs01.y + rs23.y);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_ready[g]);
    }
    // epilogue: merge (m_0, l_0, O_0) and (m_1, l_1, O_1) per row, fixed order; a group with no
    // block (or no visible key) contributes nothing (its O is never read: select, not multiply)
    xm[g][row] = m;
    xl[g][row] = l;
    named_bar_sync(2, 256);
    const float m0 = xm[0][row], m1 = xm[1][row];
    const float mt = fmaxf(m0, m1);
    const bool use0 = m0 != -INFINITY && nb > 0, use1 = m1 != -INFINITY && nb > 1;
    const float f0 = use0 ? ex2_approx(m0 - mt) : 0.f;
    const float f1 = use1 ? ex2_approx(m1 - mt) : 0.f;
    const float lt = (use0 ? xl[0][row] * f0 : 0.f) + (use1 ? xl[1][row] * f1 : 0.f);
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    const bool valid = t < a.chunk_len;
    const size_t orow = static_cast<size_t>(t) * a.n_q_heads + head;
    if (nb > 0) {
      mbar_wait(o_final, 0);
      tc_fence_after();
    }
    const float w0 = f0 * inv, w1 = f1 * inv;
    const uint32_t tO0 = tmem + lane_off + Cfg::kColO, tO1 = tO0 + 128;
    constexpr int kOCols = HD / 2;
#pragma unroll
    for (int c = 0; c < kOCols / 32; ++c) {
      const int col = g * kOCols + c * 32;
      uint32_t r0[32], r1[32];
      if (nb > 0) {
        tmem_ld32(tO0 + col, r0);
        tmem_ld32(tO1 + col, r1);
        tmem_ld_wait();
      }
      if (!valid) continue;
      float o[32];
#pragma unroll
      for (int i = 0; i < 32; ++i)
        o[i] = (use0 ? __uint_as_float(r0[i]) * w0 : 0.f) + (use1 ? __uint_as_float(r1[i]) * w1 : 0.f);
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
