// 2-SM tcgen05 GEMM (cta_group::2): the projection GEMMs of a chunk with
// more than 128 rows.
//
// A CTA pair (cluster of 2, one TPC) computes a 256 x 256 output tile: each
// CTA TMA-loads its own 128 rows of A and 128 rows of the weight tile, the
// leader issues tcgen05.mma.cta_group::2 (M = 256) that reads both CTAs'
// shared memory, and each CTA receives its 128 output rows x 256 columns in
// its own TMEM. Per SM that is 32 KB of operands per 64-deep k-block instead
// of 48 KB for the 1-SM 128 x 256 tile: at M = 512 the projections are bound
// by L2 -> SM bandwidth, so this is a 1.5x cut in the limiting resource.
//
// Pipeline (per pair): both producers wait on their own `empty` barrier,
// load their halves and count the bytes on the LEADER's `full` barrier (peer
// bit masked off); the leader's MMA thread waits `full`, issues 4 MMAs per
// k-block, and multicasts the stage release to both CTAs' `empty`. The
// accumulator handshake is the same across the pair: the leader's commit
// multicasts `tmem_full` to both CTAs; both epilogues arrive on the leader's
// `tmem_empty` (count 256). Split-K parts / stream-K partials are reduced per
// CTA exactly like the 1-SM kernel (gemm_epilogue).
#pragma once

#include "gemm.cuh"

namespace cake_dev {

#ifndef CAKE_GEMM_RING_KB
#define CAKE_GEMM_RING_KB 200
#endif
template <int BLOCK_N>
struct Gemm2Cfg {
  static_assert(BLOCK_N % 32 == 0 && BLOCK_N >= 64 && BLOCK_N <= 256, "cta_group::2 tile N");
  static constexpr int kABytes = kGemmBlockM * kGemmBlockK * 2;            // this CTA's 128 rows of A
  static constexpr int kBBytes = (BLOCK_N / 2) * kGemmBlockK * 2;          // this CTA's BLOCK_N/2 rows of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  // 6 (N 256) .. 8 (N 128). A/B of the ring budget 176 / 200 / 224 KB: within 1-2% per
  // shape, no trend (the depth is not what bounds the mainloop)
  static constexpr int kStages = (CAKE_GEMM_RING_KB * 1024) / kStageBytes;
  static constexpr int kTmemCols = (2 * BLOCK_N <= 256) ? 256 : 512;       // 2 accumulators
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
};

template <int BLOCK_N, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm2_tc_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                    const GemmArgs args) {
  using Cfg = Gemm2Cfg<BLOCK_N>;
  constexpr int kStages = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_abort;

  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const uint32_t raw_base = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_base + 1023u) & ~1023u) - raw_base);
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStages * Cfg::kABytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;       // [2] (leader's copy is the live one)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2 * 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_2sm<Cfg::kTmemCols>(tmem_slot);
  // (PDL) everything above overlaps the predecessor's tail; its outputs are read below
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) s_abort = (args.abort_flag != nullptr) ? *(volatile const int*)args.abort_flag : 0;
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // One abort decision per pair, the leader's (a lone CTA leaving would strand its peer).
  const int abort_pair = ld_shared_cluster_s32(mapa_shared(smem_u32(&s_abort), 0));
  if (abort_pair) {
    cluster_sync();
    if (warp == 1) tmem_dealloc_2sm<Cfg::kTmemCols>(tmem_base);
    return;
  }

  const int pair = blockIdx.x / 2;
  const int n_pairs = gridDim.x / 2;
  const int nk = args.num_k_blocks;
  const int m_pairs = (args.num_m_blocks + 1) / 2;
  const long long units = static_cast<long long>(m_pairs) * args.num_n_blocks * nk;
  int tile, kb0, kb1;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer (both CTAs)
      const uint64_t pol_w = gemm_policy(args.l2_hints, 1);
      const uint64_t pol_a = gemm_policy(args.l2_hints, 0);
      StreamK sk(units, nk, pair, n_pairs, args.whole_tiles);
      int stage = 0;
      uint32_t phase = 0;
      while (sk.next(tile, kb0, kb1)) {
        const int m_row = (tile % m_pairs) * 256 + static_cast<int>(rank) * 128;
        const int n_row = (tile / m_pairs) * BLOCK_N + static_cast<int>(rank) * (BLOCK_N / 2);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1u);
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::kStageBytes);
          tma_load_2d_2sm(smem_a + stage * Cfg::kABytes, &tmap_a, &full_bar[stage], kb * kGemmBlockK, m_row, pol_a);
          tma_load_2d_2sm(smem_b + stage * Cfg::kBBytes, &tmap_b, &full_bar[stage], kb * kGemmBlockK, n_row, pol_w);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------ MMA issuer (leader only)
      // converged warp, one elected lane issues (A/B against a lane-0 issuer: equal)
      constexpr uint32_t idesc = umma_idesc_bf16(256, BLOCK_N);
      StreamK sk(units, nk, pair, n_pairs, args.whole_tiles);
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
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < kGemmBlockK / 16; ++k)
              umma_bf16_ss_2sm(d_tmem, umma_desc_sw128(a_addr + k * 32), umma_desc_sw128(b_addr + k * 32), idesc,
                               (kb > kb0 || k > 0) ? 1u : 0u);
            umma_commit_2sm_mc(&empty_bar[stage], 0x3);
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (elect_one()) umma_commit_2sm_mc(&tfull_bar[acc], 0x3);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..5, both CTAs)
    const int ew = warp & 3;
    const int row = ew * 32 + static_cast<int>(lane);
    const int ep_tid = threadIdx.x - 64;
    const uint32_t leader_tempty0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    StreamK sk(units, nk, pair, n_pairs, args.whole_tiles);
    int acc = 0;
    uint32_t acc_phase = 0;
    while (sk.next(tile, kb0, kb1)) {
      const int m = (tile % m_pairs) * 256 + static_cast<int>(rank) * 128 + row;
      const int n_blk = tile / m_pairs;
      if (sk.tile_mode == 2 && tile >= sk.n_full) {
        // a part of a tail tile: its fp32 accumulator goes to the tail workspace (row-major,
        // 256 x BLOCK_N per part); gemm_tail_kernel sums the parts in order and applies the epilogue
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        const uint32_t tbase =
            tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * BLOCK_N);
        const int part = pair % sk.tail_s;
        float* dst = args.tail_ws +
                     (static_cast<size_t>((tile - sk.n_full) * sk.tail_s + part) * 256 + rank * 128 + row) * BLOCK_N;
#pragma unroll 1
        for (int c = 0; c < BLOCK_N / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tbase + c * 32, r);
          tmem_ld_wait();
          float4* d4 = reinterpret_cast<float4*>(dst + c * 32);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            __stcg(d4 + q, make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                       __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])));
        }
        tc_fence_before();
        mbar_arrive_cluster(leader_tempty0 + acc * 8);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
        continue;
      }
      EpiPre<BLOCK_N, EPI> pre;
      pre.load(args, m, n_blk, kb0 > 0);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase =
          tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * BLOCK_N);
      const bool partial = kb0 > 0;
      int first_part = 0, n_parts = 0;
      if (!partial && kb1 < nk) {
        const long long u_tile = static_cast<long long>(tile) * nk;
        first_part = sk.cta_of(u_tile) + 1;
        n_parts = sk.cta_of(u_tile + nk - 1) - first_part + 1;
      }
      gemm_epilogue<BLOCK_N, EPI>(args, tbase, row, m, n_blk, partial, blockIdx.x,
                                  first_part * 2 + static_cast<int>(rank), n_parts, 2, ep_tid, pre);
      tc_fence_before();
      mbar_arrive_cluster(leader_tempty0 + acc * 8);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  }

  __syncthreads();
  cluster_sync();  // the pair's MMAs / multicasts / remote arrives are all done
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm<Cfg::kTmemCols>(tmem_base);
  }
}

// The tail tiles of a whole_tiles == 2 gate/up GEMM: out[m, j] = silu(g) * u
// with g, u the sums (in part order) of the parts' accumulators, times the
// fused-RMSNorm row scale. One CTA per (tail tile, row), one thread per
// gate/up column pair; the row scale is reduced once per CTA.
__global__ void __launch_bounds__(128) swiglu_tail_kernel(const GemmArgs a, int n_full, int n_tail_tiles, int parts) {
  pdl_wait();
  pdl_trigger();
  if (a.abort_flag != nullptr && *(volatile const int*)a.abort_flag) return;
  __shared__ float s_rs;
  const int m_pairs = (a.num_m_blocks + 1) / 2;
  const int t = blockIdx.x / 256, r = blockIdx.x % 256;
  const int tile = n_full + t;
  const int m = (tile % m_pairs) * 256 + r;
  if (m >= a.M) return;
  if (threadIdx.x < 32) {
    float tt = 0.f;
    if (a.ss_in != nullptr)
      for (int q = threadIdx.x; q < a.ss_parts; q += 32) tt += __ldcg(a.ss_in + static_cast<size_t>(q) * a.ss_ld + m);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tt += __shfl_xor_sync(0xffffffffu, tt, o);
    if (threadIdx.x == 0) s_rs = a.ss_in != nullptr ? rsqrtf(tt / static_cast<float>(a.rms_dim) + a.rms_eps) : 1.f;
  }
  const int j = threadIdx.x;
  const float* src = a.tail_ws + (static_cast<size_t>(t) * parts * 256 + r) * 256;
  // all parts' loads in flight at once (parts <= kTailSplit), then summed in part order
  float gv[kTailSplit], uv[kTailSplit];
#pragma unroll
  for (int p = 0; p < kTailSplit; ++p)
    if (p < parts) {
      gv[p] = __ldcg(src + static_cast<size_t>(p) * 256 * 256 + j);
      uv[p] = __ldcg(src + static_cast<size_t>(p) * 256 * 256 + 128 + j);
    }
  float g = 0.f, u = 0.f;
#pragma unroll
  for (int p = 0; p < kTailSplit; ++p)
    if (p < parts) {
      g += gv[p];
      u += uv[p];
    }
  __syncthreads();
  const float rs = s_rs;
  g *= rs;
  u *= rs;
  reinterpret_cast<__nv_bfloat16*>(a.out)[static_cast<size_t>(m) * a.ldo + (tile / m_pairs) * 128 + j] =
      __float2bfloat16_rn(silu_f(g) * u);
}

}  // namespace cake_dev
