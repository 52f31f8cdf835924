// 2-SM tcgen05 GEMM in clusters of NP CTA pairs that share the A operand.
//
// At M = 512 the O / down / QKV projections (N = 4096 / 4096 / 6144) are
// bound by operand delivery from L2, not by HBM or the tensor pipe: every
// 256-row A tile is fetched once per n-block (32 times) and every weight tile
// once per m-pair (twice) — 201 MB crossing L2 -> SM for 46 MB of DRAM reads
// on the O projection (profiles/r01_ncu_summary.md). Here NP pairs that work
// on the SAME m-pair and NP consecutive n-blocks form one cluster
// (2 * NP CTAs): each CTA TMA-loads 1/NP of its half of the A k-block and
// multicasts it to the CTA of the same half in every pair of the cluster, so
// an A byte leaves L2 once per cluster instead of once per pair. The weight
// halves stay per CTA (cta_group::2 loads into the pair).
//
// Barriers, per CTA:
//   full[s]    the pair leader's copy counts every byte that lands in either
//              CTA of the pair (own A piece + NP-1 multicast pieces + B half);
//   empty[s]   count NP: stage s of THIS CTA is written by NP producers (one
//              per pair), so it is free only when every pair's MMA released
//              it — each leader's commit is multicast to the whole cluster;
//   tmem_full / tmem_empty as in gemm2.cuh, per pair (leader = rank & ~1).
// One tile (m-pair x NP n-blocks) per cluster per round, whole tiles only
// (no split-K): at M = 512 the three projections have exactly 32 cluster
// tiles at NP = 2 (128 CTAs), one round.
#pragma once

#include "gemm2.cuh"

namespace cake_dev {

// Residual epilogue through shared memory (one tile per CTA, so the operand
// ring is free once the accumulator is complete): each thread adds its row of
// the accumulator to the prefetched residual row, writes h and bf16(h) into
// 128-B-swizzled boxes, and one thread TMA-stores them — every global write a
// full line, instead of 16-B pieces of 32 rows per warp instruction
// (2.8 -> ~1 us per O / down tile, tools/gemm_trace.py).
template <int EPI>
__device__ __forceinline__ void gemm2c_staged_resid(const GemmArgs& args, const CUtensorMap* tm_h,
                                                    const CUtensorMap* tm_xb, uint8_t* stage, uint32_t tbase,
                                                    int row, int m, int m0, int n_blk, int ep_tid,
                                                    const EpiPre<128, EPI>& pre) {
  constexpr int kHBox = 128 * 128;  // bytes of one [128 rows x 32 fp32] box
  uint8_t* sh = stage;              // 4 h boxes
  uint8_t* sx = stage + 4 * kHBox;  // 2 bf16 boxes of [128 rows x 64]
  const uint32_t sw = static_cast<uint32_t>(row & 7);
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tmem_ld32(tbase + c * 32, r);
    tmem_ld_wait();
    float4 hv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 h = pre.h[c * 8 + q];
      h.x += __uint_as_float(r[q * 4]);
      h.y += __uint_as_float(r[q * 4 + 1]);
      h.z += __uint_as_float(r[q * 4 + 2]);
      h.w += __uint_as_float(r[q * 4 + 3]);
      hv[q] = h;
      ss += h.x * h.x + h.y * h.y + h.z * h.z + h.w * h.w;
      *reinterpret_cast<float4*>(sh + c * kHBox + row * 128 + ((q ^ sw) << 4)) = h;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t j = static_cast<uint32_t>((c & 1) * 4 + q);
      uint4 v = make_uint4(pack_bf16(hv[2 * q].x, hv[2 * q].y), pack_bf16(hv[2 * q].z, hv[2 * q].w),
                           pack_bf16(hv[2 * q + 1].x, hv[2 * q + 1].y), pack_bf16(hv[2 * q + 1].z, hv[2 * q + 1].w));
      *reinterpret_cast<uint4*>(sx + (c >> 1) * kHBox + row * 128 + ((j ^ sw) << 4)) = v;
    }
    // store each box as soon as it is staged: box c's TMA store drains while boxes c+1.. are computed
    fence_proxy_async();  // the generic-proxy smem writes, before the async-proxy (TMA) reads them
    named_bar_sync(1, 128);
    if (ep_tid == 0) {
      const int n0 = n_blk * 128;
      tma_store_2d(tm_h, sh + c * kHBox, n0 + c * 32, m0);
      if ((c & 1) && args.xb_out != nullptr) tma_store_2d(tm_xb, sx + (c >> 1) * kHBox, n0 + (c >> 1) * 64, m0);
    }
  }
  if (args.ss_out != nullptr && m < args.M) args.ss_out[static_cast<size_t>(n_blk) * args.ss_ld + m] = ss;
  if (ep_tid == 0) {
    bulk_commit();
    bulk_wait_read0();  // shared memory must outlive the reads
  }
}

template <int BLOCK_N, int EPI, int NP>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm2c_tc_kernel(const __grid_constant__ CUtensorMap tmap_a_piece, const __grid_constant__ CUtensorMap tmap_b,
                     const __grid_constant__ CUtensorMap tmap_h, const __grid_constant__ CUtensorMap tmap_xb,
                     const GemmArgs args) {
  static_assert(NP == 2 || NP == 4, "pairs per cluster");
  using Cfg = Gemm2Cfg<BLOCK_N>;
  constexpr int kStages = Cfg::kStages;
  constexpr int kPieceRows = kGemmBlockM / NP;
  constexpr int kPieceBytes = kPieceRows * kGemmBlockK * 2;
  constexpr int kCluster = 2 * NP;
  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_abort;

  const uint32_t rank = cluster_ctarank();
  const uint32_t half = rank & 1u;
  const uint32_t pin = rank >> 1;  // pair index inside the cluster
  const bool leader = half == 0;
  const uint32_t raw_base = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_base + 1023u) & ~1023u) - raw_base);
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStages * Cfg::kABytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;       // [2] (the pair leader's copy is the live one)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();
  if (threadIdx.x == 0) gemm_stamp(args, 0);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a_piece);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NP);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2 * 4);  // one arrive per epilogue warp of the pair
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_2sm<Cfg::kTmemCols>(tmem_slot);
  // the abort flag is written by the host (control stream), not by a predecessor kernel
  if (threadIdx.x == 0) s_abort = (args.abort_flag != nullptr) ? *(volatile const int*)args.abort_flag : 0;
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) gemm_stamp(args, 1);
  // one abort decision per cluster (rank 0's): a lone CTA leaving would strand the multicasts
  const int abort_all = ld_shared_cluster_s32(mapa_shared(smem_u32(&s_abort), 0));
  if (abort_all) {
    cluster_sync();
    if (warp == 1) tmem_dealloc_2sm<Cfg::kTmemCols>(tmem_base);
    return;
  }

  const int cluster = blockIdx.x / kCluster;
  const int n_clusters = gridDim.x / kCluster;
  const int nk = args.num_k_blocks;
  const int m_pairs = (args.num_m_blocks + 1) / 2;
  const int n_groups = args.num_n_blocks / NP;
  const int n_tiles = m_pairs * n_groups;  // tile t: m-pair t % m_pairs, n-group t / m_pairs
  const uint16_t same_half_mask = static_cast<uint16_t>((half ? 0xAAAAu : 0x5555u) & ((1u << kCluster) - 1u));
  const uint16_t all_mask = static_cast<uint16_t>((1u << kCluster) - 1u);
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * pin));
  const uint64_t pol_w = gemm_policy(args.l2_hints, 1);
  const uint64_t pol_a = gemm_policy(args.l2_hints, 0);
  auto n_row_of = [&](int tile) {
    return ((tile / m_pairs) * NP + static_cast<int>(pin)) * BLOCK_N + static_cast<int>(half) * (BLOCK_N / 2);
  };
  // The weights do not depend on the predecessor kernel: the first ring's
  // worth of weight k-blocks is requested before the PDL wait, under the
  // predecessor's tail (the activations follow once it has completed).
  int n_pre = 0;
  if (warp == 0 && lane == 0 && cluster < n_tiles) {
    n_pre = nk < kStages ? nk : kStages;
    if (args.prefetch >= 0 && args.prefetch < n_pre) n_pre = args.prefetch;
    for (int kb = 0; kb < n_pre; ++kb) {
      if (leader) mbar_arrive_expect_tx(&full_bar[kb], 2 * Cfg::kStageBytes);
      tma_load_2d_2sm(smem_b + kb * Cfg::kBBytes, &tmap_b, &full_bar[kb], kb * kGemmBlockK, n_row_of(cluster), pol_w);
    }
  }
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) gemm_stamp(args, 2);

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer (every CTA)
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cluster; tile < n_tiles; tile += n_clusters) {
        const int a_row = (tile % m_pairs) * 256 + static_cast<int>(half) * 128 + static_cast<int>(pin) * kPieceRows;
        const int n_row = n_row_of(tile);
        for (int kb = 0; kb < nk; ++kb) {
          const bool prefetched = tile == cluster && kb < n_pre;  // weights already requested
          if (!prefetched) {
            mbar_wait(&empty_bar[stage], phase ^ 1u);  // every pair consumed stage s of this CTA
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::kStageBytes);
          }
          tma_load_2d_2sm_mc(smem_a + stage * Cfg::kABytes + pin * kPieceBytes, &tmap_a_piece, &full_bar[stage],
                             kb * kGemmBlockK, a_row, same_half_mask, pol_a);
          if (!prefetched)
            tma_load_2d_2sm(smem_b + stage * Cfg::kBBytes, &tmap_b, &full_bar[stage], kb * kGemmBlockK, n_row, pol_w);
          if (kb == 0) gemm_stamp(args, 3);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------ MMA issuer (pair leaders)
      constexpr uint32_t idesc = umma_idesc_bf16(256, BLOCK_N);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = cluster; tile < n_tiles; tile += n_clusters) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BLOCK_N);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (kb == 0 && lane == 0) gemm_stamp(args, 4);
          const uint32_t a_addr = smem_u32(smem_a + stage * Cfg::kABytes);
          const uint32_t b_addr = smem_u32(smem_b + stage * Cfg::kBBytes);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < kGemmBlockK / 16; ++k)
              umma_bf16_ss_2sm(d_tmem, umma_desc_sw128(a_addr + k * 32), umma_desc_sw128(b_addr + k * 32), idesc,
                               (kb > 0 || k > 0) ? 1u : 0u);
            umma_commit_2sm_mc(&empty_bar[stage], all_mask);  // this pair is done with stage s everywhere
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (elect_one()) umma_commit_2sm_mc(&tfull_bar[acc], pair_mask);
        if (lane == 0) gemm_stamp(args, 5);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..5, every CTA)
    const int ew = warp & 3;
    const int row = ew * 32 + static_cast<int>(lane);
    const int ep_tid = threadIdx.x - 64;
    const uint32_t leader_tempty0 = mapa_shared(smem_u32(&tempty_bar[0]), rank & ~1u);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = cluster; tile < n_tiles; tile += n_clusters) {
      const int m = (tile % m_pairs) * 256 + static_cast<int>(half) * 128 + row;
      const int n_blk = (tile / m_pairs) * NP + static_cast<int>(pin);
      EpiPre<BLOCK_N, EPI> pre;
      pre.load(args, m, n_blk, false);
      if (ep_tid == 0) gemm_stamp(args, 6);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      if (ep_tid == 0) gemm_stamp(args, 7);
      const uint32_t tbase =
          tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * BLOCK_N);
      if constexpr (EPI == kEpiResid && BLOCK_N == 128) {
        if (args.staged) {
          gemm2c_staged_resid<EPI>(args, &tmap_h, &tmap_xb, smem, tbase, row, m, m - row, n_blk, ep_tid, pre);
        } else {
          gemm_epilogue<BLOCK_N, EPI>(args, tbase, row, m, n_blk, false, blockIdx.x, 0, 0, 2, ep_tid, pre);
        }
      } else {
        gemm_epilogue<BLOCK_N, EPI>(args, tbase, row, m, n_blk, false, blockIdx.x, 0, 0, 2, ep_tid, pre);
      }
      if (ep_tid == 0) gemm_stamp(args, 8);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty0 + acc * 8);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  }

  __syncthreads();
  if (threadIdx.x == 0) gemm_stamp(args, 9);
  cluster_sync();  // every multicast into this CTA and every remote arrive is done
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm<Cfg::kTmemCols>(tmem_base);
  }
  if (threadIdx.x == 64) gemm_stamp(args, 10);
}

}  // namespace cake_dev
