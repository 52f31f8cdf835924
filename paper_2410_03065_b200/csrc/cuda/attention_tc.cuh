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
// Q lives in TMEM (the A operand of QK^T, like P for PV), so each block's
// MMAs read only K and V from shared memory.
// Roles (128 + 128*NG threads): warp 0 TMA producer of K (3-stage ring, freed
// right after each QK^T), warp 2 TMA producer of V (2-stage ring, freed after
// each PV), warp 1 TMEM owner + MMA issuer, warps 4.. softmax + epilogue in
// NG column groups (warp w%4 owns TMEM lanes 32*(w%4)..; NG = 2: two softmax
// warps per sub-partition hide the MUFU / TMEM-load latency of the row chains;
// NG = 4 measured 10% slower at 32K).
#pragma once

#include "attention.cuh"
#include "ptx.cuh"

namespace cake_dev {

constexpr int kFaRows = 128;
constexpr int kFaKeys = 128;  // two pages
// 4 role warps + NG softmax groups of 4 warps
template <int NG>
constexpr int fa_threads() { return 128 + NG * 128; }

template <int HD>
struct FaCfg {
  static constexpr int kHalves = HD / 64;                    // 64-element (128 B) K slices
  static constexpr int kTileBytes = kFaRows * HD * 2;        // Q / K / V tile (128 rows)
  static constexpr int kHalfBytes = kFaRows * 128;           // one 64-wide slice of a tile
  static constexpr int kPageHalfBytes = 64 * 128;            // one page x 64 elements
  static constexpr int kKStages = 3;                          // K released right after its QK^T
  static constexpr int kVStages = 3;                          // V released after its PV
  static constexpr int kSmem = (kKStages + kVStages) * kTileBytes + 1024 + 256;
  static constexpr uint32_t kTmemCols = 512;
  // S double buffer, O accumulator, Q (bf16 pairs: HD/2 columns) as the TMEM A operand of QK^T
  static constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO = 256, kColQ = 384;
};

struct FaArgs {
  const __nv_bfloat16* q;  // [C, n_q, hd] (rows read once, into TMEM)
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
  long long* trace;  // debug (nullptr): clock64 stamps of CTA (0,0,0), tools/attn_trace.py
  int stable_pages;  // logical pages [0, stable_pages) are not written by the predecessor kernel: their
                     // K/V blocks are requested before the PDL wait (0: none)
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (degree-3 minimax of 2^f on [-0.5, 0.5], rel err 7.5e-5,
// well under bf16's 2^-8): a share of the softmax exponentials is computed here
// so the MUFU unit (16/clk/SM, the softmax bottleneck) is not the critical
// pipe next to the tensor core. x <= ~8 here; clamped below at -125 so the
// exponent add cannot wrap (2^-125 is 0 for the bf16 P and the fp32 sum).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.0f);
  const float t = __fadd_rn(x, 12582912.0f);  // 1.5 * 2^23: round(x) lands in the low mantissa bits
  const float f = __fsub_rn(x, __fsub_rn(t, 12582912.0f));
  float p = fmaf(0.05517132f, f, 0.24261054f);
  p = fmaf(p, f, 0.69326099f);
  p = fmaf(p, f, 0.99992811f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
#ifndef FA_POLY
#define FA_POLY 2
#endif
// 2^x for a pair on the FMA pipe (ex2_poly on FFMA2 / FADD2).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.0f);
  x.y = fmaxf(x.y, -125.0f);
  const float2 big = make_float2(12582912.0f, 12582912.0f);
  const float2 t = fadd2(x, big);
  const float2 u = fadd2(t, make_float2(-12582912.0f, -12582912.0f));  // round(x)
  const float2 f = ffma2(u, make_float2(-1.0f, -1.0f), x);  // x - round(x)
  float2 p = ffma2(make_float2(0.05517132f, 0.05517132f), f, make_float2(0.24261054f, 0.24261054f));
  p = ffma2(p, f, make_float2(0.69326099f, 0.69326099f));
  p = ffma2(p, f, make_float2(0.99992811f, 0.99992811f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}


template <int HD, int NG>
__global__ void __launch_bounds__(fa_threads<NG>(), 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                   const FaArgs a) {
  using Cfg = FaCfg<HD>;
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
  uint8_t* sK = smem;                                       // [kKStages][tile]
  uint8_t* sV = sK + Cfg::kKStages * Cfg::kTileBytes;      // [kVStages][tile]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + Cfg::kVStages * Cfg::kTileBytes);
  uint64_t* q_ready = bar;        // Q rows stored into TMEM by the softmax warps
  uint64_t* k_full = bar + 1;     // [3]
  uint64_t* k_empty = bar + 4;    // [3]
  uint64_t* v_full = bar + 7;     // [3]
  uint64_t* v_empty = bar + 10;   // [3]
  uint64_t* s_full = bar + 13;    // [2]
  uint64_t* p_ready = bar + 15;   // [2]
  uint64_t* pv_done = bar + 17;
  uint64_t* o_final = bar + 18;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 19);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
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
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_ready[s], 128 * NG);
    }
    mbar_init(pv_done, 1);
    mbar_init(o_final, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  // The first ring's worth of K/V blocks over stable pages (the prefix before this chunk,
  // or the whole cache for the q-only first-token pass) does not depend on the predecessor:
  // requested before the PDL wait, so the ring fills under the predecessor's tail.
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
  // (PDL) everything above overlaps the predecessor's tail; Q / the KV pool are read below
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
  auto page_row = [&](int lp, int kv) -> int32_t {  // first pool row of (page, layer, K|V, kv head)
    const long long ph = a.block_table[lp];
    return static_cast<int32_t>(((ph * planes) + (static_cast<long long>(a.layer) * 2 + kv) * a.n_kv_heads + kvh) * 64);
  };
  if (warp == 0) {
    if (lane == 0 && nb > 0) {
      // ------------------------------------------------ TMA producer: K blocks
      for (int j = n_pre; j < nb; ++j) {
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
      for (int j = n_pre; j < nb; ++j) {
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
      // ------------------------------------------------ MMA issuer
      // The whole warp runs the loop (barrier waits on every lane) and one
      // elected lane issues. In isolation a tcgen05.mma stream issued from a
      // divergent single lane loses ~200 cycles at every mbarrier wait and a
      // converged warp ~70 (profiles/r01_ncu_summary.md, "MMA issue"); in this
      // kernel both measure the same block period (the softmax bounds it).
      constexpr uint32_t idesc_s = umma_idesc_bf16(kFaRows, kFaKeys, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(kFaRows, HD, false, true);
      mbar_wait(q_ready, 0);
      tc_fence_after();
      const bool trm = a.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0;
      if (trm) a.trace[0] = clock64(), a.trace[1] = nb;
      auto issue_pv = [&](int jj) {
        const int s = jj & 1;
        const int vs = jj % Cfg::kVStages;
        if (trm && jj < 64) a.trace[64 + jj * 8 + 6] = clock64();
        mbar_wait(&p_ready[s], (jj >> 1) & 1);
        if (trm && jj < 64) a.trace[64 + jj * 8 + 7] = clock64();
        if (trm && jj < 64) a.trace[64 + 1024 + jj * 8] = clock64();
        mbar_wait(&v_full[vs], (jj / Cfg::kVStages) & 1);
        if (trm && jj < 64) a.trace[64 + 1024 + jj * 8 + 1] = clock64();
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + vs * Cfg::kTileBytes);
        const uint32_t p_col = tmem + (s ? Cfg::kColS1 : Cfg::kColS0);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kFaKeys / 16; ++kk) {
            const uint64_t bdesc = umma_desc_sw128_mn(v_addr + kk * 16 * 128, Cfg::kHalfBytes, 1024);
            umma_bf16_ts(tmem + Cfg::kColO, p_col + kk * 8, bdesc, idesc_o, (jj > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&v_empty[vs]);
          umma_commit(pv_done);
        }
        __syncwarp();
      };
      auto issue_s = [&](int jj) {
        const int s = jj & 1;
        const int ks = jj % Cfg::kKStages;
        if (trm && jj < 64) a.trace[64 + 1024 + jj * 8 + 2] = clock64();
        mbar_wait(&k_full[ks], (jj / Cfg::kKStages) & 1);
        if (trm && jj < 64) a.trace[64 + 1024 + jj * 8 + 3] = clock64();
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + ks * Cfg::kTileBytes);
        const uint32_t d = tmem + (s ? Cfg::kColS1 : Cfg::kColS0);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk >> 2) * Cfg::kHalfBytes + (kk & 3) * 32;
            umma_bf16_ts(d, tmem + Cfg::kColQ + kk * 8, umma_desc_sw128(k_addr + off), idesc_s, kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[s]);
          umma_commit(&k_empty[ks]);
        }
        __syncwarp();
      };
      // S(j+1) is issued BEFORE waiting for P(j): the tensor pipe computes the
      // next block's scores while the softmax warps work on this one. (S(j+1)
      // reuses the buffer of P(j-1), whose PV was issued earlier: in-order pipe.)
      issue_s(0);
      for (int j = 0; j < nb; ++j) {
        if (j + 1 < nb) issue_s(j + 1);
        issue_pv(j);
      }
      if (elect_one()) umma_commit(o_final);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax + epilogue
    // NG groups of 4 warps share the TMEM lanes (rows): group g owns score
    // columns [g*128/NG, (g+1)*128/NG), the matching packed P columns and O
    // columns [g*HD/NG, (g+1)*HD/NG). More groups = more warps per SM
    // sub-partition to hide the TMEM-load / MUFU latency of the row chains.
    // The row max is exchanged through shared memory once per block
    // (double-buffered by block parity), the row sum once at the end, so all
    // groups take identical rescale decisions.
    constexpr int kKeysPerG = kFaKeys / NG;
    constexpr int kOCols = HD / NG;
    constexpr int kQWords = HD / 2 / NG;  // packed bf16 pairs of Q per group
    __shared__ float xmax[2][NG][kFaRows];
    __shared__ float xsum[NG][kFaRows];
    const int g = (warp - 4) >> 2;
    const int q4 = warp & 3;
    const int row = q4 * 32 + static_cast<int>(lane);
    const int t = tok0 + row / G;
    const int head = kvh * G + row % G;
    const long long qpos = a.chunk_start + t;
    const long long kmax_valid = static_cast<long long>(p_end) * kAttnPage;  // keys past the split are absent
    const long long qpos_min = a.chunk_start + tok0;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const float sc = a.scale_log2;
    {
      // this thread's Q row, slice g (HD/NG bf16 = kQWords packed columns), into TMEM
      uint32_t qv[32];
      const bool live = t < a.chunk_len && nb > 0;
      const uint4* src = reinterpret_cast<const uint4*>(a.q + (static_cast<size_t>(t) * a.n_q_heads + head) * HD +
                                                        g * (HD / NG));
#pragma unroll
      for (int i = 0; i < kQWords / 4; ++i) {
        const uint4 v = live ? __ldg(src + i) : make_uint4(0u, 0u, 0u, 0u);
        qv[4 * i] = v.x;
        qv[4 * i + 1] = v.y;
        qv[4 * i + 2] = v.z;
        qv[4 * i + 3] = v.w;
      }
      if constexpr (kQWords == 32) {
        tmem_st32(tmem + lane_off + Cfg::kColQ + g * kQWords, qv);
      } else {
        static_assert(kQWords == 16, "Q slice per group");
        tmem_st16(tmem + lane_off + Cfg::kColQ + g * kQWords, qv);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(q_ready);
    }
    float m = -INFINITY, l = 0.f;
    const bool tr = a.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && q4 == 0 &&
                    lane == 0;
    long long* trp = tr ? a.trace + 64 + g * 8 * 64 : nullptr;  // [group][block < 64][8]
    for (int j = 0; j < nb; ++j) {
      const int s = j & 1;
      if (tr && j < 64) trp[j * 8] = clock64();
      mbar_wait(&s_full[s], (j >> 1) & 1);
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
      xmax[s][g][row] = mx;
      named_bar_sync(2, 128 * NG);
      if (tr && j < 64) trp[j * 8 + 3] = clock64();
#pragma unroll
      for (int h = 0; h < NG; ++h) mx = fmaxf(mx, xmax[s][h][row]);
      mx *= sc;  // scale > 0: max commutes
      // tcgen05.ld/st are warp-collective (.sync.aligned): when any row of the warp moves its
      // reference max the whole warp runs the rescale pass (factor 1 for the other rows)
      const bool up = mx > m + 8.0f;  // (also true on the first block with a visible key)
      const bool resc = up && m != -INFINITY;
      if (__any_sync(0xffffffffu, resc)) {
        // move the reference max: O (blocks < j, i.e. after PV(j-1)) and l scale by 2^(m - mx)
        mbar_wait(pv_done, (j - 1) & 1);
        tc_fence_after();
        const float f = resc ? ex2_approx(m - mx) : 1.f;
        const uint32_t tO = tmem + lane_off + Cfg::kColO + g * kOCols;
#pragma unroll
        for (int c = 0; c < kOCols / 32; ++c) {
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
      uint32_t pk[32];
#pragma unroll
      for (int i = 0; i < kKeysPerG / 2; ++i) {
        const float2 x = ffma2(make_float2(sv[2 * i], sv[2 * i + 1]), sc2, nb2);
        float2 p;
        if ((i & 7) >= 8 - FA_POLY) {  // FA_POLY of every 8 pairs on the FMA pipe, the rest on MUFU
          p = ex2_poly2(x);
        } else {
          p.x = ex2_approx(x.x);
          p.y = ex2_approx(x.y);
        }
        rs[i & 3] = fadd2(rs[i & 3], p);
        pk[i] = pack_bf16(p.x, p.y);
      }
      if (tr && j < 64) trp[j * 8 + 4] = clock64();
      if constexpr (kKeysPerG / 2 == 32)
        tmem_st32(tS + g * 32, pk);
      else
        tmem_st16(tS + g * 16, pk);
      const float2 rs01 = fadd2(rs[0], rs[1]), rs23 = fadd2(rs[2], rs[3]);
      l += (rs01.x + rs23.x) + (rs01.y + rs23.y);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_ready[s]);
      if (tr && j < 64) trp[j * 8 + 5] = clock64();
    }
    // epilogue: total row sum, then this group's slice of O
    xsum[g][row] = l;
    named_bar_sync(2, 128 * NG);
    l = 0.f;
#pragma unroll
    for (int h = 0; h < NG; ++h) l += xsum[h][row];
    const bool valid = t < a.chunk_len;
    const size_t orow = static_cast<size_t>(t) * a.n_q_heads + head;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    if (nb > 0) {
      mbar_wait(o_final, 0);
      tc_fence_after();
    }
    const uint32_t tO = tmem + lane_off + Cfg::kColO + g * kOCols;
#pragma unroll
    for (int c = 0; c < kOCols / 32; ++c) {
      uint32_t r[32];
      if (nb > 0) {
        tmem_ld32(tO + c * 32, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = 0u;
      }
      if (!valid) continue;
      const int col = g * kOCols + c * 32;
      if (a.num_splits == 1) {
        __nv_bfloat16* dst = a.out + orow * HD + col;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_global_v4(dst + q * 8, pack_bf16(__uint_as_float(r[q * 8]) * inv, __uint_as_float(r[q * 8 + 1]) * inv),
                       pack_bf16(__uint_as_float(r[q * 8 + 2]) * inv, __uint_as_float(r[q * 8 + 3]) * inv),
                       pack_bf16(__uint_as_float(r[q * 8 + 4]) * inv, __uint_as_float(r[q * 8 + 5]) * inv),
                       pack_bf16(__uint_as_float(r[q * 8 + 6]) * inv, __uint_as_float(r[q * 8 + 7]) * inv));
      } else {
        const size_t rows = static_cast<size_t>(a.chunk_len) * a.n_q_heads;
        float4* dst = reinterpret_cast<float4*>(a.part_o + (static_cast<size_t>(split) * rows + orow) * HD + col);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          dst[q] = make_float4(__uint_as_float(r[q * 4]) * inv, __uint_as_float(r[q * 4 + 1]) * inv,
                               __uint_as_float(r[q * 4 + 2]) * inv, __uint_as_float(r[q * 4 + 3]) * inv);
      }
    }
    if (valid && a.num_splits > 1 && g == 0) {
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
