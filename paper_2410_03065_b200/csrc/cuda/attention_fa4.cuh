// Prefix-causal attention, two Q tiles per CTA (ping-pong softmax).
//
// One CTA = 2 x 128 query rows of one KV head (rows are (token, q-head)
// pairs of the GQA group: 2 x 32 tokens at G = 4) over the keys of one split
// of the prefix. The KV block (128 keys = two 64-token pages, TMA-loaded
// through the block table) is fetched once and used by both tiles, and the
// tensor pipe alternates between them:
//
//   tensor pipe:  PV0(j) S0(j+1) | PV1(j) S1(j+1) | PV0(j+1) S0(j+2) | ...
//   softmax WG0:                 [  P0(j+1)      ]                  [ ...
//   softmax WG1:  [  P1(j)      ]                  [  P1(j+1)      ]
//
// so each softmax warpgroup has the other tile's two MMAs (1024 tensor cycles)
// to turn its 128 x 128 score block into P. A warpgroup owns all 128 TMEM
// lanes of its tile: one thread holds a whole 128-key row, so the row max
// needs no cross-warp exchange (the one-tile kernel, attention_tc.cuh, splits
// rows across two warps and pays a named barrier per block).
//
// Per block and tile:
//   S_i = Q_i K^T    tcgen05.mma, A = Q_i (smem, K-major SW128, loaded once
//                    by TMA), B = K block (smem), fp32 accumulator in TMEM
//   P_i = exp2(S_i * scale - m)   thread = row; FFMA2 for the scale/shift,
//                    3/4 of the exponentials on MUFU, 1/4 as a degree-3
//                    polynomial on the FMA pipe (FFMA2), FADD2 row sums; P
//                    (1/2 measured slower: the loop is issue-bound, not MUFU-bound)
//                    written back over S_i as packed bf16 (tcgen05.st)
//   O_i += P_i V     tcgen05.mma, A = P_i from TMEM, B = V block (smem,
//                    MN-major SW128), O_i accumulator in TMEM
// The running max moves (and O_i is rescaled in TMEM) only when it grows by
// more than 2^8. PV_i(j-1) precedes S_i(j) in the in-order tensor pipe, so
// when S_i(j) is complete O_i holds exactly blocks < j and can be rescaled
// without another wait.
//
// TMEM: S0 [0,128) S1 [128,256) O0 [256, 256+HD) O1 [256+HD, 256+2HD).
// Roles (384 threads = three warpgroups): warpgroup 0 is control (warp 0
// TMA: Q once, then K and V blocks in consumption order; warp 1 TMEM owner +
// MMA issuer) and gives its registers away (setmaxnreg 88); warpgroups 1 and
// 2 are the softmax + epilogue of tiles 0 and 1 and take them (setmaxnreg
// 200): a thread keeps its 128 scores in registers with room left for the
// exponential pipeline (warp w accesses TMEM lanes 32*(w%4)..).
//
// Split-KV: every split writes a normalised fp32 partial and its LSE; the
// last split of a (tile pair, KV head) to finish (atomic ticket) combines
// all of them in split order, so the result is independent of arrival order
// and no combine kernel is launched.
#pragma once

#include "attention.cuh"
#include "attention_tc.cuh"
#include "ptx.cuh"

// pairs of every 8 exponentials on the FMA pipe; round (cycles) at 32K for 0..5:
// 3391 / 3270 / 3167-3210 / 3404 / 3521 / 3659 (the one-tile kernel: FA_POLY,
// 0 / 1 / 2 -> 1696 / 1613 / 1622)
#ifndef FA4_POLY
#define FA4_POLY 2
#endif

namespace cake_dev {

constexpr int kF4Threads = 384;

template <int HD>
struct F4Cfg {
  static constexpr int kHalves = HD / 64;                  // 64-element (128 B) K slices
  static constexpr int kTileBytes = 128 * HD * 2;          // Q tile / K block / V block
  static constexpr int kHalfBytes = 128 * 128;             // 128 rows x 64 elements
  static constexpr int kPageHalfBytes = 64 * 128;          // one page x 64 elements
  static constexpr int kKStages = HD == 128 ? 3 : 4;
  static constexpr int kVStages = HD == 128 ? 2 : 4;
  static constexpr int kSmem = (2 + kKStages + kVStages) * kTileBytes + 1024 + 512;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColO = 256;                   // O_i at kColO + i * HD
};

struct F4Args {
  FaArgs fa;
  int* tickets;  // [gridDim.x * gridDim.y] zero at rest: split arrivals per (tile pair, KV head)
  long long* trace;  // debug (nullptr): clock64 stamps of CTA (0,0,0), see tools/fa4_trace.py
};

template <int HD>
__global__ void __launch_bounds__(kF4Threads, 1)
    attn_fa4_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                    const F4Args args) {
  using Cfg = F4Cfg<HD>;
  const FaArgs& a = args.fa;
  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_abort;
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  const bool tcta = args.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
  if (tcta && threadIdx.x == 0) args.trace[2] = clock64();
  const int kvh = blockIdx.y;
  const int split = blockIdx.z;
  const int G = a.n_q_heads / a.n_kv_heads;
  const int tpt = 128 / G;  // tokens per tile
  const int tok0 = blockIdx.x * 2 * tpt;
  const int tok_end = min(tok0 + 2 * tpt, a.chunk_len);  // exclusive
  const long long kv_end = a.chunk_start + tok_end;
  const int n_pages = static_cast<int>((kv_end + kAttnPage - 1) / kAttnPage);
  const int per_split = (n_pages + a.num_splits - 1) / a.num_splits;
  const int p_begin = split * per_split;
  const int p_end = min(n_pages, p_begin + per_split);
  const int nb = p_end > p_begin ? (p_end - p_begin + 1) / 2 : 0;  // 128-key blocks

  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sQ = smem;                                     // [2][tile]
  uint8_t* sK = sQ + 2 * Cfg::kTileBytes;                 // [kKStages][tile]
  uint8_t* sV = sK + Cfg::kKStages * Cfg::kTileBytes;     // [kVStages][tile]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + Cfg::kVStages * Cfg::kTileBytes);
  uint64_t* q_full = bar;                                 // [1]
  uint64_t* k_full = bar + 1;                             // [kKStages]
  uint64_t* k_empty = k_full + Cfg::kKStages;
  uint64_t* v_full = k_empty + Cfg::kKStages;             // [kVStages]
  uint64_t* v_empty = v_full + Cfg::kVStages;
  uint64_t* s_full = v_empty + Cfg::kVStages;             // [2]
  uint64_t* p_ready = s_full + 2;                         // [2]
  uint64_t* o_final = p_ready + 2;                        // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_final + 1);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kv);
    mbar_init(q_full, 1);
    for (int s = 0; s < Cfg::kKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < Cfg::kVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_ready[i], 128);
    }
    mbar_init(o_final, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  // (PDL) everything above overlaps the predecessor's tail; Q / the KV pool are read below
  pdl_wait();
  pdl_trigger();
  if (tcta && threadIdx.x == 0) args.trace[3] = clock64();
  if (threadIdx.x == 0) s_abort = a.abort_flag != nullptr ? *(volatile const int*)a.abort_flag : 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // an aborted (or empty) CTA still takes its split ticket below, so the
  // tickets are back at rest after every launch
  const bool skip = s_abort || tok0 >= a.chunk_len;

  const long long planes = static_cast<long long>(a.n_layers) * 2 * a.n_kv_heads;
  auto page_row = [&](int lp, int kv) -> int32_t {  // first pool row of (page, layer, K|V, kv head)
    const long long ph = a.block_table[lp];
    return static_cast<int32_t>(((ph * planes) + (static_cast<long long>(a.layer) * 2 + kv) * a.n_kv_heads + kvh) * 64);
  };

  int* ticket = args.tickets + blockIdx.y * gridDim.x + blockIdx.x;
  if (skip) {
    // nothing to compute; still take the split ticket so the tickets return to rest
    if (threadIdx.x == 0 && a.num_splits > 1 && atomicAdd(ticket, 1) == a.num_splits - 1) *ticket = 0;
  } else if (warp < 4) {
    setmaxnreg_dec<88>();
    if (warp == 0 && lane == 0 && nb > 0) {
      // ------------------------------------------------ TMA producer: Q tiles once, then K(j), V(j) in the
      // order the MMA warp consumes them (S(j) before PV(j)), so one thread can feed both rings
      mbar_arrive_expect_tx(q_full, 2 * Cfg::kTileBytes);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int h = 0; h < Cfg::kHalves; ++h)
          tma_load_3d(sQ + i * Cfg::kTileBytes + h * Cfg::kHalfBytes, &tm_q, q_full, h * 64, kvh * G, tok0 + i * tpt);
      for (int j = 0; j < nb; ++j) {
        const int lp0 = p_begin + 2 * j;
        const int lp1 = (lp0 + 1 < p_end) ? lp0 + 1 : lp0;  // odd tail: reload page 0 (its keys are masked)
        {
          const int s = j % Cfg::kKStages;
          mbar_wait(&k_empty[s], ((j / Cfg::kKStages) & 1) ^ 1u);
          const int32_t r0 = page_row(lp0, 0), r1 = page_row(lp1, 0);
          mbar_arrive_expect_tx(&k_full[s], Cfg::kTileBytes);
#pragma unroll
          for (int h = 0; h < Cfg::kHalves; ++h) {
            tma_load_2d(sK + s * Cfg::kTileBytes + h * Cfg::kHalfBytes, &tm_kv, &k_full[s], h * 64, r0);
            tma_load_2d(sK + s * Cfg::kTileBytes + h * Cfg::kHalfBytes + Cfg::kPageHalfBytes, &tm_kv, &k_full[s],
                        h * 64, r1);
          }
        }
        {
          const int s = j % Cfg::kVStages;
          mbar_wait(&v_empty[s], ((j / Cfg::kVStages) & 1) ^ 1u);
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
      // converged warp, one elected lane issues (see attn_tc_kernel: a
      // single-lane issuer drains the tensor pipe at every barrier wait)
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, HD, false, true);
      mbar_wait(q_full, 0);
      const bool tr = args.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0;
      if (tr) {
        args.trace[0] = clock64();
        args.trace[1] = nb;
      }
      auto issue_s = [&](int i, int j) {  // S_i = Q_i K(j)^T   (K(j) already waited for)
        const uint32_t q_addr = smem_u32(sQ + i * Cfg::kTileBytes);
        const uint32_t k_addr = smem_u32(sK + (j % Cfg::kKStages) * Cfg::kTileBytes);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk >> 2) * Cfg::kHalfBytes + (kk & 3) * 32;
            umma_bf16_ss(tmem + i * 128, umma_desc_sw128(q_addr + off), umma_desc_sw128(k_addr + off), idesc_s,
                         kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[i]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int i, int j) {  // O_i += P_i V(j)   (V(j) already waited for)
        if (tr && j < 64) args.trace[64 + i * 8 * 64 + j * 8 + 6] = clock64();
        mbar_wait(&p_ready[i], j & 1);
        tc_fence_after();
        if (tr && j < 64) args.trace[64 + i * 8 * 64 + j * 8 + 7] = clock64();
        const uint32_t v_addr = smem_u32(sV + (j % Cfg::kVStages) * Cfg::kTileBytes);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 128 / 16; ++kk) {
            const uint64_t bdesc = umma_desc_sw128_mn(v_addr + kk * 16 * 128, Cfg::kHalfBytes, 1024);
            umma_bf16_ts(tmem + Cfg::kColO + i * HD, tmem + i * 128 + kk * 8, bdesc, idesc_o,
                         (j > 0 || kk > 0) ? 1u : 0u);
          }
        }
        __syncwarp();
      };
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) umma_commit(bar);
        __syncwarp();
      };
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      commit(&k_empty[0]);
      for (int j = 0; j < nb; ++j) {
        const bool more = j + 1 < nb;
        mbar_wait(&v_full[j % Cfg::kVStages], (j / Cfg::kVStages) & 1);
        issue_pv(0, j);
        if (more) {
          mbar_wait(&k_full[(j + 1) % Cfg::kKStages], ((j + 1) / Cfg::kKStages) & 1);
          tc_fence_after();
          issue_s(0, j + 1);  // after PV0(j): S0(j+1) overwrites P0(j) in TMEM (in-order pipe)
        }
        issue_pv(1, j);
        commit(&v_empty[j % Cfg::kVStages]);
        if (more) {
          issue_s(1, j + 1);
          commit(&k_empty[(j + 1) % Cfg::kKStages]);
        }
      }
      commit(o_final);
    }
  } else {
    setmaxnreg_inc<200>();
    // ------------------------------------------------ softmax + epilogue of tile i
    const int i = (warp - 4) >> 2;
    const int q4 = warp & 3;
    const int row = q4 * 32 + static_cast<int>(lane);
    const int t = tok0 + i * tpt + row / G;
    const int head = kvh * G + row % G;
    const long long qpos = a.chunk_start + t;
    const long long kmax_valid = static_cast<long long>(p_end) * kAttnPage;  // keys past the split are absent
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t tS = tmem + lane_off + i * 128;
    const uint32_t tO = tmem + lane_off + Cfg::kColO + i * HD;
    const float sc = a.scale_log2;
    const float2 sc2 = make_float2(sc, sc);
    float m = -INFINITY, l = 0.f;
    const bool tr = args.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && q4 == 0 &&
                    lane == 0;
    long long* trp = tr ? args.trace + 64 + i * 8 * 64 : nullptr;  // [tile][block < 64][8]
    for (int j = 0; j < nb; ++j) {
      if (tr && j < 64) trp[j * 8 + 0] = clock64();
      mbar_wait(&s_full[i], j & 1);
      tc_fence_after();
      if (tr && j < 64) trp[j * 8 + 1] = clock64();
      // the row's 128 scores; their registers are reused for the packed P below
      uint32_t su[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&su[c * 32]));
      tmem_ld_wait();
      if (tr && j < 64) trp[j * 8 + 2] = clock64();
      const long long kbase = static_cast<long long>(p_begin + 2 * j) * kAttnPage;
      // last visible key of this row relative to the block (causal, and the split's end)
      const long long lim64 = min(qpos, kmax_valid - 1) - kbase;
      if (lim64 < 127) {
        const int lim = static_cast<int>(max(lim64, -1LL));
#pragma unroll
        for (int e = 0; e < 128; ++e)
          if (e > lim) su[e] = __float_as_uint(-INFINITY);
      }
      float mxv[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) mxv[c] = fmaxf(__uint_as_float(su[2 * c]), __uint_as_float(su[2 * c + 1]));
#pragma unroll
      for (int e = 16; e < 128; e += 16)
#pragma unroll
        for (int c = 0; c < 8; ++c)
          mxv[c] = fmaxf(mxv[c], fmaxf(__uint_as_float(su[e + 2 * c]), __uint_as_float(su[e + 2 * c + 1])));
      const float mx = fmaxf(fmaxf(fmaxf(mxv[0], mxv[1]), fmaxf(mxv[2], mxv[3])),
                             fmaxf(fmaxf(mxv[4], mxv[5]), fmaxf(mxv[6], mxv[7]))) * sc;  // scale > 0: max commutes
      // tcgen05.ld/st are warp-collective (.sync.aligned): when any row of the warp moves its
      // reference max the whole warp runs the rescale pass (factor 1 for the other rows)
      const bool up = mx > m + 8.0f;  // (also true on the first block with a visible key)
      const bool resc = up && m != -INFINITY;
      if (__any_sync(0xffffffffu, resc)) {
        // O_i holds blocks < j (PV_i(j-1) completed before S_i(j)): rescale it and l by 2^(m - mx)
        const float f = resc ? ex2_approx(m - mx) : 1.f;
        const float2 f2 = make_float2(f, f);
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tO + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float2 v = fmul2(make_float2(__uint_as_float(r[e]), __uint_as_float(r[e + 1])), f2);
            r[e] = __float_as_uint(v.x);
            r[e + 1] = __float_as_uint(v.y);
          }
          tmem_st32(tO + c * 32, r);
        }
        tmem_st_wait();
        l *= f;
      }
      if (up) m = mx;
      if (tr && j < 64) trp[j * 8 + 3] = clock64();
      const float nb_ = (m == -INFINITY) ? 0.f : -m;
      const float2 nb2 = make_float2(nb_, nb_);
      float2 rs[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      // P in key order, packed in place: word w (keys 2w, 2w+1) lands in su[w], never ahead of a read
#pragma unroll
      for (int w = 0; w < 64; ++w) {
        const float2 x = ffma2(make_float2(__uint_as_float(su[2 * w]), __uint_as_float(su[2 * w + 1])), sc2, nb2);
        float2 p;
        if ((w & 7) >= 8 - FA4_POLY) {  // FA4_POLY of every 8 pairs on the FMA pipe
          p = ex2_poly2(x);
        } else {
          p.x = ex2_approx(x.x);
          p.y = ex2_approx(x.y);
        }
        rs[w & 3] = fadd2(rs[w & 3], p);
        su[w] = pack_bf16(p.x, p.y);
      }
      if (tr && j < 64) trp[j * 8 + 4] = clock64();
      tmem_st32(tS, *reinterpret_cast<uint32_t(*)[32]>(&su[0]));
      tmem_st32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&su[32]));
      const float2 rs01 = fadd2(rs[0], rs[1]), rs23 = fadd2(rs[2], rs[3]);
      l += (rs01.x + rs23.x) + (rs01.y + rs23.y);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_ready[i]);
      if (tr && j < 64) trp[j * 8 + 5] = clock64();
    }
    if (tcta && warp == 4 && lane == 0) args.trace[4] = clock64();
    // ---- epilogue: O_i / l -> output (or this split's partial + LSE)
    const bool valid = t < a.chunk_len;
    const size_t orow = static_cast<size_t>(t) * a.n_q_heads + head;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const size_t rows = static_cast<size_t>(a.chunk_len) * a.n_q_heads;
    if (nb > 0) {
      mbar_wait(o_final, 0);
      tc_fence_after();
    }
    // split partials live in a CTA-private slot [col / 4][row][4] per tile: for a fixed
    // column quad a warp's 32 rows are 512 contiguous bytes, written and read back as float4
    const size_t n_cta = static_cast<size_t>(gridDim.x) * gridDim.y;
    const size_t cta_id = static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x;
    auto part_slot = [&](int sp) { return a.part_o + ((sp * n_cta + cta_id) * 2 + i) * (HD * 128); };
    auto lse_slot = [&](int sp) { return a.part_lse + ((sp * n_cta + cta_id) * 2 + i) * 128; };
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t r[32];
      if (nb > 0) {
        tmem_ld32(tO + c * 32, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) r[e] = 0u;
      }
      const int col = c * 32;
      if (a.num_splits == 1) {
        if (!valid) continue;
        __nv_bfloat16* dst = a.out + orow * HD + col;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_global_v4(dst + q * 8, pack_bf16(__uint_as_float(r[q * 8]) * inv, __uint_as_float(r[q * 8 + 1]) * inv),
                       pack_bf16(__uint_as_float(r[q * 8 + 2]) * inv, __uint_as_float(r[q * 8 + 3]) * inv),
                       pack_bf16(__uint_as_float(r[q * 8 + 4]) * inv, __uint_as_float(r[q * 8 + 5]) * inv),
                       pack_bf16(__uint_as_float(r[q * 8 + 6]) * inv, __uint_as_float(r[q * 8 + 7]) * inv));
      } else {
        float4* dst = reinterpret_cast<float4*>(part_slot(split)) + static_cast<size_t>(col / 4) * 128 + row;
#pragma unroll
        for (int e = 0; e < 8; ++e)
          __stcg(dst + e * 128, make_float4(__uint_as_float(r[4 * e]) * inv, __uint_as_float(r[4 * e + 1]) * inv,
                                            __uint_as_float(r[4 * e + 2]) * inv, __uint_as_float(r[4 * e + 3]) * inv));
      }
    }
    if (a.num_splits > 1) {
      __stcg(lse_slot(split) + row, l > 0.f ? m + __log2f(l) : -INFINITY);
      __threadfence();
      if (tcta && warp == 4 && lane == 0) args.trace[5] = clock64();
      // ---- the last split of this (tile pair, KV head) to arrive combines all partials in split order
      named_bar_sync(1, 256);
      if (warp == 4 && lane == 0) {
        const int prev = atomicAdd(ticket, 1);
        s_last = prev == a.num_splits - 1;
        if (s_last) *ticket = 0;  // rest state for the next launch (stream-ordered)
      }
      named_bar_sync(1, 256);
      if (tcta && warp == 4 && lane == 0) args.trace[6] = clock64();
      if (s_last && valid) {
        __threadfence();
        float mx = -INFINITY;
        for (int sp = 0; sp < a.num_splits; ++sp) mx = fmaxf(mx, __ldcg(lse_slot(sp) + row));
        float wsum = 0.f;
        for (int sp = 0; sp < a.num_splits; ++sp) {
          const float lse = __ldcg(lse_slot(sp) + row);
          wsum += (lse == -INFINITY) ? 0.f : exp2f(lse - mx);
        }
        const float winv = wsum > 0.f ? 1.f / wsum : 0.f;
        __nv_bfloat16* dst = a.out + orow * HD;
#pragma unroll 1
        for (int half = 0; half < HD / 64; ++half) {  // 64 accumulators at a time
          float acc[64];
#pragma unroll
          for (int e = 0; e < 64; ++e) acc[e] = 0.f;
          for (int sp = 0; sp < a.num_splits; ++sp) {
            const float lse = __ldcg(lse_slot(sp) + row);
            const float w = (lse == -INFINITY) ? 0.f : exp2f(lse - mx);
            const float4* po = reinterpret_cast<const float4*>(part_slot(sp)) + static_cast<size_t>(half * 16) * 128 + row;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float4 v = __ldcg(po + e * 128);
              acc[4 * e] += w * v.x;
              acc[4 * e + 1] += w * v.y;
              acc[4 * e + 2] += w * v.z;
              acc[4 * e + 3] += w * v.w;
            }
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            st_global_v4(dst + half * 64 + q * 8, pack_bf16(acc[8 * q] * winv, acc[8 * q + 1] * winv),
                         pack_bf16(acc[8 * q + 2] * winv, acc[8 * q + 3] * winv),
                         pack_bf16(acc[8 * q + 4] * winv, acc[8 * q + 5] * winv),
                         pack_bf16(acc[8 * q + 6] * winv, acc[8 * q + 7] * winv));
        }
      }
    }
  }
  if (tcta && warp == 4 && lane == 0) args.trace[7] = clock64();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem);
  }
  if (tcta && threadIdx.x == 0) args.trace[8] = clock64();
}

}  // namespace cake_dev
