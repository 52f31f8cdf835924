// Host side of the C-ABI CUDA layer (include/cake_cuda.h): device memory,
// streams/events, the Llama-shaped model (seeded weights, paged KV pool,
// activation scratch, TMA descriptors) and the launch sequence of one chunk.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "attention.cuh"
#include "attention_tc.cuh"
#include "attention_alt.cuh"
#ifdef CAKE_ATTN_VARIANTS  // experiment kernels (A/B only): make ATTN_VARIANTS=1
#include "attention_fa4.cuh"
#include "attention_dec.cuh"
#endif
#include "cake_cuda.h"
#include "elementwise.cuh"
#include "tp_peer.cuh"
#include "gemm.cuh"
#include "gemm2.cuh"
#include "gemm2c.cuh"
#include "skinny.cuh"
#include "decode_chain.cuh"

using namespace cake_dev;
using bf16 = __nv_bfloat16;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CK(expr)                                                                           \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(CAKE_ECUDA + static_cast<int>(e_), "%s: %s (%s:%d)", #expr,             \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                             \
  } while (0)

#define CKL()                                                                              \
  do {                                                                                     \
    cudaError_t e_ = cudaGetLastError();                                                   \
    if (e_ != cudaSuccess)                                                                 \
      return fail(CAKE_ECUDA + static_cast<int>(e_), "launch: %s (%s:%d)",                 \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                             \
  } while (0)

#define CKS(expr)                                                                          \
  do {                                                                                     \
    int s_ = (expr);                                                                       \
    if (s_ != CAKE_OK) return s_;                                                          \
  } while (0)

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// Programmatic dependent launch for the chunk's kernel chain (every kernel
// launched here calls pdl_wait() before touching its predecessor's outputs):
// the next kernel's CTAs become resident and run their prologue (barrier
// init, TMEM alloc, descriptor prefetch) while the previous kernel drains.
// A/B switches for measurements (cake_set_experiment); the defaults are the product.
int g_exp[CAKE_EXP_COUNT] = {1 /*PDL*/, 1 /*FUSED_NORM*/, 1 /*ATTN_MAX_WAVES*/, 0 /*GEMM_NOSPLIT*/, 1 /*DEC_CHAIN*/,
                              1 /*TP_OVERLAP*/};

// cake_set_experiment(CAKE_EXP_PDL, 0) turns programmatic dependent launch off.
bool pdl_enabled() { return g_exp[CAKE_EXP_PDL] != 0; }

template <typename... KArgs, typename... Args>
cudaError_t launch_chain(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster,
                         Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ------------------------------------------------------------ TMA maps
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Row-major bf16 [rows, cols] with a (64 x box_rows) SW128 box.
int make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(CAKE_ESTATE, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t elem[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                  elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CAKE_EINVAL, "tensor map encode failed (%d) rows=%llu cols=%llu", (int)r,
                                     (unsigned long long)rows, (unsigned long long)cols);
  return CAKE_OK;
}

// Row-major fp32 [rows, cols] with a (32 x box_rows) SW128 box (128-B rows).
int make_map_f32(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(CAKE_ESTATE, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t elem[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, elem,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CAKE_EINVAL, "fp32 tensor map encode failed (%d)", (int)r);
  return CAKE_OK;
}

// bf16 3-D tensor [d2][d1][d0] (d0 contiguous), SW128, box (64, b1, b2).
int make_map_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b1, uint32_t b2) {
  auto fn = encode_fn();
  if (!fn) return fail(CAKE_ESTATE, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * 2, d0 * d1 * 2};
  cuuint32_t box[3] = {64, b1, b2};
  cuuint32_t elem[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, elem,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CAKE_EINVAL, "3-D tensor map encode failed (%d)", (int)r);
  return CAKE_OK;
}

int g_num_sms = 0;
int g_sm_limit = 0;  // > 0: the compute stream owns this many SMs (green context); launches size to it
int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_sm_limit > 0 ? std::min(g_sm_limit, g_num_sms) : g_num_sms;
}

// Stream-K / split-K scratch, one set per launching stream: launches on one
// stream reuse it in stream order (the epoch keeps flags of consecutive
// launches apart without a reset); concurrent contexts (one compute stream
// each) never share it.
struct StreamKScratch {
  float* ws = nullptr;
  int* flags = nullptr;
  int epoch = 0;
  float* tail_ws = nullptr;  // gate/up tail-split partials (whole_tiles == 2)
  size_t tail_floats = 0;
};
std::mutex g_sk_mu;
std::unordered_map<cudaStream_t, StreamKScratch> g_sk;
int g_gemm_schedule = 0;  // 0 whole tiles (+ exact split-K when tiles < SM pairs), 1 stream-K
int g_gemm_2sm = 1;       // 1: M > 128 projections use the 2-SM (cta_group::2) kernel
int g_gemm_2sm_n128 = 1;  // O / down (N tiles of 128) on CTA pairs: down 59.9 -> 54.0 us at M = 512
int g_gemm_hints = 3;     // L2 policy of the operand loads (GemmArgs::l2_hints)
int g_gemm_tail_split = 1;  // gate/up: split the short last round along K (swiglu_tail_kernel)
int g_gemm_prefetch = -1;   // gemm2c: weight k-blocks requested before the PDL wait (-1 whole ring)
int g_gemm_pairs = 2;       // > 1: N-128/192 projections in clusters of this many CTA pairs sharing A (gemm2c)
int g_gemm_qkv192 = 1;      // QKV on CTA-pair tiles of N 192 (rope-unit weight rows) when the rows tile

// Tail-split partials of whole_tiles == 2 launches (stream-ordered reuse).
int tail_scratch(float** ws, size_t floats, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_sk_mu);
  StreamKScratch& k = g_sk[s];
  if (floats > k.tail_floats) {
    if (k.tail_ws) CK(cudaFree(k.tail_ws));
    CK(cudaMalloc(&k.tail_ws, floats * sizeof(float)));
    k.tail_floats = floats;
  }
  *ws = k.tail_ws;
  return CAKE_OK;
}

int streamk_scratch(float** ws, int** flags, int* epoch, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_sk_mu);
  StreamKScratch& k = g_sk[s];
  if (!k.ws) {
    // slots for the whole device, not the current SM budget: a stream handle
    // can be reused by a later context with a larger budget
    num_sms();
    const size_t slots = static_cast<size_t>(g_num_sms);
    CK(cudaMalloc(&k.ws, slots * kGemmBlockM * 256 * sizeof(float)));
    CK(cudaMalloc(&k.flags, slots * sizeof(int)));
    CK(cudaMemset(k.flags, 0, slots * sizeof(int)));
  }
  *ws = k.ws;
  *flags = k.flags;
  *epoch = ++k.epoch;
  return CAKE_OK;
}

// Cluster size for a chunk of M rows: its m-blocks share every weight k-block.
int g_gemm_cluster = 0;  // 1-SM kernel: multicast weight k-blocks across the chunk's m-blocks
int cluster_size_for(int M) {
  const int mb = (M + kGemmBlockM - 1) / kGemmBlockM;
  if (!g_gemm_cluster) return 1;
  return mb <= 1 ? 1 : (mb == 2 ? 2 : 4);
}
int cs_index(int cs) { return cs == 1 ? 0 : (cs == 2 ? 1 : 2); }

template <int BN, int EPI>
int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, GemmArgs a, cudaStream_t s) {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_tc_kernel<BN, EPI>;
  static bool configured = false;
  static int max_clusters[3] = {0, 0, 0};
  static int clusters_for_sms = 0;  // the SM budget max_clusters was computed for
  if (clusters_for_sms != num_sms()) {
    max_clusters[0] = max_clusters[1] = max_clusters[2] = 0;
    clusters_for_sms = num_sms();
  }
  if (!configured) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes));
    configured = true;
  }
  a.num_m_blocks = (a.M + kGemmBlockM - 1) / kGemmBlockM;
  a.num_n_blocks = a.N / BN;
  a.num_k_blocks = a.K / kGemmBlockK;
  a.cs = cluster_size_for(a.M);
  const int ci = cs_index(a.cs);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (max_clusters[ci] == 0) {
    cfg.gridDim = dim3(a.cs * 16);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = num_sms() / a.cs;
    }
    max_clusters[ci] = std::min(n, num_sms() / a.cs);
  }
  const int m_groups = (a.num_m_blocks + a.cs - 1) / a.cs;
  const long long units = static_cast<long long>(m_groups) * a.num_n_blocks * a.num_k_blocks;
  a.whole_tiles = g_gemm_schedule == 0;
  // stream-K: every cluster gets >= 8 k-blocks (>= 1 unit, so none is empty); all clusters co-resident
  const long long work = a.whole_tiles ? static_cast<long long>(m_groups) * a.num_n_blocks : units / 8;
  const int clusters = static_cast<int>(std::max<long long>(1, std::min<long long>(max_clusters[ci], work)));
  CKS(streamk_scratch(&a.sk_ws, &a.sk_flags, &a.epoch, s));
  CK(launch_chain(kern, dim3(clusters * a.cs), dim3(kGemmThreads), Cfg::kSmemBytes, s, a.cs, ta, tb, a));
  return CAKE_OK;
}

// 2-SM GEMM: pairs of CTAs on 256 x 256 tiles. Few tiles (O / down at M = 512:
// 32) are split along K into S equal parts so the pairs fill the GPU; the
// k = 0 part owns the tile and adds the others (deterministic order).
template <int BLOCK_N, int EPI>
int launch_gemm2(const CUtensorMap& ta, const CUtensorMap& tb_half, GemmArgs a, cudaStream_t s) {
  using Cfg = Gemm2Cfg<BLOCK_N>;
  auto kern = gemm2_tc_kernel<BLOCK_N, EPI>;
  static bool configured = false;
  static int max_pairs = 0;
  static int pairs_for_sms = 0;  // the SM budget max_pairs was computed for
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (!configured) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes));
    configured = true;
  }
  if (pairs_for_sms != num_sms()) {
    cfg.gridDim = dim3(32);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = num_sms() / 2;
    }
    max_pairs = std::min(n, num_sms() / 2);
    pairs_for_sms = num_sms();
  }
  a.num_m_blocks = (a.M + kGemmBlockM - 1) / kGemmBlockM;
  a.num_n_blocks = a.N / BLOCK_N;
  a.num_k_blocks = a.K / kGemmBlockK;
  a.cs = 2;
  const int m_pairs = (a.num_m_blocks + 1) / 2;
  const int tiles = m_pairs * a.num_n_blocks;
  int pairs;
  if (g_gemm_schedule == 1) {
    a.whole_tiles = 0;
    const long long units = static_cast<long long>(tiles) * a.num_k_blocks;
    pairs = static_cast<int>(std::max<long long>(1, std::min<long long>(max_pairs, units / 8)));
  } else {
    // split parts run concurrently (the owner waits for its partner): keep
    // tiles * split within the SM pairs so every part is resident together
    const int pair_budget = g_exp[CAKE_EXP_GEMM_NOSPLIT] ? 0 : num_sms() / 2;  // experiment: one pair per tile
    int split = 1;
    while (tiles * (split + 1) <= pair_budget && a.num_k_blocks % (split + 1) == 0 &&
           a.num_k_blocks / (split + 1) >= 8)
      ++split;
    a.whole_tiles = split == 1 ? 1 : 0;
    pairs = split == 1 ? std::min(tiles, max_pairs) : tiles * split;
    // gate/up (224 tiles on 74 pairs at M = 512): the short last round split along K,
    // its parts summed + SwiGLU'd by swiglu_tail_kernel
    if constexpr (EPI == kEpiSwiglu && BLOCK_N == 256) {
      const int r = tiles % pairs;
      if (split == 1 && g_gemm_tail_split && tiles > pairs && r > 0 && 2 * r <= pairs && a.num_k_blocks >= 16) {
        a.whole_tiles = 2;
        CKS(tail_scratch(&a.tail_ws, static_cast<size_t>(r) * tail_parts(r, pairs) * 256 * 256, s));
      }
    }
  }
  CKS(streamk_scratch(&a.sk_ws, &a.sk_flags, &a.epoch, s));
  CK(launch_chain(kern, dim3(2 * pairs), dim3(kGemmThreads), Cfg::kSmemBytes, s, 2, ta, tb_half, a));
  if constexpr (EPI == kEpiSwiglu) {
    if (a.whole_tiles == 2) {
      const int r = tiles % pairs;
      CK(launch_chain(swiglu_tail_kernel, dim3(r * 256), dim3(128), 0, s, 1, a, tiles - r, r,
                      tail_parts(r, pairs)));
    }
  }
  return CAKE_OK;
}

// 2-SM GEMM in clusters of NP pairs sharing the A k-block (gemm2c.cuh): one
// tile (m-pair x NP n-blocks) per cluster per round, no split. ta_piece is the
// A map with 128 / NP-row boxes.
template <int BLOCK_N, int EPI, int NP>
int launch_gemm2c(const CUtensorMap& ta_piece, const CUtensorMap& tb_half, const CUtensorMap* om, GemmArgs a,
                  cudaStream_t s) {
  using Cfg = Gemm2Cfg<BLOCK_N>;
  auto kern = gemm2c_tc_kernel<BLOCK_N, EPI, NP>;
  static bool configured = false;
  static int max_clusters = 0, for_sms = 0;
  if (!configured) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes));
    if (NP * 2 > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured = true;
  }
  if (for_sms != num_sms()) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2 * NP;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = Cfg::kSmemBytes;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(2 * NP * 16);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = num_sms() / (2 * NP);
    }
    max_clusters = std::min(n, num_sms() / (2 * NP));
    for_sms = num_sms();
  }
  a.num_m_blocks = (a.M + kGemmBlockM - 1) / kGemmBlockM;
  a.num_n_blocks = a.N / BLOCK_N;
  a.num_k_blocks = a.K / kGemmBlockK;
  a.cs = 2 * NP;
  a.whole_tiles = 1;
  const int tiles = ((a.num_m_blocks + 1) / 2) * (a.num_n_blocks / NP);
  const int clusters = std::max(1, std::min(tiles, max_clusters));
  // output maps (h fp32, bf16(h)): the staged residual epilogue, one tile per CTA
  a.prefetch = g_gemm_prefetch;
  // (the staging boxes reuse the operand ring: 4 x 16 KB of h + 2 x 16 KB of bf16(h))
  constexpr bool ring_fits = Cfg::kStages * Cfg::kStageBytes >= 6 * 128 * 128;
  a.staged = (ring_fits && EPI == kEpiResid && BLOCK_N == 128 && om != nullptr && tiles <= clusters) ? 1 : 0;
  const CUtensorMap& th = a.staged ? om[0] : ta_piece;
  const CUtensorMap& tx = a.staged ? om[1] : ta_piece;
  CK(launch_chain(kern, dim3(2 * NP * clusters), dim3(kGemmThreads), Cfg::kSmemBytes, s, 2 * NP, ta_piece, tb_half,
                  th, tx, a));
  return CAKE_OK;
}

// Whether the cluster kernel takes this projection: N-128/192 pair tiles whose
// n-blocks group by NP and whose cluster tiles fit one round of the GPU.
bool use_gemm2c(int bn, int M, int N, int np) {
  if (np <= 1 || M <= kGemmBlockM || (bn != 128 && bn != 192) || N % bn) return false;
  const int nb = N / bn;
  if (nb % np) return false;
  const int tiles = ((M + 255) / 256) * (nb / np);
  return tiles <= num_sms() / (2 * np);
}

template <int BLOCK_N, int EPI>
int launch_gemm2c_np(const CUtensorMap* ta3, const CUtensorMap& tb_half, const CUtensorMap* om, const GemmArgs& a,
                     cudaStream_t s) {
  if (g_gemm_pairs == 4) return launch_gemm2c<BLOCK_N, EPI, 4>(ta3[2], tb_half, om, a, s);
  return launch_gemm2c<BLOCK_N, EPI, 2>(ta3[1], tb_half, om, a, s);
}

long long* g_gemm_trace = nullptr;  // debug: per-launch stamp slots (cake_gemm_debug_trace)
int g_gemm_trace_n = 0, g_gemm_trace_cap = 0;

// om: optional output maps of a residual projection ([0] h fp32 32-col boxes,
// [1] bf16(h) 64-col boxes, 128 rows each) for the staged epilogue.
int gemm_dispatch(int bn, int epi, const CUtensorMap* ta3, const CUtensorMap* tb3, const GemmArgs& a_in,
                  cudaStream_t s, const CUtensorMap* om = nullptr) {
  const CUtensorMap& ta = ta3[0];
  GemmArgs a = a_in;
  if (g_gemm_trace != nullptr && g_gemm_trace_n < g_gemm_trace_cap) a.trace = g_gemm_trace + 32LL * g_gemm_trace_n++;
  a.l2_hints = g_gemm_hints;
  // Chunks of more than 128 rows run on CTA pairs (cta_group::2): the pair's
  // MMA is M = 256 x N = bn, each CTA receiving its 128 rows of A and bn/2 rows
  // of the weight tile (24 KB per 64-deep k-block at bn = 128 instead of the
  // 1-SM tile's 32 KB: the M = 512 projections are bound by L2 -> SM delivery).
  // At M = 512: QKV / gate-up 48 / 224 pair tiles of N 256, O / down 64 pair
  // tiles of N 128 (down 54.0 us against 59.9 on 1-SM 128 x 128 tiles, O 20.8
  // against 21.6; schedule bit 8 restores the 1-SM tiles).
  if (g_gemm_2sm && use_gemm2c(bn, a.M, a.N, g_gemm_pairs)) {
    // B maps: index 1 holds bn/2-row boxes (the pair kernels' weight halves)
    if (bn == 192) {
      switch (epi) {
        case kEpiBf16: return launch_gemm2c_np<192, kEpiBf16>(ta3, tb3[1], nullptr, a, s);
        case kEpiQkv: return launch_gemm2c_np<192, kEpiQkv>(ta3, tb3[1], nullptr, a, s);
      }
    } else {
      switch (epi) {
        case kEpiBf16: return launch_gemm2c_np<128, kEpiBf16>(ta3, tb3[1], nullptr, a, s);
        case kEpiF32: return launch_gemm2c_np<128, kEpiF32>(ta3, tb3[1], nullptr, a, s);
        case kEpiResid: return launch_gemm2c_np<128, kEpiResid>(ta3, tb3[1], om, a, s);
      }
    }
  }
  if (bn == 192) {
    if (a.M <= kGemmBlockM || a.N % bn) return fail(CAKE_EINVAL, "gemm: N-192 tiles need M > 128 and N %% 192 == 0");
    switch (epi) {
      case kEpiBf16: return launch_gemm2<192, kEpiBf16>(ta, tb3[1], a, s);
      case kEpiF32: return launch_gemm2<192, kEpiF32>(ta, tb3[1], a, s);
      case kEpiResid: return launch_gemm2<192, kEpiResid>(ta, tb3[1], a, s);
      case kEpiQkv: return launch_gemm2<192, kEpiQkv>(ta, tb3[1], a, s);
    }
    return fail(CAKE_EINVAL, "gemm: unsupported epi %d for N-192 tiles", epi);
  }
  if (g_gemm_2sm && a.M > kGemmBlockM && a.N % bn == 0 && (bn == 256 || g_gemm_2sm_n128)) {
    // B maps: index k holds box rows bn >> k; the pair kernel loads bn/2-row halves
    const CUtensorMap& half = tb3[1];
    if (bn == 256) {
      switch (epi) {
        case kEpiBf16: return launch_gemm2<256, kEpiBf16>(ta, half, a, s);
        case kEpiF32: return launch_gemm2<256, kEpiF32>(ta, half, a, s);
        case kEpiResid: return launch_gemm2<256, kEpiResid>(ta, half, a, s);
        case kEpiSwiglu: return launch_gemm2<256, kEpiSwiglu>(ta, half, a, s);
        case kEpiQkv: return launch_gemm2<256, kEpiQkv>(ta, half, a, s);
      }
    } else if (epi != kEpiSwiglu) {
      switch (epi) {
        case kEpiBf16: return launch_gemm2<128, kEpiBf16>(ta, half, a, s);
        case kEpiF32: return launch_gemm2<128, kEpiF32>(ta, half, a, s);
        case kEpiResid: return launch_gemm2<128, kEpiResid>(ta, half, a, s);
        case kEpiQkv: return launch_gemm2<128, kEpiQkv>(ta, half, a, s);
      }
    }
  }
  const CUtensorMap& tb = tb3[cs_index(cluster_size_for(a.M))];
  if (bn == 256) {
    switch (epi) {
      case kEpiBf16: return launch_gemm<256, kEpiBf16>(ta, tb, a, s);
      case kEpiF32: return launch_gemm<256, kEpiF32>(ta, tb, a, s);
      case kEpiResid: return launch_gemm<256, kEpiResid>(ta, tb, a, s);
      case kEpiSwiglu: return launch_gemm<256, kEpiSwiglu>(ta, tb, a, s);
      case kEpiQkv: return launch_gemm<256, kEpiQkv>(ta, tb, a, s);
    }
  } else if (bn == 128) {
    switch (epi) {
      case kEpiBf16: return launch_gemm<128, kEpiBf16>(ta, tb, a, s);
      case kEpiF32: return launch_gemm<128, kEpiF32>(ta, tb, a, s);
      case kEpiResid: return launch_gemm<128, kEpiResid>(ta, tb, a, s);
      case kEpiQkv: return launch_gemm<128, kEpiQkv>(ta, tb, a, s);
    }
  }
  return fail(CAKE_EINVAL, "gemm: unsupported block_n=%d epi=%d", bn, epi);
}

int launch_grid_for(long long work, int threads) {
  long long blocks = (work + threads - 1) / threads;
  long long cap = static_cast<long long>(num_sms()) * 8;
  return static_cast<int>(std::max<long long>(1, std::min(blocks, cap)));
}

}  // namespace

// ====================================================================== model
struct LayerWeights {
  bf16* wqkv = nullptr;  // [(nq + 2 nkv) * hd, H]   local heads
  bf16* wo = nullptr;    // [H, nq * hd]             local input columns
  bf16* wgu = nullptr;   // [2 * F, H]               gate|up interleaved per 128 rows
  bf16* wd = nullptr;    // [H, F]                   local input columns
  bf16* ln1 = nullptr;
  bf16* ln2 = nullptr;
  CUtensorMap m_qkv[3], m_o[3], m_gu[3], m_d[3];  // B box = BLOCK_N / cluster size (1, 2, 4)
  CUtensorMap m_qkv192[3];                         // QKV, box 96 rows (the pair kernel's N-192 halves)
};

struct ProfPair {
  int kind;
  cudaEvent_t a, b;
  double flops, bytes;
};

struct cake_model {
  cake_model_config cfg{};
  int nq = 0, nkv = 0, F = 0, hd = 0, H = 0, L = 0;
  int qkv_rows = 0;
  int bn_qkv = 256;
  std::vector<LayerWeights> layers;
  void* weight_arena = nullptr;
  size_t weight_bytes = 0;
  bf16* embed = nullptr;
  bf16* final_norm = nullptr;
  bf16* lm_head = nullptr;
  bf16* pool = nullptr;
  size_t pool_bytes = 0;
  int n_logical_pages = 0, n_phys_pages = 0;
  float2* rope = nullptr;
  int rows_cap = 0;  // scratch rows (multiple of 128)
  float* h = nullptr;
  bf16* xn = nullptr;
  bf16* q = nullptr;
  bf16* attn = nullptr;
  bf16* act = nullptr;
  float* part_o = nullptr;
  float* part_lse = nullptr;
  int max_splits = 16;
  size_t part_rows_cap = 0;  // splits * chunk rows * local q heads the partials hold
  float* tp_buf = nullptr;  // fp32 partial sums for the TP all-reduce
  float* ss = nullptr;      // fused RMSNorm: [H / 128][rows_cap] partial sums of squares of the residual rows
  unsigned* q8_ws = nullptr;  // quant8 encode: ordered min/max keys
  unsigned* dec_bar = nullptr;  // first-token chain kernel: grid barrier (one monotone 64-bit arrival counter)
  CUtensorMap a_xn[3], a_attn[3], a_act[3];
  CUtensorMap out_h[2];  // staged residual epilogue: h (fp32, 32-col boxes), xn = bf16(h) (64-col boxes)  // activation maps, boxes of 128 / 64 / 32 rows (gemm2c pieces)
  CUtensorMap tm_q, tm_kv;  // attention: Q rows of a GQA group, paged K/V pool
  int attn_impl = 0;        // 0 product dispatch, 1 mma.sync (cross-check), 2 one-tile / 3 two-tile tcgen05 only
  int* attn_tickets = nullptr;  // split arrival tickets of the two-tile kernel (zero at rest)
  ncclComm_t comm = nullptr;
  // peer-memory TP (tp_peer.cuh): IPC mappings of every rank's exchange buffers
  bool peer_tp = false;
  unsigned long long* tp_flags = nullptr;  // own flag block (kTpFlagWords)
  void* peer_part[kTpMaxRanks]{};
  bf16* peer_xn[kTpMaxRanks]{};
  float* peer_h[kTpMaxRanks]{};
  float* tp_logits = nullptr;  // [vocab] first-token logits, assembled from every rank's vocab shard
  float* peer_logits[kTpMaxRanks]{};
  unsigned long long* peer_flags[kTpMaxRanks]{};
  unsigned long long tp_epoch = 0;
  // micro-batch overlap of the peer reductions (prefill_overlap): the reduce stream, its
  // events, and the activation maps rebased to the second micro-batch's first row
  bool tp_defer = false;       // row_parallel: leave the partial for the caller to reduce
  int attn_stable_cap = 1 << 30;  // attention: cap on FaArgs::stable_pages (second micro-batch)
  cudaStream_t tp_rs = nullptr;
  cudaEvent_t tp_ev[9]{};
  int mb_r0 = -1;
  CUtensorMap mb_xn[3], mb_attn[3], mb_act[3], mb_q;
  bool emulated_tp = false;  // test driver sums the ranks' partials itself (cake_prefill_group)
  unsigned profile_mask = 0;  // bit k: bracket launches of kernel class k with events
  int profile_stride = 1;     // bracket every n-th launch of a class (keeps the other PDL chains intact)
  long long prof_seq[CAKE_K_COUNT]{};
  std::mutex prof_mu;  // launches come from the compute thread and the loader's pacer thread
  std::vector<ProfPair> prof;
  std::vector<cudaEvent_t> event_pool;
  cake_kernel_stat stats[CAKE_K_COUNT]{};
  long long launches = 0;
};

namespace {

cudaEvent_t pool_event(cake_model* m) {
  if (!m->event_pool.empty()) {
    cudaEvent_t e = m->event_pool.back();
    m->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Brackets a launch with events when profiling is on.
struct ProfScope {
  cake_model* m;
  int kind;
  cudaStream_t s;
  double flops, bytes;
  cudaEvent_t a = nullptr;
  ProfScope(cake_model* m_, int kind_, cudaStream_t s_, double f, double b)
      : m(m_), kind(kind_), s(s_), flops(f), bytes(b) {
    std::lock_guard<std::mutex> g(m->prof_mu);
    m->launches++;
    if ((m->profile_mask & (1u << kind)) && m->prof_seq[kind]++ % m->profile_stride == 0) {
      a = pool_event(m);
      cudaEventRecord(a, s);
    }
  }
  ~ProfScope() {
    if (a != nullptr) {
      std::lock_guard<std::mutex> g(m->prof_mu);
      cudaEvent_t b = pool_event(m);
      cudaEventRecord(b, s);
      m->prof.push_back({kind, a, b, flops, bytes});
    }
  }
};

int alloc_dev(void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  CK(cudaMalloc(p, bytes));
  return CAKE_OK;
}

int init_tensor(bf16* dst, long long rows, long long cols, long long row_off, long long col_off,
                long long logical_cols, long long group, long long group_stride, uint64_t seed,
                uint32_t tid, float scale, cudaStream_t s, int rope_hd = 0) {
  InitArgs a;
  a.rope_hd = rope_hd;
  a.dst = dst;
  a.rows = rows;
  a.cols = cols;
  a.dst_ld = cols;
  a.row_off = row_off;
  a.col_off = col_off;
  a.logical_cols = logical_cols;
  a.group = group;
  a.group_stride = group_stride;
  a.seed = seed;
  a.tensor_id = tid;
  a.scale = scale;
  init_weight_kernel<<<launch_grid_for(rows * cols, 256), 256, 0, s>>>(a);
  CKL();
  return CAKE_OK;
}

int fill(bf16* dst, long long n, float v, cudaStream_t s) {
  fill_bf16_kernel<<<launch_grid_for(n, 256), 256, 0, s>>>(dst, n, v);
  CKL();
  return CAKE_OK;
}

// Tensor ids of the seeded generator (shared with oracle/llama_ref.c).
uint32_t tid_layer(int layer, int which) { return static_cast<uint32_t>(16 * layer + which); }
constexpr uint32_t kTidEmbed = 1u << 20;
constexpr uint32_t kTidLmHead = (1u << 20) + 1;
enum { kWq = 0, kWk = 1, kWv = 2, kWo = 3, kWgate = 4, kWup = 5, kWdown = 6 };

}  // namespace

namespace {

long long* g_fa4_trace = nullptr;  // debug: clock stamps of one CTA (cake_debug_fa4_trace)
int g_fa4_trace_layer = -1;

#ifdef CAKE_ATTN_VARIANTS

// Two-tile tcgen05 attention (attention_fa4.cuh): 2 x 128 (token, head) rows
// of one KV head per CTA; splits of the prefix fill one wave of SMs, the last
// split of each tile pair combines in split order (no combine kernel).
int attention_fa4(cake_model* m, long long chunk_start, int chunk_len, int layer, const int32_t* bt,
                  const int32_t* abort_flag, cudaStream_t s) {
  const int G = m->nq / m->nkv;
  const int pair_tokens = 2 * (128 / G);
  const int qpairs = (chunk_len + pair_tokens - 1) / pair_tokens;
  const long long kv_end = chunk_start + chunk_len;
  const int n_pages = static_cast<int>((kv_end + kAttnPage - 1) / kAttnPage);
  const int base_ctas = qpairs * m->nkv;
  // partial slots: 2 tiles x 128 rows x hd fp32 per (split, tile pair, KV head)
  const int cap = static_cast<int>(m->part_rows_cap / (static_cast<size_t>(base_ctas) * 256));
  const int splits =
      std::max(1, std::min({num_sms() / std::max(1, base_ctas), std::max(1, n_pages / 4), m->max_splits, cap}));
  const double vis = static_cast<double>(chunk_len) * chunk_start + 0.5 * chunk_len * (chunk_len + 1.0);
  const double flops = 4.0 * m->hd * m->nq * vis;
  const double bytes = static_cast<double>(kv_end) * m->nkv * m->hd * 2 * 2 + 2.0 * chunk_len * m->nq * m->hd * 2;
  ProfScope ps(m, chunk_len == 1 ? CAKE_K_DEC_ATTN : CAKE_K_ATTN, s, flops, bytes);
  F4Args fa{};
  fa.fa.q = m->q;
  fa.fa.block_table = bt;
  fa.fa.out = m->attn;
  fa.fa.part_o = m->part_o;
  fa.fa.part_lse = m->part_lse;
  fa.fa.chunk_start = chunk_start;
  fa.fa.chunk_len = chunk_len;
  fa.fa.n_q_heads = m->nq;
  fa.fa.n_kv_heads = m->nkv;
  fa.fa.layer = layer;
  fa.fa.n_layers = m->L;
  fa.fa.num_splits = splits;
  fa.fa.scale_log2 = 1.4426950408889634f / std::sqrt(static_cast<float>(m->hd));
  fa.fa.abort_flag = abort_flag;
  fa.tickets = m->attn_tickets;
  fa.trace = (g_fa4_trace_layer == layer) ? g_fa4_trace : nullptr;
  const dim3 grid(qpairs, m->nkv, splits);
  if (m->hd == 128) {
    static bool cfgd = false;
    if (!cfgd) {
      CK(cudaFuncSetAttribute(attn_fa4_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, F4Cfg<128>::kSmem));
      cfgd = true;
    }
    const cudaError_t e = launch_chain(attn_fa4_kernel<128>, grid, dim3(kF4Threads), F4Cfg<128>::kSmem, s, 1,
                                       m->tm_q, m->tm_kv, fa);
    if (e != cudaSuccess) {
      cudaFuncAttributes fa_attr{};
      cudaFuncGetAttributes(&fa_attr, attn_fa4_kernel<128>);
      return fail(CAKE_ECUDA + static_cast<int>(e), "attn_fa4_kernel<128>: %s (regs %d, max threads %d, static smem %zu, "
                  "dynamic %d, max dynamic %d)", cudaGetErrorString(e), fa_attr.numRegs, fa_attr.maxThreadsPerBlock,
                  fa_attr.sharedSizeBytes, F4Cfg<128>::kSmem, fa_attr.maxDynamicSharedSizeBytes);
    }
  } else if (m->hd == 64) {
    static bool cfgd = false;
    if (!cfgd) {
      CK(cudaFuncSetAttribute(attn_fa4_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, F4Cfg<64>::kSmem));
      cfgd = true;
    }
    CK(launch_chain(attn_fa4_kernel<64>, grid, dim3(kF4Threads), F4Cfg<64>::kSmem, s, 1, m->tm_q, m->tm_kv, fa));
  } else {
    return fail(CAKE_EINVAL, "attention: head_dim %d unsupported", m->hd);
  }
  return CAKE_OK;
}
#endif  // CAKE_ATTN_VARIANTS

int attention(cake_model* m, long long chunk_start, int chunk_len, int layer, const int32_t* bt,
              const int32_t* abort_flag, cudaStream_t s) {
  // Product dispatch (impl 0): one 128-row Q tile per CTA with the softmax warpgroups on
  // alternate key blocks (attention_alt.cuh); impl 2 is the column-split one-tile kernel
  // (attention_tc.cuh), impl 1 the mma.sync cross-check; 3 / 4 are experiment builds.
#ifdef CAKE_ATTN_VARIANTS
  if (m->attn_impl == 3) return attention_fa4(m, chunk_start, chunk_len, layer, bt, abort_flag, s);
#endif
  const int G = m->nq / m->nkv;
  const bool tc = m->attn_impl != 1;
  const int rows_per_cta = tc ? kFaRows : kAttnRows;
  const int tok_per_tile = rows_per_cta / G;
  const int qtiles = (chunk_len + tok_per_tile - 1) / tok_per_tile;
  const long long kv_end = chunk_start + chunk_len;
  const int n_pages = static_cast<int>((kv_end + kAttnPage - 1) / kAttnPage);
  const int base_ctas = qtiles * m->nkv;
  const int cap = static_cast<int>(m->part_rows_cap / (static_cast<size_t>(chunk_len) * m->nq));
  int splits = 1;
  if (tc) {
    // one CTA per SM: pick the split count with the fullest last wave, >= 8 pages per split
    // at most one wave: a CTA's fixed cost (prologue, Q load, partial write) makes
    // two waves of short splits slower than one of longer splits (first-token
    // step attention 1.40 -> 1.16 ms at 32K: 18 splits instead of 37)
    const int max_s = std::max(1, std::min({n_pages / 8, m->max_splits, cap}));
    const int max_waves = std::max(1, g_exp[CAKE_EXP_ATTN_MAX_WAVES]);
    double best = 0.0;
    for (int sp = 1; sp <= max_s; ++sp) {
      const int ctas = base_ctas * sp;
      const int waves = (ctas + num_sms() - 1) / num_sms();
      if (waves > max_waves) break;
      const double eff = static_cast<double>(ctas) / (static_cast<double>(waves) * num_sms());
      if (eff > best + 0.02) {
        best = eff;
        splits = sp;
      }
    }
  } else {
    const int target = 2 * num_sms();
    splits = std::max(1, std::min({(target + base_ctas - 1) / base_ctas, std::max(1, n_pages / 4), m->max_splits, cap}));
  }
  // algorithmic work: 4 * hd * (visible keys) per (query, head)
  const double vis = static_cast<double>(chunk_len) * chunk_start + 0.5 * chunk_len * (chunk_len + 1.0);
  const double flops = 4.0 * m->hd * m->nq * vis;
  const double bytes = static_cast<double>(kv_end) * m->nkv * m->hd * 2 * 2 + 2.0 * chunk_len * m->nq * m->hd * 2;
  ProfScope ps(m, chunk_len == 1 ? CAKE_K_DEC_ATTN : CAKE_K_ATTN, s, flops, bytes);
  dim3 grid(qtiles, m->nkv, splits);
  if (tc) {
    FaArgs fa;
    fa.q = m->q;
    fa.block_table = bt;
    fa.out = m->attn;
    fa.part_o = m->part_o;
    fa.part_lse = m->part_lse;
    fa.chunk_start = chunk_start;
    fa.chunk_len = chunk_len;
    fa.n_q_heads = m->nq;
    fa.n_kv_heads = m->nkv;
    fa.layer = layer;
    fa.n_layers = m->L;
    fa.num_splits = splits;
    fa.scale_log2 = 1.4426950408889634f / std::sqrt(static_cast<float>(m->hd));
    fa.abort_flag = abort_flag;
    fa.trace = (g_fa4_trace_layer == layer) ? g_fa4_trace : nullptr;
    // pages the predecessor cannot be writing: the prefix before a (page-aligned) prefill chunk,
    // or every page for the q-only first-token pass (unaligned start, no KV write)
    fa.stable_pages = std::min(m->attn_stable_cap,
                               (chunk_start % kAttnPage) ? n_pages : static_cast<int>(chunk_start / kAttnPage));
    if (m->attn_impl == 0 || m->attn_impl == 5) {
      // product: softmax warpgroups on alternate key blocks (attention_alt.cuh; 4.5% faster than the
      // one-tile kernel at 32K, profiles/r02_attn_ab_micro.log)
      if (m->hd == 128) {
        auto kern = attn_alt_kernel<128>;
        static bool cfgd = false;
        if (!cfgd) {
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FaltCfg<128>::kSmem));
          cfgd = true;
        }
        CK(launch_chain(kern, grid, dim3(fa_threads<2>()), FaltCfg<128>::kSmem, s, 1, m->tm_q, m->tm_kv, fa));
      } else {
        auto kern = attn_alt_kernel<64>;
        static bool cfgd = false;
        if (!cfgd) {
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FaltCfg<64>::kSmem));
          cfgd = true;
        }
        CK(launch_chain(kern, grid, dim3(fa_threads<2>()), FaltCfg<64>::kSmem, s, 1, m->tm_q, m->tm_kv, fa));
      }
    } else
#ifdef CAKE_ATTN_VARIANTS
    if (m->attn_impl == 4) {  // decoupled softmax groups (attention_dec.cuh)
      if (m->hd == 128) {
        auto kern = attn_dec_kernel<128>;
        static bool cfgd = false;
        if (!cfgd) {
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FdCfg<128>::kSmem));
          cfgd = true;
        }
        CK(launch_chain(kern, grid, dim3(fa_threads<2>()), FdCfg<128>::kSmem, s, 1, m->tm_q, m->tm_kv, fa));
      } else {
        auto kern = attn_dec_kernel<64>;
        static bool cfgd = false;
        if (!cfgd) {
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FdCfg<64>::kSmem));
          cfgd = true;
        }
        CK(launch_chain(kern, grid, dim3(fa_threads<2>()), FdCfg<64>::kSmem, s, 1, m->tm_q, m->tm_kv, fa));
      }
    } else
#endif
    if (m->hd == 128) {
      // two softmax groups (384 threads): four groups measured 10% slower at 32K (512-thread max exchange)
      auto kern = attn_tc_kernel<128, 2>;
      static bool cfgd = false;
      if (!cfgd) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FaCfg<128>::kSmem));
        cfgd = true;
      }
      CK(launch_chain(kern, grid, dim3(fa_threads<2>()), FaCfg<128>::kSmem, s, 1, m->tm_q, m->tm_kv, fa));
    } else {
      auto kern = attn_tc_kernel<64, 2>;
      static bool cfgd = false;
      if (!cfgd) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FaCfg<64>::kSmem));
        cfgd = true;
      }
      CK(launch_chain(kern, grid, dim3(fa_threads<2>()), FaCfg<64>::kSmem, s, 1, m->tm_q, m->tm_kv, fa));
    }
    CKL();
  } else {
  AttnArgs a;
  a.q = m->q;
  a.pool = m->pool;
  a.block_table = bt;
  a.out = m->attn;
  a.part_o = m->part_o;
  a.part_lse = m->part_lse;
  a.chunk_start = chunk_start;
  a.chunk_len = chunk_len;
  a.n_q_heads = m->nq;
  a.n_kv_heads = m->nkv;
  a.layer = layer;
  a.n_layers = m->L;
  a.num_splits = splits;
  a.scale_log2 = 1.4426950408889634f / std::sqrt(static_cast<float>(m->hd));
  a.abort_flag = abort_flag;
  const int smem = (kAttnRows + 4 * kAttnPage) * m->hd * 2;
  if (m->hd == 128) {
    static bool cfgd = false;
    if (!cfgd) {
      CK(cudaFuncSetAttribute(attn_prefill_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      cfgd = true;
    }
    attn_prefill_kernel<128><<<grid, kAttnThreads, smem, s>>>(a);
  } else {
    static bool cfgd = false;
    if (!cfgd) {
      CK(cudaFuncSetAttribute(attn_prefill_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      cfgd = true;
    }
    attn_prefill_kernel<64><<<grid, kAttnThreads, smem, s>>>(a);
  }
  CKL();
  }
  if (splits > 1) {
    const int rows = chunk_len * m->nq;
    if (splits > kCombineMaxSplits) return fail(CAKE_EINVAL, "attention: %d splits > %d", splits, kCombineMaxSplits);
    if (m->hd == 128)
      CK(launch_chain(attn_combine_kernel<128>, dim3(rows), dim3(128), 0, s, 1,
                      static_cast<const float*>(m->part_o), static_cast<const float*>(m->part_lse), m->attn, rows,
                      splits, abort_flag));
    else
      CK(launch_chain(attn_combine_kernel<64>, dim3(rows), dim3(64), 0, s, 1,
                      static_cast<const float*>(m->part_o), static_cast<const float*>(m->part_lse), m->attn, rows,
                      splits, abort_flag));
    CKL();
  }
  return CAKE_OK;
}

template <int EPI>
int launch_skinny(cake_model* m, int kind, const SkinnyArgs& a, double rows, cudaStream_t s) {
  auto kern = skinny_kernel<EPI>;
  static bool cfgd = false;
  if (!cfgd) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cfgd = true;
  }
  const int smem = a.M * a.K * 2;
  // up to 8 CTAs per SM, warps striding over the units: the per-CTA prologue (x into
  // smem, or its RMSNorm) is paid per CTA, but these GEMVs are bound by the bytes in
  // flight (first-token step at 1 / 2 / 4 / 8 CTAs per SM: 11.6 / 7.2 / 5.39 / 5.35 ms)
  const int blocks = std::max(1, std::min((a.units + kSkinnyWarps - 1) / kSkinnyWarps, num_sms() * 8));
  ProfScope ps(m, kind, s, 2.0 * a.M * rows * a.K, 2.0 * rows * a.K);
  CK(launch_chain(kern, dim3(blocks), dim3(kSkinnyWarps * 32), smem, s, 1, a));
  CKL();
  return CAKE_OK;
}

// Peer-memory TP reduction of this rank's partial in tp_buf (tp_peer.cuh):
// slice mode (M > 1): h row slices += rank-ordered sum, RMSNorm(gamma) rows
// pushed into every rank's xn; replicated (M = 1): every rank's full h.
int tp_reduce(cake_model* m, int M, bool replicated, const bf16* gamma, cudaStream_t s) {
  TpReduceArgs a{};
  const int n = m->cfg.tp_size;
  for (int r = 0; r < n; ++r) {
    a.part[r] = m->peer_part[r];
    a.xn[r] = m->peer_xn[r];
    a.flags[r] = m->peer_flags[r];
  }
  a.h = m->h;
  a.gamma = gamma;
  a.eps = m->cfg.rms_eps;
  a.rank = m->cfg.tp_rank;
  a.nranks = n;
  a.M = M;
  a.H = m->H;
  a.replicated = replicated ? 1 : 0;
  a.epoch = ++m->tp_epoch;
  const int rows = replicated ? M : (M + n - 1) / n;
  const int grid = std::max(1, std::min(rows, num_sms()));
  // wire bytes of this rank: pulled partials of its rows (+ pushed normalized rows)
  const double elt = replicated ? 4.0 : 2.0;
  const double bytes = static_cast<double>(rows) * m->H * (elt * n + (replicated ? 0.0 : 2.0 * n) + 8.0);
  ProfScope ps(m, CAKE_K_ALLREDUCE, s, 0.0, bytes);
  tp_reduce_kernel<<<grid, kTpThreads, 0, s>>>(a);
  CKL();
  return CAKE_OK;
}

// Row-parallel skinny projection into the residual stream (TP: partials + all-reduce).
int skinny_row_parallel(cake_model* m, int kind, const bf16* W, const bf16* x, int K, cudaStream_t s) {
  SkinnyArgs a{};
  a.W = W;
  a.x = x;
  a.M = 1;
  a.K = K;
  a.units = m->H;
  if (m->cfg.tp_size == 1) {
    a.resid = m->h;
    a.ldr = m->H;
    return launch_skinny<kSkResid>(m, kind, a, m->H, s);
  }
  if (!m->comm && !m->peer_tp) return fail(CAKE_ESTATE, "tp_size > 1 but no peer mappings / NCCL communicator");
  a.out = m->tp_buf;
  a.ldo = m->H;
  CKS(launch_skinny<kSkF32>(m, kind, a, m->H, s));
  if (m->peer_tp) return tp_reduce(m, 1, true, nullptr, s);
  {
    ProfScope ps(m, CAKE_K_ALLREDUCE, s, 0.0, 4.0 * m->H);
    ncclResult_t r = ncclAllReduce(m->tp_buf, m->tp_buf, static_cast<size_t>(m->H), ncclFloat32, ncclSum, m->comm, s);
    if (r != ncclSuccess) return fail(CAKE_ENCCL + r, "allreduce: %s", ncclGetErrorString(r));
  }
  add_inplace_kernel<<<1, 256, 0, s>>>(m->h, m->tp_buf, m->H, nullptr);
  CKL();
  return CAKE_OK;
}

int rmsnorm(cake_model* m, const bf16* gamma, long long row0, int rows, const int32_t* abort_flag, cudaStream_t s);

// One launch of the first-token projection chain (decode_chain.cuh): the o,
// gate/up and down projections of `layer` (layer >= 0) and then the q
// projection of `q_layer` (q_layer >= 0), one CTA per SM, grid barriers
// between the phases. Cooperative launch: every CTA is resident before any
// spins in a barrier (two contexts' chains never split the SMs between them).
int g_dec_prefetch_kb = 64;  // L2 prefetch per CTA ahead of each chain phase (A/B: cake_dec_set_prefetch; 0/32/64/128 KB: 3.79/3.71/3.68/3.69 ms)
long long* g_dec_trace = nullptr;  // debug: cake_dec_debug_trace
int g_dec_trace_layer = -2;
int dec_chain(cake_model* m, int layer, int q_layer, long long pos, cudaStream_t s) {
  DecArgs a{};
  auto add = [&](int kind, const bf16* W, const bf16* gamma, int K, int units) {
    a.ph[a.n_phases++] = DecPhase{kind, W, gamma, K, units};
  };
  if (layer >= 0) {
    const LayerWeights& lw = m->layers[layer];
    add(kDecO, lw.wo, nullptr, m->nq * m->hd, m->H);
    add(kDecGU, lw.wgu, lw.ln2, m->H, m->F);
    add(kDecD, lw.wd, nullptr, m->F, m->H);
  }
  if (q_layer >= 0) add(kDecQ, m->layers[q_layer].wqkv, m->layers[q_layer].ln1, m->H, m->nq * m->hd / 2);
  double bytes = 0.0;
  const int ctas = num_sms();
  for (int p = 0; p < a.n_phases; ++p) {
    const int rpu = (a.ph[p].kind == kDecQ || a.ph[p].kind == kDecGU) ? 2 : 1;
    a.max_k = std::max(a.max_k, a.ph[p].K);
    a.red_rows = std::max(a.red_rows, rpu * ((a.ph[p].units + ctas - 1) / ctas));
    bytes += 2.0 * rpu * a.ph[p].K * a.ph[p].units;
    if (a.ph[p].K % 8) return fail(CAKE_EINVAL, "decode chain: row length %d not a multiple of 8", a.ph[p].K);
  }
  a.prefetch_bytes = g_dec_prefetch_kb * 1024;
  a.h = m->h;
  a.H = m->H;
  a.eps = m->cfg.rms_eps;
  a.attn = m->attn;
  a.act = m->act;
  a.q_out = m->q;
  a.rope = m->rope;
  a.pos = pos;
  a.head_dim = m->hd;
  a.gbar = reinterpret_cast<unsigned long long*>(m->dec_bar);
  if (g_dec_trace != nullptr && g_dec_trace_layer == layer) a.trace = g_dec_trace;
  const size_t smem = static_cast<size_t>(a.max_k) * 2 + sizeof(float) * a.red_rows;
  static bool cfgd = false;
  if (!cfgd) {
    CK(cudaFuncSetAttribute(dec_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cfgd = true;
  }
  if (smem > 200 * 1024) return fail(CAKE_EINVAL, "decode chain: %zu B of shared memory", smem);
  ProfScope ps(m, CAKE_K_DEC_PROJ, s, bytes, bytes);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  attr[n].id = cudaLaunchAttributeCooperative;
  attr[n].val.cooperative = 1;
  ++n;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kDecThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = n;
  CK(cudaLaunchKernelEx(&cfg, dec_chain_kernel, a));
  return CAKE_OK;
}

// First-token step on the chain kernel: embed, then per layer the attention
// between two chain launches (q(0) | attn(0) | o,gu,down(0) + q(1) | attn(1) | ...).
int last_token_chain(cake_model* m, const int32_t* d_token, long long T, const int32_t* bt, cudaStream_t s) {
  {
    ProfScope ps(m, CAKE_K_EMBED, s, 0.0, m->H * 6.0);
    embed_kernel<<<1, 128, 0, s>>>(d_token, m->embed, m->h, m->H, nullptr);
    CKL();
  }
  CKS(dec_chain(m, -1, 0, T - 1, s));
  for (int l = 0; l < m->L; ++l) {
    CKS(attention(m, T - 1, 1, l, bt, nullptr, s));
    CKS(dec_chain(m, l, l + 1 < m->L ? l + 1 : -1, T - 1, s));
  }
  return CAKE_OK;
}

// First-token step over a complete cache: the last prompt token (position
// T-1) as a q-only pass, every projection a weight stream.
int last_token_pass(cake_model* m, const int32_t* d_token, long long T, const int32_t* bt, cudaStream_t s) {
  if (m->cfg.tp_size == 1 && !m->emulated_tp && g_exp[CAKE_EXP_DEC_CHAIN]) return last_token_chain(m, d_token, T, bt, s);
  const int H = m->H;
  {
    ProfScope ps(m, CAKE_K_EMBED, s, 0.0, H * 6.0);
    embed_kernel<<<1, 128, 0, s>>>(d_token, m->embed, m->h, H, nullptr);
    CKL();
  }
  for (int l = 0; l < m->L; ++l) {
    LayerWeights& lw = m->layers[l];
    {
      SkinnyArgs a{};
      a.W = lw.wqkv;  // q rows come first
      a.x = m->xn;
      a.norm_h = m->h;  // ln1 folded into the projection (skinny.cuh)
      a.norm_gamma = lw.ln1;
      a.norm_eps = m->cfg.rms_eps;
      a.M = 1;
      a.K = H;
      a.units = m->nq * m->hd / 2;
      a.q_out = m->q;
      a.ldo = m->nq * m->hd;
      a.rope = m->rope;
      a.pos0 = T - 1;
      a.head_dim = m->hd;
      CKS(launch_skinny<kSkQRope>(m, CAKE_K_DEC_PROJ, a, m->nq * m->hd, s));
    }
    CKS(attention(m, T - 1, 1, l, bt, nullptr, s));
    CKS(skinny_row_parallel(m, CAKE_K_DEC_PROJ, lw.wo, m->attn, m->nq * m->hd, s));
    {
      SkinnyArgs a{};
      a.W = lw.wgu;
      a.x = m->xn;
      a.norm_h = m->h;  // ln2 folded in
      a.norm_gamma = lw.ln2;
      a.norm_eps = m->cfg.rms_eps;
      a.M = 1;
      a.K = H;
      a.units = m->F;
      a.act = m->act;
      a.ld_act = m->F;
      CKS(launch_skinny<kSkSwiglu>(m, CAKE_K_DEC_PROJ, a, 2.0 * m->F, s));
    }
    CKS(skinny_row_parallel(m, CAKE_K_DEC_PROJ, lw.wd, m->act, m->F, s));
  }
  return CAKE_OK;
}

// RMSNorm folded into the projections (gemm.cuh GemmArgs): the residual
// epilogues of O / down write bf16(h) and per-tile sums of squares, the next
// QKV / gate-up epilogue applies the row scale. Single-GPU only (the TP path
// adds the all-reduced partials in a separate kernel and keeps rmsnorm).
// cake_set_experiment(CAKE_EXP_FUSED_NORM, 0) restores the standalone kernel (A/B measurements).
bool fused_norm(const cake_model* m) {
  return g_exp[CAKE_EXP_FUSED_NORM] != 0 && m->cfg.tp_size == 1 && !m->emulated_tp && m->H % 128 == 0;
}

void set_norm_consumer(cake_model* m, GemmArgs& g) {
  g.ss_in = m->ss;
  g.ss_parts = m->H / 128;
  g.ss_ld = m->rows_cap;
  g.rms_dim = m->H;
  g.rms_eps = m->cfg.rms_eps;
}

int rmsnorm(cake_model* m, const bf16* gamma, long long row0, int rows, const int32_t* abort_flag, cudaStream_t s) {
  ProfScope ps(m, CAKE_K_RMSNORM, s, 0.0, static_cast<double>(rows) * m->H * 6);
  CK(launch_chain(rmsnorm_kernel, dim3((rows + kNormRowsPerCta - 1) / kNormRowsPerCta),
                  dim3(kNormThreadsPerRow * kNormRowsPerCta), 0, s, 1, static_cast<const float*>(m->h), gamma, m->xn,
                  m->H, m->cfg.rms_eps, row0, rows, abort_flag));
  CKL();
  return CAKE_OK;
}

// Row-parallel projection output: residual += acc (TP: via all-reduce of partials).
int row_parallel(cake_model* m, int kind, const CUtensorMap* ta, const CUtensorMap* tb, int K, int M,
                 const int32_t* abort_flag, cudaStream_t s, const bf16* next_gamma) {
  GemmArgs g{};
  g.M = M;
  g.N = m->H;
  g.K = K;
  g.abort_flag = abort_flag;
  const double flops = 2.0 * M * m->H * K;
  const double bytes = 2.0 * m->H * K + 2.0 * M * K + 8.0 * M * m->H;
  if (m->cfg.tp_size == 1) {
    g.resid = m->h;
    g.ldr = m->H;
    if (fused_norm(m)) {
      g.xb_out = m->xn;
      g.ss_out = m->ss;
      g.ss_ld = m->rows_cap;
    }
    ProfScope ps(m, kind, s, flops, bytes);
    return gemm_dispatch(128, kEpiResid, ta, tb, g, s, g.xb_out != nullptr ? m->out_h : nullptr);
  }
  if (!m->comm && !m->emulated_tp && !m->peer_tp)
    return fail(CAKE_ESTATE, "tp_size > 1 but no peer mappings / NCCL communicator");
  g.out = m->tp_buf;
  g.ldo = m->H;
  if (m->peer_tp) {
    // bf16 partial (half the wire bytes of fp32), then the fused reduce + RMSNorm + push
    {
      ProfScope ps(m, kind, s, flops, bytes);
      CKS(gemm_dispatch(128, kEpiBf16, ta, tb, g, s));
    }
    if (m->tp_defer) return CAKE_OK;  // prefill_overlap reduces it on the reduce stream
    return tp_reduce(m, M, false, next_gamma, s);
  }
  {
    ProfScope ps(m, kind, s, flops, bytes);
    CKS(gemm_dispatch(128, kEpiF32, ta, tb, g, s));
  }
  if (m->emulated_tp) return CAKE_OK;  // partial stays in tp_buf for the group driver
  {
    ProfScope ps(m, CAKE_K_ALLREDUCE, s, 0.0, 4.0 * M * m->H);
    ncclResult_t r = ncclAllReduce(m->tp_buf, m->tp_buf, static_cast<size_t>(M) * m->H, ncclFloat32, ncclSum,
                                   m->comm, s);
    if (r != ncclSuccess) return fail(CAKE_ENCCL + r, "allreduce: %s", ncclGetErrorString(r));
  }
  add_inplace_kernel<<<launch_grid_for(static_cast<long long>(M) * m->H / 4, 256), 256, 0, s>>>(
      m->h, m->tp_buf, static_cast<long long>(M) * m->H, abort_flag);
  CKL();
  return CAKE_OK;
}

}  // namespace

namespace {

int layer_attention_half(cake_model* m, int l, long long chunk_start, int M, const int32_t* d_block_table,
                         const int32_t* d_abort, bool no_kv, cudaStream_t s) {
  const int H = m->H;
  LayerWeights& lw = m->layers[l];
  // layer 0's input is the embedding (no producer epilogue); peer TP: the down
  // reduction of layer l-1 already wrote norm(h) rows into xn
  const bool fused = fused_norm(m) && l > 0;
  if (!fused && !(m->peer_tp && l > 0)) CKS(rmsnorm(m, lw.ln1, 0, M, d_abort, s));
  {
    GemmArgs g{};
    if (fused) set_norm_consumer(m, g);
    g.M = M;
    g.N = no_kv ? m->nq * m->hd : m->qkv_rows;
    g.K = H;
    g.q_out = m->q;
    g.kv_pool = m->pool;
    g.block_table = d_block_table;
    g.rope = m->rope;
    g.pos0 = chunk_start;
    g.n_q_heads = m->nq;
    g.n_kv_heads = no_kv ? 0 : m->nkv;
    g.head_dim = m->hd;
    g.page_tokens = m->cfg.page_tokens;
    g.layer = l;
    g.n_layers = m->L;
    g.abort_flag = d_abort;
    if (g.N % m->bn_qkv) return fail(CAKE_EINVAL, "prefill: q-only pass needs tileable q rows");
    ProfScope ps(m, CAKE_K_GEMM_QKV, s, 2.0 * M * g.N * H, 2.0 * g.N * H + 2.0 * M * H + 2.0 * M * g.N);
    // N-192 pair tiles: 32 of them at M = 512 fill 64 SM pairs, against 24 of N 256 (24.1 vs 30.1 us)
    const bool t192 = g_gemm_qkv192 && g_gemm_2sm && M > kGemmBlockM && g.N % 192 == 0;
    CKS(gemm_dispatch(t192 ? 192 : m->bn_qkv, kEpiQkv, m->a_xn, t192 ? lw.m_qkv192 : lw.m_qkv, g, s));
  }
  CKS(attention(m, chunk_start, M, l, d_block_table, d_abort, s));
  return row_parallel(m, CAKE_K_GEMM_O, m->a_attn, lw.m_o, m->nq * m->hd, M, d_abort, s, lw.ln2);
}

int layer_mlp_half(cake_model* m, int l, int M, const int32_t* d_abort, cudaStream_t s) {
  const int H = m->H;
  LayerWeights& lw = m->layers[l];
  const bool fused = fused_norm(m);
  if (!fused && !m->peer_tp) CKS(rmsnorm(m, lw.ln2, 0, M, d_abort, s));  // peer TP: the O reduction wrote xn
  {
    GemmArgs g{};
    if (fused) set_norm_consumer(m, g);
    g.M = M;
    g.N = 2 * m->F;
    g.K = H;
    g.out = m->act;
    g.ldo = m->F;
    g.abort_flag = d_abort;
    ProfScope ps(m, CAKE_K_GEMM_GU, s, 2.0 * M * g.N * H, 2.0 * g.N * H + 2.0 * M * H + 2.0 * M * m->F);
    CKS(gemm_dispatch(256, kEpiSwiglu, m->a_xn, lw.m_gu, g, s));
  }
  return row_parallel(m, CAKE_K_GEMM_D, m->a_act, lw.m_d, m->F, M, d_abort, s,
                      l + 1 < m->L ? m->layers[l + 1].ln1 : m->final_norm);
}

// ---- peer TP: two row micro-batches per chunk, reductions overlapped ----
//
// A chunk of M rows runs as micro-batches b = 0, 1 of Mb = M / 2 rows. Per layer the
// compute stream s issues QKV_0 attn_0 O_0 | QKV_1 attn_1 O_1 | GU_0 D_0 | GU_1 D_1 and the
// reduce stream r the four peer reductions R(O_0) R(O_1) R(D_0) R(D_1), each waiting on
// its projection's event; each consumer waits on its reduction's event. So R(O_0) runs
// under QKV_1 / attn_1 / O_1, R(O_1) under GU_0 / D_0, R(D_0) under GU_1 / D_1 and R(D_1)
// under the next layer's QKV_0 / attn_0 / O_0. Every rank issues the reductions in the
// same order on one stream (same epochs). Micro-batch 1 is micro-batch 0's suffix of the
// same prompt, so its attention reads micro-batch 0's K/V (written by QKV_0 on s) — the
// usual causal order. The two batches touch disjoint rows of every activation buffer, so
// the reduction of one and the projections of the other never share bytes.

// The model's row buffers seen from row r0 (the second micro-batch): pointers and TMA
// maps rebased, restored on destruction. Launches capture their arguments when enqueued.
struct RowView {
  cake_model* m;
  float *h, *tp_buf;
  bf16 *xn, *q, *attn, *act;
  void* part[kTpMaxRanks];
  bf16* pxn[kTpMaxRanks];
  CUtensorMap a_xn[3], a_attn[3], a_act[3], tm_q;
  int cap;
  RowView(cake_model* m_, int r0, int stable_cap) : m(m_) {
    h = m->h, tp_buf = m->tp_buf, xn = m->xn, q = m->q, attn = m->attn, act = m->act, cap = m->attn_stable_cap;
    for (int r = 0; r < kTpMaxRanks; ++r) part[r] = m->peer_part[r], pxn[r] = m->peer_xn[r];
    std::memcpy(a_xn, m->a_xn, sizeof(a_xn));
    std::memcpy(a_attn, m->a_attn, sizeof(a_attn));
    std::memcpy(a_act, m->a_act, sizeof(a_act));
    tm_q = m->tm_q;
    if (r0 == 0) return;
    const size_t H = m->H, QD = static_cast<size_t>(m->nq) * m->hd;
    m->h += r0 * H;
    m->tp_buf = reinterpret_cast<float*>(reinterpret_cast<bf16*>(m->tp_buf) + r0 * H);  // bf16 partial rows
    m->xn += r0 * H;
    m->q += r0 * QD;
    m->attn += r0 * QD;
    m->act += static_cast<size_t>(r0) * m->F;
    for (int r = 0; r < m->cfg.tp_size; ++r) {
      m->peer_part[r] = static_cast<bf16*>(m->peer_part[r]) + r0 * H;
      m->peer_xn[r] += r0 * H;
    }
    std::memcpy(m->a_xn, m->mb_xn, sizeof(a_xn));
    std::memcpy(m->a_attn, m->mb_attn, sizeof(a_attn));
    std::memcpy(m->a_act, m->mb_act, sizeof(a_act));
    m->tm_q = m->mb_q;
    m->attn_stable_cap = stable_cap;
  }
  ~RowView() {
    m->h = h, m->tp_buf = tp_buf, m->xn = xn, m->q = q, m->attn = attn, m->act = act, m->attn_stable_cap = cap;
    for (int r = 0; r < kTpMaxRanks; ++r) m->peer_part[r] = part[r], m->peer_xn[r] = pxn[r];
    std::memcpy(m->a_xn, a_xn, sizeof(a_xn));
    std::memcpy(m->a_attn, a_attn, sizeof(a_attn));
    std::memcpy(m->a_act, a_act, sizeof(a_act));
    m->tm_q = tm_q;
  }
};

bool overlap_ok(const cake_model* m, int M, bool no_kv) {
  if (!m->peer_tp || m->emulated_tp || !g_exp[CAKE_EXP_TP_OVERLAP] || no_kv || M % 2) return false;
  const int Mb = M / 2;
  return Mb % kGemmBlockM == 0 && Mb % m->cfg.page_tokens == 0 && Mb % kAttnPage == 0 && Mb % m->cfg.tp_size == 0;
}

int overlap_setup(cake_model* m, int Mb) {
  if (!m->tp_rs) {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&m->tp_rs, cudaStreamNonBlocking, hi));
    for (auto& e : m->tp_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (m->mb_r0 != Mb) {
    const uint64_t R = m->rows_cap - Mb, H = m->H, QD = static_cast<uint64_t>(m->nq) * m->hd;
    int st;
    for (int i = 0; i < 3; ++i) {
      if ((st = make_map(&m->mb_xn[i], m->xn + Mb * H, R, H, 128 >> i))) return st;
      if ((st = make_map(&m->mb_attn[i], m->attn + Mb * QD, R, QD, 128 >> i))) return st;
      if ((st = make_map(&m->mb_act[i], m->act + static_cast<uint64_t>(Mb) * m->F, R, m->F, 128 >> i))) return st;
    }
    const int G = m->nq / m->nkv;
    if ((st = make_map_3d(&m->mb_q, m->q + Mb * QD, m->hd, m->nq, R, G, kFaRows / G))) return st;
    m->mb_r0 = Mb;
  }
  return CAKE_OK;
}

int prefill_overlap(cake_model* m, long long chunk_start, int M, int lb, int le, const int32_t* bt,
                    const int32_t* d_abort, cudaStream_t s) {
  const int Mb = M / 2;
  CKS(overlap_setup(m, Mb));
  cudaStream_t r = m->tp_rs;
  cudaEvent_t* ev = m->tp_ev;  // [0, 4): projections O_0 O_1 D_0 D_1 done; [4, 8): their reductions; 8: entry
  const int kProj = 0, kRed = 4;
  // the reduce stream starts after everything already on s (embed, the previous call's join)
  CK(cudaEventRecord(ev[8], s));
  CK(cudaStreamWaitEvent(r, ev[8], 0));
  // micro-batch 1 must not request its chunk's K/V pages before the PDL wait: micro-batch 0
  // writes them only three kernels earlier
  const int cap1 = static_cast<int>(chunk_start / kAttnPage);
  struct Defer {
    cake_model* m;
    explicit Defer(cake_model* m_) : m(m_) { m->tp_defer = true; }
    ~Defer() { m->tp_defer = false; }
  } defer(m);
  auto reduce = [&](int b, int slot, const bf16* gamma) -> int {
    CK(cudaEventRecord(ev[kProj + slot], s));
    CK(cudaStreamWaitEvent(r, ev[kProj + slot], 0));
    RowView v(m, b * Mb, cap1);
    CKS(tp_reduce(m, Mb, false, gamma, r));
    CK(cudaEventRecord(ev[kRed + slot], r));
    return CAKE_OK;
  };
  for (int l = lb; l < le; ++l) {
    LayerWeights& lw = m->layers[l];
    const bf16* next_gamma = l + 1 < m->L ? m->layers[l + 1].ln1 : m->final_norm;
    for (int b = 0; b < 2; ++b) {
      if (l > lb) CK(cudaStreamWaitEvent(s, ev[kRed + 2 + b], 0));  // R(D_b) of layer l-1 pushed its xn rows
      {
        RowView v(m, b * Mb, cap1);
        CKS(layer_attention_half(m, l, chunk_start + static_cast<long long>(b) * Mb, Mb, bt, d_abort, false, s));
      }
      CKS(reduce(b, b, lw.ln2));
    }
    for (int b = 0; b < 2; ++b) {
      CK(cudaStreamWaitEvent(s, ev[kRed + b], 0));  // R(O_b) pushed norm(h) rows into xn
      {
        RowView v(m, b * Mb, cap1);
        CKS(layer_mlp_half(m, l, Mb, d_abort, s));
      }
      CKS(reduce(b, 2 + b, next_gamma));
    }
  }
  // join: the caller's stream sees every reduction (the reduce stream is in order)
  CK(cudaStreamWaitEvent(s, ev[kRed + 3], 0));
  return CAKE_OK;
}

}  // namespace

extern "C" {

int cake_cuda_last_error(char* buf, size_t len) {
  if (buf && len) {
    std::snprintf(buf, len, "%s", g_last_error.c_str());
  }
  return static_cast<int>(g_last_error.size());
}

int cake_cuda_version(int* runtime, int* driver) {
  CK(cudaRuntimeGetVersion(runtime));
  CK(cudaDriverGetVersion(driver));
  return CAKE_OK;
}

int cake_cuda_device_count(int* n) {
  cudaError_t e = cudaGetDeviceCount(n);
  if (e != cudaSuccess) {
    *n = 0;
    cudaGetLastError();
  }
  return CAKE_OK;
}

int cake_cuda_set_device(int device) {
  CK(cudaSetDevice(device));
  g_num_sms = 0;
  return CAKE_OK;
}

int cake_cuda_bind_thread(int device) {
  int cur = -1;
  CK(cudaGetDevice(&cur));
  if (cur != device) CK(cudaSetDevice(device));
  return CAKE_OK;
}

int cake_cuda_sm_count(int device, int* n) {
  CK(cudaDeviceGetAttribute(n, cudaDevAttrMultiProcessorCount, device));
  return CAKE_OK;
}

int cake_cuda_device_sync(void) {
  CK(cudaDeviceSynchronize());
  return CAKE_OK;
}

int cake_stream_create(void** stream, int high_priority) {
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  cudaStream_t s;
  CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, high_priority ? hi : lo));
  *stream = s;
  return CAKE_OK;
}
// A stream whose kernels run on (at least) n_sms SMs only: a green context
// over an SM partition of the device. SURVEY §8(f) item 4 / PAPER.md:331:
// the reference scales its modeled chunk latency by a GPU-share factor p; on
// the B200 the compute side gets a real fraction of the SMs instead.
int cake_stream_create_sm_share(void** stream, int n_sms, int* got_sms) {
  using GetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
  using Split = CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned);
  using GenDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned);
  using GreenCreate = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
  using GreenStream = CUresult (*)(CUstream*, CUgreenCtx, unsigned, int);
  auto entry = [](const char* name) -> void* {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      return nullptr;
    return p;
  };
  auto get_res = reinterpret_cast<GetRes>(entry("cuDeviceGetDevResource"));
  auto split = reinterpret_cast<Split>(entry("cuDevSmResourceSplitByCount"));
  auto gen = reinterpret_cast<GenDesc>(entry("cuDevResourceGenerateDesc"));
  auto gcreate = reinterpret_cast<GreenCreate>(entry("cuGreenCtxCreate"));
  auto gstream = reinterpret_cast<GreenStream>(entry("cuGreenCtxStreamCreate"));
  if (!get_res || !split || !gen || !gcreate || !gstream) return fail(CAKE_ESTATE, "green contexts unavailable");
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaFree(nullptr));  // the primary context exists
  CUdevResource all{}, group{}, rest{};
  if (get_res(static_cast<CUdevice>(dev), &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
    return fail(CAKE_ECUDA, "cuDeviceGetDevResource failed");
  if (n_sms <= 0 || static_cast<unsigned>(n_sms) >= all.sm.smCount) {
    CKS(cake_stream_create(stream, 0));
    if (got_sms) *got_sms = static_cast<int>(all.sm.smCount);
    return CAKE_OK;
  }
  unsigned nb = 1;
  if (split(&group, &nb, &all, &rest, 0, static_cast<unsigned>(n_sms)) != CUDA_SUCCESS || nb != 1)
    return fail(CAKE_ECUDA, "cuDevSmResourceSplitByCount(%d) failed", n_sms);
  CUdevResourceDesc desc;
  if (gen(&desc, &group, 1) != CUDA_SUCCESS) return fail(CAKE_ECUDA, "cuDevResourceGenerateDesc failed");
  CUgreenCtx gctx;
  if (gcreate(&gctx, desc, static_cast<CUdevice>(dev), CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
    return fail(CAKE_ECUDA, "cuGreenCtxCreate failed");
  CUstream st;
  if (gstream(&st, gctx, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS)
    return fail(CAKE_ECUDA, "cuGreenCtxStreamCreate failed");
  *stream = st;  // (the green context lives as long as the process)
  if (got_sms) *got_sms = static_cast<int>(group.sm.smCount);
  return CAKE_OK;
}

int cake_set_sm_budget(int n_sms) {
  g_sm_limit = std::max(0, n_sms);
  return CAKE_OK;
}

int cake_stream_destroy(void* stream) {
  CK(cudaStreamDestroy(S(stream)));
  return CAKE_OK;
}
int cake_stream_sync(void* stream) {
  CK(cudaStreamSynchronize(S(stream)));
  return CAKE_OK;
}
int cake_stream_wait_event(void* stream, void* event) {
  CK(cudaStreamWaitEvent(S(stream), static_cast<cudaEvent_t>(event), 0));
  return CAKE_OK;
}
int cake_event_create(void** event, int timing) {
  cudaEvent_t e;
  CK(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  *event = e;
  return CAKE_OK;
}
int cake_event_destroy(void* event) {
  CK(cudaEventDestroy(static_cast<cudaEvent_t>(event)));
  return CAKE_OK;
}
int cake_event_record(void* event, void* stream) {
  CK(cudaEventRecord(static_cast<cudaEvent_t>(event), S(stream)));
  return CAKE_OK;
}
int cake_event_query(void* event) {
  cudaError_t e = cudaEventQuery(static_cast<cudaEvent_t>(event));
  if (e == cudaSuccess) return CAKE_OK;
  if (e == cudaErrorNotReady) return CAKE_ENOTREADY;
  return fail(CAKE_ECUDA + static_cast<int>(e), "event query: %s", cudaGetErrorString(e));
}
int cake_event_sync(void* event) {
  CK(cudaEventSynchronize(static_cast<cudaEvent_t>(event)));
  return CAKE_OK;
}
int cake_event_elapsed_ms(void* start, void* stop, float* ms) {
  CK(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start), static_cast<cudaEvent_t>(stop)));
  return CAKE_OK;
}

int cake_host_alloc(void** p, size_t bytes) {
  CK(cudaHostAlloc(p, bytes ? bytes : 16, cudaHostAllocPortable));
  return CAKE_OK;
}
int cake_host_free(void* p) {
  CK(cudaFreeHost(p));
  return CAKE_OK;
}
int cake_host_register(void* p, size_t bytes) {
  CK(cudaHostRegister(p, bytes, cudaHostRegisterPortable));
  return CAKE_OK;
}
int cake_host_unregister(void* p) {
  CK(cudaHostUnregister(p));
  return CAKE_OK;
}
int cake_dev_alloc(void** p, size_t bytes) { return alloc_dev(p, bytes); }
int cake_dev_free(void* p) {
  CK(cudaFree(p));
  return CAKE_OK;
}
int cake_memset_async(void* dst, int value, size_t bytes, void* stream) {
  CK(cudaMemsetAsync(dst, value, bytes, S(stream)));
  return CAKE_OK;
}
int cake_h2d_async(void* dst, const void* src, size_t bytes, void* stream) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, S(stream)));
  return CAKE_OK;
}
int cake_d2h_async(void* dst, const void* src, size_t bytes, void* stream) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, S(stream)));
  return CAKE_OK;
}
int cake_d2d_async(void* dst, const void* src, size_t bytes, void* stream) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, S(stream)));
  return CAKE_OK;
}

// ---------------------------------------------------------------- model
int cake_model_destroy(cake_model* m) {
  if (!m) return CAKE_OK;
  cudaDeviceSynchronize();
  for (void* p : {static_cast<void*>(m->weight_arena), static_cast<void*>(m->pool),
                  static_cast<void*>(m->rope), static_cast<void*>(m->h), static_cast<void*>(m->xn),
                  static_cast<void*>(m->q), static_cast<void*>(m->attn), static_cast<void*>(m->act),
                  static_cast<void*>(m->part_o), static_cast<void*>(m->part_lse),
                  static_cast<void*>(m->tp_buf), static_cast<void*>(m->q8_ws), static_cast<void*>(m->ss),
                  static_cast<void*>(m->dec_bar), static_cast<void*>(m->tp_flags), static_cast<void*>(m->tp_logits),
                  static_cast<void*>(m->attn_tickets)})
    if (p) cudaFree(p);
  if (m->peer_tp)
    for (int r = 0; r < m->cfg.tp_size; ++r)
      if (r != m->cfg.tp_rank) {
        for (void* p : {m->peer_part[r], static_cast<void*>(m->peer_xn[r]), static_cast<void*>(m->peer_h[r]),
                        static_cast<void*>(m->peer_flags[r]), static_cast<void*>(m->peer_logits[r])})
          if (p) cudaIpcCloseMemHandle(p);
      }
  for (auto& p : m->prof) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : m->event_pool) cudaEventDestroy(e);
  for (auto e : m->tp_ev)
    if (e) cudaEventDestroy(e);
  if (m->tp_rs) cudaStreamDestroy(m->tp_rs);
  delete m;
  return CAKE_OK;
}

int cake_model_create(const cake_model_config* cfg, cake_model** out) { return cake_model_create_shared(cfg, nullptr, out); }

int cake_model_create_shared(const cake_model_config* cfg, const cake_model* parent, cake_model** out) {
  *out = nullptr;
  const cake_model_config& c = *cfg;
  if (c.n_layers < 1 || c.hidden < 64 || c.n_heads < 1 || c.n_kv_heads < 1 || c.vocab < 1)
    return fail(CAKE_EINVAL, "model: bad dimensions");
  if (c.head_dim != 64 && c.head_dim != 128) return fail(CAKE_EINVAL, "model: head_dim must be 64 or 128");
  if (c.page_tokens != kAttnPage) return fail(CAKE_EINVAL, "model: page_tokens must be %d", kAttnPage);
  if (c.tp_size < 1 || c.tp_rank < 0 || c.tp_rank >= c.tp_size) return fail(CAKE_EINVAL, "model: bad tp");
  if (c.n_heads % c.n_kv_heads || c.n_kv_heads % c.tp_size || c.n_heads % c.tp_size)
    return fail(CAKE_EINVAL, "model: heads must divide evenly (GQA groups, TP shards)");
  if (c.ffn % (128 * c.tp_size)) return fail(CAKE_EINVAL, "model: ffn / tp must be a multiple of 128");
  if (c.hidden % 128 || c.hidden > 8192) return fail(CAKE_EINVAL, "model: hidden must be a multiple of 128, <= 8192");
  if (c.max_chunk < 1 || c.max_tokens < 1) return fail(CAKE_EINVAL, "model: bad capacity");
  const int G = c.n_heads / c.n_kv_heads;
  if (kAttnRows % G) return fail(CAKE_EINVAL, "model: GQA group must divide %d", kAttnRows);

  auto* m = new cake_model();
  m->cfg = c;
  m->L = c.n_layers;
  m->H = c.hidden;
  m->hd = c.head_dim;
  m->nq = c.n_heads / c.tp_size;
  m->nkv = c.n_kv_heads / c.tp_size;
  m->F = c.ffn / c.tp_size;
  m->qkv_rows = (m->nq + 2 * m->nkv) * m->hd;
  m->bn_qkv = (m->qkv_rows % 256 == 0) ? 256 : 128;
  if (m->hd % 64) {
    delete m;
    return fail(CAKE_EINVAL, "model: head_dim %d is not a multiple of 64 (rope-unit QKV rows)", m->hd);
  }
  if (m->qkv_rows % m->bn_qkv) {
    delete m;
    return fail(CAKE_EINVAL, "model: qkv rows %d not tileable", m->qkv_rows);
  }
  cudaStream_t s = 0;
  int st = CAKE_OK;
  auto bail = [&](int code) {
    cake_model_destroy(m);
    return code;
  };

  const size_t H = m->H, F = m->F, hd = m->hd, V = c.vocab;
  if (parent != nullptr) {
    // ---- weights shared with `parent` (a concurrent request's context on the same
    // device): the sibling owns its pool, scratch and tensor maps over them only
    const cake_model_config& pc = parent->cfg;
    if (pc.n_layers != c.n_layers || pc.hidden != c.hidden || pc.n_heads != c.n_heads ||
        pc.n_kv_heads != c.n_kv_heads || pc.head_dim != c.head_dim || pc.ffn != c.ffn || pc.vocab != c.vocab ||
        pc.seed != c.seed || pc.tp_rank != c.tp_rank || pc.tp_size != c.tp_size)
      return bail(fail(CAKE_EINVAL, "model: shared weights need the same dimensions, seed and TP shard"));
    m->layers = parent->layers;  // device pointers + weight tensor maps
    m->embed = parent->embed;
    m->lm_head = parent->lm_head;
    m->final_norm = parent->final_norm;
    m->weight_bytes = 0;
  } else {
    // ---- weights (one arena, every tensor 128-B aligned)
    auto pad = [](size_t n) { return (n + 63) / 64 * 64; };
    const size_t per_layer =
        pad(m->qkv_rows * H) + pad(H * m->nq * hd) + pad(2 * F * H) + pad(H * F) + 2 * pad(H);
    m->weight_bytes = (per_layer * m->L + 2 * pad(V * H) + pad(H)) * sizeof(bf16);
    if ((st = alloc_dev(&m->weight_arena, m->weight_bytes))) return bail(st);
    bf16* w = static_cast<bf16*>(m->weight_arena);
    auto take = [&](size_t n) {
      bf16* p = w;
      w += pad(n);
      return p;
    };
    const uint64_t seed = c.seed;
    const int r = c.tp_rank;
    const float s_h = 1.0f / std::sqrt(static_cast<float>(c.hidden));
    const float s_o = 1.0f / std::sqrt(static_cast<float>(c.n_heads * c.head_dim));
    const float s_f = 1.0f / std::sqrt(static_cast<float>(c.ffn));
    m->layers.resize(m->L);
    for (int l = 0; l < m->L; ++l) {
      LayerWeights& lw = m->layers[l];
      lw.wqkv = take(m->qkv_rows * H);
      lw.wo = take(H * m->nq * hd);
      lw.wgu = take(2 * F * H);
      lw.wd = take(H * F);
      lw.ln1 = take(H);
      lw.ln2 = take(H);
      const long long qrows = static_cast<long long>(m->nq) * hd, kvrows = static_cast<long long>(m->nkv) * hd;
      // QKV rows in rope-unit order within each head (qkv_row_of, elementwise.cuh)
      if ((st = init_tensor(lw.wqkv, qrows, H, r * qrows, 0, H, 0, 0, seed, tid_layer(l, kWq), s_h, s, hd)))
        return bail(st);
      if ((st = init_tensor(lw.wqkv + qrows * H, kvrows, H, r * kvrows, 0, H, 0, 0, seed, tid_layer(l, kWk), s_h, s,
                            hd)))
        return bail(st);
      if ((st = init_tensor(lw.wqkv + (qrows + kvrows) * H, kvrows, H, r * kvrows, 0, H, 0, 0, seed,
                            tid_layer(l, kWv), s_h, s, hd)))
        return bail(st);
      if ((st = init_tensor(lw.wo, H, m->nq * hd, 0, r * qrows, c.n_heads * hd, 0, 0, seed, tid_layer(l, kWo), s_o, s)))
        return bail(st);
      // gate|up interleave: physical 256-row block b = [gate rows b*128..+128 | up rows b*128..+128]
      for (long long b = 0; b < static_cast<long long>(F) / 128; ++b) {
        if ((st = init_tensor(lw.wgu + (2 * b) * 128 * H, 128, H, r * F + b * 128, 0, H, 0, 0, seed,
                              tid_layer(l, kWgate), s_h, s)))
          return bail(st);
        if ((st = init_tensor(lw.wgu + (2 * b + 1) * 128 * H, 128, H, r * F + b * 128, 0, H, 0, 0, seed,
                              tid_layer(l, kWup), s_h, s)))
          return bail(st);
      }
      if ((st = init_tensor(lw.wd, H, F, 0, r * F, c.ffn, 0, 0, seed, tid_layer(l, kWdown), s_f, s))) return bail(st);
      if ((st = fill(lw.ln1, H, 1.0f, s))) return bail(st);
      if ((st = fill(lw.ln2, H, 1.0f, s))) return bail(st);
      for (int ci = 0; ci < 3; ++ci) {
        const uint32_t div = 1u << ci;  // cluster size 1, 2, 4
        if ((st = make_map(&lw.m_qkv[ci], lw.wqkv, m->qkv_rows, H, m->bn_qkv / div))) return bail(st);
        if (m->qkv_rows % 192 == 0 && (st = make_map(&lw.m_qkv192[ci], lw.wqkv, m->qkv_rows, H, 96))) return bail(st);
        if ((st = make_map(&lw.m_o[ci], lw.wo, H, m->nq * hd, 128 / div))) return bail(st);
        if ((st = make_map(&lw.m_gu[ci], lw.wgu, 2 * F, H, 256 / div))) return bail(st);
        if ((st = make_map(&lw.m_d[ci], lw.wd, H, F, 128 / div))) return bail(st);
      }
    }
    m->embed = take(V * H);
    m->lm_head = take(V * H);
    m->final_norm = take(H);
    if ((st = init_tensor(m->embed, V, H, 0, 0, H, 0, 0, seed, kTidEmbed, 1.0f, s))) return bail(st);
    if ((st = init_tensor(m->lm_head, V, H, 0, 0, H, 0, 0, seed, kTidLmHead, s_h, s))) return bail(st);
    if ((st = fill(m->final_norm, H, 1.0f, s))) return bail(st);
  }

  // ---- paged KV pool
  m->n_logical_pages = static_cast<int>((c.max_tokens + c.page_tokens - 1) / c.page_tokens);
  m->n_phys_pages = m->n_logical_pages + std::max(0, c.spare_pages);
  const size_t page_elems = static_cast<size_t>(m->L) * 2 * m->nkv * c.page_tokens * hd;
  m->pool_bytes = page_elems * sizeof(bf16) * m->n_phys_pages;
  if ((st = alloc_dev(reinterpret_cast<void**>(&m->pool), m->pool_bytes))) return bail(st);
  // zeroed once: keys past a chunk's end are masked (p = 0) but still read, so
  // never-written pages must hold finite values
  cudaMemset(m->pool, 0, m->pool_bytes);

  // ---- RoPE table: cos/sin(pos * theta^(-2i/hd)), computed in double.
  {
    const long long P = c.max_tokens;
    const int half = m->hd / 2;
    std::vector<float2> tab(static_cast<size_t>(P) * half);
    std::vector<double> inv(half);
    for (int i = 0; i < half; ++i) inv[i] = std::pow(static_cast<double>(c.rope_theta), -2.0 * i / m->hd);
    for (long long p = 0; p < P; ++p)
      for (int i = 0; i < half; ++i) {
        const double a = static_cast<double>(p) * inv[i];
        tab[p * half + i] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
      }
    if ((st = alloc_dev(reinterpret_cast<void**>(&m->rope), tab.size() * sizeof(float2)))) return bail(st);
    cudaError_t e = cudaMemcpy(m->rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return bail(fail(CAKE_ECUDA + e, "rope upload: %s", cudaGetErrorString(e)));
  }

  // ---- activation scratch
  m->rows_cap = std::max(128, (c.max_chunk + 127) / 128 * 128);
  const size_t R = m->rows_cap;
  if ((st = alloc_dev(reinterpret_cast<void**>(&m->h), R * H * sizeof(float)))) return bail(st);
  if ((st = alloc_dev(reinterpret_cast<void**>(&m->xn), R * H * sizeof(bf16)))) return bail(st);
  if ((st = alloc_dev(reinterpret_cast<void**>(&m->ss), R * ((H + 127) / 128) * sizeof(float)))) return bail(st);
  if ((st = alloc_dev(reinterpret_cast<void**>(&m->q), R * m->nq * hd * sizeof(bf16)))) return bail(st);
  if ((st = alloc_dev(reinterpret_cast<void**>(&m->attn), R * m->nq * hd * sizeof(bf16)))) return bail(st);
  if ((st = alloc_dev(reinterpret_cast<void**>(&m->act), R * F * sizeof(bf16)))) return bail(st);
  // split-KV partials: room for 4 splits of a full chunk, or 64 of a short one
  m->part_rows_cap = std::max<size_t>(4 * R, 64) * m->nq;
  m->max_splits = 64;
  if ((st = alloc_dev(reinterpret_cast<void**>(&m->part_o), m->part_rows_cap * hd * sizeof(float)))) return bail(st);
  if ((st = alloc_dev(reinterpret_cast<void**>(&m->part_lse), m->part_rows_cap * sizeof(float)))) return bail(st);
  if ((st = alloc_dev(reinterpret_cast<void**>(&m->attn_tickets), R * m->nkv * sizeof(int)))) return bail(st);
  cudaMemset(m->attn_tickets, 0, R * m->nkv * sizeof(int));
  if (c.tp_size > 1 && (st = alloc_dev(reinterpret_cast<void**>(&m->tp_buf), R * H * sizeof(float))))
    return bail(st);
  if (c.tp_size > 1) {
    if (c.tp_size > kTpMaxRanks) return bail(fail(CAKE_EINVAL, "model: tp_size > %d", kTpMaxRanks));
    if ((st = alloc_dev(reinterpret_cast<void**>(&m->tp_flags), kTpFlagWords * sizeof(unsigned long long))))
      return bail(st);
    if ((st = alloc_dev(reinterpret_cast<void**>(&m->tp_logits), static_cast<size_t>(c.vocab) * sizeof(float))))
      return bail(st);
    cudaMemset(m->tp_flags, 0, kTpFlagWords * sizeof(unsigned long long));
  }
  if ((st = alloc_dev(reinterpret_cast<void**>(&m->q8_ws), 2 * sizeof(unsigned)))) return bail(st);
  if ((st = alloc_dev(reinterpret_cast<void**>(&m->dec_bar), 2 * sizeof(unsigned)))) return bail(st);
  cudaMemset(m->dec_bar, 0, 2 * sizeof(unsigned));
  cudaMemset(m->xn, 0, R * H * sizeof(bf16));
  cudaMemset(m->attn, 0, R * m->nq * hd * sizeof(bf16));
  cudaMemset(m->act, 0, R * F * sizeof(bf16));
  if ((st = make_map_f32(&m->out_h[0], m->h, R, H, H, 128))) return bail(st);
  if ((st = make_map(&m->out_h[1], m->xn, R, H, 128))) return bail(st);
  for (int i = 0; i < 3; ++i) {
    if ((st = make_map(&m->a_xn[i], m->xn, R, H, 128 >> i))) return bail(st);
    if ((st = make_map(&m->a_attn[i], m->attn, R, m->nq * hd, 128 >> i))) return bail(st);
    if ((st = make_map(&m->a_act[i], m->act, R, F, 128 >> i))) return bail(st);
  }
  {
    const int G = m->nq / m->nkv;
    if ((st = make_map_3d(&m->tm_q, m->q, hd, m->nq, R, G, kFaRows / G))) return bail(st);
    const uint64_t pool_rows = static_cast<uint64_t>(m->n_phys_pages) * m->L * 2 * m->nkv * c.page_tokens;
    if ((st = make_map(&m->tm_kv, m->pool, pool_rows, hd, 64))) return bail(st);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return bail(fail(CAKE_ECUDA + e, "model init: %s", cudaGetErrorString(e)));
  *out = m;
  return CAKE_OK;
}

int cake_model_get_info(const cake_model* m, cake_model_info* o) {
  if (!m || !o) return fail(CAKE_EINVAL, "null");
  o->kv_bytes_per_token = 2LL * m->L * m->nkv * m->hd * 2;
  o->page_bytes = static_cast<long long>(m->L) * 2 * m->nkv * m->cfg.page_tokens * m->hd * 2;
  o->n_logical_pages = m->n_logical_pages;
  o->n_physical_pages = m->n_phys_pages;
  o->local_q_heads = m->nq;
  o->local_kv_heads = m->nkv;
  o->local_ffn = m->F;
  o->weight_bytes = static_cast<long long>(m->weight_bytes);
  const long long H = m->H;
  o->flops_per_token_linear =
      2LL * m->L * (static_cast<long long>(m->qkv_rows) * H + H * m->nq * m->hd + 2LL * m->F * H + H * m->F);
  o->kv_pool = m->pool;
  return CAKE_OK;
}

int cake_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(CAKE_ENCCL + r, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  std::memcpy(out128, &id, sizeof(id));
  return CAKE_OK;
}

int cake_nccl_init(void** comm, const void* id128, int nranks, int rank) {
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  ncclResult_t r = ncclCommInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return fail(CAKE_ENCCL + r, "ncclCommInitRank: %s", ncclGetErrorString(r));
  *comm = c;
  return CAKE_OK;
}

int cake_nccl_destroy(void* comm) {
  ncclResult_t r = ncclCommDestroy(static_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return fail(CAKE_ENCCL + r, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return CAKE_OK;
}

// Debug: record clock64 stamps of CTA (0,0,0) of the two-tile attention kernel
// at `layer` into dev_buf (>= 64 + 2*64*8 int64), nullptr to stop.
CAKE_API int cake_debug_fa4_trace(void* dev_buf, int layer) {
  g_fa4_trace = static_cast<long long*>(dev_buf);
  g_fa4_trace_layer = layer;
  return CAKE_OK;
}

int cake_model_set_attention_impl(cake_model* m, int impl) {
#ifndef CAKE_ATTN_VARIANTS
  if (impl == 3 || impl == 4) return fail(CAKE_EINVAL, "attention impl %d: built without ATTN_VARIANTS=1", impl);
#endif
  if (impl < 0 || impl > 5)
    return fail(CAKE_EINVAL, "attention impl must be 0 (product dispatch), 1 (mma.sync), 2 (one-tile tcgen05), "
                             "3 (two-tile tcgen05), 4 (decoupled softmax groups) or 5 (groups on alternate blocks)");
  m->attn_impl = impl;
  return CAKE_OK;
}

int cake_tp_peer_handles(cake_model* m, void* out, size_t cap) {
  if (!m || !out) return fail(CAKE_EINVAL, "tp peer: null");
  if (m->cfg.tp_size < 2) return fail(CAKE_ESTATE, "tp peer: model is not tensor-parallel");
  if (cap < CAKE_TP_PEER_HANDLE_BYTES) return fail(CAKE_EINVAL, "tp peer: need %d bytes", CAKE_TP_PEER_HANDLE_BYTES);
  static_assert(5 * sizeof(cudaIpcMemHandle_t) <= CAKE_TP_PEER_HANDLE_BYTES, "handle blob");
  auto* h = static_cast<cudaIpcMemHandle_t*>(out);
  void* bufs[5] = {m->tp_buf, m->xn, m->h, m->tp_flags, m->tp_logits};
  for (int i = 0; i < 5; ++i) CK(cudaIpcGetMemHandle(&h[i], bufs[i]));
  return CAKE_OK;
}

int cake_tp_peer_open(cake_model* m, const void* all, int nranks) {
  if (!m || !all) return fail(CAKE_EINVAL, "tp peer: null");
  if (nranks != m->cfg.tp_size) return fail(CAKE_EINVAL, "tp peer: %d handle sets for tp_size %d", nranks, m->cfg.tp_size);
  if (m->peer_tp) return fail(CAKE_ESTATE, "tp peer: already open");
  const auto* blob = static_cast<const unsigned char*>(all);
  for (int r = 0; r < nranks; ++r) {
    if (r == m->cfg.tp_rank) {
      m->peer_part[r] = m->tp_buf;
      m->peer_xn[r] = m->xn;
      m->peer_h[r] = m->h;
      m->peer_flags[r] = m->tp_flags;
      m->peer_logits[r] = m->tp_logits;
      continue;
    }
    const auto* h = reinterpret_cast<const cudaIpcMemHandle_t*>(blob + static_cast<size_t>(r) * CAKE_TP_PEER_HANDLE_BYTES);
    void* p[5] = {};
    for (int i = 0; i < 5; ++i) {
      cudaError_t e = cudaIpcOpenMemHandle(&p[i], h[i], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        for (int j = 0; j < i; ++j) cudaIpcCloseMemHandle(p[j]);
        for (int q = 0; q < r; ++q)  // and every earlier peer's mappings: open is all or nothing
          if (q != m->cfg.tp_rank)
            for (void* b : {m->peer_part[q], static_cast<void*>(m->peer_xn[q]), static_cast<void*>(m->peer_h[q]),
                            static_cast<void*>(m->peer_flags[q]), static_cast<void*>(m->peer_logits[q])})
              if (b) cudaIpcCloseMemHandle(b);
        for (int q = 0; q < kTpMaxRanks; ++q) {
          m->peer_part[q] = nullptr;
          m->peer_xn[q] = nullptr;
          m->peer_h[q] = nullptr;
          m->peer_flags[q] = nullptr;
          m->peer_logits[q] = nullptr;
        }
        return fail(CAKE_ECUDA + e, "tp peer: open rank %d buffer %d: %s", r, i, cudaGetErrorString(e));
      }
    }
    m->peer_part[r] = p[0];
    m->peer_xn[r] = static_cast<bf16*>(p[1]);
    m->peer_h[r] = static_cast<float*>(p[2]);
    m->peer_flags[r] = static_cast<unsigned long long*>(p[3]);
    m->peer_logits[r] = static_cast<float*>(p[4]);
  }
  m->peer_tp = true;
  return CAKE_OK;
}

int cake_model_set_comm(cake_model* m, void* comm) {
  m->comm = static_cast<ncclComm_t>(comm);
  return CAKE_OK;
}

int cake_model_set_profiling(cake_model* m, int mask) {
  std::lock_guard<std::mutex> g(m->prof_mu);
  m->profile_mask = static_cast<unsigned>(mask);
  return CAKE_OK;
}

int cake_model_set_profiling_stride(cake_model* m, int stride) {
  if (stride < 1) return fail(CAKE_EINVAL, "profiling stride must be >= 1");
  std::lock_guard<std::mutex> g(m->prof_mu);
  m->profile_stride = stride;
  return CAKE_OK;
}

int cake_model_kernel_stats(cake_model* m, cake_kernel_stat* out, int reset) {
  std::lock_guard<std::mutex> g(m->prof_mu);
  for (auto& p : m->prof) {
    CK(cudaEventSynchronize(p.b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p.a, p.b));
    cake_kernel_stat& st = m->stats[p.kind];
    st.launches++;
    st.total_ms += ms;
    st.flops += p.flops;
    st.bytes += p.bytes;
    m->event_pool.push_back(p.a);
    m->event_pool.push_back(p.b);
  }
  m->prof.clear();
  if (out) std::memcpy(out, m->stats, sizeof(m->stats));
  if (reset) std::memset(m->stats, 0, sizeof(m->stats));
  return CAKE_OK;
}

int cake_model_launch_count(cake_model* m, long long* n, int reset) {
  std::lock_guard<std::mutex> g(m->prof_mu);
  *n = m->launches;
  if (reset) m->launches = 0;
  return CAKE_OK;
}



int cake_prefill_chunk(cake_model* m, const int32_t* d_tokens, long long chunk_start, int chunk_len,
                       const int32_t* d_block_table, const int32_t* d_abort, int flags, void* stream) {
  if (!m) return fail(CAKE_EINVAL, "null model");
  return cake_prefill_layers(m, d_tokens, chunk_start, chunk_len, 0, m->L, d_block_table, d_abort, flags, stream);
}

int cake_prefill_layers(cake_model* m, const int32_t* d_tokens, long long chunk_start, int chunk_len, int layer_begin,
                        int layer_end, const int32_t* d_block_table, const int32_t* d_abort, int flags,
                        void* stream) {
  if (!m) return fail(CAKE_EINVAL, "null model");
  if (layer_begin < 0 || layer_end > m->L || layer_begin >= layer_end) return fail(CAKE_EINVAL, "prefill: bad layer range");
  if (chunk_len < 1 || chunk_len > m->rows_cap) return fail(CAKE_EINVAL, "prefill: chunk_len %d out of range", chunk_len);
  if (chunk_start < 0 || chunk_start + chunk_len > static_cast<long long>(m->n_logical_pages) * m->cfg.page_tokens)
    return fail(CAKE_EINVAL, "prefill: chunk beyond KV capacity");
  if (!(flags & CAKE_PREFILL_NO_KV_WRITE) && chunk_start % m->cfg.page_tokens)
    return fail(CAKE_EINVAL, "prefill: chunk must start on a page boundary");
  cudaStream_t s = S(stream);
  const int M = chunk_len;
  const int H = m->H;
  if (layer_begin == 0) {
    ProfScope ps(m, CAKE_K_EMBED, s, 0.0, static_cast<double>(M) * H * 6);
    CK(launch_chain(embed_kernel, dim3(M), dim3(128), 0, s, 1, d_tokens, static_cast<const bf16*>(m->embed), m->h, H,
                    d_abort));
    CKL();
  }
  const bool no_kv = (flags & CAKE_PREFILL_NO_KV_WRITE) != 0;
  if (overlap_ok(m, M, no_kv)) return prefill_overlap(m, chunk_start, M, layer_begin, layer_end, d_block_table, d_abort, s);
  for (int l = layer_begin; l < layer_end; ++l) {
    CKS(layer_attention_half(m, l, chunk_start, M, d_block_table, d_abort, no_kv, s));
    CKS(layer_mlp_half(m, l, M, d_abort, s));
  }
  return CAKE_OK;
}

// Test driver of head-sharded tensor parallelism on ONE device: the ranks'
// models run interleaved per half-layer on one stream and their row-parallel
// partial sums are added in rank order (a deterministic stand-in for the
// NCCL all-reduce the multi-GPU path calls at exactly the same two points).
int cake_prefill_group(cake_model** models, int n, const int32_t* d_tokens, long long chunk_start, int chunk_len,
                       const int32_t* d_block_table, void* stream) {
  if (n < 1 || !models) return fail(CAKE_EINVAL, "group: no models");
  cudaStream_t s = S(stream);
  const int M = chunk_len;
  for (int r = 0; r < n; ++r) {
    cake_model* m = models[r];
    if (m->cfg.tp_size != n || m->cfg.tp_rank != r) return fail(CAKE_EINVAL, "group: model %d is not rank %d of %d", r, r, n);
    if (chunk_start % m->cfg.page_tokens || M < 1 || M > m->rows_cap) return fail(CAKE_EINVAL, "group: bad chunk");
    m->emulated_tp = true;
    embed_kernel<<<M, 128, 0, s>>>(d_tokens, m->embed, m->h, m->H, nullptr);
    CKL();
  }
  auto reduce = [&]() -> int {
    const long long cnt = static_cast<long long>(M) * models[0]->H;
    for (int r = 0; r < n; ++r)
      for (int q = 0; q < n; ++q) {
        add_inplace_kernel<<<launch_grid_for(cnt / 4, 256), 256, 0, s>>>(models[r]->h, models[q]->tp_buf, cnt, nullptr);
        CKL();
      }
    return CAKE_OK;
  };
  int st = CAKE_OK;
  for (int l = 0; l < models[0]->L && st == CAKE_OK; ++l) {
    for (int r = 0; r < n && st == CAKE_OK; ++r)
      st = layer_attention_half(models[r], l, chunk_start, M, d_block_table, nullptr, false, s);
    if (st == CAKE_OK) st = reduce();
    for (int r = 0; r < n && st == CAKE_OK; ++r) st = layer_mlp_half(models[r], l, M, nullptr, s);
    if (st == CAKE_OK) st = reduce();
  }
  for (int r = 0; r < n; ++r) models[r]->emulated_tp = false;
  return st;
}

int cake_final_logits(cake_model* m, long long T, const int32_t* d_last_token, int recompute, int last_row,
                      const int32_t* d_block_table, float* d_logits, void* stream) {
  cudaStream_t s = S(stream);
  int row = last_row;
  if (recompute) {
    CKS(last_token_pass(m, d_last_token, T, d_block_table, s));
    row = 0;
  }
  if (row < 0 || row >= m->rows_cap) return fail(CAKE_EINVAL, "final: bad row");
  if (m->peer_tp && !recompute) {
    // prefill left h sharded by rows (row r on rank r % N): fetch the tail row
    // from its owner (final since this rank's last reduction saw every peer's B flag)
    const int owner = row % m->cfg.tp_size;
    if (owner != m->cfg.tp_rank)
      CK(cudaMemcpyAsync(m->h + static_cast<size_t>(row) * m->H, m->peer_h[owner] + static_cast<size_t>(row) * m->H,
                         m->H * sizeof(float), cudaMemcpyDeviceToDevice, s));
  }
  {
    ProfScope ps(m, CAKE_K_RMSNORM, s, 0.0, m->H * 6.0);
    rmsnorm_kernel<<<1, kNormThreadsPerRow * kNormRowsPerCta, 0, s>>>(m->h, m->final_norm, m->xn, m->H,
                                                                       m->cfg.rms_eps, row, 1, nullptr);
    CKL();
  }
  const int V = m->cfg.vocab;
  if (m->peer_tp) {
    // vocab-sharded LM head: rank r computes rows [r V / N, (r+1) V / N) and stores
    // them into every rank's logits buffer; a flag barrier, then the assembled row is copied out
    const int n = m->cfg.tp_size, r = m->cfg.tp_rank;
    TpGemvArgs g{};
    g.W = m->lm_head;
    g.x = m->xn;
    for (int q = 0; q < n; ++q) g.out[q] = m->peer_logits[q];
    g.nranks = n;
    g.n0 = static_cast<int>(static_cast<long long>(V) * r / n);
    g.n1 = static_cast<int>(static_cast<long long>(V) * (r + 1) / n);
    g.K = m->H;
    {
      const double rows = g.n1 - g.n0;
      ProfScope ps(m, CAKE_K_LMHEAD, s, 2.0 * rows * m->H, 2.0 * rows * m->H);
      const int grid = std::max(1, std::min((g.n1 - g.n0 + 7) / 8, num_sms() * 4));
      tp_gemv_kernel<<<grid, 256, m->H * sizeof(float), s>>>(g);
      CKL();
    }
    TpReduceArgs b{};
    for (int q = 0; q < n; ++q) b.flags[q] = m->peer_flags[q];
    b.rank = r;
    b.nranks = n;
    b.epoch = ++m->tp_epoch;
    tp_barrier_kernel<<<1, 32, 0, s>>>(b);
    CKL();
    CK(cudaMemcpyAsync(d_logits, m->tp_logits, static_cast<size_t>(V) * sizeof(float), cudaMemcpyDeviceToDevice, s));
    return CAKE_OK;
  }
  {
    ProfScope ps(m, CAKE_K_LMHEAD, s, 2.0 * V * m->H, 2.0 * V * m->H);
    const int threads = 256;
    const int grid = std::min((V + 7) / 8, num_sms() * 4);
    gemv_kernel<<<grid, threads, m->H * sizeof(float), s>>>(m->lm_head, m->xn, d_logits, V, m->H);
    CKL();
  }
  return CAKE_OK;
}

long long cake_kv_chunk_bytes(const cake_model* m, int chunk_len) {
  return 2LL * m->L * m->nkv * m->hd * 2 * chunk_len;
}

int cake_attention_debug(cake_model* m, const void* d_q, long long chunk_start, int chunk_len, int layer,
                         const int32_t* d_block_table, void* d_out, void* stream) {
  if (!m || !d_q || !d_out || !d_block_table) return fail(CAKE_EINVAL, "attention debug: null");
  if (layer < 0 || layer >= m->L) return fail(CAKE_EINVAL, "attention debug: bad layer");
  if (chunk_len < 1 || chunk_len > m->rows_cap) return fail(CAKE_EINVAL, "attention debug: chunk_len out of range");
  if (chunk_start < 0 || chunk_start + chunk_len > static_cast<long long>(m->n_logical_pages) * m->cfg.page_tokens)
    return fail(CAKE_EINVAL, "attention debug: beyond KV capacity");
  cudaStream_t s = S(stream);
  const size_t bytes = static_cast<size_t>(chunk_len) * m->nq * m->hd * sizeof(bf16);
  CK(cudaMemcpyAsync(m->q, d_q, bytes, cudaMemcpyDeviceToDevice, s));
  CKS(attention(m, chunk_start, chunk_len, layer, d_block_table, nullptr, s));
  CK(cudaMemcpyAsync(d_out, m->attn, bytes, cudaMemcpyDeviceToDevice, s));
  return CAKE_OK;
}

int cake_kv_poison(cake_model* m, int byte, void* stream) {
  if (!m) return fail(CAKE_EINVAL, "kv poison: null model");
  CK(cudaMemsetAsync(m->pool, byte & 0xFF, m->pool_bytes, S(stream)));
  return CAKE_OK;
}

static int kv_permute(cake_model* m, void* staging, long long chunk_start, int chunk_len, const int32_t* bt,
                      long long b0, long long b1, bool to_pool, cudaStream_t s) {
  if (chunk_start % m->cfg.page_tokens) return fail(CAKE_EINVAL, "kv: chunk must start on a page boundary");
  if (b0 % 16 || b1 % 16 || b0 < 0 || b1 > cake_kv_chunk_bytes(m, chunk_len) || b0 > b1)
    return fail(CAKE_EINVAL, "kv: byte range must be 16-B aligned and inside the chunk");
  if (b0 == b1) return CAKE_OK;
  KvLayout L{m->L, m->nkv, m->hd, m->cfg.page_tokens};
  const unsigned v0 = static_cast<unsigned>(b0 / 16), v1 = static_cast<unsigned>(b1 / 16);
  const int grid = launch_grid_for(v1 - v0, 256);
  ProfScope ps(m, CAKE_K_SCATTER, s, 0.0, 2.0 * (b1 - b0));
  if (to_pool)
    kv_permute_kernel<true><<<grid, 256, 0, s>>>(static_cast<uint4*>(staging), reinterpret_cast<uint4*>(m->pool), bt,
                                                 chunk_start / m->cfg.page_tokens, chunk_len, L, v0, v1);
  else
    kv_permute_kernel<false><<<grid, 256, 0, s>>>(static_cast<uint4*>(staging), reinterpret_cast<uint4*>(m->pool), bt,
                                                  chunk_start / m->cfg.page_tokens, chunk_len, L, v0, v1);
  CKL();
  return CAKE_OK;
}

int cake_kv_scatter(cake_model* m, const void* d_staging, long long chunk_start, int chunk_len,
                    const int32_t* d_block_table, long long byte_begin, long long byte_end, void* stream) {
  return kv_permute(m, const_cast<void*>(d_staging), chunk_start, chunk_len, d_block_table, byte_begin, byte_end,
                    true, S(stream));
}

int cake_kv_gather(cake_model* m, void* d_staging, long long chunk_start, int chunk_len,
                   const int32_t* d_block_table, void* stream) {
  return kv_permute(m, d_staging, chunk_start, chunk_len, d_block_table, 0, cake_kv_chunk_bytes(m, chunk_len),
                    false, S(stream));
}

long long cake_kv_q8_bytes(const cake_model* m, int chunk_len) { return cake_kv_chunk_bytes(m, chunk_len) / 2 + 4; }

int cake_kv_scatter_q8(cake_model* m, const void* d_encoded, long long chunk_start, int chunk_len,
                       const int32_t* d_block_table, void* stream) {
  if (chunk_start % m->cfg.page_tokens) return fail(CAKE_EINVAL, "kv q8: chunk must start on a page boundary");
  if ((reinterpret_cast<uintptr_t>(d_encoded) + 4) % 16)
    return fail(CAKE_EINVAL, "kv q8: payload (encoded + 4) must be 16-B aligned");
  const long long n = cake_kv_chunk_bytes(m, chunk_len) / 2;
  KvLayout L{m->L, m->nkv, m->hd, m->cfg.page_tokens};
  const unsigned n16 = static_cast<unsigned>(n / 16);
  const int grid = launch_grid_for(n16, 256);
  cudaStream_t s = S(stream);
  ProfScope ps(m, CAKE_K_SCATTER, s, 0.0, static_cast<double>(n) + 2.0 * n);
  const auto* enc = static_cast<const uint8_t*>(d_encoded);
  kv_scatter_q8_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const uint4*>(enc + 4), reinterpret_cast<const __half*>(enc),
                                            reinterpret_cast<uint4*>(m->pool), d_block_table,
                                            chunk_start / m->cfg.page_tokens, chunk_len, L, n16);
  CKL();
  return CAKE_OK;
}

int cake_kv_encode_q8(cake_model* m, const void* d_chunk, int chunk_len, void* d_encoded, void* stream) {
  if (reinterpret_cast<uintptr_t>(d_chunk) % 16 || reinterpret_cast<uintptr_t>(d_encoded) % 4)
    return fail(CAKE_EINVAL, "kv q8 encode: chunk 16-B / encoded 4-B alignment");
  const long long n = cake_kv_chunk_bytes(m, chunk_len) / 2;
  const unsigned n8 = static_cast<unsigned>(n / 8);
  cudaStream_t s = S(stream);
  const unsigned init[2] = {0xFFFFFFFFu, 0u};
  CK(cudaMemcpyAsync(m->q8_ws, init, sizeof(init), cudaMemcpyHostToDevice, s));
  const int grid = launch_grid_for(n8, 256);
  kv_minmax_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(d_chunk), n8, m->q8_ws);
  CKL();
  kv_quant8_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(d_chunk), n8, m->q8_ws,
                                        static_cast<uint8_t*>(d_encoded));
  CKL();
  return CAKE_OK;
}

int cake_gemm_set_schedule(int schedule) {
  // bit 0: stream-K; bit 1: disable the 2-SM kernel; bit 2: 1-SM weight multicast clusters
  g_gemm_prefetch = ((schedule >> 10) & 15) - 1;  // bits 10-13: 1 + weight stages prefetched before the PDL wait
  schedule &= 1023;
  if (schedule < 0)
    return fail(CAKE_EINVAL, "schedule bits: 1 stream-K, 2 no-2SM, 4 multicast, 8 1-SM N-128 tiles, 128 no QKV N-192, "
                             "256 no A-sharing pair clusters, 512 four pairs per cluster");
  g_gemm_pairs = (schedule & 256) ? 1 : (schedule & 512) ? 4 : 2;
  g_gemm_qkv192 = (schedule & 128) ? 0 : 1;
  g_gemm_2sm_n128 = (schedule & 8) ? 0 : 1;
  g_gemm_hints = 3 ^ ((schedule >> 4) & 3);  // bits 4/5 drop the evict_last hint of A / B
  g_gemm_tail_split = (schedule & 64) ? 0 : 1;  // bit 6: no tail split
  g_gemm_schedule = schedule & 1;
  g_gemm_2sm = (schedule & 2) ? 0 : 1;
  g_gemm_cluster = (schedule & 4) ? 1 : 0;
  return CAKE_OK;
}

int cake_dec_set_prefetch(int kb) {
  if (kb < 0) return fail(CAKE_EINVAL, "dec prefetch: kb >= 0");
  g_dec_prefetch_kb = kb;
  return CAKE_OK;
}

int cake_set_experiment(int knob, int value) {
  if (knob < 0 || knob >= CAKE_EXP_COUNT) return fail(CAKE_EINVAL, "experiment knob %d out of range", knob);
  g_exp[knob] = value;
  return CAKE_OK;
}

// Debug: %globaltimer stamps of every CTA of the decode chain launch for `layer`
// ([cta][16]: entry, after the PDL wait, then per phase: start, x staged, rows done).
CAKE_API int cake_dec_debug_trace(long long* dev_buf, int layer) {
  g_dec_trace = dev_buf;
  g_dec_trace_layer = dev_buf != nullptr ? layer : -2;
  return CAKE_OK;
}

// Debug: stamp %globaltimer at fixed points of the first / last CTA of the
// next `cap` pair-cluster GEMM launches into dev_buf[32 * launch + slot]; nullptr stops.
CAKE_API int cake_gemm_debug_trace(long long* dev_buf, int cap) {
  g_gemm_trace = dev_buf;
  g_gemm_trace_n = 0;
  g_gemm_trace_cap = cap;
  return CAKE_OK;
}

int cake_gemm(const void* dA, const void* dB, void* dC, int M, int N, int K, int epi, int block_n, void* stream) {
  if (M < 1 || N < 1 || K < 64 || K % 64 || N % block_n) return fail(CAKE_EINVAL, "gemm: bad shape");
  if (epi < 0 || epi > 2) return fail(CAKE_EINVAL, "gemm: epi must be 0..2");
  CUtensorMap ta[3], tb[3];
  for (int i = 0; i < 3; ++i)
    CKS(make_map(&ta[i], dA, static_cast<uint64_t>(M), static_cast<uint64_t>(K), static_cast<uint32_t>(128 >> i)));
  for (int ci = 0; ci < 3; ++ci)
    CKS(make_map(&tb[ci], dB, static_cast<uint64_t>(N), static_cast<uint64_t>(K), static_cast<uint32_t>(block_n >> ci)));
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.out = dC;
  g.ldo = N;
  g.resid = static_cast<float*>(dC);
  g.ldr = N;
  CUtensorMap om[2];
  if (epi == 2) {
    CKS(make_map_f32(&om[0], dC, static_cast<uint64_t>(M), static_cast<uint64_t>(N), static_cast<uint64_t>(N), 128));
    om[1] = om[0];  // no bf16 copy (xb_out == nullptr)
  }
  return gemm_dispatch(block_n, epi, ta, tb, g, S(stream), epi == 2 ? om : nullptr);
}

}  // extern "C"
