/*
 * cake_cuda.h — thin C-ABI CUDA layer underneath the cake:: host runtime.
 *
 * This is the "L3.5" layer of SURVEY.md §1: the reference (C++20, host
 * threads only) has no device code at all — its compute side sleeps for a
 * modeled latency (reference proj/src/compute.cpp:48-49) and its loader lands
 * bytes in heap buffers (proj/src/transfer.cpp:149-170). Every entry point
 * here is what the B200 build puts in place of one of those stand-ins:
 *
 *   cake_prefill_chunk      replaces sleep_for_us(compute_latency(...))
 *                           in ComputeEngine::run_forward (compute.cpp:48-49)
 *   cake_kv_scatter         replaces the heap landing of TransferEngine's
 *                           reader/pacer (transfer.cpp:149-170, 209-225) with
 *                           a staging -> paged-KV permutation on the copy stream
 *   cake_event_*            replace ResidentSet's mutex hand-off
 *                           (transfer.cpp:9-24): residency = event completed
 *   cake_final_logits       first-token step the reference never models
 *                           (its TTFT stops at KV residency, report.hpp:39)
 *
 * Conventions: plain C types only; every call returns int status
 * (0 = ok, > 0 = the cudaError_t / ncclResult_t that failed offset by
 * CAKE_ECUDA / CAKE_ENCCL, < 0 = cake validation errors); a message for the
 * last failure on the calling thread is available from cake_cuda_last_error.
 * Streams and events are opaque void* handles. All launches are
 * stream-ordered; nothing blocks except *_sync calls.
 */
#ifndef CAKE_CUDA_H_
#define CAKE_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CAKE_API __attribute__((visibility("default")))
#else
#define CAKE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  CAKE_OK = 0,
  CAKE_EINVAL = -1,
  CAKE_ENOMEM = -2,
  CAKE_ESTATE = -3,
  CAKE_ENOTREADY = 1, /* cake_event_query: work still pending */
  CAKE_ECUDA = 1000,  /* + cudaError_t */
  CAKE_ENCCL = 2000   /* + ncclResult_t */
};

CAKE_API int cake_cuda_last_error(char* buf, size_t len);
CAKE_API int cake_cuda_version(int* runtime, int* driver);
CAKE_API int cake_cuda_device_count(int* n);
CAKE_API int cake_cuda_set_device(int device);
/* Make `device` the calling thread's current device, only if it is not already (worker threads
 * of the loader start on device 0; no cached state is dropped). */
CAKE_API int cake_cuda_bind_thread(int device);
CAKE_API int cake_cuda_sm_count(int device, int* n);
CAKE_API int cake_cuda_device_sync(void);

/* ---------------------------------------------------------- streams/events */
CAKE_API int cake_stream_create(void** stream, int high_priority);
CAKE_API int cake_stream_destroy(void* stream);
/* A stream confined to (at least) n_sms SMs (green context over an SM
 * partition); n_sms <= 0 or >= the device's count gives a normal stream.
 * got_sms receives the partition size. GPU-share emulation. */
CAKE_API int cake_stream_create_sm_share(void** stream, int n_sms, int* got_sms);
/* Launch sizing (persistent grids, split counts) for an SM budget; 0 = the device. */
CAKE_API int cake_set_sm_budget(int n_sms);
CAKE_API int cake_stream_sync(void* stream);
CAKE_API int cake_stream_wait_event(void* stream, void* event);
CAKE_API int cake_event_create(void** event, int timing);
CAKE_API int cake_event_destroy(void* event);
CAKE_API int cake_event_record(void* event, void* stream);
CAKE_API int cake_event_query(void* event); /* CAKE_OK when complete, CAKE_ENOTREADY if pending */
CAKE_API int cake_event_sync(void* event);
CAKE_API int cake_event_elapsed_ms(void* start, void* stop, float* ms);

/* ---------------------------------------------------------- memory */
CAKE_API int cake_host_alloc(void** p, size_t bytes);  /* pinned, portable */
CAKE_API int cake_host_free(void* p);
CAKE_API int cake_host_register(void* p, size_t bytes);
CAKE_API int cake_host_unregister(void* p);
CAKE_API int cake_dev_alloc(void** p, size_t bytes);
CAKE_API int cake_dev_free(void* p);
CAKE_API int cake_memset_async(void* dst, int value, size_t bytes, void* stream);
CAKE_API int cake_h2d_async(void* dst, const void* src, size_t bytes, void* stream);
CAKE_API int cake_d2h_async(void* dst, const void* src, size_t bytes, void* stream);
CAKE_API int cake_d2d_async(void* dst, const void* src, size_t bytes, void* stream);

/* ---------------------------------------------------------- model */
typedef struct cake_model_config {
  int n_layers;
  int hidden;
  int n_heads;     /* query heads, whole model */
  int n_kv_heads;  /* KV heads, whole model */
  int head_dim;    /* 64 or 128 */
  int ffn;         /* MLP intermediate size, whole model */
  int vocab;
  float rope_theta;
  float rms_eps;
  int page_tokens; /* KV page size; 64 */
  int max_chunk;   /* largest chunk (rows) the activation scratch holds */
  long long max_tokens; /* KV capacity (logical pages = ceil(max_tokens / page_tokens)) */
  int spare_pages; /* extra physical pages (second page set of a contested chunk) */
  int tp_rank;
  int tp_size;
  unsigned long long seed;
} cake_model_config;

typedef struct cake_model_info {
  long long kv_bytes_per_token;   /* this rank's shard */
  long long page_bytes;           /* one physical page, all layers */
  int n_logical_pages;
  int n_physical_pages;
  int local_q_heads, local_kv_heads, local_ffn;
  long long weight_bytes;
  long long flops_per_token_linear; /* 2 * (this rank's projection weights), no LM head */
  void* kv_pool;
} cake_model_info;

typedef struct cake_model cake_model;

CAKE_API int cake_model_create(const cake_model_config* cfg, cake_model** out);
/* A model that shares `parent`'s weights (same dimensions, seed and TP shard;
 * `parent` must outlive it) and owns its own paged pool and scratch: one
 * context per concurrent request on a device, weights resident once. */
CAKE_API int cake_model_create_shared(const cake_model_config* cfg, const cake_model* parent, cake_model** out);
CAKE_API int cake_model_destroy(cake_model* m);
CAKE_API int cake_model_get_info(const cake_model* m, cake_model_info* out);
/* Attention kernel variant: 0 = product dispatch (tcgen05/TMEM flash attention,
 * softmax warpgroups on alternate key blocks, attention_alt.cuh), 1 = mma.sync
 * flash attention (independent cross-check), 2 = the column-split one-tile
 * tcgen05 kernel (attention_tc.cuh), 5 = the alternate-block kernel explicitly;
 * 3 / 4 (two-tile, decoupled groups) need an ATTN_VARIANTS=1 build. */
CAKE_API int cake_model_set_attention_impl(cake_model* m, int impl);
/* NCCL plumbing for head-sharded TP (one process per GPU): rank 0 makes the
 * 128-byte id, the launcher broadcasts it, every rank inits its communicator. */
CAKE_API int cake_nccl_unique_id(void* out128);
CAKE_API int cake_nccl_init(void** comm, const void* id128, int nranks, int rank);
CAKE_API int cake_nccl_destroy(void* comm);
/* Test driver: the n TP ranks' models (same device) run one chunk interleaved
 * per half-layer, their row-parallel partials summed in rank order in place of
 * the all-reduce. Verifies the sharding on a single GPU. */
CAKE_API int cake_prefill_group(cake_model** models, int n, const int32_t* d_tokens, long long chunk_start,
                                int chunk_len, const int32_t* d_block_table, void* stream);
/* Attach an NCCL communicator (ncclComm_t) for tp_size > 1 (the baseline
 * reduction: fp32 ncclAllReduce + add + rmsnorm kernels). */
CAKE_API int cake_model_set_comm(cake_model* m, void* nccl_comm);
/* Peer-memory TP (the product reduction, csrc/cuda/tp_peer.cuh): after each
 * row-parallel projection ONE kernel pulls the peers' bf16 partials of this
 * rank's row slice over NVLink, adds them in rank order into the residual,
 * applies the next RMSNorm and pushes the normalized rows into every rank's
 * activation buffer. Replaces the two ncclAllReduce calls per layer of the
 * north-star design (reference wiring: proj/src/scheduler.cpp:229-278 runs
 * one compute agent; here one per GPU in lockstep).
 * The first-token LM head is vocab-sharded: each rank computes V/N logits and
 * stores them into every rank's logits buffer.
 * Every rank exports CAKE_TP_PEER_HANDLE_BYTES of CUDA IPC handles; the
 * launcher all-gathers them (rank order) and every rank opens the set. */
#define CAKE_TP_PEER_HANDLE_BYTES 512
CAKE_API int cake_tp_peer_handles(cake_model* m, void* out, size_t cap);
CAKE_API int cake_tp_peer_open(cake_model* m, const void* all_handles, int nranks);

enum {
  CAKE_PREFILL_NO_KV_WRITE = 1 /* q-only pass (first-token step over a complete cache) */
};

/* One chunk of prefill through every layer on `stream`. d_tokens: the
 * chunk's chunk_len token ids (device int32). d_block_table: logical page ->
 * physical page. d_abort (optional): device int; when non-zero at a kernel's
 * start the kernel exits (lost race / cancelled chunk). */
CAKE_API int cake_prefill_chunk(cake_model* m, const int32_t* d_tokens, long long chunk_start, int chunk_len,
                       const int32_t* d_block_table, const int32_t* d_abort, int flags, void* stream);

/* Layers [layer_begin, layer_end) of one chunk (embedding runs with layer 0).
 * Lets the host record an event a few layers before the end of a chunk, which
 * is when the scheduler claims the next one. */
CAKE_API int cake_prefill_layers(cake_model* m, const int32_t* d_tokens, long long chunk_start, int chunk_len,
                                 int layer_begin, int layer_end, const int32_t* d_block_table,
                                 const int32_t* d_abort, int flags, void* stream);

/* First-token logits (fp32 [vocab]) of a prompt of T tokens whose KV is fully
 * resident. recompute = 1: run the last token as a 1-row q-only pass over the
 * cache (needed when the tail chunk was loaded, not computed); recompute = 0:
 * use row `last_row` of the hidden state the last prefill_chunk left behind. */
CAKE_API int cake_final_logits(cake_model* m, long long T, const int32_t* d_last_token, int recompute,
                      int last_row, const int32_t* d_block_table, float* d_logits, void* stream);

/* ---------------------------------------------------------- KV loader */
/* Bytes of one chunk of chunk_len tokens in the cache-tier format
 * [layer][K|V][kv_head][token][head_dim] bf16 (this rank's shard). */
CAKE_API long long cake_kv_chunk_bytes(const cake_model* m, int chunk_len);
/* Test instrumentation: fill the whole paged pool (every physical page,
 * spare set included) with `byte` on `stream` (0xFF = bf16 NaN). */
CAKE_API int cake_kv_poison(cake_model* m, int byte, void* stream);
/* staging bytes [byte_begin, byte_end) (16-B aligned) of a chunk starting at
 * token chunk_start -> paged pool through d_block_table. */
/* Test entry: the model's attention kernel alone (the product dispatch, or the
 * impl set by cake_model_set_attention_impl) for q rows d_q [chunk_len][local q
 * heads][head_dim] bf16 at positions chunk_start.., over the paged KV of `layer`
 * (keys <= each row's position); the output rows are copied to d_out (same
 * shape). Lets tests compare the kernel with a plain fp32 attention. */
CAKE_API int cake_attention_debug(cake_model* m, const void* d_q, long long chunk_start, int chunk_len, int layer,
                                  const int32_t* d_block_table, void* d_out, void* stream);
CAKE_API int cake_kv_scatter(cake_model* m, const void* d_staging, long long chunk_start, int chunk_len,
                    const int32_t* d_block_table, long long byte_begin, long long byte_end,
                    void* stream);
/* Inverse: paged pool -> staging (cache-tier format). */
CAKE_API int cake_kv_gather(cake_model* m, void* d_staging, long long chunk_start, int chunk_len,
                   const int32_t* d_block_table, void* stream);
/* quant8 cache tier (reference proj/src/codec.cpp:114-162, Codec::quant8):
 * encoded chunk = [lo fp16][hi fp16][one u8 level per element of the tier
 * format], i.e. cake_kv_chunk_bytes/2 + 4 bytes. The decode is fused into the
 * scatter (dequantise + permute into the bf16 pages, one pass); d_encoded + 4
 * must be 16-B aligned. encode: a gathered bf16 chunk -> encoded (4-B aligned). */
CAKE_API long long cake_kv_q8_bytes(const cake_model* m, int chunk_len);
CAKE_API int cake_kv_scatter_q8(cake_model* m, const void* d_encoded, long long chunk_start, int chunk_len,
                                const int32_t* d_block_table, void* stream);
CAKE_API int cake_kv_encode_q8(cake_model* m, const void* d_chunk, int chunk_len, void* d_encoded, void* stream);

/* ---------------------------------------------------------- profiling */
enum {
  CAKE_K_EMBED = 0,
  CAKE_K_RMSNORM,
  CAKE_K_GEMM_QKV,
  CAKE_K_ATTN,
  CAKE_K_GEMM_O,
  CAKE_K_GEMM_GU,
  CAKE_K_GEMM_D,
  CAKE_K_ALLREDUCE,
  CAKE_K_LMHEAD,
  CAKE_K_SCATTER,
  CAKE_K_DEC_PROJ, /* first-token step: the weight-streaming q / o / gate-up / down GEMVs */
  CAKE_K_DEC_ATTN, /* first-token step: 1-query attention over the assembled cache */
  CAKE_K_COUNT
};
typedef struct cake_kernel_stat {
  long long launches;
  double total_ms;
  double flops;  /* algorithmic */
  double bytes;  /* algorithmic */
} cake_kernel_stat;
/* mask bit k (CAKE_K_*): every launch of kernel class k is bracketed by CUDA
 * events on its stream (-1 = all, 0 = off); stats resolve (and reset) on read. */
CAKE_API int cake_model_set_profiling(cake_model* m, int mask);
/* Bracket only every n-th launch of a profiled class (n >= 1; default 1). */
CAKE_API int cake_model_set_profiling_stride(cake_model* m, int stride);
CAKE_API int cake_model_kernel_stats(cake_model* m, cake_kernel_stat* out /* [CAKE_K_COUNT] */, int reset);
CAKE_API int cake_model_launch_count(cake_model* m, long long* n, int reset);

/* ---------------------------------------------------------- unit entry points */
/* Projection GEMM schedule for subsequent launches (bit flags): bit0 stream-K
 * instead of whole tiles (+ exact split-K), bit1 disable the 2-SM
 * (cta_group::2) kernel for M > 128, bit2 weight-multicast clusters in the
 * 1-SM kernel, bit3 N-128 tiles (O / down) on the 1-SM kernel instead of CTA
 * pairs, bits 4/5 drop the L2 evict_last hint of A / B, bit6 no K-split of
 * the short last gate/up round, bit7 QKV on N-256 tiles instead of N-192. Default 0. */
CAKE_API int cake_gemm_set_schedule(int schedule);
/* A/B switches for measurements only (process-wide; the defaults are the product):
 * PDL 1 = programmatic dependent launch on; FUSED_NORM 1 = RMSNorm folded into the
 * projections; ATTN_MAX_WAVES = CTA waves the split-KV dispatch may use (1);
 * GEMM_NOSPLIT 1 = no split-K for the few-tile pair GEMMs (0). */
enum { CAKE_EXP_PDL = 0, CAKE_EXP_FUSED_NORM = 1, CAKE_EXP_ATTN_MAX_WAVES = 2, CAKE_EXP_GEMM_NOSPLIT = 3,
       CAKE_EXP_DEC_CHAIN = 4, /* 1: first-token projections on the persistent chain kernel, 0: per-projection GEMVs */
       CAKE_EXP_TP_OVERLAP = 5, /* 1: peer-TP prefill chunks run as two row micro-batches, each one's reductions
                                   overlapping the other's projections; 0: one batch, reduce in line */
       CAKE_EXP_COUNT = 6 };
CAKE_API int cake_set_experiment(int knob, int value);
/* First-token chain kernel: L2 prefetch per CTA ahead of each phase, in KB (A/B; default 128). */
CAKE_API int cake_dec_set_prefetch(int kb);
/* C = A · B^T for bf16 row-major A [M, K], B [N, K]; epi 0: bf16 C, 1: fp32 C,
 * 2: fp32 C += . block_n 128 or 256. For tests and microbenchmarks. */
CAKE_API int cake_gemm(const void* dA, const void* dB, void* dC, int M, int N, int K, int epi, int block_n,
              void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CAKE_CUDA_H_ */
