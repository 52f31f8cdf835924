/*
 * cake_c.h — C ABI over the cake:: host runtime (libcake.so), the binding
 * surface for FFI callers (the Python mirror in paper_2410_03065_b200/, and
 * any ctypes/cffi/JNI host). The reference exposes only a C++ API
 * (proj/include/cake/ headers); each entry here is a flat-argument wrapper of
 * one of those calls, cited inline, plus the B200 GPU run.
 *
 * Status: 0 ok; CAKE_C_EINVAL (std::invalid_argument), CAKE_C_ELOGIC
 * (std::logic_error), CAKE_C_EMISSING (MissingKeyError), CAKE_C_ECORRUPT
 * (CorruptChunkError), CAKE_C_ESTORE (other StoreError), CAKE_C_ERUNTIME
 * (anything else, incl. CUDA/NCCL failures). cake_last_error() returns the
 * exception message of the last failure on the calling thread.
 */
#ifndef CAKE_C_H_
#define CAKE_C_H_

#include <stddef.h>
#include <stdint.h>

#include "cake_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

enum {
  CAKE_C_EINVAL = -1,
  CAKE_C_ELOGIC = -2,
  CAKE_C_EMISSING = -3,
  CAKE_C_ECORRUPT = -4,
  CAKE_C_ESTORE = -5,
  CAKE_C_ERUNTIME = -6
};

enum { CAKE_MODE_CAKE = 0, CAKE_MODE_COMPUTE_ONLY = 1, CAKE_MODE_IO_ONLY = 2 };
enum { CAKE_SIDE_COMPUTE = 0, CAKE_SIDE_IO = 1 };

CAKE_API int cake_last_error(char* buf, size_t len);

/* ---- cost laws (reference proj/include/cake/model.hpp:79-96) ---- */
typedef struct cake_trace {
  const int64_t* at_us; /* breakpoints, first must be 0 */
  const double* mbps;
  int n;
} cake_trace;

CAKE_API int cake_time_to_transfer_bits(cake_trace trace, uint64_t bits, int64_t start_us, int64_t* out);
CAKE_API int cake_fetch_latency(cake_trace trace, uint64_t nbytes, int64_t start_us, int64_t* out);
CAKE_API int cake_compute_latency(double alpha_ms, double beta_ms_per_token, uint32_t ref_chunk, uint64_t token_start,
                                  uint32_t token_count, double power, int64_t* out);
CAKE_API int cake_kv_bytes_per_token(uint32_t n_layers, uint32_t hidden, uint32_t precision, uint32_t kv_mult,
                                     uint64_t override_or_0, uint64_t* out);
/* n_out = number of chunks; starts/counts filled up to cap */
CAKE_API int cake_split_into_chunks(uint64_t total_tokens, uint32_t chunk_size, uint32_t* n_out, uint64_t* starts,
                                    uint32_t* counts, uint32_t cap);
/* reference proj/include/cake/scheduler.hpp:68-69 */
CAKE_API int cake_oracle_best_split(const int64_t* compute_us, uint32_t n_compute, const int64_t* fetch_us,
                                    uint32_t n_fetch, uint32_t* k_star, int64_t* ttft_star);

/* ---- scheduler (reference proj/include/cake/scheduler.hpp:75-83) ---- */
typedef struct cake_record {
  uint32_t index;
  int32_t side; /* CAKE_SIDE_* */
  int64_t start_us;
  int64_t finish_us;
  uint64_t bytes;
} cake_record;

typedef struct cake_run_opts {
  int compute_enabled;
  int io_enabled;
  uint32_t token_budget;
  uint64_t throttle_quantum_bytes;
  double decode_us_per_byte;
  uint32_t jitter_max_us;
  uint64_t jitter_seed;
  int race_to_finish; /* B200 extension */
  int cached_prefix;  /* B200 extension: the tier may hold only a leading run of chunks */
  int record_slices;  /* log every released slice (TransferOptions::record_slices) */
  int race_force;     /* test instrumentation (RunOptions::race_force): 0 policy, 1 compute contests, 2 io contests */
  int race_hold;      /* test instrumentation (RunOptions::race_hold): -1 off, 0 compute waits, 1 io waits */
  void* link;         /* B200 extension: a cake_link* the loader paces through (shared with other runs), or NULL */
} cake_run_opts;

typedef struct cake_summary {
  int64_t ttft_us;
  uint32_t merge_point;
  uint32_t n_chunks;
  double computed_fraction;
  int64_t compute_busy_us;
  int64_t io_busy_us;
} cake_summary;

CAKE_API void cake_run_opts_default(cake_run_opts* o);

/* run_sim_planned over an explicit plan; records[n] in index order. */
CAKE_API int cake_sim_run(uint32_t n, const uint64_t* token_starts, const uint32_t* token_counts,
                          const uint64_t* encoded_bytes, const uint64_t* uncompressed_bytes, double alpha_ms,
                          double beta_ms_per_token, uint32_t ref_chunk, cake_trace trace, int mode, double power,
                          const cake_run_opts* opts, cake_summary* summary, cake_record* records);

/* ---- cache tier (reference proj/include/cake/store.hpp) ---- */
typedef struct cake_store cake_store;
/* root == NULL or "": memory-resident store (pinned when pinned != 0). create: 0 open, 1 create, 2 open_or_create */
CAKE_API int cake_store_open(const char* root, int create, int pinned, cake_store** out);
CAKE_API int cake_store_close(cake_store* s);
/* B200 extension: file-backed stores read aligned slices with O_DIRECT (page-cache bypass). */
CAKE_API int cake_store_set_direct_io(cake_store* s, int on);
CAKE_API int cake_store_entry_count(const cake_store* s, uint64_t* n);
/* populate(store, request, profile, codec, seed, kind) — reference proj/src/store.cpp:303-334 */
CAKE_API int cake_store_populate(cake_store* s, uint64_t total_tokens, uint32_t chunk_size, uint32_t n_layers,
                                 uint32_t hidden, uint32_t precision, const char* codec, uint64_t seed, int sparse,
                                 uint8_t* keys_out /* 32 * n_chunks or NULL */);
CAKE_API int cake_store_put(cake_store* s, const uint8_t* key32, const uint8_t* payload, uint64_t n,
                            uint32_t token_count, const char* codec, uint64_t uncompressed);
CAKE_API int cake_store_get(const cake_store* s, const uint8_t* key32, uint8_t* out, uint64_t cap, uint64_t* n_out);
CAKE_API int cake_store_make_resident(cake_store* s, int pinned);

CAKE_API int cake_chain_hash(const uint8_t* prev32_or_null, const uint32_t* tokens, uint64_t n, uint8_t* out32);
CAKE_API int cake_token_stream(uint64_t seed, uint64_t count, uint32_t* out);
CAKE_API int cake_synth_payload(uint64_t seed, uint32_t chunk_index, uint64_t nbytes, uint8_t* out);
CAKE_API int cake_codec_encoded_size(const char* codec, uint64_t raw, uint64_t* out);
CAKE_API int cake_codec_encode(const char* codec, const uint8_t* in, uint64_t n, uint8_t* out, uint64_t cap,
                               uint64_t* n_out);
CAKE_API int cake_codec_decode(const char* codec, const uint8_t* in, uint64_t n, uint64_t original_len, uint8_t* out,
                               uint64_t cap);
CAKE_API uint16_t cake_fp16_from_float(float f);
CAKE_API float cake_fp16_to_float(uint16_t h);

/* run(..., ClockMode, store, seed, options) with the modeled compute side
 * (reference proj/src/scheduler.cpp:282-294); clock 0 = sim, 1 = live. */
CAKE_API int cake_run_store(cake_store* s, uint64_t total_tokens, uint32_t chunk_size, uint32_t n_layers,
                            uint32_t hidden, uint32_t precision, const char* codec, double alpha_ms,
                            double beta_ms_per_token, uint32_t ref_chunk, cake_trace trace, int mode, int clock,
                            uint64_t seed, double power, const cake_run_opts* opts, cake_summary* summary,
                            cake_record* records);

/* ---- B200 GPU run ---- */
typedef struct cake_gpu cake_gpu;
typedef struct cake_gpu_config {
  int n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab;
  float rope_theta, rms_eps;
  int max_chunk;
  long long max_tokens;
  unsigned long long weight_seed;
  int device;
  int tp_rank, tp_size;
  void* nccl_comm;
  int lookahead_layers;
  int profile_kernels;
  int64_t race_margin_us;
  const char* tp_shm; /* POSIX shm name of the TP group's coordinator (tp_size > 1), NULL otherwise */
  int compute_sms;    /* > 0: confine the compute stream to this many SMs (GPU-share emulation) */
  const struct cake_gpu* weights_from; /* non-NULL: share this context's weights (same dims, seed, TP shard;
                                          it must outlive the new one) — concurrent requests on one device */
} cake_gpu_config;

typedef struct cake_gpu_result {
  int64_t kv_resident_us; /* reference TTFT: last chunk resident */
  int64_t first_token_us; /* logits on host: north-star TTFT */
  int64_t final_step_us;
  double device_ttft_ms;
  uint32_t merge_point;
  uint32_t n_chunks;
  int raced_chunk;
  int race_winner; /* 0 compute, 1 io, -1 none */
  int recomputed_last;
  long long kernel_launches;
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  int64_t compute_busy_us;
  int64_t io_busy_us;
} cake_gpu_result;

CAKE_API int cake_gpu_create(const cake_gpu_config* cfg, cake_gpu** out);
/* One emulated link shared by several contexts' loaders (concurrent requests
 * on one device): every slice of every attached context reserves the next slot
 * of one budget clock over `trace` (t = 0 at creation / reset). No reference
 * counterpart: the reference serves one request per process. */
typedef struct cake_link cake_link;
CAKE_API int cake_link_create(cake_trace trace, cake_link** out);
CAKE_API int cake_link_destroy(cake_link* l);
CAKE_API int cake_link_reset(cake_link* l);  /* only while no attached run is in flight */
CAKE_API int cake_link_reserved_bits(const cake_link* l, uint64_t* bits, int64_t* now_us);
/* Attach (l != NULL) or detach: later runs of g pace through l instead of their own trace. */
CAKE_API int cake_gpu_set_link(cake_gpu* g, cake_link* l);
CAKE_API int cake_gpu_destroy(cake_gpu* g);
CAKE_API int cake_gpu_kv_bytes_per_token(const cake_gpu* g, uint64_t* out);
/* Fill `store` (create it memory-resident+pinned) from a compute-only GPU pass. */
CAKE_API int cake_gpu_build_tier(cake_gpu* g, cake_store* store, uint64_t total_tokens, uint32_t chunk_size,
                                 uint64_t prompt_seed);
/* Cache-tier codec for build_tier and run: "identity" (default) or "quant8"
 * (reference codec.cpp:114-162; decode fused into the GPU scatter). */
CAKE_API int cake_gpu_set_codec(cake_gpu* g, const char* codec_id);
CAKE_API int cake_gpu_calibrate(cake_gpu* g, uint64_t total_tokens, uint32_t chunk_size, uint64_t prompt_seed,
                                double* alpha_ms, double* beta_ms_per_token);
CAKE_API int cake_gpu_run(cake_gpu* g, cake_store* store, uint64_t total_tokens, uint32_t chunk_size,
                          uint64_t prompt_seed, cake_trace trace, int mode, const cake_run_opts* opts,
                          cake_gpu_result* result, cake_record* records);
CAKE_API int cake_gpu_logits(const cake_gpu* g, float* out, int n);
CAKE_API int cake_gpu_read_chunk(const cake_gpu* g, uint64_t token_start, uint32_t token_count, uint8_t* out,
                                 uint64_t cap);
CAKE_API int cake_gpu_kernel_stats(cake_gpu* g, cake_kernel_stat* out, int reset);
/* Event-bracket kernel classes (bit CAKE_K_*; -1 all, 0 none) from now on. */
CAKE_API int cake_gpu_set_profiling(cake_gpu* g, int mask);
/* Bracket only every n-th launch of a profiled class (n >= 1). */
CAKE_API int cake_gpu_set_profiling_stride(cake_gpu* g, int stride);
/* 0 = tcgen05 attention (default), 1 = mma.sync attention (validation cross-check). */
CAKE_API int cake_gpu_set_attention_impl(cake_gpu* g, int impl);
/* Test instrumentation: fill the whole paged KV pool (spare page set
 * included) and the device staging buffers with `byte` (0xFF = bf16 NaN), so
 * a later run must write every page it references. */
CAKE_API int cake_gpu_poison(cake_gpu* g, int byte);
/* Slice log of the last run (record_slices): release time on the run clock
 * and cumulative released bits (reference transfer.hpp SliceEvent). n_out = total. */
CAKE_API int cake_gpu_slices(const cake_gpu* g, int64_t* at_us, uint64_t* cumulative_bits, uint64_t cap,
                             uint64_t* n_out);
CAKE_API void* cake_gpu_model(cake_gpu* g); /* cake_model* for direct C-ABI CUDA calls */
CAKE_API void* cake_gpu_compute_stream(cake_gpu* g);

/* ---- TP group coordination (cake/tp.hpp): leader publishes, followers mirror.
 * Exposed so the host protocol can be tested (and driven) without a GPU.
 * next_*: *has = 0 once the sequence ended. */
typedef struct cake_tp cake_tp;
CAKE_API int cake_tp_create(const char* shm_name, int rank, int size, cake_tp** out);
CAKE_API int cake_tp_destroy(cake_tp* t);
CAKE_API int cake_tp_begin_run(cake_tp* t, uint64_t run_id, uint32_t n_chunks);
CAKE_API int cake_tp_end_run(cake_tp* t);
CAKE_API int cake_tp_publish_compute(cake_tp* t, uint32_t chunk);
CAKE_API int cake_tp_end_compute(cake_tp* t);
CAKE_API int cake_tp_next_compute(cake_tp* t, uint32_t k, uint32_t* chunk, int* has);
CAKE_API int cake_tp_publish_io(cake_tp* t, uint32_t chunk);
CAKE_API int cake_tp_end_io(cake_tp* t);
CAKE_API int cake_tp_next_io(cake_tp* t, uint32_t k, uint32_t* chunk, int* has);
CAKE_API int cake_tp_shard_landed(cake_tp* t, uint32_t chunk);
CAKE_API int cake_tp_wait_all_landed(cake_tp* t, uint32_t chunk);
/* Entries of the compute / io sequences are chunk indices; the racer's entry of
 * the contested chunk carries CAKE_TP_RACE_BIT (race-to-finish mirrored). */
#define CAKE_TP_RACE_BIT (1u << 30)
/* Commit decisions: side 1 = compute, 2 = io (0 = undecided). */
CAKE_API int cake_tp_publish_decided(cake_tp* t, uint32_t chunk, int side);
CAKE_API int cake_tp_decided(cake_tp* t, uint32_t chunk, int* side);
/* race_pages: the contested chunk whose winner wrote the spare page set, or -1. */
CAKE_API int cake_tp_publish_final(cake_tp* t, int recompute, int last_row, int race_pages);
CAKE_API int cake_tp_wait_final(cake_tp* t, int* recompute, int* last_row, int* race_pages);

#ifdef __cplusplus
}
#endif
#endif /* CAKE_C_H_ */
