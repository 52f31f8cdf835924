// B200 runtime behind the cake:: API: one GPU (or one tensor-parallel rank)
// holding the model, the paged KV cache and the streams the bidirectional
// run uses. Pass a GpuContext through RunOptions::gpu and
// run(..., ClockMode::live, ...) becomes the real thing:
//
//   compute side   ComputeEngine::run_forward + GpuPrefillBackend: claimed
//                  chunks are enqueued on the compute stream (cake_cuda.h
//                  cake_prefill_layers), claims paced by a CUDA event a few
//                  layers before the running chunk ends.
//   io side        TransferEngine + GpuLoaderSink: every released slice is
//                  cudaMemcpyAsync'd from the pinned cache tier into a device
//                  staging buffer on the copy stream, then one scatter kernel
//                  permutes the chunk into its KV pages; residency = the
//                  scatter's event completed.
//   boundary       race-to-finish with a second page set for the contested
//                  chunk; first completion commits, the loser is aborted.
//   first token    q-only pass of the last prompt token over the assembled
//                  cache (or the computed tail's hidden state) -> logits.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "cake/codec.hpp"
#include "cake/compute.hpp"
#include "cake/model.hpp"
#include "cake/scheduler.hpp"
#include "cake/store.hpp"
#include "cake/tp.hpp"
#include "cake/transfer.hpp"

struct cake_model;

namespace cake {

struct GpuModelConfig {
  std::string name;
  int n_layers = 0;
  int hidden = 0;
  int n_heads = 0;
  int n_kv_heads = 0;
  int head_dim = 0;
  int ffn = 0;
  int vocab = 0;
  float rope_theta = 500000.0f;
  float rms_eps = 1e-5f;
  int page_tokens = 64;

  static GpuModelConfig llama3_8b();
  static GpuModelConfig llama3_70b();
  static GpuModelConfig tiny();  // BASELINE config 1: 2 layers, d 256, 4 heads (hd 64), FFN 1024

  // KV bytes law of one TP shard, as the reference's ModelProfile.
  ModelProfile profile(int tp_size = 1) const;
};

struct GpuOptions {
  int device = 0;
  int max_chunk = 512;
  long long max_tokens = 32768;
  std::uint64_t weight_seed = 1234;
  int tp_rank = 0;
  int tp_size = 1;
  void* nccl_comm = nullptr;  // ncclComm_t when tp_size > 1
  std::string tp_shm;         // POSIX shm name of the TP group's coordinator (cake/tp.hpp)
  int lookahead_layers = 3;   // claim the next chunk when this many layers of the current remain
  CostModel prior{5.0, 0.0002, 512};  // per-chunk duration prior (refine with calibrate())
  Micros race_margin_us = 200;        // race only when predicted to win by at least this
  bool profile_kernels = false;       // bracket tracked kernels with events (bench roofline)
  // GPU share of the compute side: > 0 confines the
  // compute stream to this many SMs (green context); 0 = the whole GPU.
  int compute_sms = 0;
  // Share this context's weights (same dimensions, seed and TP shard; it must
  // outlive the new context): one context per concurrent request on a device.
  const GpuContext* weights_from = nullptr;
};

struct GpuRunInfo {
  Micros first_token_us = 0;    // logits in host memory (run clock): the north-star TTFT
  Micros kv_resident_us = 0;    // last chunk resident (reference TTFT, report.hpp)
  Micros final_step_us = 0;     // first-token step duration (device)
  double device_ttft_ms = 0.0;  // run anchor event -> logits event
  std::uint32_t merge_point = 0;
  int raced_chunk = -1;         // contested chunk, -1 if none
  int race_winner = -1;         // 0 compute, 1 io
  bool recomputed_last = false;
  long long kernel_launches = 0;
  std::uint64_t h2d_bytes = 0;
  std::uint64_t d2h_bytes = 0;
  std::vector<float> logits;
  std::vector<SliceEvent> slices;  // RunOptions::record_slices
};

class GpuContext {
 public:
  GpuContext(const GpuModelConfig& cfg, const GpuOptions& opt);
  ~GpuContext();
  GpuContext(const GpuContext&) = delete;
  GpuContext& operator=(const GpuContext&) = delete;

  cake_model* model() const;
  void* compute_stream() const;
  void* copy_stream() const;
  void* control_stream() const;
  HostAllocator pinned_allocator() const;
  const GpuModelConfig& config() const;
  const GpuOptions& options() const;
  std::uint64_t kv_bytes_per_token() const;  // this rank's shard
  int page_tokens() const;

  // Cache tier: compute-only pass over the seeded prompt, every chunk's KV
  // gathered to the tier format and put under its chain key.
  // quant8: the chunk is encoded on the GPU (cake_kv_encode_q8), format of
  // the reference's Codec::quant8 (codec.cpp:114-162) over the bf16 KV.
  PopulateResult build_cache_tier(ChunkStore& store, const RequestSpec& request, std::uint64_t prompt_seed,
                                  const Codec& codec = Codec::identity());
  // Compute-only pass timed per chunk with events; least-squares alpha/beta.
  CostModel calibrate(const RequestSpec& request, std::uint64_t prompt_seed);
  // Assembled cache of the last run (committed pages), tier format.
  std::vector<std::byte> read_chunk_kv(const ChunkSpec& chunk) const;

  const GpuRunInfo& last_run() const;
  // Test instrumentation: fill the paged KV pool (both page sets) and the
  // device staging buffers with `byte`, so stale bytes cannot pass a check.
  void poison(int byte);
  TpCoordinator* tp() const;  // non-null for tp_size > 1 with a coordinator

  struct Impl;
  Impl* impl() const { return impl_.get(); }

 private:
  std::unique_ptr<Impl> impl_;
};

}  // namespace cake
