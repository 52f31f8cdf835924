#include <cstdio>
#include <cstdlib>
// GPU runtime: GpuContext, the compute-side PrefillBackend, the loader-side
// ChunkSink, the race-to-finish commit protocol and the live bidirectional
// run that replaces reference run_live (proj/src/scheduler.cpp:229-278).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <stdexcept>
#include <thread>

#include <nvtx3/nvToolsExt.h>

#include "cake/gpu.hpp"
#include "cake_cuda.h"
#include "internal.hpp"

namespace cake {

namespace {

void check(int st, const char* what);

// The CUDA current device is per host thread: the loader's reader / pacer threads and the TP
// follower's io thread make CUDA calls too, so each binds the context's device before its first
// call (a rank on device r > 0 would otherwise launch from device 0's context).
void bind_device(int device) {
  thread_local int bound = -1;
  if (bound == device) return;
  // through the CUDA layer (its runtime is the one whose current device matters; calling this
  // library's own cudart would initialise a second runtime inside the run), and without
  // cake_cuda_set_device's reset of the layer's cached SM count
  check(cake_cuda_bind_thread(device), "bind device");
  bound = device;
}

// NVTX annotations (header-only nvtx3: free unless a tool such as nsys is
// attached): the per-chunk, per-side timeline the reference keeps as its event
// CSV (proj/src/report.cpp:31-37), on the host threads that drive the GPU.
struct NvtxScope {
  explicit NvtxScope(const std::string& name) { nvtxRangePushA(name.c_str()); }
  ~NvtxScope() { nvtxRangePop(); }
};
void nvtx_mark(const std::string& name) { nvtxMarkA(name.c_str()); }

void check(int st, const char* what) {
  if (st == CAKE_OK) return;
  char buf[768];
  cake_cuda_last_error(buf, sizeof buf);
  throw std::runtime_error(std::string(what) + ": " + buf + " (status " + std::to_string(st) + ")");
}

void* pinned_alloc(std::size_t n, void*) {
  void* p = nullptr;
  return cake_host_alloc(&p, n) == CAKE_OK ? p : nullptr;
}
void pinned_release(void* p, void*) { cake_host_free(p); }

// Landing buffers of file-backed tiers: pinned memory kept across chunks and
// runs (a cudaHostAlloc of a 64-MiB chunk costs milliseconds; a run holds
// only the chunk the reader fills and the ones the pacer is still copying).
struct PinnedPool {
  int device = -1;  // the context's device, bound by the (reader) thread that allocates
  std::mutex mu;
  std::multimap<std::size_t, void*> free_;  // size -> buffer
  std::unordered_map<void*, std::size_t> size_of;
  ~PinnedPool() {
    for (auto& kv : free_) cake_host_free(kv.second);
  }
  static void* alloc(std::size_t n, void* ctx) {
    auto* pool = static_cast<PinnedPool*>(ctx);
    {
      std::lock_guard g(pool->mu);
      auto it = pool->free_.lower_bound(n);
      if (it != pool->free_.end() && it->first <= 2 * n) {
        void* p = it->second;
        pool->free_.erase(it);
        return p;
      }
    }
    if (pool->device >= 0) bind_device(pool->device);
    void* p = pinned_alloc(n, nullptr);
    if (p) {
      std::lock_guard g(pool->mu);
      pool->size_of[p] = n;
    }
    return p;
  }
  static void release(void* p, void* ctx) {
    auto* pool = static_cast<PinnedPool*>(ctx);
    std::lock_guard g(pool->mu);
    pool->free_.emplace(pool->size_of.at(p), p);
  }
};

struct Event {
  void* h = nullptr;
  Event() { check(cake_event_create(&h, 1), "cudaEventCreate"); }
  ~Event() {
    if (h) cake_event_destroy(h);
  }
  Event(const Event&) = delete;
  Event& operator=(const Event&) = delete;
};

template <typename T>
struct Pinned {
  T* p = nullptr;
  std::size_t n = 0;
  void reset(std::size_t count) {
    release();
    n = count;
    void* v = nullptr;
    check(cake_host_alloc(&v, std::max<std::size_t>(1, count) * sizeof(T)), "pinned alloc");
    p = static_cast<T*>(v);
  }
  void release() {
    if (p) cake_host_free(p);
    p = nullptr;
  }
  ~Pinned() { release(); }
};

template <typename T>
struct Device {
  T* p = nullptr;
  void reset(std::size_t count) {
    release();
    void* v = nullptr;
    check(cake_dev_alloc(&v, std::max<std::size_t>(1, count) * sizeof(T)), "device alloc");
    p = static_cast<T*>(v);
  }
  void release() {
    if (p) cake_dev_free(p);
    p = nullptr;
  }
  ~Device() { release(); }
};

}  // namespace

// ------------------------------------------------------------------ presets
GpuModelConfig GpuModelConfig::llama3_8b() {
  return {"llama-3-8b", 32, 4096, 32, 8, 128, 14336, 128256, 500000.0f, 1e-5f, 64};
}
GpuModelConfig GpuModelConfig::llama3_70b() {
  return {"llama-3-70b", 80, 8192, 64, 8, 128, 28672, 128256, 500000.0f, 1e-5f, 64};
}
GpuModelConfig GpuModelConfig::tiny() { return {"tiny", 2, 256, 4, 4, 64, 1024, 32000, 500000.0f, 1e-5f, 64}; }

ModelProfile GpuModelConfig::profile(int tp_size) const {
  ModelProfile p;
  p.name = name;
  p.n_layers = static_cast<std::uint32_t>(n_layers);
  p.hidden_size = static_cast<std::uint32_t>(n_kv_heads / tp_size * head_dim);  // KV width (GQA)
  p.precision_bytes = 2;
  p.kv_multiplier = 2;
  return p;
}

// ------------------------------------------------------------------ context
struct GpuContext::Impl {
  GpuModelConfig cfg;
  GpuOptions opt;
  cake_model* model = nullptr;
  cake_model_info info{};
  void* s_compute = nullptr;
  void* s_copy = nullptr;
  void* s_control = nullptr;
  int n_pages = 0;        // logical pages
  int spare_pages = 0;    // second page set for one contested chunk
  Device<std::int32_t> bt_primary, bt_race, tokens, abort_flags;
  Pinned<std::int32_t> h_bt_race, h_tokens, h_abort_one;
  Device<std::byte> staging[2];
  Pinned<std::byte> follower_landing;  // TP follower, file tier: one chunk (reused; each chunk's copies are synced)
  std::size_t staging_bytes = 0;
  Device<float> logits;
  Pinned<float> h_logits;
  const std::int32_t* final_bt = nullptr;
  std::vector<std::unique_ptr<Event>> ev_start, ev_near, ev_end, ev_io;
  std::unique_ptr<Event> ev_anchor, ev_copy_done, ev_final_start, ev_logits, ev_reset;  // created after set_device
  std::unique_ptr<Event> ev_slice[2];  // the compute racer's layer slices (GpuPrefillBackend::launch)
  GpuRunInfo last;
  std::unique_ptr<TpCoordinator> tp;
  std::uint64_t run_counter = 0;
  PinnedPool landing;  // file-tier landing buffers, reused across runs
  int compute_sms = 0;  // > 0: the compute stream's SM partition

  void ensure_events(std::size_t n) {
    for (auto* v : {&ev_start, &ev_near, &ev_end, &ev_io})
      while (v->size() < n) v->push_back(std::make_unique<Event>());
  }
  int pages_of(const ChunkSpec& c) const {
    return static_cast<int>((c.token_count + cfg.page_tokens - 1) / cfg.page_tokens);
  }
};

GpuContext::GpuContext(const GpuModelConfig& cfg, const GpuOptions& opt) : impl_(std::make_unique<Impl>()) {
  Impl& g = *impl_;
  g.cfg = cfg;
  g.opt = opt;
  check(cake_cuda_set_device(opt.device), "set device");
  g.landing.device = opt.device;
  if (opt.max_chunk % cfg.page_tokens) throw std::invalid_argument("gpu: max_chunk must be a multiple of page_tokens");
  cake_model_config mc{};
  mc.n_layers = cfg.n_layers;
  mc.hidden = cfg.hidden;
  mc.n_heads = cfg.n_heads;
  mc.n_kv_heads = cfg.n_kv_heads;
  mc.head_dim = cfg.head_dim;
  mc.ffn = cfg.ffn;
  mc.vocab = cfg.vocab;
  mc.rope_theta = cfg.rope_theta;
  mc.rms_eps = cfg.rms_eps;
  mc.page_tokens = cfg.page_tokens;
  mc.max_chunk = opt.max_chunk;
  mc.max_tokens = opt.max_tokens;
  g.spare_pages = opt.max_chunk / cfg.page_tokens;
  mc.spare_pages = g.spare_pages;
  mc.tp_rank = opt.tp_rank;
  mc.tp_size = opt.tp_size;
  mc.seed = opt.weight_seed;
  g.ev_anchor = std::make_unique<Event>();
  g.ev_copy_done = std::make_unique<Event>();
  g.ev_final_start = std::make_unique<Event>();
  g.ev_logits = std::make_unique<Event>();
  g.ev_reset = std::make_unique<Event>();
  g.ev_slice[0] = std::make_unique<Event>();
  g.ev_slice[1] = std::make_unique<Event>();
  check(opt.weights_from ? cake_model_create_shared(&mc, opt.weights_from->model(), &g.model)
                         : cake_model_create(&mc, &g.model),
        "model create");
  check(cake_model_get_info(g.model, &g.info), "model info");
  // tp_size > 1 without a communicator is allowed for the single-device
  // group driver (cake_prefill_group); a live run then fails loudly in the
  // first row-parallel projection.
  if (opt.tp_size > 1 && opt.nccl_comm) check(cake_model_set_comm(g.model, opt.nccl_comm), "set comm");
  if (opt.tp_size > 1 && !opt.tp_shm.empty())
    g.tp = std::make_unique<TpCoordinator>(opt.tp_shm, opt.tp_rank, opt.tp_size);
  check(cake_model_set_profiling(g.model, opt.profile_kernels ? -1 : 0), "profiling");
  if (opt.compute_sms > 0) {
    int got = 0;
    check(cake_stream_create_sm_share(&g.s_compute, opt.compute_sms, &got), "compute stream (SM share)");
    check(cake_set_sm_budget(got), "sm budget");
    g.compute_sms = got;
  } else {
    check(cake_set_sm_budget(0), "sm budget");
    check(cake_stream_create(&g.s_compute, 0), "stream");
  }
  check(cake_stream_create(&g.s_copy, 1), "stream");     // loader work jumps the queue for free SMs
  check(cake_stream_create(&g.s_control, 1), "stream");
  g.n_pages = g.info.n_logical_pages;
  g.bt_primary.reset(g.n_pages);
  g.bt_race.reset(g.n_pages);
  g.h_bt_race.reset(g.n_pages);
  for (int i = 0; i < g.n_pages; ++i) g.h_bt_race.p[i] = i;  // identity: logical page i -> physical i
  check(cake_h2d_async(g.bt_primary.p, g.h_bt_race.p, g.n_pages * sizeof(std::int32_t), g.s_compute), "bt upload");
  check(cake_h2d_async(g.bt_race.p, g.h_bt_race.p, g.n_pages * sizeof(std::int32_t), g.s_compute), "bt upload");
  g.tokens.reset(static_cast<std::size_t>(opt.max_tokens));
  g.h_tokens.reset(static_cast<std::size_t>(opt.max_tokens));
  g.abort_flags.reset(g.n_pages);
  g.h_abort_one.reset(1);
  g.h_abort_one.p[0] = 1;
  g.staging_bytes = static_cast<std::size_t>(cake_kv_chunk_bytes(g.model, opt.max_chunk));
  g.staging[0].reset(g.staging_bytes);
  g.staging[1].reset(g.staging_bytes);
  g.logits.reset(cfg.vocab);
  g.h_logits.reset(cfg.vocab);
  g.final_bt = g.bt_primary.p;
  check(cake_stream_sync(g.s_compute), "init sync");
}

GpuContext::~GpuContext() {
  Impl& g = *impl_;
  cake_cuda_device_sync();
  for (void* s : {g.s_compute, g.s_copy, g.s_control})
    if (s) cake_stream_destroy(s);
  if (g.model) cake_model_destroy(g.model);
  if (g.compute_sms > 0) cake_set_sm_budget(0);  // later contexts size launches for the whole device
}

cake_model* GpuContext::model() const { return impl_->model; }
void* GpuContext::compute_stream() const { return impl_->s_compute; }
void* GpuContext::copy_stream() const { return impl_->s_copy; }
void* GpuContext::control_stream() const { return impl_->s_control; }
HostAllocator GpuContext::pinned_allocator() const { return {pinned_alloc, pinned_release, nullptr}; }
const GpuModelConfig& GpuContext::config() const { return impl_->cfg; }
const GpuOptions& GpuContext::options() const { return impl_->opt; }
std::uint64_t GpuContext::kv_bytes_per_token() const {
  return static_cast<std::uint64_t>(impl_->info.kv_bytes_per_token);
}
int GpuContext::page_tokens() const { return impl_->cfg.page_tokens; }
const GpuRunInfo& GpuContext::last_run() const { return impl_->last; }
TpCoordinator* GpuContext::tp() const { return impl_->tp.get(); }

namespace {

void check_chunking(const GpuContext::Impl& g, std::span<const ChunkSpec> chunks, std::uint64_t total) {
  if (total > static_cast<std::uint64_t>(g.opt.max_tokens)) throw std::invalid_argument("gpu: prompt exceeds max_tokens");
  for (const ChunkSpec& c : chunks) {
    if (c.token_count > static_cast<std::uint32_t>(g.opt.max_chunk))
      throw std::invalid_argument("gpu: chunk exceeds max_chunk");
    if (c.token_start % g.cfg.page_tokens)
      throw std::invalid_argument("gpu: chunk_size must be a multiple of page_tokens (" +
                                  std::to_string(g.cfg.page_tokens) + ")");
  }
}

// Drain this context's streams only: another context on the same device
// (a concurrent request) keeps running.
void sync_own_streams(GpuContext::Impl& g) {
  for (void* s : {g.s_compute, g.s_copy, g.s_control}) check(cake_stream_sync(s), "pre-run sync");
}

void upload_tokens(GpuContext::Impl& g, const std::vector<std::uint32_t>& ids, void* stream) {
  for (std::size_t i = 0; i < ids.size(); ++i) {
    if (ids[i] >= static_cast<std::uint32_t>(g.cfg.vocab))
      throw std::invalid_argument("gpu: token id " + std::to_string(ids[i]) + " outside the vocabulary");
    g.h_tokens.p[i] = static_cast<std::int32_t>(ids[i]);
  }
  check(cake_h2d_async(g.tokens.p, g.h_tokens.p, ids.size() * sizeof(std::int32_t), stream), "tokens H2D");
}

// Second page set for a contested chunk: the chunk's logical pages map to
// the spare physical pages, every other page to itself. Uploaded on the
// racer's stream ahead of the racer's writes.
void upload_race_table(GpuContext::Impl& g, const ChunkSpec& c, void* stream) {
  const int first = static_cast<int>(c.token_start / g.cfg.page_tokens);
  for (int p = 0; p < g.n_pages; ++p) g.h_bt_race.p[p] = p;
  for (int p = 0; p < g.pages_of(c); ++p) g.h_bt_race.p[first + p] = g.n_pages + p;
  check(cake_h2d_async(g.bt_race.p, g.h_bt_race.p, g.n_pages * sizeof(std::int32_t), stream), "race bt");
}

}  // namespace

PopulateResult GpuContext::build_cache_tier(ChunkStore& store, const RequestSpec& request, std::uint64_t prompt_seed,
                                            const Codec& codec) {
  Impl& g = *impl_;
  request.validate();
  const auto chunks = split_into_chunks(request.total_tokens, request.chunk_size);
  check_chunking(g, chunks, request.total_tokens);
  const auto ids = token_stream(prompt_seed, request.total_tokens);
  upload_tokens(g, ids, g.s_compute);
  check(cake_memset_async(g.abort_flags.p, 0, g.n_pages * sizeof(std::int32_t), g.s_compute), "memset");
  if (codec.kind == Codec::Kind::factor) throw std::invalid_argument("gpu tier: the factor codec models bytes only");
  const bool q8 = codec.kind == Codec::Kind::quant8;
  const ModelProfile prof = g.cfg.profile(g.opt.tp_size);
  Pinned<std::byte> host;
  host.reset(g.staging_bytes);
  PopulateResult res;
  std::optional<ChunkKey> prev;
  for (const ChunkSpec& c : chunks) {
    check(cake_prefill_chunk(g.model, g.tokens.p + c.token_start, static_cast<long long>(c.token_start),
                             static_cast<int>(c.token_count), g.bt_primary.p, nullptr, 0, g.s_compute),
          "prefill");
    const auto bytes = static_cast<std::size_t>(cake_kv_chunk_bytes(g.model, static_cast<int>(c.token_count)));
    check(cake_kv_gather(g.model, g.staging[0].p, static_cast<long long>(c.token_start), static_cast<int>(c.token_count),
                         g.bt_primary.p, g.s_compute),
          "gather");
    std::size_t enc = bytes;
    if (q8) {
      enc = static_cast<std::size_t>(cake_kv_q8_bytes(g.model, static_cast<int>(c.token_count)));
      check(cake_kv_encode_q8(g.model, g.staging[0].p, static_cast<int>(c.token_count), g.staging[1].p, g.s_compute),
            "q8 encode");
      check(cake_d2h_async(host.p, g.staging[1].p, enc, g.s_compute), "D2H");
    } else {
      check(cake_d2h_async(host.p, g.staging[0].p, bytes, g.s_compute), "D2H");
    }
    check(cake_stream_sync(g.s_compute), "sync");
    const ChunkKey key =
        chain_hash(prev, std::span<const std::uint32_t>(ids.data() + c.token_start, c.token_count));
    prev = key;
    res.keys.push_back(key);
    if (bytes != chunk_bytes(prof, c)) throw std::logic_error("gpu: chunk bytes disagree with the KV profile");
    if (enc != codec.encoded_size(bytes)) throw std::logic_error("gpu: encoded size disagrees with the codec law");
    const ChunkMeta meta{c.token_count, codec.id(), enc, bytes};
    if (store.contains(key)) {
      ++res.chunks_existing;
      continue;
    }
    store.put(key, std::span<const std::byte>(host.p, enc), meta);
    res.bytes_written += enc;
    ++res.chunks_written;
  }
  return res;
}

CostModel GpuContext::calibrate(const RequestSpec& request, std::uint64_t prompt_seed) {
  Impl& g = *impl_;
  request.validate();
  const auto chunks = split_into_chunks(request.total_tokens, request.chunk_size);
  check_chunking(g, chunks, request.total_tokens);
  upload_tokens(g, token_stream(prompt_seed, request.total_tokens), g.s_compute);
  check(cake_memset_async(g.abort_flags.p, 0, g.n_pages * sizeof(std::int32_t), g.s_compute), "memset");
  g.ensure_events(chunks.size());
  for (const ChunkSpec& c : chunks) {
    check(cake_event_record(g.ev_start[c.index]->h, g.s_compute), "record");
    check(cake_prefill_chunk(g.model, g.tokens.p + c.token_start, static_cast<long long>(c.token_start),
                             static_cast<int>(c.token_count), g.bt_primary.p, nullptr, 0, g.s_compute),
          "prefill");
    check(cake_event_record(g.ev_end[c.index]->h, g.s_compute), "record");
  }
  check(cake_stream_sync(g.s_compute), "sync");
  // least squares  d_i = a + b * start_i  over full-size chunks (scaled by size otherwise)
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  int n = 0;
  for (const ChunkSpec& c : chunks) {
    float ms = 0.f;
    check(cake_event_elapsed_ms(g.ev_start[c.index]->h, g.ev_end[c.index]->h, &ms), "elapsed");
    const double y = static_cast<double>(ms) * request.chunk_size / c.token_count;
    const double x = static_cast<double>(c.token_start);
    sx += x;
    sy += y;
    sxx += x * x;
    sxy += x * y;
    ++n;
  }
  double b = 0.0, a = sy / n;
  const double den = n * sxx - sx * sx;
  if (n > 1 && den > 0) {
    b = (n * sxy - sx * sy) / den;
    a = (sy - b * sx) / n;
  }
  CostModel cm{std::max(0.0, a), std::max(0.0, b), request.chunk_size};
  g.opt.prior = cm;
  return cm;
}

void GpuContext::poison(int byte) {
  Impl& g = *impl_;
  sync_own_streams(g);  // (not the device: another context may be running)
  check(cake_kv_poison(g.model, byte, g.s_compute), "poison pool");
  for (auto& s : g.staging) check(cake_memset_async(s.p, byte & 0xFF, g.staging_bytes, g.s_compute), "poison staging");
  check(cake_stream_sync(g.s_compute), "poison: sync");
}

std::vector<std::byte> GpuContext::read_chunk_kv(const ChunkSpec& chunk) const {
  Impl& g = *impl_;
  const auto bytes = static_cast<std::size_t>(cake_kv_chunk_bytes(g.model, static_cast<int>(chunk.token_count)));
  check(cake_kv_gather(g.model, g.staging[0].p, static_cast<long long>(chunk.token_start),
                       static_cast<int>(chunk.token_count), g.final_bt, g.s_compute),
        "gather");
  std::vector<std::byte> out(bytes);
  Pinned<std::byte> host;
  host.reset(bytes);
  check(cake_d2h_async(host.p, g.staging[0].p, bytes, g.s_compute), "D2H");
  check(cake_stream_sync(g.s_compute), "sync");
  std::memcpy(out.data(), host.p, bytes);
  return out;
}

// ================================================================== live run
namespace {

constexpr int kNone = 0, kByCompute = 1, kByIo = 2;

// State one bidirectional run shares between the compute thread, the
// loader's pacer/completion threads and the final step.
struct LiveRun {
  GpuContext::Impl& g;
  const RunPlan& plan;
  const RunTimer& timer;
  Micros t0 = 0;  // run clock at the anchor event
  std::unique_ptr<std::atomic<int>[]> commit;
  std::atomic<int> race_chunk{-1};
  std::atomic<int> racer{-1};  // kByCompute / kByIo
  int hold = kNone;            // RunOptions::race_hold: this side's commit of the contested chunk waits
  std::atomic<bool> compute_done{false};  // the compute side claims nothing more
  TransferEngine* loader = nullptr;
  TpCoordinator* tp = nullptr;  // leader side of a TP group (followers run run_follower)
  std::mutex commit_mu;
  std::condition_variable commit_cv;
  std::uint32_t n_committed = 0;

  LiveRun(GpuContext::Impl& g_, const RunPlan& p, const RunTimer& t) : g(g_), plan(p), timer(t) {
    commit = std::make_unique<std::atomic<int>[]>(p.chunks.size());
    for (std::size_t i = 0; i < p.chunks.size(); ++i) commit[i].store(kNone);
  }

  Micros device_time(void* ev) const {
    float ms = 0.f;
    check(cake_event_elapsed_ms(g.ev_anchor->h, ev, &ms), "elapsed");
    return t0 + static_cast<Micros>(std::llround(static_cast<double>(ms) * 1000.0));
  }

  bool try_commit(std::uint32_t i, int who) {
    if (who == hold) {
      // test instrumentation: the held side commits nothing until the other
      // side has decided whether to contest, and lets it win a contested chunk
      const Micros deadline = timer.now_us() + 60'000'000;
      auto wait_for = [&](auto&& done) {
        while (!done()) {
          if (timer.now_us() > deadline) throw std::runtime_error("race_hold: the other side never decided");
          std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
      };
      wait_for([&] {
        if (race_chunk.load() >= 0) return true;
        return who == kByCompute ? (loader == nullptr || loader->reader_finished()) : compute_done.load();
      });
      if (race_chunk.load() == static_cast<int>(i)) wait_for([&] { return commit[i].load() != kNone; });
    }
    int expected = kNone;
    if (!commit[i].compare_exchange_strong(expected, who)) return false;
    if (tp) tp->publish_decided(i, who == kByCompute ? 1 : 2);  // followers drop the loser's work too
    nvtx_mark("commit chunk " + std::to_string(i) + (who == kByCompute ? " by compute" : " by io"));
    {
      std::lock_guard lk(commit_mu);
      ++n_committed;
    }
    commit_cv.notify_all();
    return true;
  }

  // Block until every chunk has a committed source (the first token only
  // needs that), or the loader stopped without delivering (error path).
  void wait_all_committed() {
    const auto n = static_cast<std::uint32_t>(plan.chunks.size());
    std::unique_lock lk(commit_mu);
    while (n_committed < n) {
      if (commit_cv.wait_for(lk, std::chrono::milliseconds(1), [&] { return n_committed >= n; })) break;
      if (loader == nullptr || loader->idle()) break;
    }
  }

  // One contested chunk per run: the side whose contest predicate fires
  // first takes the race slot (the spare page set and h_bt_race are single).
  bool reserve_race(std::uint32_t i, int who) {
    int expected = -1;
    if (!race_chunk.compare_exchange_strong(expected, -2)) return false;  // -2: being set up
    racer.store(who);
    race_chunk.store(static_cast<int>(i));
    return true;
  }

  // Second page set for the reserved contested chunk, uploaded on the
  // racer's stream ahead of the racer's writes.
  void start_race(const ChunkSpec& c, int who, void* stream) {
    if (race_chunk.load() != static_cast<int>(c.index) || racer.load() != who)
      throw std::logic_error("race: chunk contested without the race slot");
    upload_race_table(g, c, stream);
  }

  // Which page table each side writes a chunk through.
  const std::int32_t* table_for(std::uint32_t i, int who) const {
    return (race_chunk.load() == static_cast<int>(i) && racer.load() == who) ? g.bt_race.p : g.bt_primary.p;
  }

  void abort_compute(std::uint32_t i) {
    check(cake_h2d_async(g.abort_flags.p + i, g.h_abort_one.p, sizeof(std::int32_t), g.s_control), "abort");
  }
};

class GpuPrefillBackend final : public PrefillBackend {
 public:
  GpuPrefillBackend(LiveRun& run, const CostModel& prior) : r_(run), prior_(prior) {}

  void pace() override {
    bind_device(r_.g.opt.device);
    if (launched_.empty()) return;
    check(cake_event_sync(r_.g.ev_near[launched_.back()]->h), "pace");
    observe();
  }

  void launch(const ChunkSpec& c, bool contested) override {
    GpuContext::Impl& g = r_.g;
    bind_device(g.opt.device);
    NvtxScope nv("compute chunk " + std::to_string(c.index) + (contested ? " (contested)" : ""));
    // followers enqueue the same chunk (reduction lockstep), the racer's entry through their spare pages
    if (r_.tp) r_.tp->publish_compute(c.index | (contested ? TpCoordinator::kRaceBit : 0u));
    const Micros predicted = predict_finish(c);
    if (contested) r_.start_race(c, kByCompute, g.s_compute);
    const std::int32_t* bt = r_.table_for(c.index, kByCompute);
    const int L = g.cfg.n_layers;
    const int split = std::clamp(L - g.opt.lookahead_layers, 1, L);
    const auto start = static_cast<long long>(c.token_start);
    const auto len = static_cast<int>(c.token_count);
    const std::int32_t* tok = g.tokens.p + c.token_start;
    const std::int32_t* abort = g.abort_flags.p + c.index;
    check(cake_event_record(g.ev_start[c.index]->h, g.s_compute), "record");
    if (contested && r_.tp == nullptr) {
      // The racer is fed a few layers at a time, at most two slices ahead of the device: if the
      // loader commits the chunk first, feeding stops and the little that is queued exits on the
      // abort flag, so the first-token step is not stuck behind a whole lost chunk (a lost race
      // used to cost ~1.8 ms of TTFT that way, tools/run_timeline.py). (TP: every rank must issue
      // the same reductions, so a TP group enqueues the whole chunk.)
      constexpr int kSlice = 4;
      int k = 0;
      for (int l0 = 0; l0 < L; l0 += kSlice, ++k) {
        if (r_.commit[c.index].load() == kByIo) break;  // the loader landed it: stop feeding the device
        const int l1 = std::min(L, l0 + kSlice);
        check(cake_prefill_layers(g.model, tok, start, len, l0, l1, bt, abort, 0, g.s_compute), "prefill");
        check(cake_event_record(g.ev_slice[k & 1]->h, g.s_compute), "record");
        if (k > 0)  // keep at most two slices queued: wait for the previous one
          while (cake_event_query(g.ev_slice[(k - 1) & 1]->h) != CAKE_OK) {
            if (r_.commit[c.index].load() == kByIo) break;
            std::this_thread::sleep_for(std::chrono::microseconds(20));
          }
      }
      check(cake_event_record(g.ev_near[c.index]->h, g.s_compute), "record");  // (no next chunk paces on it)
      check(cake_event_record(g.ev_end[c.index]->h, g.s_compute), "record");
      std::lock_guard lk(mu_);
      launched_.push_back(c.index);
      predicted_end_.push_back(predicted);
      return;
    }
    check(cake_prefill_layers(g.model, tok, start, len, 0, split, bt, abort, 0, g.s_compute), "prefill");
    check(cake_event_record(g.ev_near[c.index]->h, g.s_compute), "record");
    if (split < L) check(cake_prefill_layers(g.model, tok, start, len, split, L, bt, abort, 0, g.s_compute), "prefill");
    check(cake_event_record(g.ev_end[c.index]->h, g.s_compute), "record");
    std::lock_guard lk(mu_);
    launched_.push_back(c.index);
    predicted_end_.push_back(predicted);
  }

  Micros predict_finish(const ChunkSpec& c) override {
    const Micros now = r_.timer.now_us();
    const Micros free_at = launched_.empty() ? now : expected_end(launched_.size() - 1);
    return std::max(now, free_at) + duration(c);
  }

  // Predicted completion of launched chunk `index` (for the loader's race policy).
  std::optional<Micros> expected_end_of(std::uint32_t index) {
    std::lock_guard lk(mu_);
    for (std::size_t k = 0; k < launched_.size(); ++k)
      if (launched_[k] == index) return expected_end(k);
    return std::nullopt;
  }

  std::vector<ChunkRecord> drain() override {
    std::vector<ChunkRecord> out;
    for (std::uint32_t i : launched_) {
      check(cake_event_sync(r_.g.ev_end[i]->h), "drain");
      if (!r_.try_commit(i, kByCompute)) continue;  // the loader landed it first
      out.push_back({i, Side::compute, r_.device_time(r_.g.ev_start[i]->h), r_.device_time(r_.g.ev_end[i]->h), 0});
    }
    last_launched_ = launched_.empty() ? -1 : static_cast<int>(launched_.back());
    return out;
  }

  int last_launched() const { return last_launched_; }

 private:
  // Callers on the loader thread hold mu_; the compute thread (the only
  // writer of launched_ and of the ratio, both under mu_) may read unlocked.
  Micros duration(const ChunkSpec& c) const {
    const double base = static_cast<double>(compute_latency(prior_, c, 1.0));
    const double ratio = den_ > 0 ? num_ / den_ : 1.0;
    return static_cast<Micros>(base * ratio);
  }
  Micros expected_end(std::size_t k) const {
    const std::uint32_t i = launched_[k];
    if (cake_event_query(r_.g.ev_end[i]->h) == CAKE_OK) return r_.device_time(r_.g.ev_end[i]->h);
    if (cake_event_query(r_.g.ev_start[i]->h) == CAKE_OK)
      return r_.device_time(r_.g.ev_start[i]->h) + duration(r_.plan.chunks[i]);
    return predicted_end_[k];
  }
  // Fold finished chunks into the observed/prior duration ratio.
  void observe() {
    while (observed_ < launched_.size()) {
      const std::uint32_t i = launched_[observed_];
      if (cake_event_query(r_.g.ev_end[i]->h) != CAKE_OK) break;
      float ms = 0.f;
      check(cake_event_elapsed_ms(r_.g.ev_start[i]->h, r_.g.ev_end[i]->h, &ms), "elapsed");
      std::lock_guard lk(mu_);
      num_ += static_cast<double>(ms) * 1000.0;
      den_ += static_cast<double>(compute_latency(prior_, r_.plan.chunks[i], 1.0));
      ++observed_;
    }
  }

  LiveRun& r_;
  CostModel prior_;
  std::mutex mu_;
  std::vector<std::uint32_t> launched_;
  std::vector<Micros> predicted_end_;
  std::size_t observed_ = 0;
  double num_ = 0.0, den_ = 0.0;
  int last_launched_ = -1;
};

class GpuLoaderSink final : public ChunkSink {
 public:
  GpuLoaderSink(LiveRun& run, bool q8) : r_(run), q8_(q8) {}

  ~GpuLoaderSink() override {
    if (range_) nvtxRangeEnd(range_);
  }

  void begin_chunk(const FetchTask& t) override {
    GpuContext::Impl& g = r_.g;
    bind_device(g.opt.device);
    if (range_) nvtxRangeEnd(range_);  // an abandoned chunk never reached end_chunk
    range_ = nvtxRangeStartA(("load chunk " + std::to_string(t.chunk.index) + (t.contested ? " (contested)" : "")).c_str());
    // every rank loads its shard of this chunk (the racer's entry into its spare pages)
    if (r_.tp) r_.tp->publish_io(t.chunk.index | (t.contested ? TpCoordinator::kRaceBit : 0u));
    if (t.contested) r_.start_race(t.chunk, kByIo, g.s_copy);
    // quant8: land the 4-B header at +12 so the level payload is 16-B aligned
    buf_ = g.staging[parity_].p + (q8_ ? kQ8Offset : 0);
    parity_ ^= 1;
  }

  void deliver(const FetchTask& t, std::uint64_t offset, std::span<const std::byte> bytes) override {
    bind_device(r_.g.opt.device);
    check(cake_h2d_async(buf_ + offset, bytes.data(), bytes.size(), r_.g.s_copy), "slice H2D");
    h2d_bytes_ += bytes.size();
  }

  void end_chunk(const FetchTask& t) override {
    GpuContext::Impl& g = r_.g;
    bind_device(g.opt.device);
    if (q8_)
      check(cake_kv_scatter_q8(g.model, buf_, static_cast<long long>(t.chunk.token_start),
                               static_cast<int>(t.chunk.token_count), r_.table_for(t.chunk.index, kByIo), g.s_copy),
            "q8 decode-scatter");
    else
      check(cake_kv_scatter(g.model, buf_, static_cast<long long>(t.chunk.token_start),
                            static_cast<int>(t.chunk.token_count), r_.table_for(t.chunk.index, kByIo), 0,
                            static_cast<long long>(t.encoded_bytes), g.s_copy),
            "scatter");
    check(cake_event_record(g.ev_io[t.chunk.index]->h, g.s_copy), "record");
    nvtxRangeEnd(range_);
    range_ = 0;
  }

  Micros wait_chunk(const FetchTask& t) override {
    bind_device(r_.g.opt.device);
    check(cake_event_sync(r_.g.ev_io[t.chunk.index]->h), "io wait");
    if (r_.tp) {  // resident only when every rank's KV-head shard landed
      r_.tp->shard_landed(t.chunk.index);
      if (!r_.tp->wait_all_landed(t.chunk.index)) return -1;  // compute landed it first
    }
    if (!r_.try_commit(t.chunk.index, kByIo)) return -1;  // compute landed it first
    r_.abort_compute(t.chunk.index);  // stop any compute work still queued for it
    return r_.device_time(r_.g.ev_io[t.chunk.index]->h);
  }

  bool keep_going(const FetchTask& t) override { return r_.commit[t.chunk.index].load() != kByCompute; }

  HostAllocator staging_allocator() override { return {PinnedPool::alloc, PinnedPool::release, &r_.g.landing}; }

  std::uint64_t h2d_bytes() const { return h2d_bytes_; }

 private:
  static constexpr std::size_t kQ8Offset = 12;
  LiveRun& r_;
  bool q8_;
  std::byte* buf_ = nullptr;
  int parity_ = 0;
  std::uint64_t h2d_bytes_ = 0;
  nvtxRangeId_t range_ = 0;  // the chunk being paced (pacer thread only)
};

}  // namespace

// A TP follower mirrors the leader's decisions (cake/tp.hpp): it enqueues the
// compute chunks the leader launched, loads its own KV-head shard of the
// chunks the leader's loader claimed (same throttle, its own emulated link),
// and joins the first-token step. Its collectives pair with the leader's.
RunReport run_follower(GpuContext::Impl& g, TpCoordinator& tp, const RunPlan& plan,
                       const std::vector<std::uint32_t>& tokens, const BandwidthTrace& trace, const ChunkStore& store,
                       RunMode mode, const RunOptions& opt) {
  const auto n = static_cast<std::uint32_t>(plan.chunks.size());
  g.ensure_events(n);
  tp.begin_run(++g.run_counter, n);
  sync_own_streams(g);
  RunTimer timer;
  check(cake_event_record(g.ev_anchor->h, g.s_compute), "anchor");
  const Micros t0 = timer.now_us();
  check(cake_stream_wait_event(g.s_copy, g.ev_anchor->h), "order");
  check(cake_memset_async(g.abort_flags.p, 0, g.n_pages * sizeof(std::int32_t), g.s_compute), "abort reset");
  check(cake_event_record(g.ev_reset->h, g.s_compute), "record");  // abort writes (s_control) after the reset
  check(cake_stream_wait_event(g.s_control, g.ev_reset->h), "order");
  upload_tokens(g, tokens, g.s_compute);
  auto dev_time = [&](void* ev) {
    float ms = 0.f;
    check(cake_event_elapsed_ms(g.ev_anchor->h, ev, &ms), "elapsed");
    return t0 + static_cast<Micros>(std::llround(ms * 1000.0));
  };
  std::vector<std::uint32_t> io_chunks;
  std::exception_ptr io_error;
  std::thread io([&] {
    try {
      bind_device(g.opt.device);
      const std::uint64_t quantum = std::max<std::uint64_t>(opt.throttle_quantum_bytes, 1);
      Micros budget = 0;
      for (std::uint32_t k = 0;; ++k) {
        const auto c = tp.next_io(k);
        if (!c) break;
        const std::uint32_t i = *c & ~TpCoordinator::kRaceBit;
        const bool racer = (*c & TpCoordinator::kRaceBit) != 0;
        if (racer) upload_race_table(g, plan.chunks[i], g.s_copy);
        const std::int32_t* bt = racer ? g.bt_race.p : g.bt_primary.p;
        const std::uint64_t total = plan.encoded_bytes[i];
        ChunkReader rd = store.open_reader(plan.keys[i]);
        // file tier: read the whole chunk into pinned memory (the slice H2Ds below are
        // async); memory tier: zero-copy view of the pinned tier
        const std::byte* src = nullptr;
        if (rd.in_memory()) {
          src = rd.view_next(static_cast<std::size_t>(total)).data();
        } else {
          if (g.follower_landing.n < total) g.follower_landing.reset(static_cast<std::size_t>(total));
          std::span<std::byte> host(g.follower_landing.p, static_cast<std::size_t>(total));
          if (rd.read(host) != host.size()) throw CorruptChunkError("tp follower: short read");
          src = host.data();
        }
        const bool q8 = plan.encoded_bytes[i] != plan.uncompressed_bytes[i];
        std::byte* buf = g.staging[k & 1].p + (q8 ? 12 : 0);
        bool abandoned = false;
        for (std::uint64_t off = 0; off < total;) {
          if (tp.decided(i) == 1) {  // the leader's compute side committed this chunk: drop the load
            abandoned = true;
            break;
          }
          const std::uint64_t len = std::min(quantum, total - off);
          const Micros gate = budget + time_to_transfer_bits(trace, len * 8, budget);
          timer.sleep_until_us_precise(gate);
          check(cake_h2d_async(buf + off, src + off, len, g.s_copy), "slice H2D");
          off += len;
          budget = gate;
          const Micros now = timer.now_us();
          const Micros one = time_to_transfer_bits(trace, quantum * 8, budget);
          if (budget + one < now) budget = now - one;
        }
        if (abandoned) continue;
        if (q8)
          check(cake_kv_scatter_q8(g.model, buf, static_cast<long long>(plan.chunks[i].token_start),
                                   static_cast<int>(plan.chunks[i].token_count), bt, g.s_copy),
                "q8 decode-scatter");
        else
          check(cake_kv_scatter(g.model, buf, static_cast<long long>(plan.chunks[i].token_start),
                                static_cast<int>(plan.chunks[i].token_count), bt, 0,
                                static_cast<long long>(total), g.s_copy),
                "scatter");
        check(cake_event_record(g.ev_io[i]->h, g.s_copy), "record");
        check(cake_event_sync(g.ev_io[i]->h), "io wait");
        tp.shard_landed(i);
        io_chunks.push_back(i);
      }
    } catch (...) {
      io_error = std::current_exception();
    }
  });
  std::vector<std::uint32_t> computed;
  for (std::uint32_t k = 0;; ++k) {
    const auto c = tp.next_compute(k);
    if (!c) break;
    const ChunkSpec& ch = plan.chunks[*c & ~TpCoordinator::kRaceBit];
    const bool racer = (*c & TpCoordinator::kRaceBit) != 0;
    if (racer) upload_race_table(g, ch, g.s_compute);
    check(cake_event_record(g.ev_start[ch.index]->h, g.s_compute), "record");
    check(cake_prefill_chunk(g.model, g.tokens.p + ch.token_start, static_cast<long long>(ch.token_start),
                             static_cast<int>(ch.token_count), racer ? g.bt_race.p : g.bt_primary.p,
                             g.abort_flags.p + ch.index, 0, g.s_compute),
          "prefill");
    check(cake_event_record(g.ev_end[ch.index]->h, g.s_compute), "record");
    computed.push_back(ch.index);
  }
  // the leader's loader won a chunk this rank is computing (the contested one,
  // either racer): cancel its queued kernels like the leader does (the
  // reductions still run, so the ranks stay in lockstep)
  std::vector<char> aborted(n, 0);
  auto maybe_abort = [&] {
    for (std::uint32_t i : computed)
      if (!aborted[i] && tp.decided(i) == 2) {
        check(cake_h2d_async(g.abort_flags.p + i, g.h_abort_one.p, sizeof(std::int32_t), g.s_control), "abort");
        aborted[i] = 1;
      }
  };
  const Micros final_deadline = timer.now_us() + 300'000'000;  // a leader that died must not hang its followers
  while (!tp.final_published()) {
    maybe_abort();
    if (timer.now_us() > final_deadline)
      throw std::runtime_error("tp follower: the leader never published the first-token step's inputs");
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  maybe_abort();
  const TpCoordinator::Final fin = tp.wait_final();
  const int recompute = fin.recompute, last_row = fin.last_row;
  g.final_bt = fin.race_pages >= 0 ? g.bt_race.p : g.bt_primary.p;
  io.join();
  if (io_error) std::rethrow_exception(io_error);
  const ChunkSpec& tail = plan.chunks[n - 1];
  const long long T = static_cast<long long>(tail.token_start + tail.token_count);
  check(cake_event_record(g.ev_final_start->h, g.s_compute), "record");
  check(cake_final_logits(g.model, T, g.tokens.p + (T - 1), recompute, last_row, g.final_bt, g.logits.p,
                          g.s_compute),
        "final logits");
  check(cake_d2h_async(g.h_logits.p, g.logits.p, g.cfg.vocab * sizeof(float), g.s_compute), "logits D2H");
  check(cake_event_record(g.ev_logits->h, g.s_compute), "record");
  check(cake_event_sync(g.ev_logits->h), "logits");
  GpuRunInfo info;
  info.first_token_us = timer.now_us();
  RunReport rep;
  rep.mode = mode;
  rep.n_chunks = n;
  // the leader's commits decide which side delivered each chunk (a contested one ran on both)
  for (std::uint32_t i : computed)
    if (tp.decided(i) != 2)
      rep.chunks.push_back({i, Side::compute, dev_time(g.ev_start[i]->h), dev_time(g.ev_end[i]->h), 0});
  for (std::uint32_t i : io_chunks)
    if (tp.decided(i) != 1) rep.chunks.push_back({i, Side::io, 0, dev_time(g.ev_io[i]->h), plan.encoded_bytes[i]});
  detail::finalize_report(rep, 0);
  rep.merge_point = detail::merge_from_records(rep);
  rep.computed_fraction = static_cast<double>(rep.merge_point) / n;
  float ms = 0.f;
  check(cake_event_elapsed_ms(g.ev_final_start->h, g.ev_logits->h, &ms), "elapsed");
  info.final_step_us = static_cast<Micros>(std::llround(ms * 1000.0));
  check(cake_event_elapsed_ms(g.ev_anchor->h, g.ev_logits->h, &ms), "elapsed");
  info.device_ttft_ms = ms;
  info.kv_resident_us = rep.ttft_us;
  info.merge_point = rep.merge_point;
  info.raced_chunk = fin.race_chunk;
  info.race_winner = fin.race_winner;
  info.recomputed_last = recompute != 0;
  info.d2h_bytes = g.cfg.vocab * sizeof(float);
  check(cake_model_launch_count(g.model, &info.kernel_launches, 0), "launch count");
  info.logits.assign(g.h_logits.p, g.h_logits.p + g.cfg.vocab);
  g.last = std::move(info);
  tp.end_run();
  return rep;
}

namespace detail {

RunReport run_live_gpu(const RunPlan& plan, const std::vector<std::uint32_t>& tokens, const CostModel& cost,
                       const BandwidthTrace& trace, const Codec& codec, const ChunkStore& store, RunMode mode,
                       double power, const RunOptions& opt) {
  GpuContext::Impl& g = *opt.gpu->impl();
  if (codec.kind == Codec::Kind::factor) throw std::invalid_argument("gpu run: the factor codec models bytes only");
  const auto n = static_cast<std::uint32_t>(plan.chunks.size());  // the cached prefix: bidirectional phase
  const auto n_all = static_cast<std::uint32_t>(n + plan.suffix.size());
  check_chunking(g, plan.chunks, tokens.size());
  check_chunking(g, plan.suffix, tokens.size());
  for (std::uint32_t i = 0; i < n; ++i) {
    const auto raw = static_cast<std::uint64_t>(cake_kv_chunk_bytes(g.model, plan.chunks[i].token_count));
    if (plan.encoded_bytes[i] != codec.encoded_size(raw))
      throw std::invalid_argument("gpu run: cache-tier chunk size disagrees with the model's KV layout");
  }
  const bool io_on = mode == RunMode::io_only || (mode == RunMode::cake && opt.io_enabled);
  const bool compute_on = mode == RunMode::compute_only || (mode == RunMode::cake && opt.compute_enabled);
  if (!io_on && !compute_on) throw std::invalid_argument("run: no side enabled");
  TpCoordinator* tp = g.tp.get();
  if (tp && !plan.suffix.empty()) throw std::invalid_argument("gpu run: partially cached prompts are single-GPU only");
  if (tp && !tp->leader()) return run_follower(g, *tp, plan, tokens, trace, store, mode, opt);
  const bool race = opt.race_to_finish && io_on && compute_on;  // TP: mirrored through the coordinator
  g.ensure_events(n_all);
  if (tp) tp->begin_run(++g.run_counter, n);
  sync_own_streams(g);
  long long launches0 = 0;
  check(cake_model_launch_count(g.model, &launches0, 1), "launch count");

  // ---------------------------------------------------------------- t = 0
  NvtxScope nv_run(std::string("bidirectional run: ") + (mode == RunMode::cake ? "cake" : mode == RunMode::io_only ? "io_only" : "compute_only") +
                   ", " + std::to_string(n) + " chunks");
  RunTimer timer;
  LiveRun run(g, plan, timer);
  run.tp = tp;
  check(cake_event_record(g.ev_anchor->h, g.s_compute), "anchor");
  run.t0 = timer.now_us();
  run.hold = !race ? kNone : opt.race_hold == 0 ? kByCompute : opt.race_hold == 1 ? kByIo : kNone;
  check(cake_stream_wait_event(g.s_copy, g.ev_anchor->h), "order");
  check(cake_memset_async(g.abort_flags.p, 0, g.n_pages * sizeof(std::int32_t), g.s_compute), "abort reset");
  // abort writes go on the control stream: order them after the reset
  check(cake_event_record(g.ev_reset->h, g.s_compute), "record");
  check(cake_stream_wait_event(g.s_control, g.ev_reset->h), "order");
  upload_tokens(g, tokens, g.s_compute);
  GpuRunInfo info;
  info.h2d_bytes = tokens.size() * sizeof(std::int32_t);

  ClaimTable table(n);
  GpuLoaderSink sink(run, codec.kind == Codec::Kind::quant8);
  GpuPrefillBackend backend(run, opt.gpu->options().prior);
  std::unique_ptr<TransferEngine> loader;
  if (io_on) {
    TransferOptions t;
    t.throttle_quantum_bytes = opt.throttle_quantum_bytes;
    t.jitter_max_us = opt.jitter_max_us;
    t.jitter_seed = opt.jitter_seed;
    t.record_slices = opt.record_slices;
    t.sink = &sink;
    t.link = opt.link;
    if (race) {
      t.contest = [&](const FetchTask& task, Micros io_eta) {
        if (opt.race_force == 1) return false;
        bool want = opt.race_force == 2;
        if (!want) {
          const auto c_eta = backend.expected_end_of(task.chunk.index);
          want = c_eta && io_eta + g.opt.race_margin_us < *c_eta;
        }
        return want && run.reserve_race(task.chunk.index, kByIo);
      };
    }
    loader = std::make_unique<TransferEngine>(store, trace, codec, &table, timer, std::move(t));
    run.loader = loader.get();
    std::vector<FetchTask> tasks;
    tasks.reserve(n);
    for (std::uint32_t i = n; i-- > 0;) tasks.push_back({plan.keys[i], plan.chunks[i], plan.encoded_bytes[i]});
    loader->push_seq(std::move(tasks));
    if (race && opt.race_force == 1) {
      // test hook: the compute side starts once the loader is pacing its first chunk, so
      // there is an in-flight chunk to contest however the host threads get scheduled
      const Micros deadline = timer.now_us() + 10'000'000;
      while (!loader->inflight_finish_estimate(n - 1) && timer.now_us() < deadline)
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }

  RunReport rep;
  rep.mode = mode;
  rep.n_chunks = n_all;
  if (compute_on) {
    ComputeEngine engine(cost, TokenBudget{opt.token_budget, power});
    ComputeEngine::ForwardHooks hooks;
    hooks.table = &table;
    hooks.timer = &timer;
    hooks.jitter_max_us = opt.jitter_max_us;
    hooks.jitter_seed = opt.jitter_seed + 1;
    hooks.backend = &backend;
    if (loader) {
      hooks.probe = &loader->resident_set();
      // race_force 2 (test): the loader goes on to its failing claim (and contests it) instead of
      // being stopped when the compute side runs out of chunks
      hooks.signal_stop = [&] {
        run.compute_done.store(true);
        if (opt.race_force != 2) loader->stop();
      };
    } else {
      hooks.signal_stop = [&] { run.compute_done.store(true); };
    }
    if (race) {
      hooks.contest = [&](const ChunkSpec& c, Micros c_eta) {
        if (opt.race_force == 2) return false;
        const auto io_eta = loader->inflight_finish_estimate(c.index);
        if (!io_eta) return false;  // nothing in flight to race
        const bool want = opt.race_force == 1 || c_eta + g.opt.race_margin_us < *io_eta;
        return want && run.reserve_race(c.index, kByCompute);
      };
    }
    auto recs = engine.run_forward(plan.chunks, plan.keys, hooks);
    rep.chunks.insert(rep.chunks.end(), recs.begin(), recs.end());
  }
  if (tp) tp->end_compute();
  // The first token needs every chunk committed, not the loader's threads
  // drained (a pacer may still be winding down a chunk it lost).
  run.wait_all_committed();
  if (tp) tp->end_io();
  if (run.n_committed < n && loader) loader->wait();  // surfaces the loader's error, if any
  if (run.n_committed < n) throw std::logic_error("run: chunk coverage is incomplete");

  // ---------------------------------------------------------------- first token
  const int rc = run.race_chunk.load();
  const bool racer_won = rc >= 0 && ((run.racer.load() == kByCompute && run.commit[rc].load() == kByCompute) ||
                                     (run.racer.load() == kByIo && run.commit[rc].load() == kByIo));
  g.final_bt = racer_won ? g.bt_race.p : g.bt_primary.p;
  // No stream join needed: every io-committed chunk's scatter event has
  // already completed (the commit happens after its event sync), and
  // whatever the copy stream still carries (a lost race) writes pages the
  // final block table does not reference.
  // ---------------------------------------------------------------- uncached suffix
  // Every prefix chunk is committed, so the suffix chunks (their prefix
  // attention reads all of it, through the final block table) run back to
  // back on the compute stream.
  for (const ChunkSpec& c : plan.suffix) {
    check(cake_event_record(g.ev_start[c.index]->h, g.s_compute), "record");
    check(cake_prefill_chunk(g.model, g.tokens.p + c.token_start, static_cast<long long>(c.token_start),
                             static_cast<int>(c.token_count), g.final_bt, nullptr, 0, g.s_compute),
          "suffix prefill");
    check(cake_event_record(g.ev_end[c.index]->h, g.s_compute), "record");
  }
  const ChunkSpec& tail = plan.suffix.empty() ? plan.chunks[n - 1] : plan.suffix.back();
  const bool tail_hidden = !plan.suffix.empty() || (run.commit[n - 1].load() == kByCompute &&
                                                    backend.last_launched() == static_cast<int>(n - 1));
  const long long T = static_cast<long long>(tail.token_start + tail.token_count);
  if (tp)
    tp->publish_final({tail_hidden ? 0 : 1, static_cast<int>(tail.token_count) - 1, racer_won ? rc : -1, rc,
                       rc >= 0 ? (run.commit[rc].load() == kByCompute ? 0 : 1) : -1});
  NvtxScope nv_final(std::string("first token") + (tail_hidden ? "" : " (recompute last token)"));
  check(cake_event_record(g.ev_final_start->h, g.s_compute), "record");
  check(cake_final_logits(g.model, T, g.tokens.p + (T - 1), tail_hidden ? 0 : 1, static_cast<int>(tail.token_count) - 1,
                          g.final_bt, g.logits.p, g.s_compute),
        "final logits");
  check(cake_d2h_async(g.h_logits.p, g.logits.p, g.cfg.vocab * sizeof(float), g.s_compute), "logits D2H");
  check(cake_event_record(g.ev_logits->h, g.s_compute), "record");
  check(cake_event_sync(g.ev_logits->h), "logits");
  info.first_token_us = timer.now_us();
  // ---------------------------------------------------------------- done
  if (loader) {
    loader->wait();
    rep.chunks.insert(rep.chunks.end(), loader->records().begin(), loader->records().end());
    info.slices = loader->slices();
  }
  for (const ChunkSpec& c : plan.suffix)
    rep.chunks.push_back({c.index, Side::compute, run.device_time(g.ev_start[c.index]->h),
                          run.device_time(g.ev_end[c.index]->h), 0});
  detail::finalize_report(rep, 0);
  rep.merge_point = std::min(merge_from_records(rep), n);  // within the cached prefix
  std::uint32_t computed = 0;
  for (const ChunkRecord& r : rep.chunks) computed += r.side == Side::compute ? 1u : 0u;
  rep.computed_fraction = static_cast<double>(computed) / n_all;

  info.kv_resident_us = rep.ttft_us;
  float ms = 0.f;
  check(cake_event_elapsed_ms(g.ev_final_start->h, g.ev_logits->h, &ms), "elapsed");
  info.final_step_us = static_cast<Micros>(std::llround(ms * 1000.0));
  check(cake_event_elapsed_ms(g.ev_anchor->h, g.ev_logits->h, &ms), "elapsed");
  info.device_ttft_ms = ms;
  info.merge_point = rep.merge_point;
  info.raced_chunk = rc;
  info.race_winner = rc >= 0 ? (run.commit[rc].load() == kByCompute ? 0 : 1) : -1;
  info.recomputed_last = !tail_hidden;
  info.h2d_bytes += sink.h2d_bytes();
  info.d2h_bytes = g.cfg.vocab * sizeof(float);
  check(cake_model_launch_count(g.model, &info.kernel_launches, 0), "launch count");
  info.logits.assign(g.h_logits.p, g.h_logits.p + g.cfg.vocab);
  if (rc >= 0)
    rep.events.push_back("race on chunk " + std::to_string(rc) + " won by " +
                         (info.race_winner == 0 ? "compute" : "io"));
  rep.events.push_back("first token at " + std::to_string(info.first_token_us) + "us");
  g.last = std::move(info);
  if (tp) tp->end_run();
  return rep;
}

}  // namespace detail

}  // namespace cake
