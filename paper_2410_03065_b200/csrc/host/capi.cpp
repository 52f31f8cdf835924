// Flat C ABI over the cake:: runtime (include/cake_c.h).
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <tuple>

#include "cake/codec.hpp"
#ifndef CAKE_REFERENCE_BUILD
#include "cake/gpu.hpp"
#endif
#include "cake/model.hpp"
#include "cake/scheduler.hpp"
#include "cake/store.hpp"
#include "cake_c.h"

using namespace cake;

namespace {

thread_local std::string g_err;

int guarded(const std::function<void()>& body) {
  try {
    body();
    return 0;
  } catch (const MissingKeyError& e) {
    g_err = e.what();
    return CAKE_C_EMISSING;
  } catch (const CorruptChunkError& e) {
    g_err = e.what();
    return CAKE_C_ECORRUPT;
  } catch (const StoreError& e) {
    g_err = e.what();
    return CAKE_C_ESTORE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return CAKE_C_EINVAL;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return CAKE_C_ELOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CAKE_C_ERUNTIME;
  } catch (...) {
    g_err = "unknown exception";
    return CAKE_C_ERUNTIME;
  }
}

BandwidthTrace to_trace(const cake_trace& t) {
  if (t.n < 1 || !t.at_us || !t.mbps) throw std::invalid_argument("trace: needs at least one breakpoint");
  std::vector<BandwidthTrace::Breakpoint> pts(static_cast<std::size_t>(t.n));
  for (int i = 0; i < t.n; ++i) pts[i] = {t.at_us[i], t.mbps[i]};
  return BandwidthTrace(std::move(pts));
}

#ifndef CAKE_REFERENCE_BUILD
}  // namespace
struct cake_link {
  std::shared_ptr<SharedLink> link;
};
namespace {
#endif

RunOptions to_opts(const cake_run_opts* o) {
  RunOptions r;
  if (!o) return r;
  r.compute_enabled = o->compute_enabled != 0;
  r.io_enabled = o->io_enabled != 0;
  r.token_budget = o->token_budget;
  r.throttle_quantum_bytes = o->throttle_quantum_bytes;
  r.decode_us_per_byte = o->decode_us_per_byte;
  r.jitter_max_us = o->jitter_max_us;
  r.jitter_seed = o->jitter_seed;
  r.record_slices = o->record_slices != 0;
#ifndef CAKE_REFERENCE_BUILD
  r.race_to_finish = o->race_to_finish != 0;
  r.cached_prefix = o->cached_prefix != 0;
  r.race_force = o->race_force;
  r.race_hold = o->race_hold;
  if (o->link) r.link = static_cast<const cake_link*>(o->link)->link;
#else
  if (o->link) throw std::invalid_argument("link is a B200 extension");
  if (o->race_to_finish) throw std::invalid_argument("race_to_finish is a B200 extension");
  if (o->cached_prefix) throw std::invalid_argument("cached_prefix is a B200 extension");
#endif
  return r;
}

RunMode to_mode(int m) {
  switch (m) {
    case CAKE_MODE_CAKE:
      return RunMode::cake;
    case CAKE_MODE_COMPUTE_ONLY:
      return RunMode::compute_only;
    case CAKE_MODE_IO_ONLY:
      return RunMode::io_only;
  }
  throw std::invalid_argument("bad mode");
}

void export_report(const RunReport& r, cake_summary* s, cake_record* recs) {
  if (s) {
    s->ttft_us = r.ttft_us;
    s->merge_point = r.merge_point;
    s->n_chunks = r.n_chunks;
    s->computed_fraction = r.computed_fraction;
    s->compute_busy_us = r.compute_busy_us;
    s->io_busy_us = r.io_busy_us;
  }
  if (recs)
    for (std::size_t i = 0; i < r.chunks.size(); ++i) {
      const ChunkRecord& c = r.chunks[i];
      recs[i] = {c.index, c.side == Side::io ? CAKE_SIDE_IO : CAKE_SIDE_COMPUTE, c.start_us, c.finish_us, c.bytes};
    }
}

ChunkKey key_from(const uint8_t* p) {
  ChunkKey k;
  std::memcpy(k.digest.data(), p, 32);
  return k;
}

#ifndef CAKE_REFERENCE_BUILD
void* pinned_alloc(std::size_t n, void*) {
  void* p = nullptr;
  return cake_host_alloc(&p, n) == CAKE_OK ? p : nullptr;
}
void pinned_release(void* p, void*) { cake_host_free(p); }
#endif

ModelProfile profile_of(uint32_t n_layers, uint32_t hidden, uint32_t precision) {
  ModelProfile p;
  p.name = "capi";
  p.n_layers = n_layers;
  p.hidden_size = hidden;
  p.precision_bytes = precision;
  p.kv_multiplier = 2;
  return p;
}

}  // namespace

struct cake_store {
  ChunkStore store;
};

#ifndef CAKE_REFERENCE_BUILD
struct cake_gpu {
  std::unique_ptr<GpuContext> ctx;
  Codec codec = Codec::identity();  // cache-tier codec of build_tier and run
  std::shared_ptr<SharedLink> link;  // set: runs pace through this shared link
};

#endif

extern "C" {

int cake_last_error(char* buf, size_t len) {
  if (buf && len) std::snprintf(buf, len, "%s", g_err.c_str());
  return static_cast<int>(g_err.size());
}

int cake_time_to_transfer_bits(cake_trace trace, uint64_t bits, int64_t start_us, int64_t* out) {
  return guarded([&] { *out = time_to_transfer_bits(to_trace(trace), bits, start_us); });
}

int cake_fetch_latency(cake_trace trace, uint64_t nbytes, int64_t start_us, int64_t* out) {
  return guarded([&] { *out = fetch_latency(to_trace(trace), nbytes, start_us); });
}

int cake_compute_latency(double alpha_ms, double beta, uint32_t ref_chunk, uint64_t token_start, uint32_t token_count,
                         double power, int64_t* out) {
  return guarded([&] {
    *out = compute_latency(CostModel{alpha_ms, beta, ref_chunk}, ChunkSpec{0, token_start, token_count}, power);
  });
}

int cake_kv_bytes_per_token(uint32_t n_layers, uint32_t hidden, uint32_t precision, uint32_t kv_mult,
                            uint64_t override_or_0, uint64_t* out) {
  return guarded([&] {
    ModelProfile p = profile_of(n_layers, hidden, precision);
    p.kv_multiplier = kv_mult;
    if (override_or_0) p.per_token_bytes_override = override_or_0;
    *out = kv_bytes_per_token(p);
  });
}

int cake_split_into_chunks(uint64_t total_tokens, uint32_t chunk_size, uint32_t* n_out, uint64_t* starts,
                           uint32_t* counts, uint32_t cap) {
  return guarded([&] {
    const auto cs = split_into_chunks(total_tokens, chunk_size);
    *n_out = static_cast<uint32_t>(cs.size());
    for (std::size_t i = 0; i < cs.size() && i < cap; ++i) {
      if (starts) starts[i] = cs[i].token_start;
      if (counts) counts[i] = cs[i].token_count;
    }
  });
}

int cake_oracle_best_split(const int64_t* compute_us, uint32_t n_compute, const int64_t* fetch_us, uint32_t n_fetch,
                           uint32_t* k_star, int64_t* ttft_star) {
  return guarded([&] {
    const SplitChoice s = oracle_best_split(std::span<const Micros>(compute_us, n_compute),
                                            std::span<const Micros>(fetch_us, n_fetch));
    *k_star = s.k_star;
    *ttft_star = s.ttft_star;
  });
}

void cake_run_opts_default(cake_run_opts* o) {
  const RunOptions d;
  o->compute_enabled = d.compute_enabled;
  o->io_enabled = d.io_enabled;
  o->token_budget = d.token_budget;
  o->throttle_quantum_bytes = d.throttle_quantum_bytes;
  o->decode_us_per_byte = d.decode_us_per_byte;
  o->jitter_max_us = d.jitter_max_us;
  o->jitter_seed = d.jitter_seed;
  o->race_to_finish = 0;
  o->cached_prefix = 0;
  o->record_slices = 0;
  o->race_force = 0;
  o->race_hold = -1;
}

int cake_sim_run(uint32_t n, const uint64_t* token_starts, const uint32_t* token_counts, const uint64_t* encoded_bytes,
                 const uint64_t* uncompressed_bytes, double alpha_ms, double beta, uint32_t ref_chunk,
                 cake_trace trace, int mode, double power, const cake_run_opts* opts, cake_summary* summary,
                 cake_record* records) {
  return guarded([&] {
    RunPlan plan;
    for (uint32_t i = 0; i < n; ++i) {
      plan.chunks.push_back({i, token_starts[i], token_counts[i]});
      plan.encoded_bytes.push_back(encoded_bytes[i]);
      plan.uncompressed_bytes.push_back(uncompressed_bytes[i]);
    }
    const RunReport r = run_sim_planned(plan, CostModel{alpha_ms, beta, ref_chunk}, to_trace(trace), to_mode(mode),
                                        power, to_opts(opts));
    export_report(r, summary, records);
  });
}

int cake_store_open(const char* root, int create, int pinned, cake_store** out) {
  return guarded([&] {
    if (!root || !root[0]) {
#ifndef CAKE_REFERENCE_BUILD
      *out = new cake_store{ChunkStore::in_memory(
          pinned ? HostAllocator{pinned_alloc, pinned_release, nullptr} : HostAllocator{})};
      return;
#else
      throw std::invalid_argument("memory-resident stores are a B200 extension");
#endif
    }
    if (create == 1)
      *out = new cake_store{ChunkStore::create(root)};
    else if (create == 2)
      *out = new cake_store{ChunkStore::open_or_create(root)};
    else
      *out = new cake_store{ChunkStore::open(root)};
  });
}

int cake_store_close(cake_store* s) {
  delete s;
  return 0;
}

int cake_store_set_direct_io(cake_store* s, int on) {
  return guarded([&] {
#ifndef CAKE_REFERENCE_BUILD
    s->store.set_direct_io(on != 0);
#else
    if (on) throw std::invalid_argument("direct I/O is a B200 extension");
#endif
  });
}

int cake_store_entry_count(const cake_store* s, uint64_t* n) {
  return guarded([&] { *n = s->store.entry_count(); });
}

int cake_store_populate(cake_store* s, uint64_t total_tokens, uint32_t chunk_size, uint32_t n_layers, uint32_t hidden,
                        uint32_t precision, const char* codec, uint64_t seed, int sparse, uint8_t* keys_out) {
  return guarded([&] {
    RequestSpec req;
    req.total_tokens = total_tokens;
    req.chunk_size = chunk_size;
    const PopulateResult r = populate(s->store, req, profile_of(n_layers, hidden, precision), Codec::parse(codec), seed,
                                      sparse ? PayloadKind::sparse : PayloadKind::random);
    if (keys_out)
      for (std::size_t i = 0; i < r.keys.size(); ++i) std::memcpy(keys_out + 32 * i, r.keys[i].digest.data(), 32);
  });
}

int cake_store_put(cake_store* s, const uint8_t* key32, const uint8_t* payload, uint64_t n, uint32_t token_count,
                   const char* codec, uint64_t uncompressed) {
  return guarded([&] {
    s->store.put(key_from(key32), std::span<const std::byte>(reinterpret_cast<const std::byte*>(payload), n),
                 ChunkMeta{token_count, codec, n, uncompressed});
  });
}

int cake_store_get(const cake_store* s, const uint8_t* key32, uint8_t* out, uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    const auto v = s->store.get(key_from(key32));
    *n_out = v.size();
    if (out) std::memcpy(out, v.data(), std::min<uint64_t>(cap, v.size()));
  });
}

int cake_store_make_resident(cake_store* s, int pinned) {
  return guarded([&] {
#ifndef CAKE_REFERENCE_BUILD
    s->store.make_resident(pinned ? HostAllocator{pinned_alloc, pinned_release, nullptr} : HostAllocator{});
#else
    throw std::invalid_argument("memory-resident stores are a B200 extension");
#endif
  });
}

int cake_chain_hash(const uint8_t* prev32, const uint32_t* tokens, uint64_t n, uint8_t* out32) {
  return guarded([&] {
    std::optional<ChunkKey> prev;
    if (prev32) prev = key_from(prev32);
    const ChunkKey k = chain_hash(prev, std::span<const uint32_t>(tokens, n));
    std::memcpy(out32, k.digest.data(), 32);
  });
}

int cake_token_stream(uint64_t seed, uint64_t count, uint32_t* out) {
  return guarded([&] {
    const auto v = token_stream(seed, count);
    std::memcpy(out, v.data(), v.size() * 4);
  });
}

int cake_synth_payload(uint64_t seed, uint32_t chunk_index, uint64_t nbytes, uint8_t* out) {
  return guarded([&] {
    const auto v = synth_payload(seed, chunk_index, nbytes);
    std::memcpy(out, v.data(), v.size());
  });
}

int cake_codec_encoded_size(const char* codec, uint64_t raw, uint64_t* out) {
  return guarded([&] { *out = Codec::parse(codec).encoded_size(raw); });
}

int cake_codec_encode(const char* codec, const uint8_t* in, uint64_t n, uint8_t* out, uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    const auto v = codec_encode(Codec::parse(codec), std::span<const std::byte>(reinterpret_cast<const std::byte*>(in), n));
    *n_out = v.size();
    if (v.size() > cap) throw std::invalid_argument("encode: output buffer too small");
    std::memcpy(out, v.data(), v.size());
  });
}

int cake_codec_decode(const char* codec, const uint8_t* in, uint64_t n, uint64_t original_len, uint8_t* out,
                      uint64_t cap) {
  return guarded([&] {
    const auto v = codec_decode(Codec::parse(codec), std::span<const std::byte>(reinterpret_cast<const std::byte*>(in), n),
                                original_len);
    if (v.size() > cap) throw std::invalid_argument("decode: output buffer too small");
    std::memcpy(out, v.data(), v.size());
  });
}

uint16_t cake_fp16_from_float(float f) { return fp16_from_float(f); }
float cake_fp16_to_float(uint16_t h) { return fp16_to_float(h); }

int cake_run_store(cake_store* s, uint64_t total_tokens, uint32_t chunk_size, uint32_t n_layers, uint32_t hidden,
                   uint32_t precision, const char* codec, double alpha_ms, double beta, uint32_t ref_chunk,
                   cake_trace trace, int mode, int clock, uint64_t seed, double power, const cake_run_opts* opts,
                   cake_summary* summary, cake_record* records) {
  return guarded([&] {
    RequestSpec req;
    req.total_tokens = total_tokens;
    req.chunk_size = chunk_size;
    req.power_fraction = power;
    const RunReport r = run(req, profile_of(n_layers, hidden, precision), CostModel{alpha_ms, beta, ref_chunk},
                            to_trace(trace), Codec::parse(codec), to_mode(mode), clock ? ClockMode::live : ClockMode::sim,
                            s->store, seed, to_opts(opts));
    export_report(r, summary, records);
  });
}

// ------------------------------------------------------------------ GPU
#ifndef CAKE_REFERENCE_BUILD
int cake_gpu_create(const cake_gpu_config* c, cake_gpu** out) {
  return guarded([&] {
    GpuModelConfig m;
    m.name = "custom";
    m.n_layers = c->n_layers;
    m.hidden = c->hidden;
    m.n_heads = c->n_heads;
    m.n_kv_heads = c->n_kv_heads;
    m.head_dim = c->head_dim;
    m.ffn = c->ffn;
    m.vocab = c->vocab;
    m.rope_theta = c->rope_theta;
    m.rms_eps = c->rms_eps;
    GpuOptions o;
    o.device = c->device;
    o.max_chunk = c->max_chunk;
    o.max_tokens = c->max_tokens;
    o.weight_seed = c->weight_seed;
    o.tp_rank = c->tp_rank;
    o.tp_size = c->tp_size;
    o.nccl_comm = c->nccl_comm;
    if (c->lookahead_layers > 0) o.lookahead_layers = c->lookahead_layers;
    o.profile_kernels = c->profile_kernels != 0;
    if (c->race_margin_us > 0) o.race_margin_us = c->race_margin_us;
    if (c->tp_shm) o.tp_shm = c->tp_shm;
    o.compute_sms = c->compute_sms;
    if (c->weights_from) o.weights_from = c->weights_from->ctx.get();
    auto g = std::make_unique<cake_gpu>();
    g->ctx = std::make_unique<GpuContext>(m, o);
    *out = g.release();
  });
}

int cake_link_create(cake_trace trace, cake_link** out) {
  return guarded([&] {
    auto l = std::make_unique<cake_link>();
    l->link = std::make_shared<SharedLink>(to_trace(trace));
    *out = l.release();
  });
}

int cake_link_destroy(cake_link* l) {
  delete l;
  return CAKE_OK;
}

int cake_link_reset(cake_link* l) {
  return guarded([&] { l->link->reset(); });
}

int cake_link_reserved_bits(const cake_link* l, uint64_t* bits, int64_t* now_us) {
  return guarded([&] {
    *bits = l->link->reserved_bits();
    if (now_us) *now_us = l->link->timer().now_us();
  });
}

int cake_gpu_set_link(cake_gpu* g, cake_link* l) {
  return guarded([&] { g->link = l ? l->link : nullptr; });
}

int cake_gpu_destroy(cake_gpu* g) {
  return guarded([&] { delete g; });
}

int cake_gpu_kv_bytes_per_token(const cake_gpu* g, uint64_t* out) {
  return guarded([&] { *out = g->ctx->kv_bytes_per_token(); });
}

int cake_gpu_build_tier(cake_gpu* g, cake_store* s, uint64_t total_tokens, uint32_t chunk_size, uint64_t prompt_seed) {
  return guarded([&] {
    RequestSpec req;
    req.total_tokens = total_tokens;
    req.chunk_size = chunk_size;
    g->ctx->build_cache_tier(s->store, req, prompt_seed, g->codec);
  });
}

int cake_gpu_set_codec(cake_gpu* g, const char* codec_id) {
  return guarded([&] {
    const Codec c = Codec::parse(codec_id ? codec_id : "identity");
    if (c.kind == Codec::Kind::factor) throw std::invalid_argument("gpu: the factor codec models bytes only");
    g->codec = c;
  });
}

int cake_gpu_calibrate(cake_gpu* g, uint64_t total_tokens, uint32_t chunk_size, uint64_t prompt_seed, double* alpha,
                       double* beta) {
  return guarded([&] {
    RequestSpec req;
    req.total_tokens = total_tokens;
    req.chunk_size = chunk_size;
    const CostModel cm = g->ctx->calibrate(req, prompt_seed);
    *alpha = cm.alpha_ms;
    *beta = cm.beta_ms_per_token;
  });
}

int cake_gpu_run(cake_gpu* g, cake_store* s, uint64_t total_tokens, uint32_t chunk_size, uint64_t prompt_seed,
                 cake_trace trace, int mode, const cake_run_opts* opts, cake_gpu_result* res, cake_record* records) {
  return guarded([&] {
    RequestSpec req;
    req.total_tokens = total_tokens;
    req.chunk_size = chunk_size;
    RunOptions o = to_opts(opts);
    o.gpu = g->ctx.get();
    if (!o.link) o.link = g->link;
    const GpuModelConfig& mc = g->ctx->config();
    const ModelProfile prof = mc.profile(g->ctx->options().tp_size);
    const RunReport r = run(req, prof, g->ctx->options().prior, to_trace(trace), g->codec, to_mode(mode),
                            ClockMode::live, s->store, prompt_seed, o);
    const GpuRunInfo& info = g->ctx->last_run();
    if (res) {
      res->kv_resident_us = info.kv_resident_us;
      res->first_token_us = info.first_token_us;
      res->final_step_us = info.final_step_us;
      res->device_ttft_ms = info.device_ttft_ms;
      res->merge_point = r.merge_point;
      res->n_chunks = r.n_chunks;
      res->raced_chunk = info.raced_chunk;
      res->race_winner = info.race_winner;
      res->recomputed_last = info.recomputed_last ? 1 : 0;
      res->kernel_launches = info.kernel_launches;
      res->h2d_bytes = info.h2d_bytes;
      res->d2h_bytes = info.d2h_bytes;
      res->compute_busy_us = r.compute_busy_us;
      res->io_busy_us = r.io_busy_us;
    }
    export_report(r, nullptr, records);
  });
}

int cake_gpu_logits(const cake_gpu* g, float* out, int n) {
  return guarded([&] {
    const auto& v = g->ctx->last_run().logits;
    if (static_cast<std::size_t>(n) > v.size()) throw std::invalid_argument("logits: n exceeds vocab");
    std::memcpy(out, v.data(), static_cast<std::size_t>(n) * sizeof(float));
  });
}

int cake_gpu_read_chunk(const cake_gpu* g, uint64_t token_start, uint32_t token_count, uint8_t* out, uint64_t cap) {
  return guarded([&] {
    const auto v = g->ctx->read_chunk_kv(ChunkSpec{0, token_start, token_count});
    if (v.size() > cap) throw std::invalid_argument("read_chunk: buffer too small");
    std::memcpy(out, v.data(), v.size());
  });
}

int cake_gpu_kernel_stats(cake_gpu* g, cake_kernel_stat* out, int reset) {
  return guarded([&] {
    const int st = cake_model_kernel_stats(g->ctx->model(), out, reset);
    if (st != CAKE_OK) throw std::runtime_error("kernel stats failed");
  });
}

int cake_gpu_set_profiling(cake_gpu* g, int mask) {
  return guarded([&] {
    if (cake_model_set_profiling(g->ctx->model(), mask) != CAKE_OK) throw std::runtime_error("set profiling failed");
  });
}

int cake_gpu_set_profiling_stride(cake_gpu* g, int stride) {
  return guarded([&] {
    if (cake_model_set_profiling_stride(g->ctx->model(), stride) != CAKE_OK)
      throw std::invalid_argument("profiling stride must be >= 1");
  });
}

int cake_gpu_set_attention_impl(cake_gpu* g, int impl) {
  return guarded([&] {
    if (cake_model_set_attention_impl(g->ctx->model(), impl) != CAKE_OK) throw std::invalid_argument("bad impl");
  });
}

int cake_gpu_poison(cake_gpu* g, int byte) {
  return guarded([&] { g->ctx->poison(byte); });
}

int cake_gpu_slices(const cake_gpu* g, int64_t* at_us, uint64_t* cumulative_bits, uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    const auto& s = g->ctx->last_run().slices;
    if (n_out) *n_out = s.size();
    for (std::size_t i = 0; i < s.size() && i < cap; ++i) {
      if (at_us) at_us[i] = s[i].at_us;
      if (cumulative_bits) cumulative_bits[i] = s[i].cumulative_bits;
    }
  });
}

void* cake_gpu_model(cake_gpu* g) { return g->ctx->model(); }
void* cake_gpu_compute_stream(cake_gpu* g) { return g->ctx->compute_stream(); }

struct cake_tp {
  std::unique_ptr<TpCoordinator> c;
};
int cake_tp_create(const char* shm_name, int rank, int size, cake_tp** out) {
  return guarded([&] {
    if (!shm_name || !out) throw std::invalid_argument("tp: null argument");
    auto t = std::make_unique<cake_tp>();
    t->c = std::make_unique<TpCoordinator>(shm_name, rank, size);
    *out = t.release();
  });
}
int cake_tp_destroy(cake_tp* t) {
  delete t;
  return CAKE_OK;
}
int cake_tp_begin_run(cake_tp* t, uint64_t run_id, uint32_t n) { return guarded([&] { t->c->begin_run(run_id, n); }); }
int cake_tp_end_run(cake_tp* t) { return guarded([&] { t->c->end_run(); }); }
int cake_tp_publish_compute(cake_tp* t, uint32_t chunk) { return guarded([&] { t->c->publish_compute(chunk); }); }
int cake_tp_end_compute(cake_tp* t) { return guarded([&] { t->c->end_compute(); }); }
int cake_tp_next_compute(cake_tp* t, uint32_t k, uint32_t* chunk, int* has) {
  return guarded([&] {
    const auto v = t->c->next_compute(k);
    *has = v ? 1 : 0;
    *chunk = v.value_or(0);
  });
}
int cake_tp_publish_io(cake_tp* t, uint32_t chunk) { return guarded([&] { t->c->publish_io(chunk); }); }
int cake_tp_end_io(cake_tp* t) { return guarded([&] { t->c->end_io(); }); }
int cake_tp_next_io(cake_tp* t, uint32_t k, uint32_t* chunk, int* has) {
  return guarded([&] {
    const auto v = t->c->next_io(k);
    *has = v ? 1 : 0;
    *chunk = v.value_or(0);
  });
}
int cake_tp_shard_landed(cake_tp* t, uint32_t chunk) { return guarded([&] { t->c->shard_landed(chunk); }); }
int cake_tp_wait_all_landed(cake_tp* t, uint32_t chunk) { return guarded([&] { (void)t->c->wait_all_landed(chunk); }); }
int cake_tp_publish_decided(cake_tp* t, uint32_t chunk, int side) {
  return guarded([&] { t->c->publish_decided(chunk, side); });
}
int cake_tp_decided(cake_tp* t, uint32_t chunk, int* side) { return guarded([&] { *side = t->c->decided(chunk); }); }
int cake_tp_publish_final(cake_tp* t, int recompute, int last_row, int race_pages) {
  return guarded([&] { t->c->publish_final({recompute, last_row, race_pages}); });
}
int cake_tp_wait_final(cake_tp* t, int* recompute, int* last_row, int* race_pages) {
  return guarded([&] {
    const auto f = t->c->wait_final();
    *recompute = f.recompute;
    *last_row = f.last_row;
    *race_pages = f.race_pages;
  });
}
#endif  // CAKE_REFERENCE_BUILD

}  // extern "C"
