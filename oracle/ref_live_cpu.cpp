// TEST INFRASTRUCTURE (the CPU baseline of bench.py / tests): the REFERENCE's
// own live bidirectional run — its claim table, throttled loader, store and
// scheduler, compiled from /root/reference/proj/src (oracle/Makefile) — with
// the compute side's modeled sleep (proj/src/compute.cpp:48-49) replaced by a
// real CPU forward of each claimed chunk (oracle/llama_ref.c, fp32, OpenMP).
// Nothing here is extrapolated: one request of BASELINE config 1 (tiny
// 2-layer d=256 transformer, 2K prompt, 256-token chunks, cached prefix on a
// file tier behind a throttled link) is served end to end on the host cores,
// then its first token is produced:
//   * the cache tier is the oracle's own KV of the prompt, written in the
//     reference's store format under the reference's chain keys;
//   * run(..., ClockMode::live) (proj/src/scheduler.cpp:229-278) races the
//     forward against the loader; its TTFT is the reference's (last chunk
//     resident);
//   * the first token: the final norm + LM head of the last computed row when
//     compute produced the tail, else the loaded chunks are installed (the
//     tier's bytes) and the last token is recomputed over the cache.
//
//   ref_live_cpu <tokens> <chunk> <mbps> <threads> <store-dir> [mode: cake|compute_only|io_only]
// prints one JSON object.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "cake/compute.hpp"
#include "cake/scheduler.hpp"
#include "cake/store.hpp"
#include "llama_ref.h"

namespace {
// the forward the live loop runs for a claimed chunk (set by main)
std::function<void(const cake::ChunkSpec&)> g_forward;
}  // namespace

namespace cake {

// proj/src/compute.cpp:8-25, restated (the live loop below does not use the step law).
ComputeEngine::ComputeEngine(CostModel model, TokenBudget budget) : model_(model), budget_(budget) {
  model_.validate();
  if (budget_.budget_per_step < 1) throw std::invalid_argument("compute engine: token budget must be >= 1");
  if (!(budget_.share_for_request > 0.0) || budget_.share_for_request > 1.0)
    throw std::invalid_argument("compute engine: share_for_request must be in (0, 1]");
}

PrefillStep ComputeEngine::prefill_chunk(const ChunkSpec& chunk, Micros start_us) {
  if (chunk.index != next_index_) throw std::logic_error("prefill_chunk: prefix dependency violated");
  if (chunk.token_count > budget_.budget_per_step) throw std::invalid_argument("prefill_chunk: chunk exceeds budget");
  ++next_index_;
  const Micros dur = compute_latency(model_, chunk, budget_.share_for_request);
  return {chunk, budget_.share_for_request, start_us, start_us + dur};
}

// proj/src/compute.cpp:27-55: residency probe, claim, then the chunk — the
// sleep of its modeled latency replaced by the real CPU forward.
std::vector<ChunkRecord> ComputeEngine::run_forward(std::span<const ChunkSpec> chunks, std::span<const ChunkKey> keys,
                                                    const ForwardHooks& hooks) {
  if (!hooks.table || !hooks.timer) throw std::invalid_argument("run_forward: missing table/timer");
  std::mt19937_64 jitter_rng(hooks.jitter_seed ^ 0xA24BAED4963EE407ULL);
  std::vector<ChunkRecord> records;
  for (const auto& chunk : chunks) {
    if (hooks.jitter_max_us > 0)
      hooks.timer->sleep_for_us(static_cast<Micros>(jitter_rng() % (hooks.jitter_max_us + 1)));
    if (hooks.probe && !keys.empty() && hooks.probe->is_resident(keys[chunk.index])) {
      if (hooks.signal_stop) hooks.signal_stop();
      break;
    }
    if (!hooks.table->claim(Side::compute, chunk.index, hooks.timer->now_us())) {
      if (hooks.signal_stop) hooks.signal_stop();
      break;
    }
    const Micros start = hooks.timer->now_us();
    g_forward(chunk);
    records.push_back({chunk.index, Side::compute, start, hooks.timer->now_us(), 0});
    ++next_index_;
  }
  if (hooks.signal_stop) hooks.signal_stop();
  return records;
}

}  // namespace cake

int main(int argc, char** argv) {
  using namespace cake;
  if (argc < 6) {
    std::fprintf(stderr, "usage: %s tokens chunk mbps threads store-dir [mode]\n", argv[0]);
    return 2;
  }
  const std::uint64_t T = std::stoull(argv[1]);
  const std::uint32_t C = static_cast<std::uint32_t>(std::stoul(argv[2]));
  const double mbps = std::stod(argv[3]);
  const int threads = std::stoi(argv[4]);
  const std::filesystem::path dir = argv[5];
  const std::string mode_s = argc > 6 ? argv[6] : "cake";
  const RunMode mode = mode_s == "io_only" ? RunMode::io_only : mode_s == "compute_only" ? RunMode::compute_only
                                                                                          : RunMode::cake;
  const std::uint64_t seed = 42;
  // BASELINE config 1: 2 layers, d = 256, 4 heads (head_dim 64), the "tiny" preset of the GPU runtime
  ref_config cfg{2, 256, 4, 4, 64, 1024, 32000, 500000.0f, 1e-5f, 1234ull, threads};
  const int L = cfg.n_layers, nkv = cfg.n_kv_heads, hd = cfg.head_dim;
  ModelProfile profile{"tiny", static_cast<std::uint32_t>(L), static_cast<std::uint32_t>(nkv * hd), 2, 2, {}};
  RequestSpec request;
  request.total_tokens = T;
  request.chunk_size = C;
  const auto chunks = split_into_chunks(T, C);
  const auto ids = token_stream(seed, T);
  std::vector<int32_t> toks(ids.begin(), ids.end());

  // ---- the cache tier: the oracle's KV of the whole prompt, reference store format
  ref_model* m = ref_create(&cfg, static_cast<long long>(T), 0);
  std::filesystem::remove_all(dir);
  ChunkStore store = ChunkStore::create(dir);
  {
    std::optional<ChunkKey> prev;
    for (const ChunkSpec& c : chunks) {
      ref_begin_chunk(m, toks.data() + c.token_start, static_cast<long long>(c.token_start),
                      static_cast<int>(c.token_count));
      ref_run_layers(m, 0, L);
      const ChunkKey key = chain_hash(prev, std::span<const std::uint32_t>(ids.data() + c.token_start, c.token_count));
      prev = key;
      // [layer][K|V][kv_head][token][head_dim] bf16 of this chunk
      std::vector<std::uint16_t> tier(static_cast<size_t>(L) * 2 * nkv * c.token_count * hd);
      const float* kv = ref_kv(m);
      const long long P = ref_max_tokens(m);
      size_t o = 0;
      for (int l = 0; l < L; ++l)
        for (int k = 0; k < 2; ++k)
          for (int h = 0; h < nkv; ++h)
            for (std::uint32_t t = 0; t < c.token_count; ++t)
              for (int d = 0; d < hd; ++d)
                tier[o++] = ref_bf16_from_float(
                    kv[((((static_cast<size_t>(l) * 2 + k) * nkv + h) * P) + c.token_start + t) * hd + d]);
      const auto bytes = std::as_bytes(std::span<const std::uint16_t>(tier));
      store.put(key, bytes, ChunkMeta{c.token_count, "identity", bytes.size(), bytes.size()});
    }
  }
  ref_destroy(m);

  // ---- the live run: a fresh oracle whose cache only holds what the run produces
  m = ref_create(&cfg, static_cast<long long>(T), 0);
  int last_computed = -1;
  g_forward = [&](const ChunkSpec& c) {
    ref_begin_chunk(m, toks.data() + c.token_start, static_cast<long long>(c.token_start),
                    static_cast<int>(c.token_count));
    ref_run_layers(m, 0, L);
    last_computed = static_cast<int>(c.index);
  };
  // modeled cost: only its validation is used on the live path (the forward is real)
  const CostModel cost{1.0, 0.0, C};
  RunOptions opt;
  opt.token_budget = C;
  opt.throttle_quantum_bytes = 64 << 10;
  const auto t0 = std::chrono::steady_clock::now();
  const RunReport rep =
      run(request, profile, cost, BandwidthTrace::constant(mbps), Codec::identity(), mode, ClockMode::live, store, seed, opt);
  // ---- first token
  std::vector<float> logits(static_cast<size_t>(cfg.vocab));
  const std::uint32_t n = static_cast<std::uint32_t>(chunks.size());
  bool recompute = last_computed != static_cast<int>(n - 1);
  if (recompute) {
    for (const ChunkRecord& r : rep.chunks) {
      if (r.side != Side::io) continue;
      const ChunkSpec& c = chunks[r.index];
      std::optional<ChunkKey> prev;
      ChunkKey key{};
      for (std::uint32_t i = 0; i <= r.index; ++i) {
        key = chain_hash(prev, std::span<const std::uint32_t>(ids.data() + chunks[i].token_start, chunks[i].token_count));
        prev = key;
      }
      const auto payload = store.get(key);
      ref_load_chunk(m, reinterpret_cast<const std::uint16_t*>(payload.data()), static_cast<long long>(c.token_start),
                     static_cast<int>(c.token_count));
    }
    ref_last_token_logits(m, toks[T - 1], static_cast<long long>(T), logits.data());
  } else {
    ref_final_logits(m, static_cast<int>(chunks.back().token_count) - 1, logits.data());
  }
  const double first_token_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  int top = 0;
  for (int v = 1; v < cfg.vocab; ++v)
    if (logits[v] > logits[top]) top = v;
  std::uint32_t computed = 0;
  for (const ChunkRecord& r : rep.chunks) computed += r.side == Side::compute ? 1u : 0u;
  std::printf("{\"mode\": \"%s\", \"tokens\": %llu, \"chunk\": %u, \"mbps\": %g, \"threads\": %d, "
              "\"ttft_ms\": %.3f, \"first_token_ms\": %.3f, \"merge_point\": %u, \"computed_chunks\": %u, "
              "\"n_chunks\": %u, \"chunks_reported\": %zu, \"recomputed_last\": %s, \"top1\": %d, \"logit_top1\": %.6f}\n",
              mode_s.c_str(), static_cast<unsigned long long>(T), C, mbps, threads, rep.ttft_us / 1e3, first_token_ms,
              rep.merge_point, computed, n, rep.chunks.size(), recompute ? "true" : "false", top, logits[top]);
  ref_destroy(m);
  std::filesystem::remove_all(dir);
  return 0;
}
