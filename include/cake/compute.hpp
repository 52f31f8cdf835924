// The forward-order chunked-prefill worker.
// Drop-in for reference proj/include/cake/compute.hpp: TokenBudget,
// PrefillStep, ComputeEngine::{prefill_chunk, run_forward, ForwardHooks}.
//
// Reference behaviour (kept for the virtual clock and modeled runs): a chunk
// "computes" by sleeping compute_latency() (proj/src/compute.cpp:48-49).
// B200: ForwardHooks::backend plugs in the real GPU prefill — each claimed
// chunk is enqueued on the compute stream (32 layers of tcgen05 GEMMs +
// paged attention) and its record carries CUDA-event timestamps.
#pragma once

#include <cstdint>
#include <functional>
#include <span>
#include <vector>

#include "cake/claim.hpp"
#include "cake/model.hpp"
#include "cake/report.hpp"
#include "cake/store.hpp"
#include "cake/transfer.hpp"

namespace cake {

struct TokenBudget {
  std::uint32_t budget_per_step = 512;  // caps the chunk size
  double share_for_request = 1.0;       // effective power fraction
};

struct PrefillStep {
  ChunkSpec chunk;
  double power_fraction = 1.0;
  Micros started_at_us = 0;
  Micros finished_at_us = 0;
};

// Device-side chunk prefill used by run_forward (implemented by the GPU
// runtime, include/cake/gpu.hpp). Called from the compute (caller) thread.
class PrefillBackend {
 public:
  virtual ~PrefillBackend() = default;
  // Returns when the device is about to need its next chunk; the claim for
  // that chunk is made right after, so it reflects the real frontier.
  virtual void pace() = 0;
  // Enqueue the chunk (asynchronous). contested: the io side owns it and the
  // compute side is racing it into a second page set.
  virtual void launch(const ChunkSpec& chunk, bool contested) = 0;
  // Predicted completion (run clock) of `chunk` if launched next.
  virtual Micros predict_finish(const ChunkSpec& chunk) = 0;
  // Wait for every launched chunk; records of the chunks the compute side
  // committed (a contested chunk it lost is omitted).
  virtual std::vector<ChunkRecord> drain() = 0;
};

class ComputeEngine {
 public:
  ComputeEngine(CostModel model, TokenBudget budget);

  // Virtual-clock step: [start, start + compute_latency). Chunks must come in
  // index order (std::logic_error otherwise) and fit the token budget.
  PrefillStep prefill_chunk(const ChunkSpec& chunk, Micros start_us);

  void reset() { next_index_ = 0; }

  const CostModel& model() const { return model_; }
  const TokenBudget& budget() const { return budget_; }

  struct ForwardHooks {
    ClaimTable* table = nullptr;         // required
    const ResidentSet* probe = nullptr;  // optional residency check before each claim
    std::function<void()> signal_stop;   // tells the loader to wind down
    const RunTimer* timer = nullptr;     // required
    std::uint32_t jitter_max_us = 0;
    std::uint64_t jitter_seed = 0;
    // ---- B200 extensions
    PrefillBackend* backend = nullptr;   // real GPU prefill instead of the modeled sleep
    // Race-to-finish policy for a chunk the io side owns: (chunk, predicted
    // compute finish) -> compute it anyway into the second page set?
    std::function<bool(const ChunkSpec&, Micros)> contest;
  };

  // Walks chunks from index 0: residency probe, claim, work, record; stops at
  // the first chunk the loader owns (or, racing, right after contesting it).
  std::vector<ChunkRecord> run_forward(std::span<const ChunkSpec> chunks, std::span<const ChunkKey> keys,
                                       const ForwardHooks& hooks);

 private:
  CostModel model_;
  TokenBudget budget_;
  std::uint32_t next_index_ = 0;
};

}  // namespace cake
