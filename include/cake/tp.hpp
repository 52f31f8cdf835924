// Cross-process coordination of one head-sharded tensor-parallel group
// (one process per GPU, all on one node) during a bidirectional run.
//
// The reference is single-process (no parallelism); this is the
// B200 build's §8(e) design: ONE scheduler. Rank 0 (the leader) runs the
// ClaimTable / TransferEngine / ComputeEngine exactly as on one GPU and
// publishes every decision; followers mirror them:
//   compute sequence  chunks in launch order -> every rank enqueues the same
//                     chunks, so the per-layer NCCL all-reduces line up;
//   io sequence       chunks the leader's loader claimed -> every rank loads
//                     its own KV-head shard of them (its own emulated link);
//   shard landed      per-chunk counters: a chunk is io-committed only when
//                     every rank's shard is in HBM;
//   final step        recompute flag / tail row of the first-token step, and
//                     whether the contested chunk's pages are the spare set;
//   race-to-finish    the racer's entry carries kRaceBit (followers write that
//                     chunk through their own spare page set); every commit is
//                     published (decided), so followers abort the losing
//                     side's work on the contested chunk the same way.
// State lives in a POSIX shared-memory segment of lock-free atomics.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <utility>

namespace cake {

class TpCoordinator {
 public:
  static constexpr int kMaxChunks = 8192;

  // Rank 0 creates (and zeroes) the segment, the others open it (retrying
  // until it exists). `name` is a POSIX shm name ("/cake_tp_<job>").
  TpCoordinator(const std::string& name, int rank, int size);
  ~TpCoordinator();
  TpCoordinator(const TpCoordinator&) = delete;
  TpCoordinator& operator=(const TpCoordinator&) = delete;

  int rank() const { return rank_; }
  int size() const { return size_; }
  bool leader() const { return rank_ == 0; }

  // Run framing: the leader resets the per-run state once every follower has
  // finished the previous run, then opens run `run_id`; followers block until
  // that run is open.
  void begin_run(std::uint64_t run_id, std::uint32_t n_chunks);
  void end_run();

  // Leader publishes, followers consume entry k (blocking; nullopt = sequence ended).
  // Entries are chunk indices, or'ed with kRaceBit for the racer's entry of the
  // contested chunk.
  static constexpr std::uint32_t kRaceBit = 1u << 30;
  void publish_compute(std::uint32_t chunk);
  void end_compute();
  std::optional<std::uint32_t> next_compute(std::uint32_t k);
  void publish_io(std::uint32_t chunk);
  void end_io();
  std::optional<std::uint32_t> next_io(std::uint32_t k);

  // Every rank reports its shard of `chunk` landed; the leader waits for all
  // (false: the compute side committed the chunk first, the loads were dropped).
  void shard_landed(std::uint32_t chunk);
  bool wait_all_landed(std::uint32_t chunk);

  // Commit decisions (side 1 = compute, 2 = io); 0 = undecided.
  void publish_decided(std::uint32_t chunk, int side);
  int decided(std::uint32_t chunk) const;
  struct Final {
    int recompute = 0, last_row = 0;
    int race_pages = -1;  // contested chunk whose winner wrote the spare page set, or -1
    int race_chunk = -1, race_winner = -1;  // the run's contest (0 compute, 1 io won), for the report
  };
  void publish_final(const Final& f);
  Final wait_final();
  bool final_published() const;

 private:
  struct Shared;
  Shared* sh_ = nullptr;
  std::string name_;
  int rank_, size_;
};

}  // namespace cake
