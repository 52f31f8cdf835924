// Shared-memory protocol of a TP group's run (include/cake/tp.hpp).
#include "cake/tp.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <thread>

namespace cake {

struct TpCoordinator::Shared {
  std::atomic<std::uint64_t> run_id;
  std::atomic<std::uint32_t> n_chunks;
  std::atomic<std::int32_t> followers_ready;
  std::atomic<std::int32_t> followers_done;
  std::atomic<std::int32_t> compute_count, compute_end;
  std::atomic<std::int32_t> io_count, io_end;
  std::atomic<std::int32_t> final_set;
  std::atomic<std::int32_t> final_recompute, final_last_row, final_race_pages, final_race_chunk, final_race_winner;
  std::atomic<std::int32_t> compute_seq[kMaxChunks];
  std::atomic<std::int32_t> io_seq[kMaxChunks];
  std::atomic<std::int32_t> landed[kMaxChunks];
  std::atomic<std::int32_t> decided[kMaxChunks];
};

namespace {
static_assert(std::atomic<std::int32_t>::is_always_lock_free && std::atomic<std::uint64_t>::is_always_lock_free,
              "shared-memory atomics must be lock-free");

template <typename Pred>
void spin_until(Pred p) {
  int spins = 0;
  while (!p()) {
    if (++spins < 256) continue;
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}
}  // namespace

TpCoordinator::TpCoordinator(const std::string& name, int rank, int size) : name_(name), rank_(rank), size_(size) {
  if (size < 1 || rank < 0 || rank >= size) throw std::invalid_argument("tp: bad rank/size");
  const std::size_t bytes = sizeof(Shared);
  int fd = -1;
  if (rank == 0) {
    shm_unlink(name.c_str());
    fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) throw std::runtime_error("tp: shm_open(create) failed for " + name);
    if (ftruncate(fd, static_cast<off_t>(bytes)) != 0) throw std::runtime_error("tp: ftruncate failed");
  } else {
    for (int attempt = 0; attempt < 60000 && fd < 0; ++attempt) {  // up to ~60 s for the leader
      fd = shm_open(name.c_str(), O_RDWR, 0600);
      if (fd < 0) std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    if (fd < 0) throw std::runtime_error("tp: shm segment " + name + " never appeared");
    for (int attempt = 0; attempt < 60000; ++attempt) {  // leader may not have sized it yet
      off_t end = lseek(fd, 0, SEEK_END);
      if (end >= static_cast<off_t>(bytes)) break;
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
  }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) throw std::runtime_error("tp: mmap failed");
  sh_ = static_cast<Shared*>(p);
  if (rank == 0) {
    // fresh segment is zero-filled by ftruncate; make the atomics' state explicit
    sh_->run_id.store(0);
    sh_->followers_done.store(size - 1);  // "previous run" finished by everyone
  }
}

TpCoordinator::~TpCoordinator() {
  if (sh_) munmap(sh_, sizeof(Shared));
  if (rank_ == 0) shm_unlink(name_.c_str());
}

void TpCoordinator::begin_run(std::uint64_t run_id, std::uint32_t n_chunks) {
  if (n_chunks > static_cast<std::uint32_t>(kMaxChunks)) throw std::invalid_argument("tp: too many chunks");
  if (leader()) {
    spin_until([&] { return sh_->followers_done.load(std::memory_order_acquire) >= size_ - 1; });
    sh_->followers_done.store(0);
    sh_->followers_ready.store(0);
    sh_->compute_count.store(0);
    sh_->compute_end.store(0);
    sh_->io_count.store(0);
    sh_->io_end.store(0);
    sh_->final_set.store(0);
    for (std::uint32_t i = 0; i < n_chunks; ++i) {
      sh_->landed[i].store(0, std::memory_order_relaxed);
      sh_->decided[i].store(0, std::memory_order_relaxed);
    }
    sh_->n_chunks.store(n_chunks);
    sh_->run_id.store(run_id, std::memory_order_release);
    spin_until([&] { return sh_->followers_ready.load(std::memory_order_acquire) >= size_ - 1; });
  } else {
    spin_until([&] { return sh_->run_id.load(std::memory_order_acquire) == run_id; });
    if (sh_->n_chunks.load() != n_chunks) throw std::logic_error("tp: ranks disagree on the chunk count");
    sh_->followers_ready.fetch_add(1, std::memory_order_acq_rel);
  }
}

void TpCoordinator::end_run() {
  if (!leader()) sh_->followers_done.fetch_add(1, std::memory_order_acq_rel);
}

void TpCoordinator::publish_compute(std::uint32_t chunk) {
  const int k = sh_->compute_count.load(std::memory_order_relaxed);
  sh_->compute_seq[k].store(static_cast<std::int32_t>(chunk), std::memory_order_relaxed);
  sh_->compute_count.store(k + 1, std::memory_order_release);
}
void TpCoordinator::end_compute() { sh_->compute_end.store(1, std::memory_order_release); }

std::optional<std::uint32_t> TpCoordinator::next_compute(std::uint32_t k) {
  std::optional<std::uint32_t> out;
  spin_until([&] {
    if (sh_->compute_count.load(std::memory_order_acquire) > static_cast<std::int32_t>(k)) {
      out = static_cast<std::uint32_t>(sh_->compute_seq[k].load(std::memory_order_relaxed));
      return true;
    }
    // end is published after the last entry: re-check the count after seeing it
    return sh_->compute_end.load(std::memory_order_acquire) != 0 &&
           sh_->compute_count.load(std::memory_order_acquire) <= static_cast<std::int32_t>(k);
  });
  return out;
}

void TpCoordinator::publish_io(std::uint32_t chunk) {
  const int k = sh_->io_count.load(std::memory_order_relaxed);
  sh_->io_seq[k].store(static_cast<std::int32_t>(chunk), std::memory_order_relaxed);
  sh_->io_count.store(k + 1, std::memory_order_release);
}
void TpCoordinator::end_io() { sh_->io_end.store(1, std::memory_order_release); }

std::optional<std::uint32_t> TpCoordinator::next_io(std::uint32_t k) {
  std::optional<std::uint32_t> out;
  spin_until([&] {
    if (sh_->io_count.load(std::memory_order_acquire) > static_cast<std::int32_t>(k)) {
      out = static_cast<std::uint32_t>(sh_->io_seq[k].load(std::memory_order_relaxed));
      return true;
    }
    return sh_->io_end.load(std::memory_order_acquire) != 0 &&
           sh_->io_count.load(std::memory_order_acquire) <= static_cast<std::int32_t>(k);
  });
  return out;
}

void TpCoordinator::shard_landed(std::uint32_t chunk) { sh_->landed[chunk].fetch_add(1, std::memory_order_acq_rel); }

bool TpCoordinator::wait_all_landed(std::uint32_t chunk) {
  bool all = false;
  spin_until([&] {
    all = sh_->landed[chunk].load(std::memory_order_acquire) >= size_;
    return all || sh_->decided[chunk].load(std::memory_order_acquire) == 1;
  });
  return all;
}

void TpCoordinator::publish_decided(std::uint32_t chunk, int side) {
  sh_->decided[chunk].store(side, std::memory_order_release);
}

int TpCoordinator::decided(std::uint32_t chunk) const { return sh_->decided[chunk].load(std::memory_order_acquire); }

void TpCoordinator::publish_final(const Final& f) {
  sh_->final_recompute.store(f.recompute, std::memory_order_relaxed);
  sh_->final_last_row.store(f.last_row, std::memory_order_relaxed);
  sh_->final_race_pages.store(f.race_pages, std::memory_order_relaxed);
  sh_->final_race_chunk.store(f.race_chunk, std::memory_order_relaxed);
  sh_->final_race_winner.store(f.race_winner, std::memory_order_relaxed);
  sh_->final_set.store(1, std::memory_order_release);
}

bool TpCoordinator::final_published() const { return sh_->final_set.load(std::memory_order_acquire) != 0; }

TpCoordinator::Final TpCoordinator::wait_final() {
  spin_until([&] { return sh_->final_set.load(std::memory_order_acquire) != 0; });
  return {sh_->final_recompute.load(), sh_->final_last_row.load(), sh_->final_race_pages.load(),
          sh_->final_race_chunk.load(), sh_->final_race_winner.load()};
}

}  // namespace cake
