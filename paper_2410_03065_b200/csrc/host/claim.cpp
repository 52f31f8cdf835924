// Lock-free ClaimTable (semantics of reference proj/src/claim.cpp:9-47).
#include "cake/claim.hpp"

#include <stdexcept>

namespace cake {

namespace {
constexpr std::uint64_t kTaken = 1ull << 63;
constexpr std::uint64_t kIoBit = 1ull << 62;
constexpr std::uint64_t kTimeMask = kIoBit - 1;
}  // namespace

const char* to_string(Side side) { return side == Side::io ? "io" : "compute"; }

ClaimTable::ClaimTable(std::uint32_t n_chunks) : n_(n_chunks), state_(0) {
  if (n_chunks == 0) throw std::invalid_argument("claim table: need at least one chunk");
  state_.store(static_cast<std::uint64_t>(n_chunks) << 32, std::memory_order_relaxed);  // io_next = n - 1
  slots_ = std::make_unique<std::atomic<std::uint64_t>[]>(n_chunks);
  for (std::uint32_t i = 0; i < n_chunks; ++i) slots_[i].store(0, std::memory_order_relaxed);
}

bool ClaimTable::claim(Side side, std::uint32_t index, Micros now_us) {
  std::uint64_t s = state_.load(std::memory_order_acquire);
  for (;;) {
    const std::int64_t c = lo(s);
    const std::int64_t io = io_ptr(s);
    const std::int64_t mine = side == Side::compute ? c : io;
    if (static_cast<std::int64_t>(index) != mine)
      throw std::logic_error("claim: side attempted non-adjacent index");
    if (c > io) return false;  // pointers met: the other side holds this chunk
    const std::uint64_t next = side == Side::compute ? s + 1 : s - (1ull << 32);
    if (state_.compare_exchange_weak(s, next, std::memory_order_acq_rel, std::memory_order_acquire)) {
      const std::uint64_t t = static_cast<std::uint64_t>(now_us < 0 ? 0 : now_us) & kTimeMask;
      slots_[index].store(kTaken | (side == Side::io ? kIoBit : 0) | t, std::memory_order_release);
      return true;
    }
  }
}

std::optional<std::uint32_t> ClaimTable::next_index(Side side) const {
  const std::uint64_t s = state_.load(std::memory_order_acquire);
  const std::int64_t c = lo(s), io = io_ptr(s);
  if (c > io) return std::nullopt;
  return static_cast<std::uint32_t>(side == Side::compute ? c : io);
}

bool ClaimTable::all_claimed() const {
  const std::uint64_t s = state_.load(std::memory_order_acquire);
  return static_cast<std::int64_t>(lo(s)) > io_ptr(s);
}

std::optional<ClaimRecord> ClaimTable::record(std::uint32_t index) const {
  if (index >= n_) throw std::out_of_range("claim table: index out of range");
  // Taken-ness comes from the pointer word (the linearization point of a
  // claim); the slot is stored right after the CAS, so a reader that sees the
  // pointer past `index` waits out that window instead of reporting "free".
  const std::uint64_t s = state_.load(std::memory_order_acquire);
  if (!(index < lo(s) || static_cast<std::int64_t>(index) > io_ptr(s))) return std::nullopt;
  std::uint64_t v;
  while (!((v = slots_[index].load(std::memory_order_acquire)) & kTaken)) {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
  }
  return ClaimRecord{(v & kIoBit) ? Side::io : Side::compute, static_cast<Micros>(v & kTimeMask)};
}

std::uint32_t ClaimTable::merge_point() const {
  return static_cast<std::uint32_t>(io_ptr(state_.load(std::memory_order_acquire)) + 1);
}

}  // namespace cake
