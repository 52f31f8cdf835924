// Chunk ownership between the forward compute worker and the reverse loader.
// Drop-in for reference proj/include/cake/claim.hpp (ClaimTable API and
// semantics identical; see proj/src/claim.cpp:14-47).
//
// B200 build: one 64-bit atomic word packs both pointers, so a claim is a
// single CAS (no mutex on the compute thread's per-chunk decision path) and
// the table can live in memory shared by several rank processes.
#pragma once

#include <atomic>
#include <cstdint>
#include <memory>
#include <optional>

#include "cake/time.hpp"

namespace cake {

enum class Side { compute, io };

const char* to_string(Side side);

struct ClaimRecord {
  Side side;
  Micros at_us;
};

// compute claims 0, 1, 2, ... ; io claims n-1, n-2, ... Each side may only
// claim the chunk its own pointer names, so the claimed set is a prefix plus
// a suffix and the one chunk both pointers can name goes to exactly one side.
class ClaimTable {
 public:
  explicit ClaimTable(std::uint32_t n_chunks);  // std::invalid_argument if 0

  // true: this side now owns `index` and its pointer moved. false: the
  // pointers have met (the other side owns it) — stop. std::logic_error if
  // `index` is not this side's current pointer.
  bool claim(Side side, std::uint32_t index, Micros now_us);

  std::optional<std::uint32_t> next_index(Side side) const;  // nullopt once crossed
  bool all_claimed() const;
  std::uint32_t n_chunks() const { return n_; }
  std::optional<ClaimRecord> record(std::uint32_t index) const;

  // Lowest io-owned index (n when io owns nothing): [0, merge) computed,
  // [merge, n) loaded.
  std::uint32_t merge_point() const;

 private:
  // state_ = compute_next | (io_next + 1) << 32
  static std::uint32_t lo(std::uint64_t s) { return static_cast<std::uint32_t>(s); }
  static std::int64_t io_ptr(std::uint64_t s) { return static_cast<std::int64_t>(s >> 32) - 1; }

  std::uint32_t n_;
  std::atomic<std::uint64_t> state_;
  // per chunk: 0 = free, else bit63 set | side << 62 | at_us
  std::unique_ptr<std::atomic<std::uint64_t>[]> slots_;
};

}  // namespace cake
