// memplan — B200 extension: how model-state bytes of chunks are charged.
//
// The reference charges every persistent chunk 8 x s_chunk device bytes and
// every buffer s_chunk bytes (proj/src/cost.cpp:10, proj/include/memplan/
// cost.hpp:17-21), and every offloaded chunk 8 x s_chunk host bytes
// (proj/src/search.cpp:135-145), whatever the chunk actually holds. That is
// the default here too (byte-identical plans). The B200 runtime allocates a
// chunk's state for its USED bytes (16 B per parameter: bf16 param + grad,
// fp32 master/m/v) and sizes buffer slots for the largest non-persistent
// chunk, so when chunks are far from full (llama-13b: 634 MB of every 1 GiB
// chunk) the reference accounting leaves a third of the 180 GB of HBM unused.
// `ScopedUsedBytesAccounting` switches the state terms of the peak-memory
// model, the search's feasibility test and the simulator's ledger to the
// physical bytes of a given layout for its lifetime (opt-in:
// `memplan plan --chunk-bytes used`).
#pragma once

#include <cstdint>
#include <vector>

#include "memplan/layout.hpp"

namespace memplan {

// Device bytes of the model states of `c`: n_persist persistent chunks plus
// n_buffer buffers (reference: 8*s_chunk*np + s_chunk*nb).
std::int64_t device_state_bytes(const PlanConfig& c);
// Host bytes of the offloaded chunks (reference: 8*s_chunk*(N - np)).
std::int64_t host_state_bytes(const PlanConfig& c);

bool used_bytes_accounting();

// While alive (one at a time; set before any concurrent search), state bytes
// are charged from `layout`'s used bytes: persistent chunk c = 8*used_c,
// buffer = max used_c over the non-persistent chunks, offloaded chunk c =
// 8*used_c. Throws InvariantViolation when a config's n_chunk differs from
// the layout's.
class ScopedUsedBytesAccounting {
 public:
  explicit ScopedUsedBytesAccounting(const ChunkLayout& layout);
  ~ScopedUsedBytesAccounting();
  ScopedUsedBytesAccounting(const ScopedUsedBytesAccounting&) = delete;
  ScopedUsedBytesAccounting& operator=(const ScopedUsedBytesAccounting&) = delete;
};

}  // namespace memplan
