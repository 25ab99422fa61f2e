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

namespace memplan {

// B200 extension: host-memory bandwidth shared by the host optimizer and the
// PCIe copies (opt-in; `memplan simulate|plan|validate --host-mem-bw B`).
// The reference's simulator gives the host Adam its own rate and the h2d/d2h
// links their own bandwidth (proj/src/sim.cpp:25-81,552-562); on a real host
// all three stream through the same DRAM. With bw > 0 every consumer that is
// active at a moment demands its nominal rate -- the host Adam
// cpu_bytes_per_param * cpu_optim_rate, an active h2d link h2d_bw, an active
// d2h link d2h_bw -- and when the sum exceeds bw all of them are slowed by the
// same factor bw / demand. bw == 0 (the default) is the reference model.
struct HostMemoryModel {
  double bw = 0.0;                  // bytes/s; 0 = off
  double cpu_bytes_per_param = 28;  // host Adam: fp32 master/m/v read+write, bf16 grad in, param out
};

const HostMemoryModel& host_memory_model();

class ScopedHostMemoryModel {
 public:
  explicit ScopedHostMemoryModel(double bw, double cpu_bytes_per_param = 28.0);
  ~ScopedHostMemoryModel();
  ScopedHostMemoryModel(const ScopedHostMemoryModel&) = delete;
  ScopedHostMemoryModel& operator=(const ScopedHostMemoryModel&) = delete;
};

}  // namespace memplan
