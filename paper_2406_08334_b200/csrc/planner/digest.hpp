// Internal to the planner: per-(trace, layout) and per-schedule invariants
// of the cost model, computed once and shared by the public estimate_* entry
// points and the search's hot loop. Every value is produced with exactly the
// operation order of the reference cost model (proj/src/cost.cpp:24-66), so a
// cost evaluated from the digest is bit-identical to one evaluated directly.
#pragma once

#include <cstdint>
#include <vector>

#include "memplan/cost.hpp"
#include "memplan/hardware.hpp"
#include "memplan/layout.hpp"
#include "memplan/trace.hpp"

namespace memplan::detail {

struct Window {
  double begin = 0;
  double end = 0;
  bool overlaps(const Window& o) const { return begin < o.end && o.begin < end; }
};

struct TraceDigest {
  int n_chunk = 0;
  int n_block = 0;
  std::vector<double> comp_fwd;        // [1..n_chunk], chunk span sums of t_fwd
  std::vector<double> comp_bwd;        // [1..n_chunk]
  std::vector<double> cum_fwd;         // [0..n_chunk], prefix of comp_fwd
  std::vector<double> rev_bwd;         // [1..n_chunk+1], suffix of comp_bwd
  std::vector<std::int64_t> chunk_bytes;  // [1..n_chunk]
  std::vector<double> block_fwd_end;   // per block, on the pure forward timeline
  std::vector<double> block_bwd_start; // per block, on the pure backward timeline
  std::vector<std::int64_t> block_act; // per block retained activation bytes
  std::vector<double> block_fwd;       // per block forward seconds (recompute cost)
  std::vector<std::vector<int>> chunk_blocks;  // [1..n_chunk]

  TraceDigest(const ModelTrace& trace, const ChunkLayout& layout);
};

// Per (schedule, hardware): contention of each prefetch window and the
// recompute charge of each chunk.
struct ScheduleDigest {
  std::vector<char> fwd_contended;  // [1..n_chunk]: stage-s prefetch overlaps a swap-out
  std::vector<char> bwd_contended;  // [1..n_chunk]: chunk-c backward prefetch overlaps a swap-in
  std::vector<double> recomp;       // [1..n_chunk]

  // `fwd` / `bwd` select which half is needed: the forward half reads only
  // the D2H bandwidth (swap-outs), the backward half only H2D (swap-ins),
  // exactly like the reference's estimate_fwd / estimate_bwd.
  ScheduleDigest(const TraceDigest& d, const BlockSchedule& schedule, const HardwareProfile& hw,
                 bool fwd = true, bool bwd = true);
};

// Per (layout, hardware): the prefetch / drain terms of every chunk.
struct LinkDigest {
  std::vector<double> pf_plain;  // gather + upload at full H2D
  std::vector<double> pf_half;   // gather + upload at contended (half) H2D
  std::vector<double> reduce;    // reduce only (persistent chunk drain)
  std::vector<double> drain;     // reduce + offload (non-persistent chunk drain)
  bool upload_ok = true;         // H2D bandwidth valid (else a needed upload throws)
  bool offload_ok = true;        // D2H bandwidth valid

  LinkDigest(const TraceDigest& d, const HardwareProfile& hw);
};

double fwd_time(const TraceDigest& d, const ScheduleDigest& s, const LinkDigest& l,
                int n_persist, std::vector<StageTerm>* stages);
double bwd_time(const TraceDigest& d, const ScheduleDigest& s, const LinkDigest& l,
                int n_persist, int n_buffer, std::vector<StageTerm>* stages);

// Activation replay peak of the backward pass for a schedule (Eq.8-11
// without model states and alpha).
std::int64_t replay_peak(const ModelTrace& trace, const BlockSchedule& schedule, int n_swap,
                         int n_checkpoint);

// The feasible candidates in enumerate_candidates order (what
// `validate` samples from), with each peak taken from the cached replay of
// the candidate stream instead of a fresh estimate_peak_memory per config.
std::vector<PlanConfig> feasible_candidates(const ChunkLayout& layout, const ModelTrace& trace,
                                            const HardwareProfile& hw, const CostOptions& opts);

}  // namespace memplan::detail
