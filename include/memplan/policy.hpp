// memplan — B200 extension: THE chunk-runtime policy, one implementation.
//
// The reference states its runtime policy only inside the simulator
// (proj/src/sim.cpp:99-562). Here the decisions live in two small state
// machines that every driver shares:
//
//   * ChunkBufferPool — where each chunk is (away / arriving / resident /
//     draining), which of the n_buffer device slots it occupies, the fetch
//     queue with ONE fetch in flight, and the eviction rule (the idle
//     resident non-persistent chunk whose next use is farthest, strictly
//     later than the incoming chunk's, never a pinned chunk; lower id on
//     ties) — proj/src/sim.cpp:275-343,427-451;
//   * IterationCore — the ordered job list of one iteration (forward ops,
//     backward ops with each checkpointed block's recompute before its last
//     op, one device optimizer job per persistent chunk), job readiness, the
//     device-memory ledger, the drain trigger after a chunk's last backward
//     job, and the activation swap chains / swap-in release rule —
//     proj/src/sim.cpp:203-273,345-425,453-550.
//
// Drivers: `simulate` (modelled time, csrc/planner/simulator.cpp), `execute`
// (the device runtime with measured time, csrc/runtime/executor.cpp) and the
// training-time chunk pool (paper_2406_08334_b200/offload.py through the
// ptk_pool_* C-ABI). Drivers own the mechanism (links, streams, copies,
// logging); the policy owns every decision. Chunk ids are 1-based here, as in
// the reference simulator; chunks 1..n_persist are persistent.
#pragma once

#include <algorithm>
#include <cstdint>
#include <deque>
#include <optional>
#include <vector>

#include "memplan/layout.hpp"
#include "memplan/sim.hpp"
#include "memplan/trace.hpp"

namespace memplan {

enum class Residency { Away, Arriving, Resident, Draining };

// Pipeline positions of one iteration over N chunks: chunk c is used in
// forward at position c and in backward at 2N - c + 1; the device optimizer
// runs at 2N + 1 and 2N + 2 means "iteration over".
struct PipelinePositions {
  int n = 0;
  int forward(int c) const { return c; }
  int backward(int c) const { return 2 * n - c + 1; }
  int chunk_at(int p) const { return p <= n ? p : 2 * n - p + 1; }
  int optimizer() const { return 2 * n + 1; }
  int past_end() const { return 2 * n + 2; }
  // First use of c at or after position `now`; INT_MAX when none is left.
  int next_use(int c, int now) const;
};

class ChunkBufferPool {
 public:
  ChunkBufferPool(int n_chunk, int n_persist, int n_buffer);

  struct Grant {
    int chunk = 0;    // the chunk that got a slot
    int slot = -1;    // its device slot, 0..n_buffer-1
    int evicted = 0;  // the chunk that gave the slot up (0: a free slot was used)
  };

  // A slot for chunk c (away) at position `now`. Takes the lowest-numbered
  // free slot, else evicts the farthest-next-use candidate -- for a prefetch
  // only one needed strictly later than c itself (the simulator's rule); on
  // `demand` (c is needed right now, e.g. a use the position model does not
  // list, like a tied head) any unpinned resident chunk. nullopt when no
  // chunk may be evicted for c. On success c is Arriving.
  std::optional<Grant> grant(int c, int now, const std::vector<int>& pinned, bool demand = false);
  void arrived(int c);       // Arriving -> Resident (ends the fetch in flight)
  void drain_started(int c); // non-persistent Resident -> Draining
  int drain_finished(int c); // Draining/Resident -> Away; returns the freed slot

  // The fetch queue: every away chunk used at a position up to `position`
  // is queued (once, in position order).
  void want_through(int position);
  enum class FetchStep { Nothing, Skipped, Started };
  struct FetchDecision {
    FetchStep step = FetchStep::Nothing;
    Grant grant;
  };
  // Next step of the prefetch pipeline: Nothing when a fetch is in flight,
  // the queue is empty or no slot can be granted; Skipped when the queue head
  // was already on the device (dropped from the queue); Started with the
  // grant otherwise (the chunk is now the fetch in flight).
  FetchDecision next_fetch(int now, const std::vector<int>& pinned);

  Residency where(int c) const { return state_[c]; }
  bool usable(int c) const {
    return state_[c] == Residency::Resident || state_[c] == Residency::Draining;
  }
  bool persistent(int c) const { return c <= n_persist_; }
  int slot_of(int c) const { return slot_[c]; }
  int chunk_in_slot(int s) const { return owner_[s]; }  // 0 = free
  int n_slots() const { return static_cast<int>(owner_.size()); }
  int free_slots() const;
  int fetch_in_flight() const { return fetching_; }
  int n_chunk() const { return pos_.n; }
  const PipelinePositions& positions() const { return pos_; }

 private:
  int pick_victim(int c, int now, const std::vector<int>& pinned, bool demand) const;

  PipelinePositions pos_;
  int n_persist_ = 0;
  std::vector<Residency> state_;  // 1-based
  std::vector<int> slot_;         // 1-based; -1 = none
  std::vector<int> owner_;        // per slot; 0 = free
  std::deque<int> queue_;
  int queued_through_ = 0;
  int fetching_ = 0;
};

// One device-memory ledger: bytes held, the high-water mark, and the sampled
// trace (one sample per distinct time).
class MemoryLedger {
 public:
  void change(std::int64_t t_ns, std::int64_t delta);
  void peek(std::int64_t extra) { high_ = std::max(high_, held_ + extra); }
  std::int64_t held() const { return held_; }
  std::int64_t high() const { return high_; }
  std::vector<MemSample>& samples() { return samples_; }

 private:
  std::int64_t held_ = 0, high_ = 0;
  std::vector<MemSample> samples_;
};

class IterationCore {
 public:
  struct Job {
    enum Kind { Forward, Backward, Recompute, Optimizer } kind;
    int op = -1;
    int block = -1;
    int chunk = 0;
    double seconds = 0;  // modelled duration
    int position = 0;
  };

  // gpu_optim_rate <= 0 leaves the optimizer jobs' modelled time at 0.
  IterationCore(const ModelTrace& trace, const ChunkLayout& layout, const BlockSchedule& schedule,
                const PlanConfig& cfg, double gpu_optim_rate);

  const std::vector<Job>& jobs() const { return jobs_; }
  std::size_t cursor() const { return cursor_; }  // oldest unfinished job
  bool finished() const { return cursor_ >= jobs_.size(); }
  int position() const {
    return finished() ? pool_.positions().past_end() : jobs_[cursor_].position;
  }
  // The chunk the next job needs (never evicted); 0 when done.
  int head_chunk() const { return finished() ? 0 : jobs_[cursor_].chunk; }

  bool ready(const Job& j) const;
  // Job j starts at t: queues fetches one position ahead, enters backward,
  // charges its memory.
  void start(const Job& j, std::int64_t t);

  struct Finished {
    Job job;
    int swap_out_block = -1;  // a swap block's forward just ended: stream it out
    int drain_chunk = 0;      // the chunk's last backward job just ended
  };
  // The job at the cursor ended at t.
  Finished finish(std::int64_t t);

  // After the chunk's reduce: true when its shard must go to the host (a
  // non-persistent chunk); a persistent chunk's optimizer job becomes ready.
  bool reduced(int c);
  // The chunk's gradient shard reached the host: its slot is free again.
  int offloaded(int c) { return pool_.drain_finished(c); }

  // Swap chains: the next activation-holding op of block b from op i on
  // (forward order out, reverse order in); -1 when the chain is complete
  // (swap-out: the block is then out; swap-in: zero-byte ops are marked back).
  int swap_out_next(int b, int i);
  int swap_in_next(int b, int i);
  void swapped_out(int op, std::int64_t t);
  void swapped_in(int op, std::int64_t t);
  // Swap blocks whose activations should start coming back now (marked issued).
  std::vector<int> swap_ins_due();

  ChunkBufferPool& pool() { return pool_; }
  const ChunkBufferPool& pool() const { return pool_; }
  MemoryLedger& ledger() { return ledger_; }
  std::int64_t chunk_used(int c) const { return used_[c]; }
  int block_first(int b) const { return first_[b]; }
  int block_last(int b) const { return last_[b]; }
  BlockStrategy strategy(int b) const { return sch_.strategies[b]; }

 private:
  BlockStrategy strategy_of(const OperatorRecord& op) const {
    return op.block_id ? sch_.strategies[*op.block_id] : BlockStrategy::None;
  }

  const ModelTrace& tr_;
  const BlockSchedule& sch_;
  const PlanConfig& cfg_;
  ChunkBufferPool pool_;
  MemoryLedger ledger_;
  std::vector<Job> jobs_;
  std::size_t cursor_ = 0;
  std::vector<std::int64_t> used_;       // 1-based chunk used bytes
  std::vector<int> bwd_left_;            // 1-based: backward jobs still to run
  std::vector<char> reduce_done_;        // 1-based
  std::vector<std::int64_t> block_act_;  // per block
  std::vector<int> first_, last_;        // per block
  std::vector<char> out_done_, in_issued_, act_back_;
  int lowest_entered_;
  bool backward_ = false;
};

}  // namespace memplan
