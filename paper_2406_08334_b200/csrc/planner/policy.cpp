// The chunk-runtime policy shared by the simulator, the device executor and
// the training-time chunk pool (include/memplan/policy.hpp). Decisions follow
// the reference simulator's semantics (proj/src/sim.cpp, cited per rule);
// the code is organised as two reusable state machines instead of one
// simulation object so that every driver runs the same rules.
#include "memplan/policy.hpp"

#include <algorithm>
#include <limits>

#include "memplan/accounting.hpp"
#include "memplan/errors.hpp"

namespace memplan {

namespace {
constexpr int kNoUse = std::numeric_limits<int>::max();
}

int PipelinePositions::next_use(int c, int now) const {
  // proj/src/sim.cpp:286-291: the forward use if it is still ahead, else the
  // backward use, else never
  for (const int p : {forward(c), backward(c)})
    if (p >= now) return p;
  return kNoUse;
}

// ------------------------------------------------------------------ pool --

ChunkBufferPool::ChunkBufferPool(int n_chunk, int n_persist, int n_buffer)
    : n_persist_(n_persist) {
  if (n_chunk < 0 || n_persist < 0 || n_persist > n_chunk || n_buffer < 0)
    throw InvariantViolation("ChunkBufferPool: need 0 <= n_persist <= n_chunk, n_buffer >= 0");
  pos_.n = n_chunk;
  state_.assign(n_chunk + 1, Residency::Away);
  slot_.assign(n_chunk + 1, -1);
  owner_.assign(n_buffer, 0);
  for (int c = 1; c <= n_persist; ++c) state_[c] = Residency::Resident;  // sim.cpp:260
}

int ChunkBufferPool::free_slots() const {
  return static_cast<int>(std::count(owner_.begin(), owner_.end(), 0));
}

// Farthest next use among idle resident non-persistent chunks that are not
// pinned; the first such chunk in id order wins a tie (proj/src/sim.cpp:314-325).
int ChunkBufferPool::pick_victim(int c, int now, const std::vector<int>& pinned,
                                 bool demand) const {
  int best = 0, best_use = -1;
  for (int v = n_persist_ + 1; v <= pos_.n; ++v) {
    if (v == c || state_[v] != Residency::Resident) continue;
    if (std::find(pinned.begin(), pinned.end(), v) != pinned.end()) continue;
    const int use = pos_.next_use(v, now);
    if (use > best_use) {
      best = v;
      best_use = use;
    }
  }
  // only a chunk needed strictly later than the incoming one may give way
  // (sim.cpp:326)
  if (best == 0 || (!demand && best_use <= pos_.next_use(c, now))) return 0;
  return best;
}

std::optional<ChunkBufferPool::Grant> ChunkBufferPool::grant(int c, int now,
                                                             const std::vector<int>& pinned,
                                                             bool demand) {
  if (c <= n_persist_ || c > pos_.n) throw InvariantViolation("grant: not a pooled chunk");
  if (state_[c] != Residency::Away) throw InvariantViolation("grant: chunk is not away");
  Grant g;
  g.chunk = c;
  const auto free_it = std::find(owner_.begin(), owner_.end(), 0);
  if (free_it != owner_.end()) {
    g.slot = static_cast<int>(free_it - owner_.begin());
  } else {
    g.evicted = pick_victim(c, now, pinned, demand);
    if (g.evicted == 0) return std::nullopt;
    g.slot = slot_[g.evicted];
    state_[g.evicted] = Residency::Away;
    slot_[g.evicted] = -1;
  }
  owner_[g.slot] = c;
  slot_[c] = g.slot;
  state_[c] = Residency::Arriving;
  return g;
}

void ChunkBufferPool::arrived(int c) {
  if (state_[c] != Residency::Arriving) throw InvariantViolation("arrived: chunk was not arriving");
  state_[c] = Residency::Resident;
  if (fetching_ == c) fetching_ = 0;
}

void ChunkBufferPool::drain_started(int c) {
  if (!persistent(c)) state_[c] = Residency::Draining;  // sim.cpp:529-532
}

int ChunkBufferPool::drain_finished(int c) {
  const int s = slot_[c];
  if (s >= 0) owner_[s] = 0;
  slot_[c] = -1;
  state_[c] = Residency::Away;  // sim.cpp:445-450
  return s;
}

void ChunkBufferPool::want_through(int position) {
  // proj/src/sim.cpp:270-277: positions are considered once, in order
  const int last = std::min(position, 2 * pos_.n);
  for (; queued_through_ < last; ++queued_through_) {
    const int c = pos_.chunk_at(queued_through_ + 1);
    if (state_[c] == Residency::Away && std::find(queue_.begin(), queue_.end(), c) == queue_.end())
      queue_.push_back(c);
  }
}

ChunkBufferPool::FetchDecision ChunkBufferPool::next_fetch(int now,
                                                           const std::vector<int>& pinned) {
  FetchDecision d;
  if (fetching_ != 0 || queue_.empty()) return d;  // one fetch in flight (sim.cpp:307-308)
  const int c = queue_.front();
  if (state_[c] != Residency::Away) {  // came back on its own meanwhile
    queue_.pop_front();
    d.step = FetchStep::Skipped;
    return d;
  }
  const std::optional<Grant> g = grant(c, now, pinned);
  if (!g) return d;
  queue_.pop_front();
  fetching_ = c;
  d.step = FetchStep::Started;
  d.grant = *g;
  return d;
}

// ---------------------------------------------------------------- ledger --

void MemoryLedger::change(std::int64_t t_ns, std::int64_t delta) {
  held_ += delta;
  if (held_ < 0) throw LedgerUnderflow("allocated bytes went negative");
  high_ = std::max(high_, held_);
  if (!samples_.empty() && samples_.back().time_ns == t_ns)
    samples_.back().bytes = held_;
  else
    samples_.push_back({t_ns, held_});
}

// ------------------------------------------------------------- iteration --

IterationCore::IterationCore(const ModelTrace& trace, const ChunkLayout& layout,
                             const BlockSchedule& schedule, const PlanConfig& cfg,
                             double gpu_optim_rate)
    : tr_(trace),
      sch_(schedule),
      cfg_(cfg),
      pool_(layout.n_chunk(), cfg.n_persist, cfg.n_buffer),
      lowest_entered_(std::numeric_limits<int>::max()) {
  const int n_ops = static_cast<int>(trace.ops.size());
  const int n_chunk = layout.n_chunk();
  const std::size_t n_blk = static_cast<std::size_t>(std::max(1, trace.n_blocks));
  const PipelinePositions& pos = pool_.positions();

  used_.assign(n_chunk + 1, 0);
  for (const Chunk& ch : layout.chunks) used_[ch.chunk_id + 1] = ch.used_bytes;
  std::vector<int> chunk_of(n_ops);
  for (int i = 0; i < n_ops; ++i) chunk_of[i] = layout.chunk_of_op(i);

  block_act_.assign(n_blk, 0);
  first_.assign(n_blk, -1);
  last_.assign(n_blk, -1);
  std::vector<double> block_fwd(n_blk, 0.0);
  for (const OperatorRecord& op : trace.ops) {
    if (!op.block_id) continue;
    const std::size_t b = static_cast<std::size_t>(*op.block_id);
    block_act_[b] += op.act_bytes;
    if (first_[b] < 0) first_[b] = op.index;
    last_[b] = op.index;
    block_fwd[b] += op.t_fwd;
  }

  // proj/src/sim.cpp:227-248: forward in op order; backward in reverse with a
  // checkpointed block's recompute just before its last op's backward; then a
  // device optimizer job per persistent chunk (gated on its reduce)
  for (int i = 0; i < n_ops; ++i)
    jobs_.push_back({Job::Forward, i, trace.ops[i].block_id.value_or(-1), chunk_of[i],
                     trace.ops[i].t_fwd, pos.forward(chunk_of[i])});
  for (int i = n_ops - 1; i >= 0; --i) {
    const OperatorRecord& op = trace.ops[i];
    const int c = chunk_of[i];
    if (strategy_of(op) == BlockStrategy::Checkpoint && i == last_[*op.block_id])
      jobs_.push_back({Job::Recompute, -1, *op.block_id, c, block_fwd[*op.block_id],
                       pos.backward(c)});
    jobs_.push_back({Job::Backward, i, op.block_id.value_or(-1), c, op.t_bwd, pos.backward(c)});
  }
  for (int c = 1; c <= cfg.n_persist; ++c) {
    const double t = gpu_optim_rate > 0.0 ? static_cast<double>(used_[c]) /
                                                layout.bytes_per_param / gpu_optim_rate
                                          : 0.0;
    jobs_.push_back({Job::Optimizer, -1, -1, c, t, pos.optimizer()});
  }

  bwd_left_.assign(n_chunk + 1, 0);
  for (const Job& j : jobs_)
    if (j.kind == Job::Backward || j.kind == Job::Recompute) ++bwd_left_[j.chunk];
  reduce_done_.assign(n_chunk + 1, 0);
  out_done_.assign(n_blk, 0);
  in_issued_.assign(n_blk, 0);
  act_back_.assign(n_ops, 0);
  // model states + the residual floor are held for the whole iteration
  ledger_.change(0, device_state_bytes(cfg) + trace.m_fwd);
  pool_.want_through(1);
}

bool IterationCore::ready(const Job& j) const {
  switch (j.kind) {
    case Job::Optimizer:
      return reduce_done_[j.chunk] != 0;  // sim.cpp:470-471
    case Job::Forward:
    case Job::Recompute:
      return pool_.usable(j.chunk);
    case Job::Backward:
      // a swapped block's activations must be back first (sim.cpp:462-467)
      return pool_.usable(j.chunk) &&
             !(j.block >= 0 && sch_.strategies[j.block] == BlockStrategy::Swap &&
               tr_.ops[j.op].act_bytes > 0 && !act_back_[j.op]);
  }
  return false;
}

void IterationCore::start(const Job& j, std::int64_t t) {
  pool_.want_through(j.position + 1);  // sim.cpp:481
  if (j.kind == Job::Backward || j.kind == Job::Recompute) {
    backward_ = true;
    if (j.block >= 0) lowest_entered_ = std::min(lowest_entered_, j.block);
  }
  if (j.kind == Job::Recompute) {
    // the block's activations are rebuilt; its boundary input was kept
    ledger_.change(t, block_act_[j.block] - tr_.ops[first_[j.block]].act_bytes);
  } else if (j.kind == Job::Backward) {
    const OperatorRecord& op = tr_.ops[j.op];
    ledger_.peek(op.d_peak_prior);
    if (op.d_cur_prior != 0) ledger_.change(t, op.d_cur_prior);
    ledger_.peek(op.d_peak_op);
  }
}

IterationCore::Finished IterationCore::finish(std::int64_t t) {
  Finished f;
  f.job = jobs_[cursor_++];
  const Job& j = f.job;
  if (j.kind == Job::Forward) {
    const OperatorRecord& op = tr_.ops[j.op];
    const BlockStrategy st = strategy_of(op);
    const bool opens_block = op.block_id && j.op == first_[*op.block_id];
    // activations kept: not checkpointed, or a checkpointed block's input (sim.cpp:507-512)
    if (op.act_bytes > 0 && (st != BlockStrategy::Checkpoint || opens_block))
      ledger_.change(t, op.act_bytes);
    if (st == BlockStrategy::Swap && j.op == last_[*op.block_id]) f.swap_out_block = *op.block_id;
  } else if (j.kind == Job::Backward || j.kind == Job::Recompute) {
    if (j.kind == Job::Backward) {
      const OperatorRecord& op = tr_.ops[j.op];
      if (op.d_cur_op != 0) ledger_.change(t, op.d_cur_op);
      if (op.act_bytes > 0) ledger_.change(t, -op.act_bytes);
    }
    if (--bwd_left_[j.chunk] == 0) {  // the chunk's gradients are complete
      pool_.drain_started(j.chunk);
      f.drain_chunk = j.chunk;
    }
  }
  return f;
}

bool IterationCore::reduced(int c) {
  if (pool_.persistent(c)) {
    reduce_done_[c] = 1;  // sim.cpp:438-442
    return false;
  }
  return true;
}

int IterationCore::swap_out_next(int b, int i) {
  for (; i <= last_[b]; ++i)
    if (tr_.ops[i].act_bytes != 0) return i;
  out_done_[b] = 1;
  return -1;
}

int IterationCore::swap_in_next(int b, int i) {
  for (; i >= first_[b]; --i) {
    if (tr_.ops[i].act_bytes != 0) return i;
    act_back_[i] = 1;  // nothing to move for this op
  }
  return -1;
}

void IterationCore::swapped_out(int op, std::int64_t t) { ledger_.change(t, -tr_.ops[op].act_bytes); }

void IterationCore::swapped_in(int op, std::int64_t t) {
  ledger_.change(t, tr_.ops[op].act_bytes);
  act_back_[op] = 1;
}

std::vector<int> IterationCore::swap_ins_due() {
  // proj/src/sim.cpp:397-412: within n_interval blocks of the backward front
  // with one block of headroom under the high-water mark, or needed next
  std::vector<int> due;
  const int n_blk = tr_.n_blocks;
  const int front = backward_ ? std::min(lowest_entered_, n_blk) : std::numeric_limits<int>::max();
  const Job* head = finished() ? nullptr : &jobs_[cursor_];
  for (int b = 0; b < n_blk; ++b) {
    if (sch_.strategies[b] != BlockStrategy::Swap || in_issued_[b] || !out_done_[b]) continue;
    const bool close = front <= b + cfg_.n_interval;
    const bool room = ledger_.high() - ledger_.held() >= block_act_[b];
    const bool next = head != nullptr && head->kind == Job::Backward && head->block == b;
    if ((close && room) || next) {
      in_issued_[b] = 1;
      due.push_back(b);
    }
  }
  return due;
}

}  // namespace memplan
