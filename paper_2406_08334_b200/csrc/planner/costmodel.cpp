// Analytic cost model: forward / backward stage sums (paper Eq.3-7), the
// optimizer split, the backward-replay peak memory (Eq.8-11) and the
// iteration estimate (Eq.2).
//
// Behavioural sources (clean-room restatement, bit-identical doubles):
//   chunk compute / timelines    proj/src/cost.cpp:24-66
//   forward stages               proj/src/cost.cpp:91-134
//   backward stages              proj/src/cost.cpp:136-204
//   optimizer split              proj/src/cost.cpp:206-219
//   peak-memory replay           proj/src/cost.cpp:221-274
//   iteration                    proj/src/cost.cpp:276-291
// The per-trace / per-schedule invariants live in detail::*Digest so the
// search can reuse them across ~10^6 candidates (search.cpp).
#include <algorithm>
#include <cmath>

#include "digest.hpp"
#include "memplan/accounting.hpp"
#include "memplan/cost.hpp"
#include "memplan/errors.hpp"

namespace memplan {

std::int64_t persistent_chunk_bytes(std::int64_t s_chunk) { return 8 * s_chunk; }

namespace detail {

TraceDigest::TraceDigest(const ModelTrace& trace, const ChunkLayout& layout)
    : n_chunk(layout.n_chunk()), n_block(trace.n_blocks) {
  const int n = n_chunk;
  comp_fwd.assign(n + 1, 0.0);
  comp_bwd.assign(n + 1, 0.0);
  chunk_bytes.assign(n + 1, 0);
  chunk_blocks.assign(n + 1, {});
  for (const Chunk& c : layout.chunks) {
    double f = 0, b = 0;
    for (int i = c.first_op; i <= c.last_op; ++i) {
      f += trace.ops[i].t_fwd;
      b += trace.ops[i].t_bwd;
    }
    comp_fwd[c.chunk_id + 1] = f;
    comp_bwd[c.chunk_id + 1] = b;
    chunk_bytes[c.chunk_id + 1] = c.used_bytes;
    chunk_blocks[c.chunk_id + 1] = c.block_ids;
  }
  cum_fwd.assign(n + 1, 0.0);
  for (int i = 1; i <= n; ++i) cum_fwd[i] = cum_fwd[i - 1] + comp_fwd[i];
  rev_bwd.assign(n + 3, 0.0);
  for (int c = n; c >= 1; --c) rev_bwd[c] = rev_bwd[c + 1] + comp_bwd[c];

  const std::size_t nb = static_cast<std::size_t>(std::max(0, n_block));
  block_fwd_end.assign(nb, 0.0);
  block_bwd_start.assign(nb, 0.0);
  block_act.assign(nb, 0);
  block_fwd.assign(nb, 0.0);
  double t = 0;
  for (const OperatorRecord& op : trace.ops) {
    t += op.t_fwd;
    if (!op.block_id) continue;
    block_fwd_end[*op.block_id] = t;
    block_act[*op.block_id] += op.act_bytes;
    block_fwd[*op.block_id] += op.t_fwd;
  }
  t = 0;
  for (auto it = trace.ops.rbegin(); it != trace.ops.rend(); ++it) {
    if (it->block_id) block_bwd_start[*it->block_id] = t;
    t += it->t_bwd;
  }
}

ScheduleDigest::ScheduleDigest(const TraceDigest& d, const BlockSchedule& schedule,
                               const HardwareProfile& hw, bool fwd, bool bwd) {
  const int n = d.n_chunk;
  std::vector<Window> outs, ins;
  const int nb = static_cast<int>(schedule.strategies.size());
  for (int b = 0; fwd && b < nb; ++b) {
    if (schedule.strategies[b] != BlockStrategy::Swap) continue;
    const double leave = transfer_time(d.block_act[b], hw.d2h_bw);
    outs.push_back({d.block_fwd_end[b], d.block_fwd_end[b] + leave});
  }
  for (int b = 0; bwd && b < nb; ++b) {
    if (schedule.strategies[b] != BlockStrategy::Swap) continue;
    const double back = transfer_time(d.block_act[b], hw.h2d_bw);
    ins.push_back({std::max(0.0, d.block_bwd_start[b] - back), d.block_bwd_start[b]});
  }
  const auto hits = [](const Window& w, const std::vector<Window>& set) {
    for (const Window& x : set)
      if (w.overlaps(x)) return true;
    return false;
  };
  fwd_contended.assign(n + 1, 0);
  bwd_contended.assign(n + 1, 0);
  for (int s = 1; s <= n; ++s) {
    // chunk s is fetched while chunk s-1 computes
    const Window w = s >= 2 ? Window{d.cum_fwd[s - 2], d.cum_fwd[s - 1]} : Window{0.0, 0.0};
    fwd_contended[s] = hits(w, outs);
    // in backward, chunk s is fetched during chunk s+1's stage
    bwd_contended[s] = hits(Window{d.rev_bwd[s + 2], d.rev_bwd[s + 1]}, ins);
  }
  recomp.assign(n + 1, 0.0);
  for (int c = 1; c <= n; ++c)
    for (int b : d.chunk_blocks[c])
      if (schedule.strategies[b] == BlockStrategy::Checkpoint) recomp[c] += d.block_fwd[b];
}

LinkDigest::LinkDigest(const TraceDigest& d, const HardwareProfile& hw) {
  const int n = d.n_chunk;
  pf_plain.assign(n + 1, 0.0);
  pf_half.assign(n + 1, 0.0);
  reduce.assign(n + 1, 0.0);
  drain.assign(n + 1, 0.0);
  // Bandwidth errors surface only when a term is actually used (fwd/bwd_time),
  // as in the reference where transfer_time is called lazily.
  upload_ok = hw.h2d_bw > 0;
  offload_ok = hw.d2h_bw > 0;
  const double half_h2d = hw.h2d_bw / 2.0;  // contended_bandwidth(h2d, 2)
  for (int c = 1; c <= n; ++c) {
    const std::int64_t bytes = d.chunk_bytes[c];
    const std::int64_t shard = bytes / hw.world_size;  // modeled shard: floor(used / w)
    if (upload_ok) {
      pf_plain[c] = gather_time(bytes, hw) + transfer_time(shard, hw.h2d_bw);
      pf_half[c] = gather_time(bytes, hw) + transfer_time(shard, half_h2d);
    }
    reduce[c] = reduce_time(bytes, hw);
    if (offload_ok) {
      double t = reduce_time(bytes, hw);
      t += transfer_time(shard, hw.d2h_bw);
      drain[c] = t;
    }
  }
}

namespace {
[[noreturn]] void no_bandwidth() { throw ZeroBandwidth("transfer bandwidth must be positive"); }
}  // namespace

double fwd_time(const TraceDigest& d, const ScheduleDigest& s, const LinkDigest& l, int n_persist,
                std::vector<StageTerm>* stages) {
  const int n = d.n_chunk;
  double total = 0;
  if (stages) stages->clear();
  for (int st = 1; st <= n + 1; ++st) {
    const double comp = st >= 2 ? d.comp_fwd[st - 1] : 0.0;
    double pf = 0;
    if (st > n_persist && st <= n) {
      if (!l.upload_ok) no_bandwidth();
      pf = s.fwd_contended[st] ? l.pf_half[st] : l.pf_plain[st];
    }
    const double chosen = std::max(comp, pf);
    total += chosen;
    if (stages) stages->push_back({st - 1, comp, 0, pf, 0, chosen});
  }
  return total;
}

double bwd_time(const TraceDigest& d, const ScheduleDigest& s, const LinkDigest& l, int n_persist,
                int n_buffer, std::vector<StageTerm>* stages) {
  const int n = d.n_chunk;
  // chunk c's backward prefetch: none if persistent or still buffered
  const auto prefetch = [&](int c) -> double {
    if (c < 1 || c > n || c <= n_persist || c > n - n_buffer) return 0.0;
    if (!l.upload_ok) no_bandwidth();
    return s.bwd_contended[c] ? l.pf_half[c] : l.pf_plain[c];
  };
  const auto drain = [&](int c) -> double {
    if (c < 1 || c > n) return 0.0;
    if (c <= n_persist) return l.reduce[c];
    if (!l.offload_ok) no_bandwidth();
    return l.drain[c];
  };
  double total = 0;
  if (stages) stages->clear();
  for (int p = 1; p <= n + 1; ++p) {
    const int c = n + 1 - p;  // chunk computing in this stage, 0 = final drain stage
    const double comp = c >= 1 ? d.comp_bwd[c] : 0.0;
    const double rc = c >= 1 ? s.recomp[c] : 0.0;
    const double pf = prefetch(c - 1);
    const double ro = drain(c + 1);
    const double chosen = std::max({comp + rc, pf, ro});
    total += chosen;
    if (stages) stages->push_back({c, comp, rc, pf, ro, chosen});
  }
  return total;
}

std::int64_t replay_peak(const ModelTrace& trace, const BlockSchedule& schedule, int n_swap,
                         int n_checkpoint) {
  const std::int64_t save_swap = mean_block_act_bytes(trace);
  const std::int64_t save_ckpt = save_swap - mean_block_boundary_bytes(trace);
  std::int64_t cur =
      trace.m_fwd + trace.total_act_bytes() - save_swap * n_swap - save_ckpt * n_checkpoint;
  std::int64_t peak = cur;
  const auto policy = [&](const OperatorRecord& op) {
    return op.block_id ? schedule.strategies[*op.block_id] : BlockStrategy::None;
  };
  // Walk backward; a checkpointed block re-materialises its activations when
  // its first replayed operator (its backward entry) runs.
  int last_block = -1;
  for (auto it = trace.ops.rbegin(); it != trace.ops.rend(); ++it) {
    const OperatorRecord& op = *it;
    const BlockStrategy pol = policy(op);
    const bool entry = op.block_id && pol == BlockStrategy::Checkpoint && *op.block_id != last_block;
    const std::int64_t bump = entry ? save_ckpt : 0;
    if (op.block_id) last_block = *op.block_id;
    peak = std::max(peak, cur + op.d_peak_prior);
    peak = std::max(peak, cur + op.d_cur_prior + op.d_peak_op + bump);
    cur += op.d_cur_prior + op.d_cur_op;
    if (pol == BlockStrategy::None) cur -= op.act_bytes;
  }
  return peak;
}

}  // namespace detail

std::int64_t mean_block_act_bytes(const ModelTrace& trace) {
  if (trace.n_blocks == 0) return 0;
  std::int64_t total = 0;
  for (const OperatorRecord& op : trace.ops)
    if (op.block_id) total += op.act_bytes;
  return total / trace.n_blocks;
}

std::int64_t mean_block_boundary_bytes(const ModelTrace& trace) {
  // the first operator's activation of each block is its boundary input
  if (trace.n_blocks == 0) return 0;
  std::int64_t total = 0;
  int prev = -1;
  for (const OperatorRecord& op : trace.ops) {
    if (!op.block_id || *op.block_id == prev) continue;
    total += op.act_bytes;
    prev = *op.block_id;
  }
  return total / trace.n_blocks;
}

double estimate_fwd(const ModelTrace& trace, const ChunkLayout& layout,
                    const BlockSchedule& schedule, const PlanConfig& config,
                    const HardwareProfile& hw, std::vector<StageTerm>* stages) {
  config.validate();
  const detail::TraceDigest d(trace, layout);
  const detail::ScheduleDigest s(d, schedule, hw, /*fwd=*/true, /*bwd=*/false);
  const detail::LinkDigest l(d, hw);
  return detail::fwd_time(d, s, l, config.n_persist, stages);
}

double estimate_bwd(const ModelTrace& trace, const ChunkLayout& layout,
                    const BlockSchedule& schedule, const PlanConfig& config,
                    const HardwareProfile& hw, std::vector<StageTerm>* stages) {
  config.validate();
  const detail::TraceDigest d(trace, layout);
  const detail::ScheduleDigest s(d, schedule, hw, /*fwd=*/false, /*bwd=*/true);
  const detail::LinkDigest l(d, hw);
  return detail::bwd_time(d, s, l, config.n_persist, config.n_buffer, stages);
}

std::pair<double, double> estimate_optim(const ChunkLayout& layout, const PlanConfig& config,
                                         const HardwareProfile& hw) {
  std::int64_t persistent = 0;
  const int upto = std::min(config.n_persist, layout.n_chunk());
  for (int i = 0; i < upto; ++i) persistent += layout.chunks[i].used_bytes;
  const std::int64_t offloaded = layout.used_total() - persistent;
  const double gpu_params = static_cast<double>(persistent) / layout.bytes_per_param;
  const double cpu_params = static_cast<double>(offloaded) / layout.bytes_per_param;
  return {gpu_params / hw.gpu_optim_rate, cpu_params / hw.cpu_optim_rate};
}

PeakMemoryBreakdown estimate_peak_memory(const ModelTrace& trace, const BlockSchedule& schedule,
                                         const PlanConfig& config, const HardwareProfile& hw,
                                         const CostOptions& opts) {
  (void)hw;
  config.validate();
  if (static_cast<int>(schedule.strategies.size()) != trace.n_blocks)
    throw InvariantViolation("schedule size does not match trace block count");
  if (schedule.n_swap() != config.n_swap || schedule.n_checkpoint() != config.n_checkpoint)
    throw InvariantViolation("schedule strategy counts disagree with config");
  PeakMemoryBreakdown out;
  out.replay_peak = detail::replay_peak(trace, schedule, config.n_swap, config.n_checkpoint);
  out.model_state_bytes = device_state_bytes(config);
  out.before_alpha = out.replay_peak + out.model_state_bytes;
  out.total =
      static_cast<std::int64_t>(std::llround(opts.alpha * static_cast<double>(out.before_alpha)));
  return out;
}

CostEstimate estimate_iteration(const ModelTrace& trace, const ChunkLayout& layout,
                                const BlockSchedule& schedule, const PlanConfig& config,
                                const HardwareProfile& hw, const CostOptions& opts) {
  CostEstimate e;
  e.t_fwd = estimate_fwd(trace, layout, schedule, config, hw, &e.fwd_stages);
  e.t_bwd = estimate_bwd(trace, layout, schedule, config, hw, &e.bwd_stages);
  const auto [gpu, cpu] = estimate_optim(layout, config, hw);
  e.t_gpu_optim = gpu;
  e.t_cpu_optim = cpu;
  e.t_iter = e.t_fwd + std::max(e.t_bwd + e.t_gpu_optim, e.t_cpu_optim);
  const PeakMemoryBreakdown mem = estimate_peak_memory(trace, schedule, config, hw, opts);
  e.m_peak = mem.total;
  e.m_peak_before_alpha = mem.before_alpha;
  return e;
}

}  // namespace memplan
