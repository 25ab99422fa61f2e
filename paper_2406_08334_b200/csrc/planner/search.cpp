// Cost-model configuration search over {n_persist, n_buffer, n_swap,
// n_checkpoint}.
//
// Behavioural sources (clean-room restatement; same winner, counters and
// frontier as the reference):
//   swap caps                    proj/src/search.cpp:13-37
//   candidate stream + ordering  proj/src/search.cpp:45-121
//   feasibility / preference     proj/src/search.cpp:135-155
//   memory-ordered walk          proj/src/search.cpp:157-226
//
// What is different (B200 build): the reference
// re-derives every per-trace quantity inside each of ~10^6 estimate calls.
// Here the trace / layout / link terms are digested once (digest.hpp), the
// schedule terms once per (n_swap, n_checkpoint), and the surviving prefix of
// the memory-ordered stream is evaluated by a pool of threads. Each
// candidate's t_iter is computed with the reference's exact operation order,
// the argmin under config_preferred (a total order) is unique, and the
// frontier is built by the same std::sort over the same sequence, so the
// result is bit-identical and independent of the thread count.
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <limits>
#include <map>
#include <memory>
#include <thread>

#include "digest.hpp"
#include "memplan/accounting.hpp"
#include "memplan/errors.hpp"
#include "memplan/search.hpp"
#include "memplan/sim.hpp"

namespace memplan {

namespace {

std::atomic<int> g_threads{0};

struct Candidate {
  PlanConfig config;
  std::int64_t m_peak = 0;
  std::int64_t m_peak_before_alpha = 0;
};

// Largest swap count whose swap positions j*(k+1) stay inside the model.
int swap_cap_layout(int n_block, int n_interval) {
  return n_block <= 0 ? 0 : (n_block - 1) / (n_interval + 1) + 1;
}

// Largest swap count whose block swap-outs all fit inside the forward pass at
// half (contended) D2H bandwidth.
int swap_cap_bandwidth(const ModelTrace& trace, const HardwareProfile& hw) {
  const std::int64_t act = mean_block_act_bytes(trace);
  if (act <= 0) return trace.n_blocks;
  double fwd = 0;
  for (const OperatorRecord& op : trace.ops)
    if (op.block_id) fwd += op.t_fwd;
  const double one_swap = static_cast<double>(act) / contended_bandwidth(hw.d2h_bw, 2);
  if (one_swap <= 0) return trace.n_blocks;
  return static_cast<int>(std::floor(fwd / one_swap));
}

std::int64_t largest_block_act(const ModelTrace& trace) {
  std::vector<std::int64_t> act(static_cast<std::size_t>(std::max(1, trace.n_blocks)), 0);
  for (const OperatorRecord& op : trace.ops)
    if (op.block_id) act[*op.block_id] += op.act_bytes;
  return *std::max_element(act.begin(), act.end());
}

// config_feasible with the per-trace largest block activation passed in
bool feasible_with(const PlanConfig& c, std::int64_t m_peak, const HardwareProfile& hw,
                   std::int64_t biggest_block) {
  if (m_peak >= hw.gpu_mem) return false;
  // swap-ins need one block of activation headroom on the device
  if (c.n_swap > 0 && hw.gpu_mem - m_peak < biggest_block) return false;
  return host_state_bytes(c) <= hw.cpu_mem;
}

// The memory-ordered candidate stream. Peaks come from one activation replay
// per (n_swap, n_checkpoint) plus the model-state bytes of (n_persist,
// n_buffer).
// Sorts v by `less` on up to worker_count threads: sorted runs, then pairwise
// merges. `less` must be a strict total order (the result is then unique).
template <typename T, typename Less>
void sort_unique_keys(std::vector<T>& v, Less less);

// With `cap`, only candidates whose peak is below it are materialised (the
// walk never passes the first one at or above capacity); `total` receives the
// size of the full stream.
std::vector<Candidate> candidate_stream(const ChunkLayout& layout, const ModelTrace& trace,
                                        const HardwareProfile& hw, const CostOptions& opts,
                                        std::int64_t cap = std::numeric_limits<std::int64_t>::max(),
                                        std::size_t* total = nullptr) {
  const int n_chunk = layout.n_chunk();
  const int n_block = trace.n_blocks;
  const int n_interval = compute_interval(trace, hw);
  const int max_swaps = std::min(swap_cap_layout(n_block, n_interval), swap_cap_bandwidth(trace, hw));
  const int ns_hi = std::min(max_swaps, n_block);

  // replay[ns][nc]: activation peak of one schedule (independent of np, nb)
  std::vector<std::vector<std::int64_t>> replay(static_cast<std::size_t>(ns_hi) + 1);
  for (int ns = 0; ns <= ns_hi; ++ns) {
    const int nc_lo = ns > 1 ? (ns - 1) * n_interval : 0;
    replay[ns].assign(static_cast<std::size_t>(std::max(0, n_block - ns)) + 1, 0);
    for (int nc = nc_lo; nc <= n_block - ns; ++nc) {
      const BlockSchedule sched = build_block_schedule(n_block, ns, nc, n_interval);
      replay[ns][nc] = detail::replay_peak(trace, sched, ns, nc);
    }
  }

  // Sort compact keys (peak, then np/nb/ns/nc packed in 16-bit fields, which
  // orders exactly like candidate_before) and build the candidates after.
  struct Key {
    std::int64_t peak;
    std::uint64_t rest;
    std::int64_t before_alpha;
  };
  std::vector<Key> keys;
  std::size_t n_all = 0;
  for (int np = 0; np <= n_chunk; ++np) {
    const int nb_lo = np == n_chunk ? 0 : std::min(3, n_chunk - np);
    const int nb_hi = np == n_chunk ? 0 : n_chunk - np;
    for (int nb = nb_lo; nb <= nb_hi; ++nb) {
      PlanConfig pc;
      pc.s_chunk = layout.s_chunk;
      pc.n_chunk = n_chunk;
      pc.n_persist = np;
      pc.n_buffer = nb;
      const std::int64_t states = device_state_bytes(pc);
      for (int ns = 0; ns <= ns_hi; ++ns) {
        const int nc_lo = ns > 1 ? (ns - 1) * n_interval : 0;
        for (int nc = nc_lo; nc <= n_block - ns; ++nc) {
          const std::int64_t before = replay[ns][nc] + states;
          const auto peak = static_cast<std::int64_t>(
              std::llround(opts.alpha * static_cast<double>(before)));
          ++n_all;
          if (peak >= cap) continue;
          keys.push_back({peak,
                          (static_cast<std::uint64_t>(np) << 48) |
                              (static_cast<std::uint64_t>(nb) << 32) |
                              (static_cast<std::uint64_t>(ns) << 16) | static_cast<std::uint64_t>(nc),
                          before});
        }
      }
    }
  }
  if (n_chunk >= (1 << 16) || n_block >= (1 << 16))
    throw InvariantViolation("candidate_stream: more than 65535 chunks or blocks");
  // All five keys together identify a candidate, so any correct sort yields
  // the reference's stable order.
  sort_unique_keys(keys, [](const Key& a, const Key& b) {
    return a.peak != b.peak ? a.peak < b.peak : a.rest < b.rest;
  });
  if (total) *total = n_all;
  std::vector<Candidate> out(keys.size());
  for (std::size_t i = 0; i < keys.size(); ++i) {
    const std::uint64_t r = keys[i].rest;
    Candidate& c = out[i];
    c.config = PlanConfig{layout.s_chunk, n_chunk, static_cast<int>(r >> 48),
                          static_cast<int>((r >> 32) & 0xffff), n_block, n_interval,
                          static_cast<int>((r >> 16) & 0xffff), static_cast<int>(r & 0xffff)};
    c.m_peak = keys[i].peak;
    c.m_peak_before_alpha = keys[i].before_alpha;
  }
  return out;
}

int worker_count(std::size_t work) {
  int n = g_threads.load();
  if (n <= 0) {  // not set by the caller: MEMPLAN_THREADS, else every core
    const char* e = std::getenv("MEMPLAN_THREADS");
    n = e ? std::atoi(e) : 0;
  }
  if (n <= 0) n = static_cast<int>(std::thread::hardware_concurrency());
  if (n <= 0) n = 1;
  const int by_work = static_cast<int>(work / 4096) + 1;  // tiny searches stay serial
  return std::max(1, std::min(n, by_work));
}

template <typename T, typename Less>
void sort_unique_keys(std::vector<T>& v, Less less) {
  const int workers = worker_count(v.size() / 16);
  if (workers <= 1) {
    std::sort(v.begin(), v.end(), less);
    return;
  }
  const std::size_t per = (v.size() + workers - 1) / workers;
  std::vector<std::size_t> bounds;
  for (std::size_t lo = 0; lo < v.size(); lo += per) bounds.push_back(lo);
  bounds.push_back(v.size());
  {
    std::vector<std::thread> pool;
    for (std::size_t k = 0; k + 1 < bounds.size(); ++k)
      pool.emplace_back([&, k] { std::sort(v.begin() + bounds[k], v.begin() + bounds[k + 1], less); });
    for (auto& t : pool) t.join();
  }
  while (bounds.size() > 2) {  // merge neighbouring runs, in parallel per level
    std::vector<std::size_t> next;
    std::vector<std::thread> pool;
    for (std::size_t k = 0; k + 1 < bounds.size(); k += 2) {
      next.push_back(bounds[k]);
      if (k + 2 < bounds.size())
        pool.emplace_back([&, k] {
          std::inplace_merge(v.begin() + bounds[k], v.begin() + bounds[k + 1],
                             v.begin() + bounds[k + 2], less);
        });
    }
    next.push_back(v.size());
    for (auto& t : pool) t.join();
    bounds = std::move(next);
  }
}

}  // namespace

void set_search_threads(int n) { g_threads.store(n); }

std::vector<PlanConfig> enumerate_candidates(const ChunkLayout& layout, const ModelTrace& trace,
                                             const HardwareProfile& hw, const CostOptions& opts) {
  std::vector<PlanConfig> out;
  for (const Candidate& c : candidate_stream(layout, trace, hw, opts)) out.push_back(c.config);
  return out;
}

namespace detail {

std::vector<PlanConfig> feasible_candidates(const ChunkLayout& layout, const ModelTrace& trace,
                                            const HardwareProfile& hw, const CostOptions& opts) {
  const std::int64_t biggest_block = largest_block_act(trace);
  std::vector<PlanConfig> out;
  for (const Candidate& c : candidate_stream(layout, trace, hw, opts, hw.gpu_mem))
    if (feasible_with(c.config, c.m_peak, hw, biggest_block)) out.push_back(c.config);
  return out;
}

}  // namespace detail

bool config_feasible(const ModelTrace& trace, const PlanConfig& config, std::int64_t m_peak,
                     const HardwareProfile& hw) {
  return feasible_with(config, m_peak, hw, largest_block_act(trace));
}

bool config_preferred(double t_iter_a, const PlanConfig& a, std::int64_t peak_a, double t_iter_b,
                      const PlanConfig& b, std::int64_t peak_b) {
  if (t_iter_a != t_iter_b) return t_iter_a < t_iter_b;
  if (a.n_swap != b.n_swap) return a.n_swap < b.n_swap;
  if (a.n_checkpoint != b.n_checkpoint) return a.n_checkpoint < b.n_checkpoint;
  if (a.n_persist != b.n_persist) return a.n_persist > b.n_persist;
  if (a.n_buffer != b.n_buffer) return a.n_buffer > b.n_buffer;
  return peak_a < peak_b;
}

SearchOutcome find_optimal(const ModelTrace& trace, const ChunkLayout& layout,
                           const HardwareProfile& hw, const CostOptions& opts) {
  hw.validate();
  // Memory-ordered: the first candidate past capacity ends the walk, so only
  // the candidates below it are materialised.
  std::size_t stream_size = 0;
  const std::vector<Candidate> stream =
      candidate_stream(layout, trace, hw, opts, hw.gpu_mem, &stream_size);
  const std::size_t walk = stream.size();

  // Shared digests; one schedule digest per (n_swap, n_checkpoint).
  const detail::TraceDigest digest(trace, layout);
  const detail::LinkDigest links(digest, hw);
  std::map<std::pair<int, int>, std::unique_ptr<detail::ScheduleDigest>> sched_digest;
  std::map<std::pair<int, int>, BlockSchedule> schedules;
  const std::int64_t biggest_block = largest_block_act(trace);
  std::vector<char> feasible(walk, 0);
  for (std::size_t i = 0; i < walk; ++i) {
    const PlanConfig& c = stream[i].config;
    const bool ok = feasible_with(c, stream[i].m_peak, hw, biggest_block);
    feasible[i] = ok;
    if (!ok) continue;
    const auto key = std::make_pair(c.n_swap, c.n_checkpoint);
    if (!sched_digest.count(key)) {
      auto it = schedules.emplace(key, build_block_schedule(c.n_block, c.n_swap, c.n_checkpoint,
                                                            c.n_interval)).first;
      sched_digest.emplace(key, std::make_unique<detail::ScheduleDigest>(digest, it->second, hw));
    }
  }

  // Evaluate the feasible prefix in parallel (each t_iter in reference order).
  std::vector<double> t_iter(walk, 0.0);
  // estimate_optim depends on n_persist only: one call per value
  std::vector<std::pair<double, double>> optim(static_cast<std::size_t>(layout.n_chunk()) + 1);
  for (int np = 0; np <= layout.n_chunk(); ++np) {
    PlanConfig c = walk ? stream[0].config : PlanConfig{};
    c.n_persist = np;
    optim[np] = estimate_optim(layout, c, hw);
  }
  std::vector<const detail::ScheduleDigest*> sd_of(walk, nullptr);
  for (std::size_t i = 0; i < walk; ++i)
    if (feasible[i])
      sd_of[i] = sched_digest.at({stream[i].config.n_swap, stream[i].config.n_checkpoint}).get();
  const auto eval_range = [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      if (!feasible[i]) continue;
      const PlanConfig& c = stream[i].config;
      const detail::ScheduleDigest& sd = *sd_of[i];
      const double f = detail::fwd_time(digest, sd, links, c.n_persist, nullptr);
      const double b = detail::bwd_time(digest, sd, links, c.n_persist, c.n_buffer, nullptr);
      const auto [gpu, cpu] = optim[c.n_persist];
      t_iter[i] = f + std::max(b + gpu, cpu);
    }
  };
  const int workers = worker_count(walk);
  if (workers == 1) {
    eval_range(0, walk);
  } else {
    std::vector<std::thread> pool;
    const std::size_t per = (walk + workers - 1) / workers;
    for (int w = 0; w < workers; ++w) {
      const std::size_t lo = std::min(walk, w * per), hi = std::min(walk, lo + per);
      pool.emplace_back(eval_range, lo, hi);
    }
    for (auto& t : pool) t.join();
  }

  // Deterministic merge in stream order.
  SearchOutcome outcome;
  bool have = false;
  double best_t = 0;
  std::int64_t best_peak = 0;
  std::vector<std::pair<PlanConfig, double>> ranked;
  for (std::size_t i = 0; i < walk; ++i) {
    if (!feasible[i]) {
      ++outcome.n_pruned;
      continue;
    }
    ++outcome.n_evaluated;
    const Candidate& cand = stream[i];
    ranked.emplace_back(cand.config, t_iter[i]);
    if (!have || config_preferred(t_iter[i], cand.config, cand.m_peak, best_t, outcome.best,
                                  best_peak)) {
      have = true;
      best_t = t_iter[i];
      best_peak = cand.m_peak;
      outcome.best = cand.config;
    }
  }
  outcome.n_pruned += static_cast<std::int64_t>(stream_size - walk);
  if (!have) throw NoFeasibleConfig("even the maximum-savings configuration exceeds device memory");

  // Frontier: the same (unstable) introsort over the same sequence as the
  // reference, then the 16 fastest.
  std::sort(ranked.begin(), ranked.end(),
            [](const auto& a, const auto& b) { return a.second < b.second; });
  if (ranked.size() > 16) ranked.resize(16);
  outcome.frontier = std::move(ranked);

  const BlockSchedule best_sched = build_block_schedule(
      outcome.best.n_block, outcome.best.n_swap, outcome.best.n_checkpoint, outcome.best.n_interval);
  outcome.estimate = estimate_iteration(trace, layout, best_sched, outcome.best, hw, opts);
  return outcome;
}

namespace {

// The analytically fastest feasible candidate for every n_persist value: the
// frontier alone is blind to plans that Eq.2 under-rates (e.g. keeping every
// chunk on the device and checkpointing more, when the host optimizer cannot
// hide behind the backward pass).
std::vector<std::pair<PlanConfig, double>> best_per_persist(const ModelTrace& trace,
                                                            const ChunkLayout& layout,
                                                            const HardwareProfile& hw) {
  const std::vector<Candidate> stream = candidate_stream(layout, trace, hw, CostOptions{}, hw.gpu_mem);
  const detail::TraceDigest digest(trace, layout);
  const detail::LinkDigest links(digest, hw);
  std::map<std::pair<int, int>, std::unique_ptr<detail::ScheduleDigest>> sdig;
  std::map<int, std::pair<PlanConfig, double>> best;
  std::map<int, std::int64_t> best_peak;
  for (const Candidate& cand : stream) {
    if (cand.m_peak >= hw.gpu_mem) break;
    if (!config_feasible(trace, cand.config, cand.m_peak, hw)) continue;
    const PlanConfig& c = cand.config;
    const auto key = std::make_pair(c.n_swap, c.n_checkpoint);
    if (!sdig.count(key)) {
      const BlockSchedule s = build_block_schedule(c.n_block, c.n_swap, c.n_checkpoint, c.n_interval);
      sdig.emplace(key, std::make_unique<detail::ScheduleDigest>(digest, s, hw));
    }
    const detail::ScheduleDigest& sd = *sdig.at(key);
    const auto [gpu, cpu] = estimate_optim(layout, c, hw);
    const double t = detail::fwd_time(digest, sd, links, c.n_persist, nullptr) +
                     std::max(detail::bwd_time(digest, sd, links, c.n_persist, c.n_buffer, nullptr) +
                                  gpu,
                              cpu);
    auto it = best.find(c.n_persist);
    if (it == best.end() || config_preferred(t, c, cand.m_peak, it->second.second, it->second.first,
                                             best_peak[c.n_persist])) {
      best[c.n_persist] = {c, t};
      best_peak[c.n_persist] = cand.m_peak;
    }
  }
  std::vector<std::pair<PlanConfig, double>> out;
  for (auto& [np, v] : best) out.push_back(v);
  return out;
}

bool same_config(const PlanConfig& a, const PlanConfig& b) {
  return a.n_persist == b.n_persist && a.n_buffer == b.n_buffer && a.n_swap == b.n_swap &&
         a.n_checkpoint == b.n_checkpoint;
}

}  // namespace

std::vector<RefinedChoice> refine_with_simulation(const ModelTrace& trace, const ChunkLayout& layout,
                                                  const HardwareProfile& hw,
                                                  const SearchOutcome& outcome, int top_k) {
  std::vector<std::pair<PlanConfig, double>> pool;
  const int k = std::min<int>(top_k, static_cast<int>(outcome.frontier.size()));
  for (int i = 0; i < k; ++i) pool.push_back(outcome.frontier[i]);
  for (const auto& cand : best_per_persist(trace, layout, hw)) {
    bool dup = false;
    for (const auto& p : pool) dup = dup || same_config(p.first, cand.first);
    if (!dup) pool.push_back(cand);
  }
  std::vector<RefinedChoice> out;
  for (const auto& [cfg, t_est] : pool) {
    const BlockSchedule sched =
        build_block_schedule(cfg.n_block, cfg.n_swap, cfg.n_checkpoint, cfg.n_interval);
    const SimulationResult sim = simulate(trace, layout, sched, cfg, hw);
    out.push_back({cfg, t_est, sim.t_iter, sim.m_peak});
  }
  std::stable_sort(out.begin(), out.end(), [](const RefinedChoice& a, const RefinedChoice& b) {
    return config_preferred(a.simulated_t_iter, a.config, a.simulated_m_peak, b.simulated_t_iter,
                            b.config, b.simulated_m_peak);
  });
  return out;
}

}  // namespace memplan
