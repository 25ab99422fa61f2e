// Profiler re-feed: measure the HardwareProfile fields
// the reference takes as calibration constants (proj/include/memplan/hardware.hpp:15-27,
// presets flagged "for calibration" in proj/src/presets.cpp:154-159) on this
// machine, with the same primitives the runtime uses:
//   h2d_bw / d2h_bw      pinned cudaMemcpyAsync of 512 MiB, best of 5
//   coll_alpha/coll_bw   NCCL all-gather of 8 KiB (alpha) and 512 MiB (beta)
//   gpu_optim_rate       fused chunk Adam over 256 Mi params (params/s)
//   cpu_optim_rate       host Adam over 32 Mi params, all threads (params/s)
//   gpu_mem / cpu_mem    cudaMemGetInfo total / physical host pages
// and the C-ABI used by Python to run the executor and the profiler.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <fstream>
#include <sstream>
#include <vector>

#include <json.hpp>

#include "memplan/cli.hpp"
#include "memplan/errors.hpp"
#include "memplan/execute.hpp"
#include "../ptk_common.h"

namespace memplan {

namespace {

struct Timer {
  void *a = nullptr, *b = nullptr;
  Timer() {
    ptk_event_create(&a);
    ptk_event_create(&b);
  }
  ~Timer() {
    ptk_event_destroy(a);
    ptk_event_destroy(b);
  }
  template <typename F>
  double best_seconds(void* stream, int reps, F&& body) {
    double best = 1e30;
    for (int i = 0; i < reps; ++i) {
      ptk_event_record(a, stream);
      body();
      ptk_event_record(b, stream);
      ptk_stream_synchronize(stream);
      float ms = 0;
      ptk_event_elapsed_ms(a, b, &ms);
      best = std::min(best, static_cast<double>(ms) * 1e-3);
    }
    return best;
  }
};

}  // namespace

HardwareProfile measure_profile(const HardwareProfile& base, void* comm, int world) {
  HardwareProfile hw = base;
  void* s = nullptr;
  ptk_stream_create(&s, 0);
  Timer timer;
  const std::size_t copy_bytes = 512ull << 20;
  void *host = nullptr, *dev = nullptr;
  ptk_host_alloc_pinned(&host, copy_bytes);
  cudaMalloc(&dev, copy_bytes);
  std::memset(host, 1, copy_bytes);
  hw.h2d_bw = copy_bytes / timer.best_seconds(s, 5, [&] { ptk_memcpy_h2d_async(dev, host, copy_bytes, s); });
  hw.d2h_bw = copy_bytes / timer.best_seconds(s, 5, [&] { ptk_memcpy_d2h_async(host, dev, copy_bytes, s); });

  if (comm != nullptr && world > 1) {
    auto* c = static_cast<ptk_comm*>(comm);
    const std::int64_t small = 4096, large = static_cast<std::int64_t>(copy_bytes / 2 / world);
    const double t_small = timer.best_seconds(s, 10, [&] { ptk_chunk_allgather(c, dev, small, 0, s); });
    const double t_large = timer.best_seconds(s, 5, [&] { ptk_chunk_allgather(c, dev, large, 0, s); });
    hw.coll_alpha = t_small;
    const double moved = 2.0 * large * world * (world - 1) / world;  // bytes*(w-1)/w of the chunk
    hw.coll_bw = moved / std::max(1e-9, t_large - t_small);
    hw.world_size = world;
  }

  // device Adam rate on a 256 Mi-parameter chunk
  const std::int64_t n = 256ll << 20;
  float *master, *m, *v;
  uint16_t *g, *p;
  cudaMalloc(&master, 4 * n);
  cudaMalloc(&m, 4 * n);
  cudaMalloc(&v, 4 * n);
  cudaMalloc(&g, 2 * n);
  cudaMalloc(&p, 2 * n);
  cudaMemsetAsync(m, 0, 4 * n, static_cast<cudaStream_t>(s));
  cudaMemsetAsync(v, 0, 4 * n, static_cast<cudaStream_t>(s));
  ptk_fill_uniform_f32(master, n, 1, 0, 0.05f, s);
  ptk_fill_uniform_bf16(g, n, 2, 0, 1e-3f, s);
  int step = 0;
  const double t_adam = timer.best_seconds(s, 5, [&] {
    const ptk_adam_config cfg{1e-3, 0.9, 0.999, 1e-8, 0.0, 0, ++step, 1.0};
    ptk_chunk_adam(&cfg, master, m, v, g, p, n, nullptr, nullptr, nullptr, nullptr, s);
  });
  hw.gpu_optim_rate = n / t_adam;
  for (void* q : {static_cast<void*>(master), static_cast<void*>(m), static_cast<void*>(v),
                  static_cast<void*>(g), static_cast<void*>(p)})
    cudaFree(q);

  // host Adam rate
  const std::int64_t hn = 32ll << 20;
  std::vector<float> hmaster(hn, 0.01f), hm(hn, 0.0f), hv(hn, 0.0f);
  std::vector<uint16_t> hg(hn, 0x3a83), hp(hn, 0);
  double best = 1e30;
  for (int r = 1; r <= 3; ++r) {
    const ptk_adam_config cfg{1e-3, 0.9, 0.999, 1e-8, 0.0, 0, r, 1.0};
    const auto t0 = std::chrono::steady_clock::now();
    ptk_cpu_adam(&cfg, hmaster.data(), hm.data(), hv.data(), hg.data(), hp.data(), hn, 0, nullptr,
                 nullptr);
    best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  hw.cpu_optim_rate = hn / best;

  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  hw.gpu_mem = static_cast<std::int64_t>(total_b);
  hw.cpu_mem = static_cast<std::int64_t>(sysconf(_SC_PHYS_PAGES)) * sysconf(_SC_PAGE_SIZE);
  cudaFree(dev);
  ptk_host_free_pinned(host);
  ptk_stream_destroy(s);
  hw.validate();
  return hw;
}

}  // namespace memplan

// ------------------------------------------------------------------ C-ABI --

namespace {

std::string slurp(const char* path) {
  std::ifstream in(path);
  if (!in) throw memplan::MalformedTrace(std::string("cannot open ") + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

int report(const std::exception& e) {
  ptk::set_error(e.what());  // surfaces through ptk_last_error()
  return PTK_EINVAL;
}

}  // namespace

extern "C" {

int ptk_execute_plan(const char* trace_path, const char* plan_path, const char* profile_path,
                     void* comm, int32_t rank, double compute_scale, int32_t iterations,
                     const char* result_json_path, const char* timeline_csv_path) {
  try {
    std::istringstream tin(slurp(trace_path));
    const memplan::ModelTrace trace = memplan::load_trace(tin);
    std::istringstream pin(slurp(plan_path));
    const memplan::PlanConfig cfg = memplan::plan_config_from_json(pin);
    std::istringstream hin(slurp(profile_path));
    const memplan::HardwareProfile hw = memplan::load_profile(hin);
    const memplan::ChunkLayout layout = memplan::pack_chunks(trace, cfg.s_chunk);
    const memplan::BlockSchedule sched =
        memplan::build_block_schedule(cfg.n_block, cfg.n_swap, cfg.n_checkpoint, cfg.n_interval);
    memplan::ExecOptions opt;
    opt.rank = rank;
    opt.comm = comm;
    opt.compute_scale = compute_scale;
    opt.iterations = iterations;
    const memplan::ExecutionResult r = memplan::execute(trace, layout, sched, cfg, hw, opt);
    const memplan::CostEstimate est = memplan::estimate_iteration(trace, layout, sched, cfg, hw);
    nlohmann::ordered_json j = nlohmann::ordered_json::parse(memplan::simulation_to_json(r.measured));
    j["estimate_t_iter"] = est.t_iter;
    j["estimate_m_peak"] = est.m_peak;
    j["h2d_bytes"] = r.stats.h2d_bytes;
    j["d2h_bytes"] = r.stats.d2h_bytes;
    j["coll_bytes"] = r.stats.coll_bytes;
    j["gpu_optim_ns"] = r.stats.gpu_optim_ns;
    j["cpu_optim_ns"] = r.stats.cpu_optim_ns;
    j["device_bytes"] = r.stats.device_bytes;
    j["pinned_host_bytes"] = r.stats.pinned_host_bytes;
    if (result_json_path) {
      std::ofstream out(result_json_path);
      out << j.dump(2) << "\n";
    }
    if (timeline_csv_path) {
      std::ofstream out(timeline_csv_path);
      memplan::timeline_to_csv(r.measured.timeline, out);
    }
    return PTK_OK;
  } catch (const std::exception& e) {
    return report(e);
  }
}

int ptk_measure_profile(const char* base_profile_path, void* comm, int32_t world,
                        const char* out_path) {
  try {
    std::istringstream in(slurp(base_profile_path));
    const memplan::HardwareProfile base = memplan::load_profile(in);
    const memplan::HardwareProfile hw = memplan::measure_profile(base, comm, world);
    std::ofstream out(out_path);
    memplan::save_profile(hw, out);
    return PTK_OK;
  } catch (const std::exception& e) {
    return report(e);
  }
}

}  // extern "C"
