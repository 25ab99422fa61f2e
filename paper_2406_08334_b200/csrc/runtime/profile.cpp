// Profiler re-feed: measure the HardwareProfile fields
// the reference takes as calibration constants (proj/include/memplan/hardware.hpp:15-27,
// presets flagged "for calibration" in proj/src/presets.cpp:154-159) on this
// machine, with the same primitives the runtime uses. Each field has its own
// C-ABI probe (the `ptk_profile_*` set of SURVEY §8(b)):
//   h2d_bw / d2h_bw      ptk_profile_copy_bw       pinned cudaMemcpyAsync, best of 5
//   coll_alpha/coll_bw   ptk_profile_collective    NCCL all-gather of 8 KiB (alpha) and
//                                                  a large shard (beta)
//   gpu_optim_rate       ptk_profile_gpu_adam_rate fused chunk Adam (params/s)
//   cpu_optim_rate       ptk_profile_cpu_adam_rate host Adam, all threads (params/s)
//   gpu_mem / cpu_mem    cudaMemGetInfo total / physical host pages
// and, outside the reference's HardwareProfile schema, the host-memory
// bandwidth of the simulator extension (ptk_profile_host_memory_bw).
// measure_profile composes them; the C-ABI also runs the executor.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <vector>

#include <json.hpp>

#include "memplan/cli.hpp"
#include "memplan/errors.hpp"
#include "memplan/execute.hpp"
#include "../ptk_common.h"

namespace {

void check(int rc, const char* what) {
  if (rc != PTK_OK) throw std::runtime_error(std::string(what) + ": " + ptk_last_error());
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

struct Stream {
  void* s = nullptr;
  Stream() { check(ptk_stream_create(&s, 0), "stream"); }
  ~Stream() { ptk_stream_destroy(s); }
};

struct DeviceBuf {
  void* p = nullptr;
  explicit DeviceBuf(std::size_t bytes) { check_cuda(cudaMalloc(&p, bytes), "cudaMalloc"); }
  ~DeviceBuf() { cudaFree(p); }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

struct PinnedBuf {
  void* p = nullptr;
  explicit PinnedBuf(std::size_t bytes) { check(ptk_host_alloc_pinned(&p, bytes), "pinned"); }
  ~PinnedBuf() { ptk_host_free_pinned(p); }
};

struct Timer {
  void *a = nullptr, *b = nullptr;
  Timer() {
    check(ptk_event_create(&a), "event");
    check(ptk_event_create(&b), "event");
  }
  ~Timer() {
    ptk_event_destroy(a);
    ptk_event_destroy(b);
  }
  template <typename F>
  double best_seconds(void* stream, int reps, F&& body) {
    double best = 1e30;
    for (int i = 0; i < reps; ++i) {
      check(ptk_event_record(a, stream), "record");
      body();
      check(ptk_event_record(b, stream), "record");
      check(ptk_stream_synchronize(stream), "synchronize");
      float ms = 0;
      check(ptk_event_elapsed_ms(a, b, &ms), "elapsed");
      best = std::min(best, static_cast<double>(ms) * 1e-3);
    }
    return best;
  }
};

void copy_bw(std::size_t bytes, double* h2d, double* d2h) {
  Stream s;
  Timer timer;
  PinnedBuf host(bytes);
  DeviceBuf dev(bytes);
  std::memset(host.p, 1, bytes);
  *h2d = bytes / timer.best_seconds(s.s, 5, [&] {
    check(ptk_memcpy_h2d_async(dev.p, host.p, bytes, s.s), "h2d");
  });
  *d2h = bytes / timer.best_seconds(s.s, 5, [&] {
    check(ptk_memcpy_d2h_async(host.p, dev.p, bytes, s.s), "d2h");
  });
}

// alpha = time of a tiny all-gather; beta = wire bytes (chunk * (w-1)/w)
// over the large all-gather's time above alpha -- the reference's
// gather_time model alpha + b*(w-1)/(w*beta) (proj/src/hardware.cpp:29-34)
void collective(ptk_comm* c, int world, std::size_t chunk_bytes, double* alpha, double* bw) {
  Stream s;
  Timer timer;
  DeviceBuf dev(chunk_bytes);
  const std::int64_t small = 4096;
  const std::int64_t large = static_cast<std::int64_t>(chunk_bytes / 2 / world);
  const double t_small = timer.best_seconds(s.s, 10, [&] {
    check(ptk_chunk_allgather(c, dev.p, small, 0, s.s), "allgather");
  });
  const double t_large = timer.best_seconds(s.s, 5, [&] {
    check(ptk_chunk_allgather(c, dev.p, large, 0, s.s), "allgather");
  });
  *alpha = t_small;
  const double moved = 2.0 * large * world * (world - 1) / world;
  *bw = moved / std::max(1e-9, t_large - t_small);
}

double gpu_adam_rate(std::int64_t n) {
  Stream s;
  Timer timer;
  DeviceBuf master(4 * n), m(4 * n), v(4 * n), g(2 * n), p(2 * n);
  auto* cs = static_cast<cudaStream_t>(s.s);
  check_cuda(cudaMemsetAsync(m.p, 0, 4 * n, cs), "memset");
  check_cuda(cudaMemsetAsync(v.p, 0, 4 * n, cs), "memset");
  check(ptk_fill_uniform_f32(master.as<float>(), n, 1, 0, 0.05f, s.s), "fill");
  check(ptk_fill_uniform_bf16(g.as<uint16_t>(), n, 2, 0, 1e-3f, s.s), "fill");
  int step = 0;
  const double t = timer.best_seconds(s.s, 5, [&] {
    const ptk_adam_config cfg{1e-3, 0.9, 0.999, 1e-8, 0.0, 0, ++step, 1.0};
    check(ptk_chunk_adam(&cfg, master.as<float>(), m.as<float>(), v.as<float>(),
                         g.as<uint16_t>(), p.as<uint16_t>(), n, nullptr, nullptr, nullptr,
                         nullptr, s.s),
          "chunk_adam");
  });
  return n / t;
}

double cpu_adam_rate(std::int64_t n) {
  std::vector<float> master(n, 0.01f), m(n, 0.0f), v(n, 0.0f);
  std::vector<uint16_t> g(n, 0x3a83), p(n, 0);
  double best = 1e30;
  for (int r = 1; r <= 3; ++r) {
    const ptk_adam_config cfg{1e-3, 0.9, 0.999, 1e-8, 0.0, 0, r, 1.0};
    const auto t0 = std::chrono::steady_clock::now();
    check(ptk_cpu_adam(&cfg, master.data(), m.data(), v.data(), g.data(), p.data(), n, 0,
                       nullptr, nullptr),
          "cpu_adam");
    best = std::min(best,
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  return n / best;
}

// Host-memory bandwidth (the --host-mem-bw of the simulator extension): the
// host Adam on `threads` threads runs while pinned H2D and D2H copies of
// 256 MiB loop on two streams; bw = (cpu_bytes_per_param * params updated +
// bytes copied) / elapsed, over about `seconds` of wall time.
double host_memory_bw(std::int64_t n, int threads, double seconds, double cpu_bytes_per_param) {
  const std::size_t bytes = 256ull << 20;
  PinnedBuf up(bytes), down(bytes);
  DeviceBuf dev(bytes);
  Stream s1, s2;
  std::memset(up.p, 1, bytes);
  std::atomic<bool> stop{false};
  std::atomic<long long> copied{0};
  std::atomic<int> errors{0};
  std::thread dma([&] {
    while (!stop.load()) {
      if (ptk_memcpy_h2d_async(dev.p, up.p, bytes, s1.s) != PTK_OK ||
          ptk_memcpy_d2h_async(down.p, dev.p, bytes, s2.s) != PTK_OK ||
          ptk_stream_synchronize(s1.s) != PTK_OK || ptk_stream_synchronize(s2.s) != PTK_OK) {
        errors.fetch_add(1);
        return;
      }
      copied.fetch_add(2ll * static_cast<long long>(bytes));
    }
  });
  std::vector<float> master(n, 0.01f), m(n, 0.0f), v(n, 0.0f);
  std::vector<uint16_t> g(n, 0x3a83), p(n, 0);
  std::this_thread::sleep_for(std::chrono::milliseconds(50));
  const long long c0 = copied.load();
  const auto t0 = std::chrono::steady_clock::now();
  long long params = 0;
  double el = 0.0;
  for (int r = 1; el < seconds; ++r) {
    const ptk_adam_config cfg{1e-3, 0.9, 0.999, 1e-8, 0.0, 0, r, 1.0};
    const int rc = ptk_cpu_adam(&cfg, master.data(), m.data(), v.data(), g.data(), p.data(), n,
                                threads, nullptr, nullptr);
    if (rc != PTK_OK) {
      stop.store(true);
      dma.join();
      check(rc, "cpu_adam");
    }
    params += n;
    el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  const long long moved = copied.load() - c0;   // whole copies finished in the window
  stop.store(true);
  dma.join();
  if (errors.load() != 0) throw std::runtime_error("host memory probe: copy failed");
  return (cpu_bytes_per_param * static_cast<double>(params) + static_cast<double>(moved)) / el;
}

}  // namespace

namespace memplan {

HardwareProfile measure_profile(const HardwareProfile& base, void* comm, int world) {
  HardwareProfile hw = base;
  const std::size_t chunk_bytes = 512ull << 20;
  copy_bw(chunk_bytes, &hw.h2d_bw, &hw.d2h_bw);
  if (comm != nullptr && world > 1) {
    collective(static_cast<ptk_comm*>(comm), world, chunk_bytes, &hw.coll_alpha, &hw.coll_bw);
    hw.world_size = world;
  }
  hw.gpu_optim_rate = gpu_adam_rate(256ll << 20);
  hw.cpu_optim_rate = cpu_adam_rate(32ll << 20);
  size_t free_b = 0, total_b = 0;
  check_cuda(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  hw.gpu_mem = static_cast<std::int64_t>(total_b);
  hw.cpu_mem = static_cast<std::int64_t>(sysconf(_SC_PHYS_PAGES)) * sysconf(_SC_PAGE_SIZE);
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

int ptk_profile_copy_bw(int64_t bytes, double* h2d_bw, double* d2h_bw) {
  if (bytes <= 0 || !h2d_bw || !d2h_bw) return ptk::fail(PTK_EINVAL, "ptk_profile_copy_bw: bad argument");
  try {
    copy_bw(static_cast<std::size_t>(bytes), h2d_bw, d2h_bw);
    return PTK_OK;
  } catch (const std::exception& e) {
    return report(e);
  }
}

int ptk_profile_collective(ptk_comm* comm, int32_t world, int64_t chunk_bytes, double* alpha,
                           double* bw) {
  if (!comm || world < 2 || chunk_bytes < 16 * world || !alpha || !bw)
    return ptk::fail(PTK_EINVAL, "ptk_profile_collective: bad argument");
  try {
    collective(comm, world, static_cast<std::size_t>(chunk_bytes), alpha, bw);
    return PTK_OK;
  } catch (const std::exception& e) {
    return report(e);
  }
}

int ptk_profile_gpu_adam_rate(int64_t n, double* params_per_s) {
  if (n <= 0 || !params_per_s) return ptk::fail(PTK_EINVAL, "ptk_profile_gpu_adam_rate: bad argument");
  try {
    *params_per_s = gpu_adam_rate(n);
    return PTK_OK;
  } catch (const std::exception& e) {
    return report(e);
  }
}

int ptk_profile_host_memory_bw(int64_t n, int32_t threads, double seconds, double* bytes_per_s) {
  if (n <= 0 || seconds <= 0.0 || !bytes_per_s)
    return ptk::fail(PTK_EINVAL, "ptk_profile_host_memory_bw: bad argument");
  try {
    const long hc = sysconf(_SC_NPROCESSORS_ONLN);
    const int t = threads > 0 ? threads : static_cast<int>(std::max(1L, hc - 2));
    *bytes_per_s = host_memory_bw(n, t, seconds, 28.0);
    return PTK_OK;
  } catch (const std::exception& e) {
    return report(e);
  }
}

int ptk_profile_cpu_adam_rate(int64_t n, double* params_per_s) {
  if (n <= 0 || !params_per_s) return ptk::fail(PTK_EINVAL, "ptk_profile_cpu_adam_rate: bad argument");
  try {
    *params_per_s = cpu_adam_rate(n);
    return PTK_OK;
  } catch (const std::exception& e) {
    return report(e);
  }
}

}  // extern "C"
