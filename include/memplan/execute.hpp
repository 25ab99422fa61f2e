// memplan — B200 extension: EXECUTE a plan instead of simulating it.
//
// `simulate` (sim.hpp, proj/src/sim.cpp:689-699) models one iteration;
// `execute` runs the same iteration on the device with the same decisions —
// one prefetch in flight, farthest-next-use eviction from a pool of n_buffer
// chunk slots, upload (+ all-gather) before use, reduce-scatter -> offload ->
// host Adam for non-persistent chunks, reduce-scatter -> device Adam for
// persistent chunks, swap-out / swap-in chains of activation bytes,
// recompute before a checkpointed block's backward — and returns the MEASURED
// timeline in the simulator's schema (SURVEY §8(b) "runtime execute").
//
// Bytes are real: chunk shards live in pinned host memory (fp32 master/m/v +
// bf16 parameters) or on the device, uploads/offloads are pinned
// cudaMemcpyAsync on side streams, collectives are NCCL, the optimizer
// updates are the real fused chunk Adam (ptk_chunk_adam) and host Adam
// (ptk_cpu_adam). Operator compute, which needs the model, is a stand-in
// that occupies the compute stream for the trace's t_fwd / t_bwd.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "memplan/sim.hpp"

namespace memplan {

struct ExecOptions {
  int rank = 0;                // this process's data-parallel rank
  void* comm = nullptr;        // ptk_comm* (required when hw.world_size > 1)
  double compute_scale = 1.0;  // stand-in compute = scale * trace time
  int cpu_threads = 0;         // host Adam threads (0 = all)
  int iterations = 1;          // iterations run; the result is the last one
};

struct ExecutionStats {
  std::int64_t h2d_bytes = 0;   // uploads + swap-ins
  std::int64_t d2h_bytes = 0;   // offloads + swap-outs
  std::int64_t coll_bytes = 0;  // all-gather + reduce-scatter payload
  std::int64_t gpu_optim_ns = 0;
  std::int64_t cpu_optim_ns = 0;
  std::int64_t device_bytes = 0;      // allocated by the runtime on the device
  std::int64_t pinned_host_bytes = 0;  // allocated by the runtime on the host
};

struct ExecutionResult {
  SimulationResult measured;  // same schema as simulate(); times are measured
  ExecutionStats stats;
};

ExecutionResult execute(const ModelTrace& trace, const ChunkLayout& layout,
                        const BlockSchedule& schedule, const PlanConfig& config,
                        const HardwareProfile& hw, const ExecOptions& opts = {});

// Measure this machine's HardwareProfile fields (pinned H2D/D2H bandwidth,
// NCCL all-gather alpha/beta when comm != nullptr, device and host Adam
// rates, memory capacities). Fields that cannot be measured are taken from
// `base`.
HardwareProfile measure_profile(const HardwareProfile& base, void* comm, int world);

}  // namespace memplan
