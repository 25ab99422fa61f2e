// The chunk runtime: executes one training iteration of a plan on the
// device with the simulator's decisions and measured times (execute.hpp).
//
// Policy: the shared chunk-runtime policy (include/memplan/policy.hpp), the
// same code the simulator (csrc/planner/simulator.cpp) and the training-time
// chunk pool run -- proj/src/sim.cpp's semantics:
//   * positions: forward of chunk c at c, backward at 2N-c+1, optimizer 2N+1
//   * fetch queue filled one position ahead of the GPU; ONE fetch in flight
//   * a fetch needs a free slot of the n_buffer pool, else evicts the idle
//     resident chunk with the farthest next use (strictly later than the
//     incoming chunk's, never the chunk of the next GPU task)
//   * after a chunk's last backward task: reduce-scatter, then either device
//     Adam (persistent) or offload + host Adam (non-persistent)
//   * swap blocks stream their activations out after the block's forward and
//     back in when backward is within n_interval blocks (and one block of
//     headroom is free) or when the block is needed next
// Mechanism (B200): streams compute / h2d / d2h / coll, CUDA events for every
// start/end, one host worker thread for the host Adam queue, NCCL for the
// collectives, pinned host shards, and a pool of device chunk slots.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <limits>
#include <map>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <thread>

#include "memplan/accounting.hpp"
#include "memplan/errors.hpp"
#include "memplan/execute.hpp"
#include "memplan/policy.hpp"
#include "ptk.h"

namespace memplan {

namespace {

void must(int rc, const char* what) {
  if (rc != PTK_OK) throw std::runtime_error(std::string(what) + ": " + ptk_last_error());
}
void must_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

std::int64_t host_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

struct DeviceBuf {
  void* p = nullptr;
  std::size_t bytes = 0;
  DeviceBuf() = default;
  explicit DeviceBuf(std::size_t n) : bytes(n) {
    if (n) must_cuda(cudaMalloc(&p, n), "cudaMalloc");
  }
  DeviceBuf(DeviceBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; }
  DeviceBuf& operator=(DeviceBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
    return *this;
  }
  ~DeviceBuf() {
    if (p) cudaFree(p);
  }
};

struct HostBuf {
  void* p = nullptr;
  std::size_t bytes = 0;
  HostBuf() = default;
  explicit HostBuf(std::size_t n) : bytes(n) {
    if (n) must(ptk_host_alloc_pinned(&p, n), "ptk_host_alloc_pinned");
  }
  HostBuf(HostBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; }
  HostBuf& operator=(HostBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
    return *this;
  }
  ~HostBuf() {
    if (p) ptk_host_free_pinned(p);
  }
};

// Storage of one chunk on this rank.
struct ChunkStore {
  std::int64_t numel = 0;  // real parameters
  std::int64_t shard = 0;  // padded per-rank shard (elements)
  bool persistent = false;
  // persistent: device param/grad (n_pad) + device fp32 state (shard)
  DeviceBuf d_param, d_grad, d_master, d_m, d_v;
  // non-persistent: pinned host shard state
  HostBuf h_param, h_grad, h_master, h_m, h_v;
};

// The host Adam queue: one worker, FIFO, like the simulator's serial CPU.
class HostOptimizer {
 public:
  explicit HostOptimizer(int threads) : threads_(threads), worker_([this] { loop(); }) {}
  ~HostOptimizer() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    worker_.join();
  }
  void submit(int chunk, ChunkStore* s, ptk_adam_config cfg) {
    std::lock_guard<std::mutex> g(mu_);
    queue_.push_back({chunk, s, cfg});
    cv_.notify_all();
  }
  // (chunk, start_ns, end_ns) of finished updates since the last call
  std::vector<std::tuple<int, std::int64_t, std::int64_t>> drain_done() {
    std::lock_guard<std::mutex> g(mu_);
    auto out = std::move(done_);
    done_.clear();
    return out;
  }
  bool idle() {
    std::lock_guard<std::mutex> g(mu_);
    return queue_.empty() && !busy_;
  }

 private:
  struct Job {
    int chunk;
    ChunkStore* s;
    ptk_adam_config cfg;
  };
  void loop() {
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || !queue_.empty(); });
        if (stop_ && queue_.empty()) return;
        j = queue_.front();
        queue_.pop_front();
        busy_ = true;
      }
      const std::int64_t t0 = host_ns();
      ptk_cpu_adam(&j.cfg, static_cast<float*>(j.s->h_master.p), static_cast<float*>(j.s->h_m.p),
                   static_cast<float*>(j.s->h_v.p), static_cast<const uint16_t*>(j.s->h_grad.p),
                   static_cast<uint16_t*>(j.s->h_param.p), j.s->shard, threads_, nullptr, nullptr);
      const std::int64_t t1 = host_ns();
      std::lock_guard<std::mutex> g(mu_);
      done_.emplace_back(j.chunk, t0, t1);
      busy_ = false;
    }
  }
  int threads_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Job> queue_;
  std::vector<std::tuple<int, std::int64_t, std::int64_t>> done_;
  bool busy_ = false;
  bool stop_ = false;
  std::thread worker_;
};

class Runtime {
 public:
  Runtime(const ModelTrace& t, const ChunkLayout& l, const BlockSchedule& s, const PlanConfig& c,
          const HardwareProfile& hw, const ExecOptions& o)
      : tr_(t), lay_(l), sch_(s), cfg_(c), hw_(hw), opt_(o), host_opt_(o.cpu_threads) {
    w_ = hw.world_size;
    if (w_ > 1 && !o.comm) throw InvariantViolation("execute: world_size > 1 needs a ptk_comm");
    must(ptk_stream_create(&s_gpu_, 1), "stream");
    must(ptk_stream_create(&s_h2d_, 0), "stream");
    must(ptk_stream_create(&s_d2h_, 0), "stream");
    must(ptk_stream_create(&s_coll_, 0), "stream");
    allocate();
  }
  ~Runtime() {
    cudaDeviceSynchronize();
    for (void* e : events_) ptk_event_destroy(e);
    for (void* s : {s_gpu_, s_h2d_, s_d2h_, s_coll_}) ptk_stream_destroy(s);
  }

  ExecutionResult run(int iterations) {
    ExecutionResult out;
    for (int it = 0; it < std::max(1, iterations); ++it) {
      step_ = it + 1;
      stats_ = {};
      out.measured = iterate();
    }
    stats_.device_bytes = device_bytes_;
    stats_.pinned_host_bytes = host_bytes_;
    out.stats = stats_;
    return out;
  }

 private:
  // an asynchronous device operation whose completion the loop waits for
  struct Pending {
    enum What { Gpu, Upload, Gather, Reduce, Offload, SwapOut, SwapIn } what;
    int chunk = 0, block = -1, op = -1;
    void* start = nullptr;
    void* end = nullptr;
    int start_note = -1;  // log_ index of the "_start" event, re-stamped with device time
  };

  // ------------------------------------------------------------ set-up --
  void allocate() {
    nops_ = static_cast<int>(tr_.ops.size());
    nc_ = lay_.n_chunk();
    nblk_ = tr_.n_blocks;
    store_.resize(nc_ + 1);
    std::int64_t max_pad = 0;
    for (const Chunk& ch : lay_.chunks) {
      const int c = ch.chunk_id + 1;
      ChunkStore& st = store_[c];
      st.numel = ch.used_bytes / lay_.bytes_per_param;
      st.shard = ptk_shard_elems(st.numel, w_);
      const std::int64_t n_pad = st.shard * w_;
      st.persistent = c <= cfg_.n_persist;
      if (st.persistent) {
        st.d_param = DeviceBuf(2 * n_pad);
        st.d_grad = DeviceBuf(2 * n_pad);
        st.d_master = DeviceBuf(4 * st.shard);
        st.d_m = DeviceBuf(4 * st.shard);
        st.d_v = DeviceBuf(4 * st.shard);
        device_bytes_ += 4 * n_pad + 12 * st.shard;
        must(ptk_fill_uniform_f32(static_cast<float*>(st.d_master.p), st.shard, 1000 * c,
                                  opt_.rank * st.shard, 0.05f, s_gpu_), "fill");
        must(ptk_fill_uniform_bf16(static_cast<uint16_t*>(st.d_param.p), n_pad, 1000 * c, 0,
                                   0.05f, s_gpu_), "fill");
        must(ptk_fill_uniform_bf16(static_cast<uint16_t*>(st.d_grad.p), n_pad,
                                   1000 * c + 1 + opt_.rank, 0, 1e-3f, s_gpu_), "fill");
        must_cuda(cudaMemsetAsync(st.d_m.p, 0, 4 * st.shard, static_cast<cudaStream_t>(s_gpu_)), "memset");
        must_cuda(cudaMemsetAsync(st.d_v.p, 0, 4 * st.shard, static_cast<cudaStream_t>(s_gpu_)), "memset");
      } else {
        max_pad = std::max(max_pad, n_pad);
        st.h_param = HostBuf(2 * st.shard);
        st.h_grad = HostBuf(2 * st.shard);
        st.h_master = HostBuf(4 * st.shard);
        st.h_m = HostBuf(4 * st.shard);
        st.h_v = HostBuf(4 * st.shard);
        host_bytes_ += 16 * st.shard;
        // host state initialised with the same counter-based generator
        std::vector<float> tmp;
        auto* hm = static_cast<float*>(st.h_master.p);
        for (std::int64_t i = 0; i < st.shard; ++i) hm[i] = 0.0f;
        std::fill_n(static_cast<float*>(st.h_m.p), st.shard, 0.0f);
        std::fill_n(static_cast<float*>(st.h_v.p), st.shard, 0.0f);
        std::fill_n(static_cast<uint16_t*>(st.h_param.p), st.shard, uint16_t{0x3c00});
        std::fill_n(static_cast<uint16_t*>(st.h_grad.p), st.shard, uint16_t{0});
      }
    }
    slots_.clear();
    for (int i = 0; i < cfg_.n_buffer; ++i) slots_.emplace_back(2 * std::max<std::int64_t>(max_pad, 8));
    device_bytes_ += static_cast<std::int64_t>(cfg_.n_buffer) * 2 * max_pad;
    // swap arena: a device + pinned host region per activation-holding op of a swap block
    act_dev_.assign(nops_, nullptr);
    act_host_.assign(nops_, nullptr);
    std::int64_t swap_bytes = 0;
    for (const OperatorRecord& op : tr_.ops)
      if (op.block_id && sch_.strategies[*op.block_id] == BlockStrategy::Swap) swap_bytes += op.act_bytes;
    if (swap_bytes > 0) {
      swap_dev_ = DeviceBuf(swap_bytes);
      swap_host_ = HostBuf(swap_bytes);
      device_bytes_ += swap_bytes;
      host_bytes_ += swap_bytes;
      std::int64_t off = 0;
      for (const OperatorRecord& op : tr_.ops)
        if (op.block_id && sch_.strategies[*op.block_id] == BlockStrategy::Swap) {
          act_dev_[op.index] = static_cast<char*>(swap_dev_.p) + off;
          act_host_[op.index] = static_cast<char*>(swap_host_.p) + off;
          off += op.act_bytes;
        }
    }
    ws_ = DeviceBuf(static_cast<std::size_t>(ptk_stats_workspace_bytes()));
    stats_dev_ = DeviceBuf(sizeof(ptk_grad_stats_t));
    cudaMemset(ws_.p, 0, ws_.bytes);
    must(ptk_stream_synchronize(s_gpu_), "sync");
  }

  void* new_event() {
    if (free_events_.empty()) {
      void* e = nullptr;
      must(ptk_event_create(&e), "event");
      events_.push_back(e);
      return e;
    }
    void* e = free_events_.back();
    free_events_.pop_back();
    return e;
  }

  ptk_adam_config adam(double grad_scale) const {
    return ptk_adam_config{1e-3, 0.9, 0.999, 1e-8, 0.0, 0, step_, grad_scale};
  }

  // ------------------------------------------------------- one iteration --
  using Job = IterationCore::Job;
  SimulationResult iterate();
  void prepare_iteration();
  void note(const char* res, const std::string& ev, const std::string& subj, std::int64_t t) {
    log_.push_back({t, res, ev, subj});
  }
  std::int64_t dev_ns(void* ev) const {
    float ms = 0;
    must(ptk_event_elapsed_ms(base_, ev, &ms), "elapsed");
    return static_cast<std::int64_t>(static_cast<double>(ms) * 1e6);
  }
  void* chunk_slot(int c) {
    // non-persistent chunks reuse the gathered slot for gradients (quirk Q5:
    // the model charges a buffer only for the working copy)
    const ChunkStore& st = store_[c];
    return st.persistent ? nullptr : slots_[core_->pool().slot_of(c)].p;
  }
  void* chunk_dev_params(int c) { return store_[c].persistent ? store_[c].d_param.p : chunk_slot(c); }
  void* chunk_dev_grads(int c) { return store_[c].persistent ? store_[c].d_grad.p : chunk_slot(c); }

  Pending& launch(Pending::What what, void* stream, int chunk, int block, int op) {
    pending_.push_back({what, chunk, block, op, new_event(), new_event()});
    must(ptk_event_record(pending_.back().start, stream), "record");
    return pending_.back();
  }
  void finish_launch(Pending& p, void* stream) { must(ptk_event_record(p.end, stream), "record"); }

  bool issue_prefetch(std::int64_t t);
  void swap_out_from(int b, int i, std::int64_t t);
  void swap_in_from(int b, int i, std::int64_t t);
  void release_swap_ins(std::int64_t t);
  void drain(int c, std::int64_t t);
  void reduced(int c, std::int64_t t);
  bool start_gpu(std::int64_t t);
  void finish_gpu(std::int64_t t);
  bool start_cpu(std::int64_t t);
  void complete(const Pending& p, std::int64_t t_end);

  const ModelTrace& tr_;
  const ChunkLayout& lay_;
  const BlockSchedule& sch_;
  const PlanConfig& cfg_;
  const HardwareProfile& hw_;
  ExecOptions opt_;
  HostOptimizer host_opt_;
  int w_ = 1;
  int step_ = 1;
  void *s_gpu_ = nullptr, *s_h2d_ = nullptr, *s_d2h_ = nullptr, *s_coll_ = nullptr;
  std::vector<void*> events_, free_events_;
  void* base_ = nullptr;

  int nops_ = 0, nc_ = 0, nblk_ = 0;
  std::vector<ChunkStore> store_;
  std::vector<DeviceBuf> slots_;
  DeviceBuf swap_dev_, ws_, stats_dev_;
  HostBuf swap_host_;
  std::vector<void*> act_dev_, act_host_;
  std::int64_t device_bytes_ = 0, host_bytes_ = 0;
  ExecutionStats stats_;

  // iteration state: every decision is the shared policy's (policy.hpp)
  std::optional<IterationCore> core_;
  std::size_t next_launch_ = 0;  // next GPU job to put on the compute stream
  static constexpr std::size_t kRunAhead = 4;  // GPU jobs queued ahead (hides launch gaps)
  int fetch_parts_left_ = 0;
  bool gpu_busy_ = false;
  std::deque<int> host_queue_;
  bool cpu_busy_ = false;
  std::int64_t cpu_first_ = -1, cpu_last_ = 0;
  std::int64_t fwd_end_ = 0, bwd_end_ = 0, gpu_end_ = 0;
  std::vector<TimelineEvent> log_;
  std::deque<Pending> pending_;
  std::int64_t t0_host_ = 0;
  int cpu_start_note_ = -1;
};

void Runtime::prepare_iteration() {
  // the optimizer jobs' time is measured, not modelled (rate 0)
  core_.emplace(tr_, lay_, sch_, cfg_, 0.0);
  next_launch_ = 0;
  log_.clear();
  fetch_parts_left_ = 0;
  gpu_busy_ = cpu_busy_ = false;
  host_queue_.clear();
  cpu_first_ = -1;
  cpu_last_ = fwd_end_ = bwd_end_ = gpu_end_ = 0;
}

bool Runtime::issue_prefetch(std::int64_t t) {
  // the chunks of every GPU job already on the stream (and the next one) stay
  std::vector<int> pinned;
  const auto& jobs = core_->jobs();
  for (std::size_t k = core_->cursor(); k <= next_launch_ && k < jobs.size(); ++k)
    pinned.push_back(jobs[k].chunk);
  const auto d = core_->pool().next_fetch(core_->position(), pinned);
  if (d.step == ChunkBufferPool::FetchStep::Nothing) return false;
  if (d.step == ChunkBufferPool::FetchStep::Skipped) return true;
  if (d.grant.evicted != 0) note("gpu", "evict", "chunk=" + std::to_string(d.grant.evicted), t);
  const int c = d.grant.chunk;
  ChunkStore& st = store_[c];
  // upload this rank's shard into its place in the slot, then all-gather
  char* dst = static_cast<char*>(chunk_dev_params(c)) + 2 * st.shard * opt_.rank;
  Pending& up = launch(Pending::Upload, s_h2d_, c, -1, -1);
  must(ptk_memcpy_h2d_async(dst, st.h_param.p, 2 * st.shard, s_h2d_), "upload");
  finish_launch(up, s_h2d_);
  stats_.h2d_bytes += 2 * st.shard;
  note("h2d", "upload_start", "chunk=" + std::to_string(c), t);
  up.start_note = static_cast<int>(log_.size()) - 1;
  fetch_parts_left_ = 1;
  if (w_ > 1) {
    must(ptk_stream_wait_event(s_coll_, up.end), "wait");
    Pending& ag = launch(Pending::Gather, s_coll_, c, -1, -1);
    must(ptk_chunk_allgather(static_cast<ptk_comm*>(opt_.comm), chunk_dev_params(c), st.shard, 0,
                             s_coll_), "allgather");
    finish_launch(ag, s_coll_);
    stats_.coll_bytes += 2 * st.shard * (w_ - 1);
    note("coll", "gather_start", "chunk=" + std::to_string(c), t);
    ag.start_note = static_cast<int>(log_.size()) - 1;
    fetch_parts_left_ = 2;
  }
  return true;
}

void Runtime::swap_out_from(int b, int i, std::int64_t t) {
  const int op = core_->swap_out_next(b, i);
  if (op < 0) {
    note("d2h", "swap_out_done", "block=" + std::to_string(b), t);
    return;
  }
  Pending& p = launch(Pending::SwapOut, s_d2h_, 0, b, op);
  must(ptk_memcpy_d2h_async(act_host_[op], act_dev_[op], tr_.ops[op].act_bytes, s_d2h_), "swap out");
  finish_launch(p, s_d2h_);
  stats_.d2h_bytes += tr_.ops[op].act_bytes;
  note("d2h", "swap_out_start", "block=" + std::to_string(b) + " op=" + std::to_string(op), t);
  p.start_note = static_cast<int>(log_.size()) - 1;
}

void Runtime::swap_in_from(int b, int i, std::int64_t t) {
  const int op = core_->swap_in_next(b, i);
  if (op < 0) {
    note("h2d", "swap_in_done", "block=" + std::to_string(b), t);
    return;
  }
  Pending& p = launch(Pending::SwapIn, s_h2d_, 0, b, op);
  must(ptk_memcpy_h2d_async(act_dev_[op], act_host_[op], tr_.ops[op].act_bytes, s_h2d_), "swap in");
  finish_launch(p, s_h2d_);
  stats_.h2d_bytes += tr_.ops[op].act_bytes;
  note("h2d", "swap_in_start", "block=" + std::to_string(b) + " op=" + std::to_string(op), t);
  p.start_note = static_cast<int>(log_.size()) - 1;
}

void Runtime::release_swap_ins(std::int64_t t) {
  for (const int b : core_->swap_ins_due()) swap_in_from(b, core_->block_last(b), t);
}

void Runtime::drain(int c, std::int64_t t) {
  ChunkStore& st = store_[c];
  if (w_ > 1) {
    // the gradient chunk is complete on the compute stream: reduce-scatter it
    void* ready = new_event();
    must(ptk_event_record(ready, s_gpu_), "record");
    must(ptk_stream_wait_event(s_coll_, ready), "wait");
    free_events_.push_back(ready);
    Pending& rs = launch(Pending::Reduce, s_coll_, c, -1, -1);
    must(ptk_chunk_reduce_scatter(static_cast<ptk_comm*>(opt_.comm), chunk_dev_grads(c), st.shard,
                                  0, s_coll_), "reduce_scatter");
    finish_launch(rs, s_coll_);
    stats_.coll_bytes += 2 * st.shard * (w_ - 1);
    note("coll", "reduce_start", "chunk=" + std::to_string(c), t);
    rs.start_note = static_cast<int>(log_.size()) - 1;
  } else {
    reduced(c, t);
  }
}

void Runtime::reduced(int c, std::int64_t t) {
  if (!core_->reduced(c)) return;  // persistent: its device optimizer job is now ready
  ChunkStore& st = store_[c];
  void* after = new_event();
  must(ptk_event_record(after, w_ > 1 ? s_coll_ : s_gpu_), "record");
  must(ptk_stream_wait_event(s_d2h_, after), "wait");
  free_events_.push_back(after);
  const char* src = static_cast<const char*>(chunk_dev_grads(c)) + 2 * st.shard * opt_.rank;
  Pending& off = launch(Pending::Offload, s_d2h_, c, -1, -1);
  must(ptk_memcpy_d2h_async(st.h_grad.p, src, 2 * st.shard, s_d2h_), "offload");
  finish_launch(off, s_d2h_);
  stats_.d2h_bytes += 2 * st.shard;
  note("d2h", "offload_start", "chunk=" + std::to_string(c), t);
  off.start_note = static_cast<int>(log_.size()) - 1;
}

// Queues the next GPU job if it is ready. Up to kRunAhead jobs sit on the
// compute stream at once (stream order keeps them serial, as the simulator's
// single GPU queue); readiness can only be lost by eviction, and queued jobs'
// chunks are pinned against eviction.
bool Runtime::start_gpu(std::int64_t t) {
  const auto& jobs = core_->jobs();
  if (next_launch_ >= jobs.size() || next_launch_ - core_->cursor() >= kRunAhead) return false;
  const Job& j = jobs[next_launch_];
  if (!core_->ready(j)) return false;
  ++next_launch_;
  core_->start(j, t);
  Pending& p = launch(Pending::Gpu, s_gpu_, j.chunk, j.block, j.op);
  const auto busy = [&](double sec) {
    must(ptk_busy_wait(static_cast<std::int64_t>(sec * opt_.compute_scale * 1e9), s_gpu_), "busy");
  };
  switch (j.kind) {
    case Job::Recompute:
      note("gpu", "recompute_start", "block=" + std::to_string(j.block), t);
      busy(j.seconds);
      break;
    case Job::Backward:
      note("gpu", "bwd_start", "op=" + std::to_string(j.op), t);
      busy(j.seconds);
      break;
    case Job::Forward:
      note("gpu", "fwd_start", "op=" + std::to_string(j.op), t);
      busy(j.seconds);
      break;
    case Job::Optimizer: {
      note("gpu", "optim_start", "chunk=" + std::to_string(j.chunk), t);
      ChunkStore& st = store_[j.chunk];
      const ptk_adam_config a = adam(1.0 / w_);
      must(ptk_chunk_adam(&a, static_cast<float*>(st.d_master.p), static_cast<float*>(st.d_m.p),
                          static_cast<float*>(st.d_v.p),
                          static_cast<const uint16_t*>(st.d_grad.p) + st.shard * opt_.rank,
                          static_cast<uint16_t*>(st.d_param.p) + st.shard * opt_.rank, st.shard,
                          static_cast<ptk_grad_stats_t*>(stats_dev_.p), ws_.p, nullptr, nullptr,
                          s_gpu_), "chunk adam");
      if (w_ > 1)
        must(ptk_chunk_allgather(static_cast<ptk_comm*>(opt_.comm), st.d_param.p, st.shard, 0,
                                 s_gpu_), "allgather");
      break;
    }
  }
  p.start_note = static_cast<int>(log_.size()) - 1;
  finish_launch(p, s_gpu_);
  gpu_busy_ = true;
  return true;
}

void Runtime::finish_gpu(std::int64_t t) {
  const IterationCore::Finished f = core_->finish(t);
  gpu_busy_ = core_->cursor() < next_launch_;
  gpu_end_ = t;
  const Job& j = f.job;
  switch (j.kind) {
    case Job::Forward:
      if (f.swap_out_block >= 0) swap_out_from(f.swap_out_block, core_->block_first(f.swap_out_block), t);
      note("gpu", "fwd_end", "op=" + std::to_string(j.op), t);
      fwd_end_ = t;
      break;
    case Job::Backward:
      note("gpu", "bwd_end", "op=" + std::to_string(j.op), t);
      bwd_end_ = t;
      break;
    case Job::Recompute:
      note("gpu", "recompute_end", "block=" + std::to_string(j.block), t);
      bwd_end_ = t;
      break;
    case Job::Optimizer:
      note("gpu", "optim_end", "chunk=" + std::to_string(j.chunk), t);
      break;
  }
  if (f.drain_chunk != 0) drain(f.drain_chunk, t);
}

bool Runtime::start_cpu(std::int64_t t) {
  if (cpu_busy_ || host_queue_.empty()) return false;
  const int c = host_queue_.front();
  host_queue_.pop_front();
  cpu_busy_ = true;
  if (cpu_first_ < 0) cpu_first_ = t;
  note("cpu", "update_start", "chunk=" + std::to_string(c), t);
  cpu_start_note_ = static_cast<int>(log_.size()) - 1;
  host_opt_.submit(c, &store_[c], adam(1.0 / w_));
  return true;
}

void Runtime::complete(const Pending& p, std::int64_t t) {
  const std::string tag = "chunk=" + std::to_string(p.chunk);
  switch (p.what) {
    case Pending::Gpu:
      finish_gpu(t);
      break;
    case Pending::Upload:
    case Pending::Gather:
      note(p.what == Pending::Upload ? "h2d" : "coll",
           p.what == Pending::Upload ? "upload_end" : "gather_end", tag, t);
      if (--fetch_parts_left_ == 0) core_->pool().arrived(p.chunk);
      break;
    case Pending::Reduce:
      note("coll", "reduce_end", tag, t);
      reduced(p.chunk, t);
      break;
    case Pending::Offload:
      note("d2h", "offload_end", tag, t);
      core_->offloaded(p.chunk);  // the slot is free again
      host_queue_.push_back(p.chunk);
      break;
    case Pending::SwapOut:
      core_->swapped_out(p.op, t);
      note("d2h", "swap_out_end", "block=" + std::to_string(p.block) + " op=" + std::to_string(p.op), t);
      swap_out_from(p.block, p.op + 1, t);
      break;
    case Pending::SwapIn:
      core_->swapped_in(p.op, t);
      note("h2d", "swap_in_end", "block=" + std::to_string(p.block) + " op=" + std::to_string(p.op), t);
      swap_in_from(p.block, p.op - 1, t);
      break;
  }
}

SimulationResult Runtime::iterate() {
  must(ptk_device_synchronize(), "sync");
  prepare_iteration();
  base_ = new_event();
  must(ptk_event_record(base_, s_gpu_), "record");
  must(ptk_stream_synchronize(s_gpu_), "sync");
  t0_host_ = host_ns();
  std::int64_t now = 0;
  for (;;) {
    for (bool moved = true; moved;) {
      moved = false;
      moved |= start_gpu(now);
      moved |= start_cpu(now);
      moved |= issue_prefetch(now);
      release_swap_ins(now);
    }
    const bool work_left = !core_->finished() || !host_queue_.empty() || cpu_busy_ ||
                           !pending_.empty();
    if (!work_left) break;
    if (pending_.empty() && !cpu_busy_)
      throw DeadlockDetected("executor: no runnable operation with the iteration incomplete");
    // wait for the earliest completion (device events or the host optimizer)
    for (;;) {
      bool any = false;
      std::int64_t best_t = std::numeric_limits<std::int64_t>::max();
      std::size_t best_i = pending_.size();
      for (std::size_t i = 0; i < pending_.size(); ++i) {
        if (cudaEventQuery(static_cast<cudaEvent_t>(pending_[i].end)) != cudaSuccess) continue;
        const std::int64_t t = dev_ns(pending_[i].end);
        if (!any || t < best_t) {
          any = true;
          best_t = t;
          best_i = i;
        }
      }
      auto done = host_opt_.drain_done();
      for (auto& [c, s, e] : done) {
        const std::int64_t te = e - t0_host_;
        stats_.cpu_optim_ns += e - s;
        if (cpu_start_note_ >= 0) log_[cpu_start_note_].time_ns = s - t0_host_;
        if (cpu_first_ >= 0 && cpu_first_ > s - t0_host_) cpu_first_ = s - t0_host_;
        now = std::max(now, te);
        cpu_busy_ = false;
        cpu_last_ = te;
        note("cpu", "update_end", "chunk=" + std::to_string(c), te);
        any = true;
        best_i = pending_.size();  // handle the host completion first
        break;
      }
      if (!done.empty()) break;
      if (any) {
        Pending p = pending_[best_i];
        pending_.erase(pending_.begin() + static_cast<std::ptrdiff_t>(best_i));
        now = std::max(now, best_t);
        if (p.what == Pending::Gpu && !core_->finished() &&
            core_->jobs()[core_->cursor()].kind == Job::Optimizer)
          stats_.gpu_optim_ns += dev_ns(p.end) - dev_ns(p.start);
        if (p.start_note >= 0) log_[p.start_note].time_ns = dev_ns(p.start);
        complete(p, best_t);
        free_events_.push_back(p.start);
        free_events_.push_back(p.end);
        break;
      }
      std::this_thread::yield();  // busy-poll: completions are usually microseconds apart
    }
  }
  free_events_.push_back(base_);
  SimulationResult r;
  r.t_fwd = static_cast<double>(fwd_end_) * 1e-9;
  r.t_bwd = static_cast<double>(std::max<std::int64_t>(0, bwd_end_ - fwd_end_)) * 1e-9;
  r.t_iter = static_cast<double>(std::max(gpu_end_, cpu_last_)) * 1e-9;
  r.t_cpu_optim_span = cpu_first_ >= 0 ? static_cast<double>(cpu_last_ - cpu_first_) * 1e-9 : 0.0;
  r.m_peak = core_->ledger().high();
  std::stable_sort(log_.begin(), log_.end(),
                   [](const TimelineEvent& a, const TimelineEvent& b) { return a.time_ns < b.time_ns; });
  r.timeline = log_;
  r.mem_trace = core_->ledger().samples();
  return r;
}

}  // namespace

ExecutionResult execute(const ModelTrace& trace, const ChunkLayout& layout,
                        const BlockSchedule& schedule, const PlanConfig& config,
                        const HardwareProfile& hw, const ExecOptions& opts) {
  hw.validate();
  config.validate();
  if (static_cast<int>(schedule.strategies.size()) != trace.n_blocks)
    throw InvariantViolation("schedule size does not match trace block count");
  if (config.n_chunk != layout.n_chunk())
    throw InvariantViolation("config n_chunk does not match layout");
  Runtime rt(trace, layout, schedule, config, hw, opts);
  return rt.run(opts.iterations);
}

}  // namespace memplan
