// The chunk runtime: executes one training iteration of a plan on the
// device with the simulator's decisions and measured times (execute.hpp).
//
// Policy (identical decisions to the simulator, csrc/planner/simulator.cpp,
// which restates proj/src/sim.cpp:99-685):
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
#include <stdexcept>
#include <thread>

#include "memplan/accounting.hpp"
#include "memplan/errors.hpp"
#include "memplan/execute.hpp"
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

enum class Where { Away, Arriving, Here, Leaving };

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
  enum class Kind { Fwd, Bwd, Recompute, Optim };
  struct Job {
    Kind kind;
    int op;
    int block;
    int chunk;
    double seconds;
    int slot;
  };
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
  SimulationResult iterate();
  void prepare_iteration();
  int fwd_slot(int c) const { return c; }
  int bwd_slot(int c) const { return 2 * nc_ - c + 1; }
  int chunk_in_slot(int p) const { return p <= nc_ ? p : 2 * nc_ - p + 1; }
  int slot_now() const { return next_ < jobs_.size() ? jobs_[next_].slot : 2 * nc_ + 2; }
  int next_use(int c) const {
    const int p = slot_now();
    if (fwd_slot(c) >= p) return fwd_slot(c);
    if (bwd_slot(c) >= p) return bwd_slot(c);
    return std::numeric_limits<int>::max();
  }
  BlockStrategy policy(const OperatorRecord& op) const {
    return op.block_id ? sch_.strategies[*op.block_id] : BlockStrategy::None;
  }
  void note(const char* res, const std::string& ev, const std::string& subj, std::int64_t t) {
    log_.push_back({t, res, ev, subj});
  }
  void alloc(std::int64_t d, std::int64_t t) {
    held_ += d;
    if (held_ < 0) throw LedgerUnderflow("allocated bytes went negative");
    high_ = std::max(high_, held_);
    if (!mem_.empty() && mem_.back().time_ns == t)
      mem_.back().bytes = held_;
    else
      mem_.push_back({t, held_});
  }
  std::int64_t dev_ns(void* ev) const {
    float ms = 0;
    must(ptk_event_elapsed_ms(base_, ev, &ms), "elapsed");
    return static_cast<std::int64_t>(static_cast<double>(ms) * 1e6);
  }
  void* chunk_dev_params(int c) {
    ChunkStore& st = store_[c];
    return st.persistent ? st.d_param.p : slots_[slot_of_[c]].p;
  }
  void* chunk_dev_grads(int c) {
    // non-persistent chunks reuse the gathered slot for gradients (quirk Q5:
    // the model charges a buffer only for the working copy)
    ChunkStore& st = store_[c];
    return st.persistent ? st.d_grad.p : slots_[slot_of_[c]].p;
  }

  Pending& launch(Pending::What what, void* stream, int chunk, int block, int op) {
    pending_.push_back({what, chunk, block, op, new_event(), new_event()});
    must(ptk_event_record(pending_.back().start, stream), "record");
    return pending_.back();
  }
  void finish_launch(Pending& p, void* stream) { must(ptk_event_record(p.end, stream), "record"); }

  void enqueue_until(int slot);
  bool issue_prefetch(std::int64_t t);
  void swap_out_from(int b, int i, std::int64_t t);
  void swap_in_from(int b, int i, std::int64_t t);
  void release_swap_ins(std::int64_t t);
  void drain(int c, std::int64_t t);
  void reduced(int c, std::int64_t t);
  bool ready(const Job& j) const;
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
  std::vector<int> free_slot_ids_;
  std::vector<int> slot_of_;
  DeviceBuf swap_dev_, ws_, stats_dev_;
  HostBuf swap_host_;
  std::vector<void*> act_dev_, act_host_;
  std::int64_t device_bytes_ = 0, host_bytes_ = 0;
  ExecutionStats stats_;

  // iteration state (mirrors the simulator)
  std::vector<Job> jobs_;
  std::size_t next_ = 0;         // oldest unfinished GPU job (the simulator's next_task)
  std::size_t next_launch_ = 0;  // next GPU job to put on the compute stream
  static constexpr std::size_t kRunAhead = 4;  // GPU jobs queued ahead (hides launch gaps)
  std::vector<Where> where_;
  std::vector<int> bwd_left_;
  std::vector<char> reduce_done_;
  std::deque<int> fetch_queue_;
  int fetching_ = 0;
  int fetch_parts_left_ = 0;
  int enqueued_ = 0;
  std::vector<std::int64_t> blk_act_;
  std::vector<int> blk_first_, blk_last_;
  std::vector<double> blk_fwd_;
  std::vector<char> out_done_, in_issued_, act_back_;
  int lowest_entered_ = std::numeric_limits<int>::max();
  bool in_backward_ = false;
  bool gpu_busy_ = false;
  std::deque<int> host_queue_;
  bool cpu_busy_ = false;
  std::int64_t cpu_first_ = -1, cpu_last_ = 0;
  std::int64_t fwd_end_ = 0, bwd_end_ = 0, gpu_end_ = 0;
  std::int64_t held_ = 0, high_ = 0;
  std::vector<MemSample> mem_;
  std::vector<TimelineEvent> log_;
  std::deque<Pending> pending_;
  std::int64_t t0_host_ = 0;
  int cpu_start_note_ = -1;
};

void Runtime::prepare_iteration() {
  jobs_.clear();
  next_ = 0;
  next_launch_ = 0;
  log_.clear();
  mem_.clear();
  held_ = high_ = 0;
  const std::size_t nb = static_cast<std::size_t>(std::max(1, nblk_));
  blk_act_.assign(nb, 0);
  blk_first_.assign(nb, -1);
  blk_last_.assign(nb, -1);
  blk_fwd_.assign(nb, 0.0);
  for (const OperatorRecord& op : tr_.ops) {
    if (!op.block_id) continue;
    const int b = *op.block_id;
    blk_act_[b] += op.act_bytes;
    if (blk_first_[b] < 0) blk_first_[b] = op.index;
    blk_last_[b] = op.index;
    blk_fwd_[b] += op.t_fwd;
  }
  std::vector<int> op_chunk(nops_);
  for (int i = 0; i < nops_; ++i) op_chunk[i] = lay_.chunk_of_op(i);
  for (int i = 0; i < nops_; ++i)
    jobs_.push_back({Kind::Fwd, i, tr_.ops[i].block_id.value_or(-1), op_chunk[i], tr_.ops[i].t_fwd,
                     fwd_slot(op_chunk[i])});
  for (int i = nops_ - 1; i >= 0; --i) {
    const OperatorRecord& op = tr_.ops[i];
    if (op.block_id && policy(op) == BlockStrategy::Checkpoint && i == blk_last_[*op.block_id])
      jobs_.push_back({Kind::Recompute, -1, *op.block_id, op_chunk[i], blk_fwd_[*op.block_id],
                       bwd_slot(op_chunk[i])});
    jobs_.push_back({Kind::Bwd, i, op.block_id.value_or(-1), op_chunk[i], op.t_bwd,
                     bwd_slot(op_chunk[i])});
  }
  for (int c = 1; c <= cfg_.n_persist; ++c) jobs_.push_back({Kind::Optim, -1, -1, c, 0.0, 2 * nc_ + 1});
  where_.assign(nc_ + 1, Where::Away);
  for (int c = 1; c <= cfg_.n_persist; ++c) where_[c] = Where::Here;
  bwd_left_.assign(nc_ + 1, 0);
  for (const Job& j : jobs_)
    if (j.kind == Kind::Bwd || j.kind == Kind::Recompute) ++bwd_left_[j.chunk];
  reduce_done_.assign(nc_ + 1, 0);
  fetch_queue_.clear();
  fetching_ = 0;
  enqueued_ = 0;
  out_done_.assign(nb, 0);
  in_issued_.assign(nb, 0);
  act_back_.assign(nops_, 0);
  lowest_entered_ = std::numeric_limits<int>::max();
  in_backward_ = false;
  gpu_busy_ = cpu_busy_ = false;
  host_queue_.clear();
  cpu_first_ = -1;
  cpu_last_ = fwd_end_ = bwd_end_ = gpu_end_ = 0;
  slot_of_.assign(nc_ + 1, -1);
  free_slot_ids_.clear();
  for (int i = cfg_.n_buffer - 1; i >= 0; --i) free_slot_ids_.push_back(i);
}

void Runtime::enqueue_until(int slot) {
  const int upto = std::min(slot, 2 * nc_);
  for (int p = enqueued_ + 1; p <= upto; ++p) {
    const int c = chunk_in_slot(p);
    if (where_[c] == Where::Away &&
        std::find(fetch_queue_.begin(), fetch_queue_.end(), c) == fetch_queue_.end())
      fetch_queue_.push_back(c);
  }
  enqueued_ = std::max(enqueued_, upto);
}

bool Runtime::issue_prefetch(std::int64_t t) {
  if (fetching_ != 0 || fetch_queue_.empty()) return false;
  const int c = fetch_queue_.front();
  if (where_[c] != Where::Away) {
    fetch_queue_.pop_front();
    return true;
  }
  if (free_slot_ids_.empty()) {
    // never evict a chunk a queued or next-to-queue GPU job uses
    const auto pinned = [&](int v) {
      for (std::size_t k = next_; k <= next_launch_ && k < jobs_.size(); ++k)
        if (jobs_[k].chunk == v) return true;
      return false;
    };
    int victim = 0, victim_use = -1;
    for (int v = cfg_.n_persist + 1; v <= nc_; ++v) {
      if (where_[v] != Where::Here || pinned(v)) continue;
      const int use = next_use(v);
      if (use > victim_use) {
        victim_use = use;
        victim = v;
      }
    }
    if (victim == 0 || victim_use <= next_use(c)) return false;
    where_[victim] = Where::Away;
    free_slot_ids_.push_back(slot_of_[victim]);
    slot_of_[victim] = -1;
    note("gpu", "evict", "chunk=" + std::to_string(victim), t);
  }
  fetch_queue_.pop_front();
  slot_of_[c] = free_slot_ids_.back();
  free_slot_ids_.pop_back();
  where_[c] = Where::Arriving;
  fetching_ = c;
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
  while (i <= blk_last_[b] && tr_.ops[i].act_bytes == 0) ++i;
  if (i > blk_last_[b]) {
    out_done_[b] = 1;
    note("d2h", "swap_out_done", "block=" + std::to_string(b), t);
    return;
  }
  Pending& p = launch(Pending::SwapOut, s_d2h_, 0, b, i);
  must(ptk_memcpy_d2h_async(act_host_[i], act_dev_[i], tr_.ops[i].act_bytes, s_d2h_), "swap out");
  finish_launch(p, s_d2h_);
  stats_.d2h_bytes += tr_.ops[i].act_bytes;
  note("d2h", "swap_out_start", "block=" + std::to_string(b) + " op=" + std::to_string(i), t);
  p.start_note = static_cast<int>(log_.size()) - 1;
}

void Runtime::swap_in_from(int b, int i, std::int64_t t) {
  for (; i >= blk_first_[b] && tr_.ops[i].act_bytes == 0; --i) act_back_[i] = 1;
  if (i < blk_first_[b]) {
    note("h2d", "swap_in_done", "block=" + std::to_string(b), t);
    return;
  }
  Pending& p = launch(Pending::SwapIn, s_h2d_, 0, b, i);
  must(ptk_memcpy_h2d_async(act_dev_[i], act_host_[i], tr_.ops[i].act_bytes, s_h2d_), "swap in");
  finish_launch(p, s_h2d_);
  stats_.h2d_bytes += tr_.ops[i].act_bytes;
  note("h2d", "swap_in_start", "block=" + std::to_string(b) + " op=" + std::to_string(i), t);
  p.start_note = static_cast<int>(log_.size()) - 1;
}

void Runtime::release_swap_ins(std::int64_t t) {
  for (int b = 0; b < nblk_; ++b) {
    if (sch_.strategies[b] != BlockStrategy::Swap || in_issued_[b] || !out_done_[b]) continue;
    const int entered =
        in_backward_ ? std::min(lowest_entered_, nblk_) : std::numeric_limits<int>::max();
    const bool near = entered <= b + cfg_.n_interval;
    const bool room = (high_ - held_) >= blk_act_[b];
    const bool needed = next_ < jobs_.size() && jobs_[next_].kind == Kind::Bwd && jobs_[next_].block == b;
    if ((near && room) || needed) {
      in_issued_[b] = 1;
      swap_in_from(b, blk_last_[b], t);
    }
  }
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
  ChunkStore& st = store_[c];
  if (st.persistent) {
    reduce_done_[c] = 1;
    return;
  }
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

bool Runtime::ready(const Job& j) const {
  const auto present = [&](int c) { return where_[c] == Where::Here || where_[c] == Where::Leaving; };
  switch (j.kind) {
    case Kind::Fwd:
    case Kind::Recompute:
      return present(j.chunk);
    case Kind::Bwd:
      if (!present(j.chunk)) return false;
      return !(j.block >= 0 && sch_.strategies[j.block] == BlockStrategy::Swap &&
               tr_.ops[j.op].act_bytes > 0 && !act_back_[j.op]);
    case Kind::Optim:
      return reduce_done_[j.chunk] != 0;
  }
  return false;
}

// Queues the next GPU job if it is ready. Up to kRunAhead jobs sit on the
// compute stream at once (stream order keeps them serial, as the simulator's
// single GPU queue); readiness can only be lost by eviction, and queued jobs'
// chunks are pinned against eviction.
bool Runtime::start_gpu(std::int64_t t) {
  if (next_launch_ >= jobs_.size() || next_launch_ - next_ >= kRunAhead) return false;
  const Job& j = jobs_[next_launch_];
  if (!ready(j)) return false;
  ++next_launch_;
  enqueue_until(j.slot + 1);
  if (j.kind == Kind::Bwd || j.kind == Kind::Recompute) {
    in_backward_ = true;
    if (j.block >= 0) lowest_entered_ = std::min(lowest_entered_, j.block);
  }
  Pending& p = launch(Pending::Gpu, s_gpu_, j.chunk, j.block, j.op);
  const auto busy = [&](double sec) {
    must(ptk_busy_wait(static_cast<std::int64_t>(sec * opt_.compute_scale * 1e9), s_gpu_), "busy");
  };
  switch (j.kind) {
    case Kind::Recompute:
      alloc(blk_act_[j.block] - tr_.ops[blk_first_[j.block]].act_bytes, t);
      note("gpu", "recompute_start", "block=" + std::to_string(j.block), t);
      busy(j.seconds);
      break;
    case Kind::Bwd: {
      const OperatorRecord& op = tr_.ops[j.op];
      high_ = std::max(high_, held_ + op.d_peak_prior);
      if (op.d_cur_prior != 0) alloc(op.d_cur_prior, t);
      high_ = std::max(high_, held_ + op.d_peak_op);
      note("gpu", "bwd_start", "op=" + std::to_string(j.op), t);
      busy(j.seconds);
      break;
    }
    case Kind::Fwd:
      note("gpu", "fwd_start", "op=" + std::to_string(j.op), t);
      busy(j.seconds);
      break;
    case Kind::Optim: {
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
  const Job j = jobs_[next_];
  ++next_;
  gpu_busy_ = next_ < next_launch_;
  gpu_end_ = t;
  const auto chunk_done = [&](int c) {
    if (--bwd_left_[c] != 0) return;
    if (c > cfg_.n_persist) where_[c] = Where::Leaving;
    drain(c, t);
  };
  switch (j.kind) {
    case Kind::Fwd: {
      const OperatorRecord& op = tr_.ops[j.op];
      const BlockStrategy pol = policy(op);
      const bool first = op.block_id && j.op == blk_first_[*op.block_id];
      const bool keep = pol == BlockStrategy::None || pol == BlockStrategy::Swap ||
                        (pol == BlockStrategy::Checkpoint && first);
      if (keep && op.act_bytes > 0) alloc(op.act_bytes, t);
      if (op.block_id && j.op == blk_last_[*op.block_id] && pol == BlockStrategy::Swap)
        swap_out_from(*op.block_id, blk_first_[*op.block_id], t);
      note("gpu", "fwd_end", "op=" + std::to_string(j.op), t);
      fwd_end_ = t;
      break;
    }
    case Kind::Bwd: {
      const OperatorRecord& op = tr_.ops[j.op];
      if (op.d_cur_op != 0) alloc(op.d_cur_op, t);
      if (op.act_bytes > 0) alloc(-op.act_bytes, t);
      note("gpu", "bwd_end", "op=" + std::to_string(j.op), t);
      bwd_end_ = t;
      chunk_done(j.chunk);
      break;
    }
    case Kind::Recompute:
      note("gpu", "recompute_end", "block=" + std::to_string(j.block), t);
      bwd_end_ = t;
      chunk_done(j.chunk);
      break;
    case Kind::Optim:
      note("gpu", "optim_end", "chunk=" + std::to_string(j.chunk), t);
      break;
  }
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
      if (--fetch_parts_left_ == 0) {
        where_[p.chunk] = Where::Here;
        if (fetching_ == p.chunk) fetching_ = 0;
      }
      break;
    case Pending::Reduce:
      note("coll", "reduce_end", tag, t);
      reduced(p.chunk, t);
      break;
    case Pending::Offload:
      note("d2h", "offload_end", tag, t);
      where_[p.chunk] = Where::Away;
      free_slot_ids_.push_back(slot_of_[p.chunk]);
      slot_of_[p.chunk] = -1;
      host_queue_.push_back(p.chunk);
      break;
    case Pending::SwapOut:
      alloc(-tr_.ops[p.op].act_bytes, t);
      note("d2h", "swap_out_end", "block=" + std::to_string(p.block) + " op=" + std::to_string(p.op), t);
      swap_out_from(p.block, p.op + 1, t);
      break;
    case Pending::SwapIn:
      alloc(tr_.ops[p.op].act_bytes, t);
      act_back_[p.op] = 1;
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
  // model states + residual floor
  alloc(device_state_bytes(cfg_) + tr_.m_fwd,
        0);
  enqueue_until(1);
  std::int64_t now = 0;
  for (;;) {
    for (bool moved = true; moved;) {
      moved = false;
      moved |= start_gpu(now);
      moved |= start_cpu(now);
      moved |= issue_prefetch(now);
      release_swap_ins(now);
    }
    const bool work_left = next_ < jobs_.size() || !host_queue_.empty() || cpu_busy_ ||
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
        if (p.what == Pending::Gpu && tr_.ops.size() && jobs_[next_].kind == Kind::Optim)
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
  r.m_peak = high_;
  std::stable_sort(log_.begin(), log_.end(),
                   [](const TimelineEvent& a, const TimelineEvent& b) { return a.time_ns < b.time_ns; });
  r.timeline = log_;
  r.mem_trace = mem_;
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
