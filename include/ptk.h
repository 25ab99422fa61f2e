/* ptk.h — C-ABI of the B200 chunk data plane (libptk.so, sm_100a).
 *
 * This is the drop-in boundary BELOW the reference's planner API. The
 * reference (memplan, /root/reference/proj) only MODELS these operations; each
 * entry point replaces one modeled quantity with the real byte movement:
 *
 *   ptk_chunk_adam            <- GPU optimizer time `persist_params / gpu_optim_rate`
 *                                (proj/src/cost.cpp:206-219) and the Sim `GpuOptim`
 *                                task per persistent chunk (proj/src/sim.cpp:245-250)
 *   ptk_grad_prep/_stats      <- "gradient-chunk cast/scale" of north_star (not modeled)
 *   ptk_chunk_allgather       <- `gather_time(used_bytes)` (proj/src/hardware.cpp:29-34),
 *                                Sim Gather (proj/src/sim.cpp:335-338)
 *   ptk_chunk_reduce_scatter  <- `reduce_time(used_bytes)` (proj/src/hardware.cpp:36-38),
 *                                Sim Reduce (proj/src/sim.cpp:428-436)
 *   ptk_fused_rs_adam_ag      <- reduce_time + GpuOptim + next gather, as ONE kernel
 *                                over NVLink peer memory (P2P loads / stores)
 *   ptk_cpu_adam              <- CPU optimizer `nonpersist_params / cpu_optim_rate`
 *                                (proj/src/cost.cpp:213-218, proj/src/sim.cpp:446-451)
 *   ptk_memcpy_h2d/d2h_async  <- `transfer_time(shard_bytes, h2d/d2h)` upload/offload
 *                                (proj/src/cost.cpp:126-127,186-187; sim.cpp:352-368)
 *   ptk_profile_*             <- the calibration constants of HardwareProfile
 *                                (proj/include/memplan/hardware.hpp:15-27)
 *   ptk_execute_plan          <- memplan::simulate (proj/include/memplan/sim.hpp:48-50),
 *                                executed with real transfers and kernels
 *
 * Conventions: plain pointers and sizes only; the caller owns
 * all memory; every call is asynchronous and stream-ordered on the given
 * cudaStream_t (passed as void*; NULL = legacy default stream) and performs no
 * host synchronisation unless its name says so. Every function returns 0 on
 * success or a negative PTK_E* code; ptk_last_error() returns the message of
 * the last failure on the calling thread. Element buffers must be 16-byte
 * aligned; chunk shards are padded to a multiple of world*8 elements
 * (ptk_shard_elems) so every shard is 16-byte aligned. bf16 values are
 * passed as uint16_t bit patterns.
 */
#ifndef PTK_H
#define PTK_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define PTK_OK 0
#define PTK_EINVAL -1
#define PTK_ECUDA -2
#define PTK_ENCCL -3
#define PTK_EUNSUPPORTED -4

#define PTK_MAX_PEERS 8

/* Adam / AdamW hyper-parameters of one step (host doubles; the library
 * derives fp32 scalars exactly once, see ptk_adam_scalars). */
typedef struct ptk_adam_config {
  double lr;
  double beta1;
  double beta2;
  double eps;
  double weight_decay;
  int32_t adamw;     /* 1: decoupled decay p *= 1-lr*wd; 0: L2 g += wd*p */
  int32_t step;      /* 1-based step count used for bias correction */
  double grad_scale; /* multiplies every gradient: 1/(world*loss_scale)*clip */
} ptk_adam_config;

/* fp32 scalars actually used by the kernels (exposed for the tests). */
typedef struct ptk_adam_scalars {
  float gscale, wd, decay, w1, b2, w2, eps, neg_step_size, bc2_sqrt;
  int32_t adamw;
} ptk_adam_scalars;

/* Gradient statistics accumulated on the device: sum of squares of the
 * scaled gradient (fp64) and the count of non-finite elements. */
typedef struct ptk_grad_stats_t {
  double sumsq;
  unsigned long long nonfinite;
} ptk_grad_stats_t;

/* ---- library ---------------------------------------------------------- */
const char* ptk_last_error(void);
const char* ptk_version(void);
int ptk_adam_derive(const ptk_adam_config* cfg, ptk_adam_scalars* out);
/* elements per rank shard for a chunk of n elements: roundup(n, 8w)/w */
int64_t ptk_shard_elems(int64_t n, int32_t world);
/* name of the chunk-Adam kernel shape in use (PTK_ADAM_VARIANT or default) */
const char* ptk_adam_kernel_name(void);
/* how the fused RS->Adam->AG kernel is chosen (PTK_FUSED_KERNEL=tma|ldg, or per table) */
const char* ptk_fused_kernel_name(void);
/* scratch: CTA partial buffer the reducing kernels need (bytes) */
int64_t ptk_stats_workspace_bytes(void);

/* ---- K1 + K2: fused chunk Adam ----------------------------------------
 * master/exp_avg/exp_avg_sq: fp32[n]; grad: bf16[n] (or fp32[n] for the
 * _f32grad variant); param_out: bf16[n] (nullable). If stats != NULL the
 * statistics of this launch are ADDED to *stats (device memory; zero it
 * with ptk_stats_reset); workspace = device scratch of
 * ptk_stats_workspace_bytes() (required when stats != NULL).
 * gscale_dev (nullable, device float): extra multiplier read on device
 * (e.g. a clip coefficient from ptk_clip_coef). skip_dev (nullable, device
 * int): when nonzero the launch is a no-op (overflow skip). */
int ptk_chunk_adam(const ptk_adam_config* cfg, float* master, float* exp_avg,
                   float* exp_avg_sq, const uint16_t* grad, uint16_t* param_out,
                   int64_t n, ptk_grad_stats_t* stats, void* workspace,
                   const float* gscale_dev, const int32_t* skip_dev, void* stream);
int ptk_chunk_adam_f32grad(const ptk_adam_config* cfg, float* master,
                           float* exp_avg, float* exp_avg_sq, const float* grad,
                           uint16_t* param_out, int64_t n,
                           ptk_grad_stats_t* stats, void* workspace,
                           const float* gscale_dev, const int32_t* skip_dev,
                           void* stream);

/* ---- K1 + K2 over a chunk TABLE: one launch per step --------------------
 * The persistent TMA kernel walks every chunk of the table in one launch, so
 * its shared-memory ring is filled and drained once per step instead of once
 * per chunk (small chunks: ProTrain's 32-128 MiB chunk sizes). The table is
 * built once (device copy owned by the handle) and may be used inside CUDA
 * graph capture. Same per-element rule, statistics and device-side
 * gscale/skip semantics as ptk_chunk_adam, bit-identical results. Replaces
 * the per-chunk GpuOptim tasks of one iteration (proj/src/sim.cpp:245-250,
 * 470-471) with one kernel. */
typedef struct ptk_chunk_desc {
  float* master;
  float* exp_avg;
  float* exp_avg_sq;
  const uint16_t* grad;
  uint16_t* param_out; /* nullable */
  int64_t n;
} ptk_chunk_desc;
typedef struct ptk_chunk_table ptk_chunk_table;
int ptk_chunk_table_create(const ptk_chunk_desc* descs, int32_t n_chunks, ptk_chunk_table** out);
int ptk_chunk_table_destroy(ptk_chunk_table* table);
int64_t ptk_chunk_table_params(const ptk_chunk_table* table);
int ptk_chunk_adam_table(const ptk_adam_config* cfg, const ptk_chunk_table* table,
                         ptk_grad_stats_t* stats, void* workspace, const float* gscale_dev,
                         const int32_t* skip_dev, void* stream);

/* ---- K2 standalone: gradient statistics (+ optional fp32 scaled copy) --- */
int ptk_grad_stats(const uint16_t* grad, int64_t n, float scale,
                   float* out_f32 /* nullable */, ptk_grad_stats_t* stats,
                   void* workspace, void* stream);
/* K2 as SURVEY §8(b) names it: out_f32[i] = float(grad[i]) * scale (the
 * bf16 -> fp32 cast with scale = 1/(world*loss_scale)), plus the same
 * statistics; out_f32 is required. */
int ptk_grad_prep(const uint16_t* grad, int64_t n, float scale, float* out_f32,
                  ptk_grad_stats_t* stats, void* workspace, void* stream);
int ptk_stats_reset(ptk_grad_stats_t* stats, void* stream);
/* coef_out = max_norm > 0 ? min(1, max_norm / (sqrt(sumsq) + 1e-6)) : 1;
 * skip_out (nullable) = nonfinite != 0 */
int ptk_clip_coef(const ptk_grad_stats_t* stats, double max_norm,
                  float* coef_out, int32_t* skip_out, void* stream);

/* ---- fused reduce-scatter -> Adam -> all-gather over peer memory -------
 * grad_peers[r]: rank r's full bf16 gradient chunk (n_pad elements);
 * param_peers[r]: rank r's full bf16 parameter chunk buffer. This rank
 * owns elements [rank*shard, (rank+1)*shard). Reduction is an fp32 sum in
 * rank order 0..world-1 (deterministic), then Adam on the local fp32
 * master/m/v shard, then the bf16 result is stored into every peer's
 * parameter buffer. Pointers may be NVLink peer mappings (ptk_ipc_*) or,
 * for single-GPU validation, local buffers standing in for virtual ranks.
 * The caller brackets the launch with ptk_peer_barrier. Replaces the
 * reference's modeled reduce (proj/src/hardware.cpp:36-38, sim Reduce),
 * GPU optimizer task (proj/src/cost.cpp:206-219) and gather
 * (proj/src/hardware.cpp:29-34) of one chunk with ONE kernel: by default a
 * TMA ring (cp.async.bulk of the local state and of every rank's gradient
 * tile into shared memory, bulk stores of the bf16 tile into every rank,
 * tiles claimed dynamically by the CTAs when a workspace is given);
 * PTK_FUSED_KERNEL=ldg selects the register-staged variant (128-bit peer
 * loads / stores). Both are bit-identical. shard must be a multiple of 8
 * elements. */
int ptk_fused_rs_adam_ag(const ptk_adam_config* cfg, const uint16_t* const* grad_peers,
                         uint16_t* const* param_peers, int32_t world, int32_t rank,
                         int64_t shard, float* master, float* exp_avg,
                         float* exp_avg_sq, ptk_grad_stats_t* stats,
                         void* workspace, void* stream);

/* Table form of the fused step: every chunk of a rank in ONE launch (the
 * ring stays full across chunks). kernel: PTK_FUSED_AUTO (PTK_FUSED_KERNEL
 * env if set, else the TMA ring -- decided once, here), PTK_FUSED_TMA or
 * PTK_FUSED_LDG (register-staged 128-bit peer loads / stores). gscale_dev / skip_dev as for ptk_chunk_adam (a device
 * clip coefficient / overflow flag from ptk_stats_collect).
 * ptk_fused_grad_stats_table is phase 1 of a clipped or overflow-checked
 * step: the statistics of this rank's reduced, scaled gradient shards (the
 * same fp32 rank-order sums), ADDED to *stats, no update. */
#define PTK_FUSED_AUTO 0
#define PTK_FUSED_TMA 1
#define PTK_FUSED_LDG 2
typedef struct ptk_fused_desc {
  const uint16_t* grad_peers[PTK_MAX_PEERS];
  uint16_t* param_peers[PTK_MAX_PEERS];
  float* master;
  float* exp_avg;
  float* exp_avg_sq;
  int64_t shard;
} ptk_fused_desc;
typedef struct ptk_fused_table ptk_fused_table;
int ptk_fused_table_create(const ptk_fused_desc* descs, int32_t n_chunks, int32_t world,
                           int32_t rank, int32_t kernel, ptk_fused_table** out);
int ptk_fused_table_destroy(ptk_fused_table* table);
/* the resolved kernel of a table: PTK_FUSED_TMA or PTK_FUSED_LDG */
int32_t ptk_fused_table_kernel(const ptk_fused_table* table);
int ptk_fused_step_table(const ptk_adam_config* cfg, const ptk_fused_table* table,
                         ptk_grad_stats_t* stats, void* workspace, const float* gscale_dev,
                         const int32_t* skip_dev, void* stream);
int ptk_fused_grad_stats_table(const ptk_adam_config* cfg, const ptk_fused_table* table,
                               ptk_grad_stats_t* stats, void* workspace, void* stream);

/* Statistics exchange over peer memory (global grad norm / overflow of the
 * fused path, no NCCL): a mailbox is ptk_stats_mailbox_bytes() of device
 * memory per rank (zeroed once, 32-byte aligned, peer-mapped like the
 * signal slots). ptk_stats_publish stores this rank's *stats into slot
 * [rank] of every rank's mailbox with a release-stored epoch;
 * ptk_stats_collect waits (device-side, PTK_PEER_BARRIER_TIMEOUT_MS) for
 * all `world` slots of the local mailbox to reach `epoch`, sums them in
 * rank order (identical bits on every rank) into *global_out (nullable) and
 * writes coef_out / skip_out (nullable) like ptk_clip_coef. */
int64_t ptk_stats_mailbox_bytes(void);
int ptk_stats_publish(const ptk_grad_stats_t* stats, void* const* mailbox_peers, int32_t world,
                      int32_t rank, int32_t epoch, void* stream);
int ptk_stats_collect(const void* mailbox, int32_t world, int32_t epoch, double max_norm,
                      ptk_grad_stats_t* global_out, float* coef_out, int32_t* skip_out,
                      void* stream);

/* ---- synthetic inputs (SURVEY §8(d) counter-based generator) ----------- */
/* out[i] = scale * u(seed, index0 + i), u in [-1, 1) exact in fp32 */
int ptk_fill_uniform_f32(float* out, int64_t n, uint64_t seed, int64_t index0, float scale,
                         void* stream);
int ptk_fill_uniform_bf16(uint16_t* out, int64_t n, uint64_t seed, int64_t index0, float scale,
                          void* stream);

/* Occupies `stream` for ns nanoseconds of device time: the stand-in for an
 * operator's compute when a trace is executed without its model. */
int ptk_busy_wait(int64_t ns, void* stream);

/* ---- K3 / K4: NCCL chunk collectives --------------------------------- */
typedef struct ptk_comm ptk_comm;
#define PTK_UNIQUE_ID_BYTES 128
int ptk_comm_unique_id(uint8_t out[PTK_UNIQUE_ID_BYTES]);
int ptk_comm_init(ptk_comm** out, int32_t world, int32_t rank,
                  const uint8_t id[PTK_UNIQUE_ID_BYTES]);
int ptk_comm_destroy(ptk_comm* comm);
/* dtype: 0 = bf16, 1 = fp32. In place: this rank's shard lives at
 * buf + rank*shard_elems; after the call buf holds all world shards. */
int ptk_chunk_allgather(ptk_comm* comm, void* buf, int64_t shard_elems,
                        int32_t dtype, void* stream);
/* In place: buf holds world*shard_elems local gradients; afterwards
 * buf + rank*shard_elems holds the sum over ranks of that shard. */
int ptk_chunk_reduce_scatter(ptk_comm* comm, void* buf, int64_t shard_elems,
                             int32_t dtype, void* stream);
/* Sums a ptk_grad_stats_t (sumsq fp64, nonfinite u64) over all ranks, in
 * place on the device (global gradient norm / overflow across the world). */
int ptk_stats_allreduce(ptk_comm* comm, ptk_grad_stats_t* stats, void* stream);
/* Device-side barrier over the communicator (an 1-element all-reduce). */
int ptk_comm_barrier(ptk_comm* comm, void* stream);
/* Failure detection (the reference simulator's DeadlockDetected,
 * proj/src/sim.cpp:640-647, for the real exchange): ptk_comm_wait blocks the
 * host until `stream` has drained, polling ncclCommGetAsyncError; on an
 * asynchronous NCCL error, or when timeout_ms (> 0) elapses first (a hung or
 * dead peer), it aborts the communicator (ncclCommAbort) and returns
 * PTK_ENCCL. ptk_comm_async_error returns PTK_ENCCL if NCCL reported an
 * asynchronous error. After ptk_comm_abort every collective call on the
 * communicator fails with PTK_ENCCL; ptk_comm_destroy still frees it. */
int ptk_comm_wait(ptk_comm* comm, void* stream, int64_t timeout_ms);
int ptk_comm_async_error(ptk_comm* comm);
int ptk_comm_abort(ptk_comm* comm);

/* NCCL symmetric memory for the library baseline's chunk buffers. The
 * NVLink-optimised NCCL kernels for all-gather / reduce-scatter engage when
 * the send / receive buffers lie in a window registered with
 * NCCL_WIN_COLL_SYMMETRIC on every rank; such windows must come from
 * ncclMemAlloc (cuMem, multicast-capable granularity).
 * ptk_comm_mem_alloc / _free: ncclMemAlloc / ncclMemFree of `bytes`.
 * ptk_comm_window_register: COLLECTIVE over the communicator (every rank, same
 * order, same size); *win_out is an opaque handle for _deregister (also
 * collective). Replaces nothing in the reference (its coll_bw is a modelled
 * constant, proj/src/hardware.cpp:29-38); it makes the NCCL comparison leg
 * the strongest NCCL path. */
int ptk_comm_mem_alloc(void** ptr_out, int64_t bytes);
int ptk_comm_mem_free(void* ptr);
int ptk_comm_window_register(ptk_comm* comm, void* buf, int64_t bytes, void** win_out);
int ptk_comm_window_deregister(ptk_comm* comm, void* win);

/* ---- NVLink peer memory for the fused path ---------------------------- */
#define PTK_IPC_HANDLE_BYTES 64
/* Handle of the allocation containing dev_ptr; *offset_out = dev_ptr - base
 * (buffers carved from a caching allocator are sub-ranges of an allocation). */
int ptk_ipc_get_handle(void* dev_ptr, uint8_t out[PTK_IPC_HANDLE_BYTES], int64_t* offset_out);
/* Maps a peer allocation; *dev_ptr = its base (add the peer's offset). */
int ptk_ipc_open_handle(const uint8_t handle[PTK_IPC_HANDLE_BYTES], void** dev_ptr);
int ptk_ipc_close_handle(void* dev_ptr);
/* signal_peers[r]: rank r's int32[PTK_MAX_PEERS] signal slots (zeroed once).
 * Each call bumps `epoch` (monotone, identical on all ranks), stores it into
 * slot [rank] of every peer and spins until all slots of its own array
 * reached epoch. Orders all prior stream work before later stream work
 * across the world. A peer that does not arrive within
 * PTK_PEER_BARRIER_TIMEOUT_MS (env, default 60000) of device time makes the
 * barrier trap: the launch fails instead of hanging the device. */
int ptk_peer_barrier(int32_t* const* signal_peers, int32_t world, int32_t rank,
                     int32_t epoch, void* stream);

/* ---- K3 / K4 over peer memory for NON-persistent chunks --------------
 * The offload path's exchange without a library collective (the gather
 * before a block's use and the reduce after its backward, proj/src/
 * sim.cpp:335-350,426-436; modelled as gather_time / reduce_time,
 * proj/src/hardware.cpp:29-38). Both are collective over the ranks and are
 * bracketed by ptk_peer_barrier on the calling stream (one signal array per
 * stream that issues them).
 * ptk_peer_reduce_scatter_f32: out[i] = sum over r = 0..world-1, in that
 *   order, of bf16 grad_peers[r][rank * shard + i] in fp32 (shard elements,
 *   16-byte aligned): the same sum ptk_fused_step_table feeds its Adam, kept
 *   in fp32 for the host Adam (ptk_cpu_adam_f32grad).
 * ptk_peer_allgather: for every q != rank, copies bytes
 *   [q * shard_bytes, (q+1) * shard_bytes) of buf_peers[q] to the same range
 *   of buf_peers[rank]: copy-engine peer transfers over NVLink, the W-1 pulls
 *   concurrent on internal side streams forked from and joined back into
 *   `stream` (stream-ordered for the caller). */
int ptk_peer_reduce_scatter_f32(const uint16_t* const* grad_peers, int32_t world, int32_t rank,
                                int64_t shard, float* out, void* stream);
int ptk_peer_allgather(void* const* buf_peers, int32_t world, int32_t rank, int64_t shard_bytes,
                       void* stream);

/* ---- K5: pinned host <-> device chunk copies on side streams ---------- */
int ptk_host_alloc_pinned(void** out, size_t bytes);
int ptk_host_free_pinned(void* ptr);
int ptk_memcpy_h2d_async(void* dst, const void* src, size_t bytes, void* stream);
int ptk_memcpy_d2h_async(void* dst, const void* src, size_t bytes, void* stream);

/* ---- K6: host Adam over an offloaded shard (OpenMP) -------------------
 * n_threads <= 0: the OpenMP default (OMP_NUM_THREADS if set -- torchrun sets
 * it to 1 -- else every core). The same update rule as ptk_chunk_adam, bit
 * for bit; optional statistics of the scaled gradient. */
int ptk_cpu_adam(const ptk_adam_config* cfg, float* master, float* exp_avg,
                 float* exp_avg_sq, const uint16_t* grad, uint16_t* param_out,
                 int64_t n, int32_t n_threads, double* sumsq_out,
                 int64_t* nonfinite_out);
/* fp32 gradients (a reduce-scattered sum kept in fp32, ptk_peer_reduce_scatter_f32) */
int ptk_cpu_adam_f32grad(const ptk_adam_config* cfg, float* master, float* exp_avg,
                         float* exp_avg_sq, const float* grad, uint16_t* param_out,
                         int64_t n, int32_t n_threads, double* sumsq_out,
                         int64_t* nonfinite_out);

/* ---- the chunk runtime (memplan::execute) and the profiler re-feed ----- */
/* Executes `iterations` iterations of a plan (plan JSON as written by
 * `memplan plan`, or a bare PlanConfig) for a trace (trace JSON) on this
 * device with the hardware profile (profile JSON): real chunk storage,
 * uploads/offloads, collectives and optimizer updates; stand-in compute of
 * compute_scale x the trace's op times. Writes the measured result (the
 * simulator's summary schema + estimate_t_iter + byte counters) as JSON and
 * the measured event timeline as CSV (either path may be NULL). */
int ptk_execute_plan(const char* trace_path, const char* plan_path, const char* profile_path,
                     void* comm, int32_t rank, double compute_scale, int32_t iterations,
                     const char* result_json_path, const char* timeline_csv_path);
/* Measures this machine's HardwareProfile (H2D/D2H, NCCL alpha/beta when
 * comm != NULL, device/host Adam rates, memory) starting from a base profile
 * JSON and writes the measured profile JSON to out_path. */
int ptk_measure_profile(const char* base_profile_path, void* comm, int32_t world,
                        const char* out_path);
/* The individual probes measure_profile composes (host-synchronising; best
 * of several repetitions on a private stream):
 *   ptk_profile_copy_bw        pinned H2D / D2H bytes/s of a `bytes` copy
 *                              -> HardwareProfile::h2d_bw / d2h_bw
 *   ptk_profile_collective     alpha (s) of an 8 KiB all-gather and beta
 *                              (wire bytes/s) of a chunk_bytes all-gather,
 *                              the gather_time model of proj/src/hardware.cpp:29-34
 *                              -> coll_alpha / coll_bw
 *   ptk_profile_gpu_adam_rate  ptk_chunk_adam params/s over n params -> gpu_optim_rate
 *   ptk_profile_cpu_adam_rate  ptk_cpu_adam params/s over n params   -> cpu_optim_rate */
int ptk_profile_copy_bw(int64_t bytes, double* h2d_bw, double* d2h_bw);
int ptk_profile_collective(ptk_comm* comm, int32_t world, int64_t chunk_bytes, double* alpha,
                           double* bw);
int ptk_profile_gpu_adam_rate(int64_t n, double* params_per_s);
int ptk_profile_cpu_adam_rate(int64_t n, double* params_per_s);
/* Host-memory bandwidth shared by the host Adam and PCIe copies (the
 * simulator extension's --host-mem-bw): the host Adam over n params on
 * `threads` threads (<= 0: cores - 2, the ChunkPool default) runs for about
 * `seconds` while pinned H2D + D2H copies loop; returns
 * (28 * params updated + bytes copied) / elapsed. Host-synchronising. */
int ptk_profile_host_memory_bw(int64_t n, int32_t threads, double seconds, double* bytes_per_s);

/* ---- the chunk buffer pool: the runtime's ONE residency policy --------- */
/* memplan::ChunkBufferPool (include/memplan/policy.hpp) -- the same decisions
 * the simulator (memplan::simulate, proj/src/sim.cpp:275-343,427-451) and the
 * device executor (ptk_execute_plan) make -- for a host runtime that moves the
 * chunk bytes itself (the training loop's chunk pool, offload.py). Chunk ids
 * are 1-based, chunks 1..n_persist are persistent (never pooled); positions:
 * forward of chunk c = c, backward = 2N - c + 1. Not thread-safe.
 *   ptk_pool_grant     a slot for chunk c (away) at position `now`: the
 *                      lowest free slot, else the slot of the idle resident
 *                      chunk whose next use is farthest, pinned chunks
 *                      excluded -- for a prefetch (demand = 0) only a chunk
 *                      needed strictly later than c; demand != 0 (c is needed
 *                      now) takes any candidate. *slot = -1 when no slot can
 *                      be granted now; *evicted = the chunk that gave its slot
 *                      up (0 = a free slot). c is then arriving.
 *   ptk_pool_arrived   the chunk's bytes are in its slot (stream-ordered)
 *   ptk_pool_release   drain: the chunk leaves the device, its slot is free */
typedef struct ptk_pool ptk_pool;
int ptk_pool_create(int32_t n_chunk, int32_t n_persist, int32_t n_buffer, ptk_pool** out);
void ptk_pool_destroy(ptk_pool* pool);
int ptk_pool_grant(ptk_pool* pool, int32_t c, int32_t now, const int32_t* pinned,
                   int32_t n_pinned, int32_t demand, int32_t* slot, int32_t* evicted);
int ptk_pool_arrived(ptk_pool* pool, int32_t c);
int ptk_pool_release(ptk_pool* pool, int32_t c, int32_t* slot);
int32_t ptk_pool_slot_of(const ptk_pool* pool, int32_t c);       /* -1: none */
int32_t ptk_pool_chunk_in_slot(const ptk_pool* pool, int32_t s);  /* 0: free */
int32_t ptk_pool_residency(const ptk_pool* pool, int32_t c);      /* 0 away, 1 arriving,
                                                                     2 resident, 3 draining */

/* ---- the planner in process ------------------------------------------- */
/* memplan::run_cli (proj/include/memplan/cli.hpp:20-35) with argv = the memplan
 * command line without the program name; returns its exit code (0 ok, 1 domain
 * error, 2 usage error) and malloc'ed stdout / stderr text (free with ptk_free). */
int ptk_memplan_run(int32_t argc, const char* const* argv, char** out, char** err);
void ptk_free(void* p);

/* ---- streams / events / timing helpers used by the host runtime ------- */
int ptk_stream_create(void** out, int32_t high_priority);
int ptk_stream_destroy(void* stream);
int ptk_event_create(void** out);
int ptk_event_destroy(void* ev);
int ptk_event_record(void* ev, void* stream);
int ptk_stream_wait_event(void* stream, void* ev);
int ptk_event_elapsed_ms(void* start, void* end, float* ms);
int ptk_stream_synchronize(void* stream);
int ptk_device_synchronize(void);
/* number of ptk kernels launched by this process so far */
int64_t ptk_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* PTK_H */
