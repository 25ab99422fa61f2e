// K3 / K4: in-place chunk all-gather and reduce-scatter over NCCL (NVLink 5 /
// NVSwitch on a B200 box). One communicator per device, created from a
// unique id the host runtime distributes (torch.distributed store). These
// are the library-collective baseline of the data plane; the fused
// peer-memory kernel in ptk_kernels.cu is the B200-native path.
//
// Modeled counterparts: gather_time / reduce_time, `alpha + bytes*(w-1)/(w*bw)`
// (proj/src/hardware.cpp:29-38); Sim gather/reduce on the coll link
// (proj/src/sim.cpp:335-350,428-436).
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <string>
#include <thread>

#include "ptk_common.h"

struct ptk_comm {
  ncclComm_t comm = nullptr;
  int world = 1;
  int rank = 0;
  void* scratch = nullptr;  // 1 float for the barrier all-reduce
  bool aborted = false;     // after ptk_comm_abort / a failed ptk_comm_wait
};

namespace {

int check_nccl(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return PTK_OK;
  return ptk::fail(PTK_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

ncclDataType_t to_nccl(int32_t dtype) { return dtype == 1 ? ncclFloat32 : ncclBfloat16; }
size_t elem_bytes(int32_t dtype) { return dtype == 1 ? 4 : 2; }

// Every collective entry point refuses an aborted communicator loudly.
int usable(const ptk_comm* c, const char* what) {
  if (!c) return ptk::fail(PTK_EINVAL, std::string(what) + ": null comm");
  if (c->aborted || !c->comm)
    return ptk::fail(PTK_ENCCL, std::string(what) + ": communicator was aborted");
  return PTK_OK;
}

}  // namespace

#define PTK_TRY_USABLE(c, what)                 \
  do {                                          \
    int ptk_rc_ = usable((c), (what));          \
    if (ptk_rc_ != PTK_OK) return ptk_rc_;      \
  } while (0)

#define PTK_TRY_NCCL(expr)                                \
  do {                                                    \
    int ptk_rc_ = check_nccl((expr), #expr);              \
    if (ptk_rc_ != PTK_OK) return ptk_rc_;                \
  } while (0)

extern "C" {

int ptk_comm_unique_id(uint8_t out[PTK_UNIQUE_ID_BYTES]) {
  static_assert(sizeof(ncclUniqueId) == PTK_UNIQUE_ID_BYTES, "nccl unique id size");
  if (!out) return ptk::fail(PTK_EINVAL, "ptk_comm_unique_id: null out");
  ncclUniqueId id;
  PTK_TRY_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return PTK_OK;
}

int ptk_comm_init(ptk_comm** out, int32_t world, int32_t rank,
                  const uint8_t id_bytes[PTK_UNIQUE_ID_BYTES]) {
  if (!out || !id_bytes || world < 1 || rank < 0 || rank >= world)
    return ptk::fail(PTK_EINVAL, "ptk_comm_init: bad arguments");
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof(id));
  auto* c = new ptk_comm;
  c->world = world;
  c->rank = rank;
  const int rc = check_nccl(ncclCommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
  if (rc != PTK_OK) {
    delete c;
    return rc;
  }
  if (cudaMalloc(&c->scratch, 16) != cudaSuccess) {
    ncclCommDestroy(c->comm);
    delete c;
    return ptk::fail(PTK_ECUDA, "ptk_comm_init: scratch allocation failed");
  }
  cudaMemset(c->scratch, 0, 16);
  *out = c;
  return PTK_OK;
}

int ptk_comm_destroy(ptk_comm* c) {
  if (!c) return PTK_OK;
  if (c->scratch) cudaFree(c->scratch);
  const int rc = c->comm ? check_nccl(ncclCommDestroy(c->comm), "ncclCommDestroy") : PTK_OK;
  delete c;
  return rc;
}

// Failure detection of the NCCL path (the analogue of the reference
// simulator's DeadlockDetected, proj/src/sim.cpp:640-647): a hung or failed
// peer must not hang the job. ptk_comm_wait polls the stream and the
// communicator's asynchronous error state; on an async error or after
// timeout_ms it aborts the communicator (ncclCommAbort releases the NCCL
// kernels still waiting on the stream) and returns PTK_ENCCL.
int ptk_comm_abort(ptk_comm* c) {
  if (!c) return ptk::fail(PTK_EINVAL, "ptk_comm_abort: null comm");
  if (c->comm) {
    const ncclResult_t r = ncclCommAbort(c->comm);
    c->comm = nullptr;
    c->aborted = true;
    return check_nccl(r, "ncclCommAbort");
  }
  c->aborted = true;
  return PTK_OK;
}

int ptk_comm_async_error(ptk_comm* c) {
  PTK_TRY_USABLE(c, "ptk_comm_async_error");
  ncclResult_t async = ncclSuccess;
  PTK_TRY_NCCL(ncclCommGetAsyncError(c->comm, &async));
  if (async == ncclSuccess || async == ncclInProgress) return PTK_OK;
  return ptk::fail(PTK_ENCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(async));
}

int ptk_comm_wait(ptk_comm* c, void* stream, int64_t timeout_ms) {
  PTK_TRY_USABLE(c, "ptk_comm_wait");
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(ptk::as_stream(stream));
    if (q == cudaSuccess) return PTK_OK;
    if (q != cudaErrorNotReady) return ptk::check_cuda(q, "ptk_comm_wait: stream");
    ncclResult_t async = ncclSuccess;
    if (ncclCommGetAsyncError(c->comm, &async) != ncclSuccess ||
        (async != ncclSuccess && async != ncclInProgress)) {
      const std::string why = ncclGetErrorString(async);
      ptk_comm_abort(c);
      return ptk::fail(PTK_ENCCL, "ptk_comm_wait: NCCL asynchronous error (" + why +
                                      "); communicator aborted");
    }
    const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(
                        std::chrono::steady_clock::now() - t0).count();
    if (timeout_ms > 0 && ms > timeout_ms) {
      ptk_comm_abort(c);
      return ptk::fail(PTK_ENCCL, "ptk_comm_wait: stream not drained after " +
                                      std::to_string(timeout_ms) +
                                      " ms (hung peer?); communicator aborted");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

int ptk_comm_mem_alloc(void** ptr_out, int64_t bytes) {
  if (!ptr_out || bytes <= 0) return ptk::fail(PTK_EINVAL, "ptk_comm_mem_alloc: bad arguments");
  *ptr_out = nullptr;
  PTK_TRY_NCCL(ncclMemAlloc(ptr_out, static_cast<size_t>(bytes)));
  return PTK_OK;
}

int ptk_comm_mem_free(void* ptr) {
  if (!ptr) return PTK_OK;
  PTK_TRY_NCCL(ncclMemFree(ptr));
  return PTK_OK;
}

int ptk_comm_window_register(ptk_comm* c, void* buf, int64_t bytes, void** win_out) {
  PTK_TRY_USABLE(c, "ptk_comm_window_register");
  if (!buf || bytes <= 0 || !win_out)
    return ptk::fail(PTK_EINVAL, "ptk_comm_window_register: bad arguments");
  ncclWindow_t win = nullptr;
  PTK_TRY_NCCL(ncclCommWindowRegister(c->comm, buf, static_cast<size_t>(bytes), &win,
                                      NCCL_WIN_COLL_SYMMETRIC));
  *win_out = static_cast<void*>(win);
  return PTK_OK;
}

int ptk_comm_window_deregister(ptk_comm* c, void* win) {
  PTK_TRY_USABLE(c, "ptk_comm_window_deregister");
  if (!win) return PTK_OK;
  PTK_TRY_NCCL(ncclCommWindowDeregister(c->comm, static_cast<ncclWindow_t>(win)));
  return PTK_OK;
}

int ptk_chunk_allgather(ptk_comm* c, void* buf, int64_t shard_elems, int32_t dtype,
                        void* stream) {
  PTK_TRY_USABLE(c, "ptk_chunk_allgather");
  if (!buf || shard_elems < 0) return ptk::fail(PTK_EINVAL, "ptk_chunk_allgather: bad arguments");
  if (shard_elems == 0) return PTK_OK;  // w = 1 still goes through NCCL (a local copy)
  char* base = static_cast<char*>(buf);
  const void* send = base + static_cast<size_t>(c->rank) * shard_elems * elem_bytes(dtype);
  PTK_TRY_NCCL(ncclAllGather(send, buf, static_cast<size_t>(shard_elems), to_nccl(dtype), c->comm,
                             ptk::as_stream(stream)));
  return PTK_OK;
}

int ptk_chunk_reduce_scatter(ptk_comm* c, void* buf, int64_t shard_elems, int32_t dtype,
                             void* stream) {
  PTK_TRY_USABLE(c, "ptk_chunk_reduce_scatter");
  if (!buf || shard_elems < 0)
    return ptk::fail(PTK_EINVAL, "ptk_chunk_reduce_scatter: bad arguments");
  if (shard_elems == 0) return PTK_OK;  // w = 1 still goes through NCCL (a local copy)
  char* base = static_cast<char*>(buf);
  void* recv = base + static_cast<size_t>(c->rank) * shard_elems * elem_bytes(dtype);
  PTK_TRY_NCCL(ncclReduceScatter(buf, recv, static_cast<size_t>(shard_elems), to_nccl(dtype),
                                 ncclSum, c->comm, ptk::as_stream(stream)));
  return PTK_OK;
}

int ptk_stats_allreduce(ptk_comm* c, ptk_grad_stats_t* stats, void* stream) {
  PTK_TRY_USABLE(c, "ptk_stats_allreduce");
  if (!stats) return ptk::fail(PTK_EINVAL, "ptk_stats_allreduce: null argument");
  PTK_TRY_NCCL(ncclGroupStart());
  PTK_TRY_NCCL(ncclAllReduce(&stats->sumsq, &stats->sumsq, 1, ncclFloat64, ncclSum, c->comm,
                             ptk::as_stream(stream)));
  PTK_TRY_NCCL(ncclAllReduce(&stats->nonfinite, &stats->nonfinite, 1, ncclUint64, ncclSum,
                             c->comm, ptk::as_stream(stream)));
  PTK_TRY_NCCL(ncclGroupEnd());
  return PTK_OK;
}

int ptk_comm_barrier(ptk_comm* c, void* stream) {
  PTK_TRY_USABLE(c, "ptk_comm_barrier");
  PTK_TRY_NCCL(ncclAllReduce(c->scratch, c->scratch, 1, ncclFloat32, ncclSum, c->comm,
                             ptk::as_stream(stream)));
  return PTK_OK;
}

}  // extern "C"
