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

#include <cstring>
#include <string>

#include "ptk_common.h"

struct ptk_comm {
  ncclComm_t comm = nullptr;
  int world = 1;
  int rank = 0;
  void* scratch = nullptr;  // 1 float for the barrier all-reduce
};

namespace {

int check_nccl(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return PTK_OK;
  return ptk::fail(PTK_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

ncclDataType_t to_nccl(int32_t dtype) { return dtype == 1 ? ncclFloat32 : ncclBfloat16; }
size_t elem_bytes(int32_t dtype) { return dtype == 1 ? 4 : 2; }

}  // namespace

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

int ptk_chunk_allgather(ptk_comm* c, void* buf, int64_t shard_elems, int32_t dtype,
                        void* stream) {
  if (!c || !buf || shard_elems < 0) return ptk::fail(PTK_EINVAL, "ptk_chunk_allgather: bad arguments");
  if (shard_elems == 0) return PTK_OK;  // w = 1 still goes through NCCL (a local copy)
  char* base = static_cast<char*>(buf);
  const void* send = base + static_cast<size_t>(c->rank) * shard_elems * elem_bytes(dtype);
  PTK_TRY_NCCL(ncclAllGather(send, buf, static_cast<size_t>(shard_elems), to_nccl(dtype), c->comm,
                             ptk::as_stream(stream)));
  return PTK_OK;
}

int ptk_chunk_reduce_scatter(ptk_comm* c, void* buf, int64_t shard_elems, int32_t dtype,
                             void* stream) {
  if (!c || !buf || shard_elems < 0)
    return ptk::fail(PTK_EINVAL, "ptk_chunk_reduce_scatter: bad arguments");
  if (shard_elems == 0) return PTK_OK;  // w = 1 still goes through NCCL (a local copy)
  char* base = static_cast<char*>(buf);
  void* recv = base + static_cast<size_t>(c->rank) * shard_elems * elem_bytes(dtype);
  PTK_TRY_NCCL(ncclReduceScatter(buf, recv, static_cast<size_t>(shard_elems), to_nccl(dtype),
                                 ncclSum, c->comm, ptk::as_stream(stream)));
  return PTK_OK;
}

int ptk_stats_allreduce(ptk_comm* c, ptk_grad_stats_t* stats, void* stream) {
  if (!c || !stats) return ptk::fail(PTK_EINVAL, "ptk_stats_allreduce: null argument");
  PTK_TRY_NCCL(ncclGroupStart());
  PTK_TRY_NCCL(ncclAllReduce(&stats->sumsq, &stats->sumsq, 1, ncclFloat64, ncclSum, c->comm,
                             ptk::as_stream(stream)));
  PTK_TRY_NCCL(ncclAllReduce(&stats->nonfinite, &stats->nonfinite, 1, ncclUint64, ncclSum,
                             c->comm, ptk::as_stream(stream)));
  PTK_TRY_NCCL(ncclGroupEnd());
  return PTK_OK;
}

int ptk_comm_barrier(ptk_comm* c, void* stream) {
  if (!c) return ptk::fail(PTK_EINVAL, "ptk_comm_barrier: null comm");
  PTK_TRY_NCCL(ncclAllReduce(c->scratch, c->scratch, 1, ncclFloat32, ncclSum, c->comm,
                             ptk::as_stream(stream)));
  return PTK_OK;
}

}  // extern "C"
