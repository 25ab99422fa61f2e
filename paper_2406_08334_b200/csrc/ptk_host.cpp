// libptk host plumbing: error state, scalar derivation, streams/events,
// pinned host memory and the K5 side-stream copies.
//
// The scalar derivation is the single place where the Adam hyper-parameters
// are rounded to fp32; the CUDA kernels (ptk_kernels.cu) and the host Adam
// (ptk_cpu_adam.cpp) both consume the result, which is what makes the GPU
// and CPU update rules agree bit for bit.
#include <cmath>
#include <cstring>

#include "ptk_common.h"

namespace ptk {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

std::atomic<int64_t>& launch_counter() {
  static std::atomic<int64_t> counter{0};
  return counter;
}

ptk_adam_scalars derive_scalars(const ptk_adam_config& c) {
  const double bc1 = 1.0 - std::pow(c.beta1, static_cast<double>(c.step));
  const double bc2 = 1.0 - std::pow(c.beta2, static_cast<double>(c.step));
  ptk_adam_scalars s{};
  s.gscale = static_cast<float>(c.grad_scale);
  s.adamw = c.adamw ? 1 : 0;
  s.wd = c.adamw ? 0.0f : static_cast<float>(c.weight_decay);
  s.decay = c.adamw ? static_cast<float>(1.0 - c.lr * c.weight_decay) : 1.0f;
  s.w1 = static_cast<float>(1.0 - c.beta1);
  s.b2 = static_cast<float>(c.beta2);
  s.w2 = static_cast<float>(1.0 - c.beta2);
  s.eps = static_cast<float>(c.eps);
  s.neg_step_size = static_cast<float>(-(c.lr / bc1));
  s.bc2_sqrt = static_cast<float>(std::sqrt(bc2));
  return s;
}

}  // namespace ptk

using ptk::fail;

extern "C" {

const char* ptk_last_error(void) { return ptk::g_last_error.c_str(); }

const char* ptk_version(void) { return "ptk 0.1 sm_100a"; }

int ptk_adam_derive(const ptk_adam_config* cfg, ptk_adam_scalars* out) {
  if (!cfg || !out) return fail(PTK_EINVAL, "ptk_adam_derive: null argument");
  if (cfg->step < 1) return fail(PTK_EINVAL, "ptk_adam_derive: step must be >= 1");
  *out = ptk::derive_scalars(*cfg);
  return PTK_OK;
}

int64_t ptk_shard_elems(int64_t n, int32_t world) {
  if (n < 0 || world < 1) return -1;
  const int64_t q = static_cast<int64_t>(world) * 8;
  return (n + q - 1) / q * q / world;
}

int ptk_host_alloc_pinned(void** out, size_t bytes) {
  if (!out) return fail(PTK_EINVAL, "ptk_host_alloc_pinned: null out");
  PTK_TRY_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocPortable));
  return PTK_OK;
}

int ptk_host_free_pinned(void* ptr) {
  PTK_TRY_CUDA(cudaFreeHost(ptr));
  return PTK_OK;
}

int ptk_memcpy_h2d_async(void* dst, const void* src, size_t bytes, void* stream) {
  PTK_TRY_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ptk::as_stream(stream)));
  return PTK_OK;
}

int ptk_memcpy_d2h_async(void* dst, const void* src, size_t bytes, void* stream) {
  PTK_TRY_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ptk::as_stream(stream)));
  return PTK_OK;
}

int ptk_stream_create(void** out, int32_t high_priority) {
  if (!out) return fail(PTK_EINVAL, "ptk_stream_create: null out");
  int lo = 0, hi = 0;
  PTK_TRY_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  cudaStream_t s;
  PTK_TRY_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, high_priority ? hi : lo));
  *out = s;
  return PTK_OK;
}

int ptk_stream_destroy(void* stream) {
  PTK_TRY_CUDA(cudaStreamDestroy(ptk::as_stream(stream)));
  return PTK_OK;
}

int ptk_event_create(void** out) {
  if (!out) return fail(PTK_EINVAL, "ptk_event_create: null out");
  cudaEvent_t e;
  PTK_TRY_CUDA(cudaEventCreate(&e));
  *out = e;
  return PTK_OK;
}

int ptk_event_destroy(void* ev) {
  PTK_TRY_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(ev)));
  return PTK_OK;
}

int ptk_event_record(void* ev, void* stream) {
  PTK_TRY_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev), ptk::as_stream(stream)));
  return PTK_OK;
}

int ptk_stream_wait_event(void* stream, void* ev) {
  PTK_TRY_CUDA(cudaStreamWaitEvent(ptk::as_stream(stream), static_cast<cudaEvent_t>(ev), 0));
  return PTK_OK;
}

int ptk_event_elapsed_ms(void* start, void* end, float* ms) {
  if (!ms) return fail(PTK_EINVAL, "ptk_event_elapsed_ms: null out");
  PTK_TRY_CUDA(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start), static_cast<cudaEvent_t>(end)));
  return PTK_OK;
}

int ptk_stream_synchronize(void* stream) {
  PTK_TRY_CUDA(cudaStreamSynchronize(ptk::as_stream(stream)));
  return PTK_OK;
}

int ptk_device_synchronize(void) {
  PTK_TRY_CUDA(cudaDeviceSynchronize());
  return PTK_OK;
}

int64_t ptk_kernel_launch_count(void) { return ptk::launch_counter().load(); }

int ptk_ipc_get_handle(void* dev_ptr, uint8_t out[PTK_IPC_HANDLE_BYTES], int64_t* offset_out) {
  static_assert(sizeof(cudaIpcMemHandle_t) <= PTK_IPC_HANDLE_BYTES, "ipc handle size");
  if (!dev_ptr || !out || !offset_out) return fail(PTK_EINVAL, "ptk_ipc_get_handle: null argument");
  // Allocation base through the driver entry point (no link-time libcuda
  // dependency, so the library still loads on a machine without a driver).
  using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
  static GetRange get_range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<GetRange>(nullptr);
    return reinterpret_cast<GetRange>(fn);
  }();
  if (!get_range) return fail(PTK_ECUDA, "ptk_ipc_get_handle: cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0)
    return fail(PTK_ECUDA, "ptk_ipc_get_handle: cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  PTK_TRY_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memset(out, 0, PTK_IPC_HANDLE_BYTES);
  std::memcpy(out, &h, sizeof(h));
  *offset_out = static_cast<int64_t>(reinterpret_cast<unsigned long long>(dev_ptr) - base);
  return PTK_OK;
}

int ptk_ipc_open_handle(const uint8_t handle[PTK_IPC_HANDLE_BYTES], void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(PTK_EINVAL, "ptk_ipc_open_handle: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  PTK_TRY_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return PTK_OK;
}

int ptk_ipc_close_handle(void* dev_ptr) {
  PTK_TRY_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return PTK_OK;
}

}  // extern "C"
