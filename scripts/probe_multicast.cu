// Probe: can this box's GPU bind a CUDA multicast (NVLS) object and run
// multimem.ld_reduce / multimem.st on it?  Prints one line per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o build/probe_multicast scripts/probe_multicast.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_ = nullptr; \
  cuGetErrorString(r_, &s_); std::printf("FAIL %s -> %d %s\n", #x, (int)r_, s_ ? s_ : "?"); return 1; } } while (0)

__global__ void mm_kernel(float* mc, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * i + 3 >= n) return;
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc + 4 * i) : "memory");
  v.x += 1.f; v.y += 1.f; v.z += 1.f; v.w += 1.f;
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(mc + 4 * i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  reinterpret_cast<float4*>(out)[i] = v;
}

int main() {
  CK(cuInit(0));
  int ndev = 0; CK(cuDeviceGetCount(&ndev));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  int mc = 0, fab = 0, fd = 0;
  CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev));
  std::printf("devices=%d multicast_supported=%d fabric_handle=%d posix_fd=%d\n", ndev, mc, fab, fd);
  if (!mc) { std::printf("RESULT no-multicast\n"); return 0; }
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));

  const size_t n = 1 << 20, bytes = n * sizeof(float);
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1; mp.size = bytes; mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  size_t sz = (bytes + gran - 1) / gran * gran; mp.size = sz;
  std::printf("mc granularity=%zu size=%zu\n", gran, sz);
  CUmemGenericAllocationHandle mch;
  {
    // which handle types / sizes does cuMulticastCreate accept on this box?
    const CUmemAllocationHandleType types[] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                               CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_NONE};
    const char* names[] = {"posix_fd", "fabric", "none"};
    bool ok = false;
    for (int nd = 1; nd <= 2 && !ok; ++nd)
      for (int t = 0; t < 3 && !ok; ++t) {
        CUmulticastObjectProp q = mp; q.numDevices = nd; q.handleTypes = types[t];
        CUresult r = cuMulticastCreate(&mch, &q);
        const char* es = nullptr; cuGetErrorString(r, &es);
        std::printf("cuMulticastCreate numDevices=%d handle=%s -> %d %s\n", nd, names[t], (int)r, es ? es : "?");
        if (r == CUDA_SUCCESS && nd == 1) { ok = true; mp = q; }
      }
    if (!ok) { std::printf("RESULT multicast-create-refused\n"); return 0; }
  }
  CK(cuMulticastAddDevice(mch, dev));

  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0; ap.requestedHandleTypes = static_cast<CUmemAllocationHandleType>(mp.handleTypes);
  CUmemGenericAllocationHandle ph; CK(cuMemCreate(&ph, sz, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, ph, 0, sz, 0));

  CUdeviceptr uc, mcp;
  CK(cuMemAddressReserve(&uc, sz, gran, 0, 0)); CK(cuMemMap(uc, sz, 0, ph, 0));
  CK(cuMemAddressReserve(&mcp, sz, gran, 0, 0)); CK(cuMemMap(mcp, sz, 0, mch, 0));
  CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, sz, &ad, 1)); CK(cuMemSetAccess(mcp, sz, &ad, 1));

  std::vector<float> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = float(i % 1000) * 0.5f;
  CK(cuMemcpyHtoD(uc, h.data(), bytes));
  float* out; cudaMalloc(&out, bytes);
  mm_kernel<<<(n / 4 + 255) / 256, 256>>>((float*)mcp, out, (int)n);
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("kernel: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) { std::printf("RESULT kernel-failed\n"); return 1; }
  std::vector<float> o(n), u(n);
  cudaMemcpy(o.data(), out, bytes, cudaMemcpyDeviceToHost);
  CK(cuMemcpyDtoH(u.data(), uc, bytes));
  size_t bad = 0;
  for (size_t i = 0; i < n; ++i) if (o[i] != h[i] + 1.f || u[i] != h[i] + 1.f) ++bad;
  std::printf("RESULT multimem %s (mismatches=%zu)\n", bad ? "WRONG" : "OK", bad);
  return 0;
}
