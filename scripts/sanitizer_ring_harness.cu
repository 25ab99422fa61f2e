// Standalone TMA-ring harness used to tell compute-sanitizer artifacts from
// real hazards (profiles/r01_sanitizer.txt). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -lineinfo -o ring scripts/sanitizer_ring_harness.cu
// Run: compute-sanitizer --tool synccheck ./ring <0..4>
// minimal TMA ring (same protocol as chunk_adam_tma_kernel) for the sanitizer:
// kStages mbarriers, producer thread 0 runs kStages-2 tiles ahead.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int kStages, int kTile>
__global__ void ring(const float* src, float* dst, int tiles_per_cta) {
  extern __shared__ __align__(128) float sbuf[];
  __shared__ __align__(8) unsigned long long full[kStages];
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[i])), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int k) {
    const int st = k % kStages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(kTile * 4) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su(sbuf + st * kTile)), "l"(src + ((long)blockIdx.x * tiles_per_cta + k) * kTile), "r"(kTile * 4), "r"(su(&full[st])) : "memory");
  };
  constexpr int kAhead = kStages - 2;
  if (threadIdx.x == 0) for (int k = 0; k < kAhead && k < tiles_per_cta; ++k) issue(k);
  for (int k = 0; k < tiles_per_cta; ++k) {
    if (threadIdx.x == 0 && k + kAhead < tiles_per_cta) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue(k + kAhead);
    }
    const int st = k % kStages;
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n"
                 ::"r"(su(&full[st])), "r"((k / kStages) & 1) : "memory");
    for (int e = threadIdx.x; e < kTile; e += blockDim.x) sbuf[st * kTile + e] *= 2.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + ((long)blockIdx.x * tiles_per_cta + k) * kTile), "r"(su(sbuf + st * kTile)), "r"(kTile * 4) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
template <int S>
void run(const float* a, float* b, int tiles) {
  const int smem = S * 1024 * 4;
  cudaFuncSetAttribute(ring<S, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ring<S, 1024><<<148, 256, smem>>>(a, b, tiles);
  printf("stages=%d tiles=%d %s\n", S, tiles, cudaGetErrorString(cudaDeviceSynchronize()));
}
int main(int argc, char** argv) {
  float *a, *b;
  cudaMalloc(&a, 148L * 12 * 4096); cudaMalloc(&b, 148L * 12 * 4096);
  cudaMemset(a, 0, 148L * 12 * 4096);
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  if (which == 0) { run<9>(a, b, 3); }
  if (which == 1) { run<9>(a, b, 12); }
  if (which == 2) { run<4>(a, b, 3); }
  if (which == 3) { run<6>(a, b, 3); }
  if (which == 4) { run<6>(a, b, 5); }
  return 0;
}
