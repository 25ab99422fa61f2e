// Shared host-side helpers of libptk (error state, launch accounting).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "ptk.h"

namespace ptk {

void set_error(const std::string& msg);
std::atomic<int64_t>& launch_counter();

inline int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

inline int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PTK_OK;
  return fail(PTK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Host derivation of the fp32 kernel scalars (one rounding per scalar).
ptk_adam_scalars derive_scalars(const ptk_adam_config& cfg);

}  // namespace ptk

#define PTK_TRY_CUDA(expr)                                   \
  do {                                                       \
    int ptk_rc_ = ::ptk::check_cuda((expr), #expr);          \
    if (ptk_rc_ != PTK_OK) return ptk_rc_;                   \
  } while (0)
