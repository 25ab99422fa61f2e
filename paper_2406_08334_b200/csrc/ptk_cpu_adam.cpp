// K6: host Adam over an offloaded (non-persistent) chunk shard.
//
// The reference charges `nonpersist_params / cpu_optim_rate` for this
// (proj/src/cost.cpp:213-218) and runs it as a serial CPU queue that drains
// while the GPU continues backward (proj/src/sim.cpp:446-451,552-562). Here it
// is real work: OpenMP across all host cores, the same fp32 update rule and
// the same scalars (ptk::derive_scalars) as the GPU kernel, so a chunk
// updated on the CPU is bit-identical to one updated on the GPU.
#include <omp.h>

#include <cmath>
#include <cstring>

#include "ptk_common.h"

namespace {

inline float bf16_to_f32(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

inline uint16_t f32_to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fff;
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

}  // namespace

extern "C" int ptk_cpu_adam(const ptk_adam_config* cfg, float* master, float* exp_avg,
                            float* exp_avg_sq, const uint16_t* grad, uint16_t* param_out,
                            int64_t n, int32_t n_threads, double* sumsq_out,
                            int64_t* nonfinite_out) {
  if (!cfg || !master || !exp_avg || !exp_avg_sq || !grad || n < 0)
    return ptk::fail(PTK_EINVAL, "ptk_cpu_adam: bad arguments");
  if (cfg->step < 1) return ptk::fail(PTK_EINVAL, "ptk_cpu_adam: step must be >= 1");
  const ptk_adam_scalars s = ptk::derive_scalars(*cfg);
  const int threads = n_threads > 0 ? n_threads : omp_get_max_threads();
  double sq = 0.0;
  int64_t bad = 0;
#pragma omp parallel for num_threads(threads) schedule(static) reduction(+ : sq, bad)
  for (int64_t i = 0; i < n; ++i) {
    float g = bf16_to_f32(grad[i]) * s.gscale;
    sq += static_cast<double>(g) * static_cast<double>(g);
    bad += std::isfinite(g) ? 0 : 1;
    float p = master[i];
    if (s.wd != 0.0f) g = g + s.wd * p;
    if (s.adamw) p = p * s.decay;
    float m = exp_avg[i];
    m = m + s.w1 * (g - m);
    float v = exp_avg_sq[i];
    v = v * s.b2 + s.w2 * (g * g);
    const float d = std::sqrt(v) / s.bc2_sqrt + s.eps;
    p = p + s.neg_step_size * (m / d);
    master[i] = p;
    exp_avg[i] = m;
    exp_avg_sq[i] = v;
    if (param_out) param_out[i] = f32_to_bf16(p);
  }
  if (sumsq_out) *sumsq_out = sq;
  if (nonfinite_out) *nonfinite_out = bad;
  return PTK_OK;
}
