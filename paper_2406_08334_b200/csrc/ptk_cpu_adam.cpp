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
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

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

// The element loop, branch-free inside so it vectorises (IEEE vdivps /
// vsqrtps keep it bit-exact with the GPU rule; no FMA contraction).
template <bool kL2, bool kDecay, bool kOut>
inline __attribute__((always_inline)) void update_run(const ptk_adam_scalars& s, float* __restrict__ pm,
                                                       float* __restrict__ mm, float* __restrict__ vm,
                                                       const uint16_t* __restrict__ gr,
                                                       uint16_t* __restrict__ out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    float g = bf16_to_f32(gr[i]) * s.gscale;
    float p = pm[i];
    if (kL2) g = g + s.wd * p;
    if (kDecay) p = p * s.decay;
    float m = mm[i];
    m = m + s.w1 * (g - m);
    float v = vm[i];
    v = v * s.b2 + s.w2 * (g * g);
    const float d = std::sqrt(v) / s.bc2_sqrt + s.eps;
    p = p + s.neg_step_size * (m / d);
    pm[i] = p;
    mm[i] = m;
    vm[i] = v;
    if (kOut) out[i] = f32_to_bf16(p);
  }
}

// One block of the shard, compiled for AVX-512, AVX2 and baseline x86-64
// (resolved once at load time), so the library runs on any host CPU.
__attribute__((target_clones("avx512f", "avx2", "default"))) void update_block(
    const ptk_adam_scalars& s, float* pm, float* mm, float* vm, const uint16_t* gr, uint16_t* out,
    int64_t n) {
  const bool l2 = s.wd != 0.0f, decay = s.adamw != 0, has_out = out != nullptr;
  if (l2) {
    if (has_out) update_run<true, false, true>(s, pm, mm, vm, gr, out, n);
    else update_run<true, false, false>(s, pm, mm, vm, gr, out, n);
  } else if (decay) {
    if (has_out) update_run<false, true, true>(s, pm, mm, vm, gr, out, n);
    else update_run<false, true, false>(s, pm, mm, vm, gr, out, n);
  } else {
    if (has_out) update_run<false, false, true>(s, pm, mm, vm, gr, out, n);
    else update_run<false, false, false>(s, pm, mm, vm, gr, out, n);
  }
}

constexpr int64_t kBlock = 1 << 16;

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
  const bool stats = sumsq_out != nullptr || nonfinite_out != nullptr;
  const int64_t blocks = (n + kBlock - 1) / kBlock;
  // Per-block statistics summed in block order afterwards: the result does
  // not depend on which thread ran which block.
  std::vector<double> part_sq(stats ? blocks : 0);
  std::vector<int64_t> part_bad(stats ? blocks : 0);
  // Dynamic scheduling by default: the host Adam shares the cores with the
  // launching threads and the copy engines' host traffic, and under that
  // oversubscription a static split waits for its slowest (preempted) thread.
  // PTK_CPU_ADAM_SCHEDULE=static restores the static split.
  static const bool kStatic = [] {
    const char* e = std::getenv("PTK_CPU_ADAM_SCHEDULE");
    return e && std::string(e) == "static";
  }();
  auto body = [&](int64_t b) {
    const int64_t lo = b * kBlock, len = std::min(kBlock, n - lo);
    if (stats) {  // statistics of this block's scaled gradient (still in cache after)
      double sq = 0.0;
      int64_t bad = 0;
      for (int64_t i = lo; i < lo + len; ++i) {
        const float g = bf16_to_f32(grad[i]) * s.gscale;
        sq += static_cast<double>(g) * static_cast<double>(g);
        bad += std::isfinite(g) ? 0 : 1;
      }
      part_sq[b] = sq;
      part_bad[b] = bad;
    }
    update_block(s, master + lo, exp_avg + lo, exp_avg_sq + lo, grad + lo,
                 param_out ? param_out + lo : nullptr, len);
  };
  if (kStatic) {
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t b = 0; b < blocks; ++b) body(b);
  } else {
#pragma omp parallel for num_threads(threads) schedule(dynamic, 2)
    for (int64_t b = 0; b < blocks; ++b) body(b);
  }
  double sq = 0.0;
  int64_t bad = 0;
  for (int64_t b = 0; b < static_cast<int64_t>(part_sq.size()); ++b) {
    sq += part_sq[b];
    bad += part_bad[b];
  }
  if (sumsq_out) *sumsq_out = sq;
  if (nonfinite_out) *nonfinite_out = bad;
  return PTK_OK;
}
