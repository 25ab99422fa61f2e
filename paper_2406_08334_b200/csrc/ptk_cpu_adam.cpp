// K6: host Adam over an offloaded (non-persistent) chunk shard.
//
// The reference charges `nonpersist_params / cpu_optim_rate` for this
// (proj/src/cost.cpp:213-218) and runs it as a serial CPU queue that drains
// while the GPU continues backward (proj/src/sim.cpp:446-451,552-562). Here it
// is real work: OpenMP across all host cores, the same fp32 update rule and
// the same scalars (ptk::derive_scalars) as the GPU kernel, so a chunk
// updated on the CPU is bit-identical to one updated on the GPU.
#include <immintrin.h>
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

inline float grad_f32(uint16_t g) { return bf16_to_f32(g); }
inline float grad_f32(float g) { return g; }

// The element loop, branch-free inside so it vectorises (IEEE vdivps /
// vsqrtps keep it bit-exact with the GPU rule; no FMA contraction). G is the
// gradient type: bf16 bits, or fp32 (a reduce-scattered sum kept in fp32).
template <bool kL2, bool kDecay, bool kOut, class G>
inline __attribute__((always_inline)) void update_run(const ptk_adam_scalars& s, float* __restrict__ pm,
                                                       float* __restrict__ mm, float* __restrict__ vm,
                                                       const G* __restrict__ gr,
                                                       uint16_t* __restrict__ out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    float g = grad_f32(gr[i]) * s.gscale;
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
template <class G>
inline __attribute__((always_inline)) void update_block_body(
    const ptk_adam_scalars& s, float* pm, float* mm, float* vm, const G* gr, uint16_t* out,
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

__attribute__((target_clones("avx512f", "avx2", "default"))) void update_block(
    const ptk_adam_scalars& s, float* pm, float* mm, float* vm, const uint16_t* gr, uint16_t* out,
    int64_t n) {
  update_block_body(s, pm, mm, vm, gr, out, n);
}

__attribute__((target_clones("avx512f", "avx2", "default"))) void update_block(
    const ptk_adam_scalars& s, float* pm, float* mm, float* vm, const float* gr, uint16_t* out,
    int64_t n) {
  update_block_body(s, pm, mm, vm, gr, out, n);
}

// AVX-512 variant with the bf16 parameter output written by non-temporal
// stores: the output is write-only, so streaming it saves the read-for-
// ownership of its cache lines (2 of ~30 host DRAM bytes per parameter --
// host DRAM is what the offloaded iteration is bound by). The arithmetic is
// the same sequence of IEEE single operations as update_run (no FMA), so the
// result is bit-identical; the rounding to bf16 is f32_to_bf16's.
template <class G>
__attribute__((target("avx512f,avx512bw"))) inline __m512 load_grad16(const G* gr) {
  if constexpr (sizeof(G) == 2) {
    const __m256i gb = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(gr));
    return _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(gb), 16));
  } else {
    return _mm512_loadu_ps(reinterpret_cast<const float*>(gr));
  }
}

template <bool kL2, bool kDecay, class G>
__attribute__((target("avx512f,avx512bw"))) void update_run_nt(
    const ptk_adam_scalars& s, float* __restrict__ pm, float* __restrict__ mm,
    float* __restrict__ vm, const G* __restrict__ gr, uint16_t* __restrict__ out,
    int64_t n) {
  int64_t i = 0;
  // scalar head until the output is 32-byte aligned (stream stores need it)
  while (i < n && (reinterpret_cast<uintptr_t>(out + i) & 31u) != 0) {
    update_run<kL2, kDecay, true>(s, pm + i, mm + i, vm + i, gr + i, out + i, 1);
    ++i;
  }
  const __m512 gscale = _mm512_set1_ps(s.gscale), wd = _mm512_set1_ps(s.wd),
               decay = _mm512_set1_ps(s.decay), w1 = _mm512_set1_ps(s.w1),
               b2 = _mm512_set1_ps(s.b2), w2 = _mm512_set1_ps(s.w2),
               bc2 = _mm512_set1_ps(s.bc2_sqrt), eps = _mm512_set1_ps(s.eps),
               step = _mm512_set1_ps(s.neg_step_size);
  const __m512i abs_mask = _mm512_set1_epi32(0x7fffffff), inf = _mm512_set1_epi32(0x7f800000),
                round = _mm512_set1_epi32(0x7fff), one = _mm512_set1_epi32(1),
                qnan = _mm512_set1_epi32(0x7fff);
  for (; i + 16 <= n; i += 16) {
    __m512 g = _mm512_mul_ps(load_grad16(gr + i), gscale);
    __m512 p = _mm512_loadu_ps(pm + i);
    if (kL2) g = _mm512_add_ps(g, _mm512_mul_ps(wd, p));
    if (kDecay) p = _mm512_mul_ps(p, decay);
    __m512 m = _mm512_loadu_ps(mm + i);
    m = _mm512_add_ps(m, _mm512_mul_ps(w1, _mm512_sub_ps(g, m)));
    __m512 v = _mm512_loadu_ps(vm + i);
    v = _mm512_add_ps(_mm512_mul_ps(v, b2), _mm512_mul_ps(w2, _mm512_mul_ps(g, g)));
    const __m512 d = _mm512_add_ps(_mm512_div_ps(_mm512_sqrt_ps(v), bc2), eps);
    p = _mm512_add_ps(p, _mm512_mul_ps(step, _mm512_div_ps(m, d)));
    _mm512_storeu_ps(pm + i, p);
    _mm512_storeu_ps(mm + i, m);
    _mm512_storeu_ps(vm + i, v);
    const __m512i u = _mm512_castps_si512(p);
    __m512i r = _mm512_add_epi32(_mm512_add_epi32(u, round),
                                 _mm512_and_si512(_mm512_srli_epi32(u, 16), one));
    r = _mm512_srli_epi32(r, 16);
    const __mmask16 nan = _mm512_cmpgt_epu32_mask(_mm512_and_si512(u, abs_mask), inf);
    r = _mm512_mask_mov_epi32(r, nan, qnan);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + i), _mm512_cvtepi32_epi16(r));
  }
  if (i < n) update_run<kL2, kDecay, true>(s, pm + i, mm + i, vm + i, gr + i, out + i, n - i);
  _mm_sfence();  // the streamed output is visible before the caller publishes it
}

bool use_nt_path() {
  static const bool ok = [] {
    const char* e = std::getenv("PTK_CPU_ADAM_NT");
    if (e && std::string(e) == "0") return false;
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");
  }();
  return ok;
}

template <class G>
void update_block_dispatch(const ptk_adam_scalars& s, float* pm, float* mm, float* vm,
                           const G* gr, uint16_t* out, int64_t n) {
  if (out != nullptr && use_nt_path()) {
    if (s.wd != 0.0f) update_run_nt<true, false>(s, pm, mm, vm, gr, out, n);
    else if (s.adamw != 0) update_run_nt<false, true>(s, pm, mm, vm, gr, out, n);
    else update_run_nt<false, false>(s, pm, mm, vm, gr, out, n);
    return;
  }
  update_block(s, pm, mm, vm, gr, out, n);
}

constexpr int64_t kBlock = 1 << 16;

template <class G>
int cpu_adam(const char* what, const ptk_adam_config* cfg, float* master, float* exp_avg,
             float* exp_avg_sq, const G* grad, uint16_t* param_out, int64_t n,
             int32_t n_threads, double* sumsq_out, int64_t* nonfinite_out) {
  if (!cfg || !master || !exp_avg || !exp_avg_sq || !grad || n < 0)
    return ptk::fail(PTK_EINVAL, std::string(what) + ": bad arguments");
  if (cfg->step < 1) return ptk::fail(PTK_EINVAL, std::string(what) + ": step must be >= 1");
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
        const float g = grad_f32(grad[i]) * s.gscale;
        sq += static_cast<double>(g) * static_cast<double>(g);
        bad += std::isfinite(g) ? 0 : 1;
      }
      part_sq[b] = sq;
      part_bad[b] = bad;
    }
    update_block_dispatch(s, master + lo, exp_avg + lo, exp_avg_sq + lo, grad + lo,
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

}  // namespace

extern "C" int ptk_cpu_adam(const ptk_adam_config* cfg, float* master, float* exp_avg,
                            float* exp_avg_sq, const uint16_t* grad, uint16_t* param_out,
                            int64_t n, int32_t n_threads, double* sumsq_out,
                            int64_t* nonfinite_out) {
  return cpu_adam("ptk_cpu_adam", cfg, master, exp_avg, exp_avg_sq, grad, param_out, n,
                  n_threads, sumsq_out, nonfinite_out);
}

extern "C" int ptk_cpu_adam_f32grad(const ptk_adam_config* cfg, float* master, float* exp_avg,
                                    float* exp_avg_sq, const float* grad, uint16_t* param_out,
                                    int64_t n, int32_t n_threads, double* sumsq_out,
                                    int64_t* nonfinite_out) {
  return cpu_adam("ptk_cpu_adam_f32grad", cfg, master, exp_avg, exp_avg_sq, grad, param_out, n,
                  n_threads, sumsq_out, nonfinite_out);
}
