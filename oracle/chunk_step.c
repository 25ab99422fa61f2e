/* CPU ORACLE for the chunk data plane — TEST INFRASTRUCTURE, NOT PRODUCT.
 * See chunk_step.h for what is restated and from where (parity of the data
 * plane is unpinned by the reference; cross-checked against torch.optim.Adam).
 * Build: oracle/Makefile (`make port`), -O3 -fopenmp -ffp-contract=off. */
#include "chunk_step.h"

#include <math.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* torchrun exports OMP_NUM_THREADS=1 to every rank; the CPU baseline arm
 * sets the thread count it actually uses explicitly. */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

static inline uint16_t to_bf16(float f) {
  uint32_t u = f2u(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fff; /* canonical NaN */
  u += 0x7fffu + ((u >> 16) & 1u);                    /* round to nearest even */
  return (uint16_t)(u >> 16);
}

static inline float from_bf16(uint16_t h) { return u2f((uint32_t)h << 16); }

/* exported wrappers (internal loops use the inline forms so they vectorise) */
uint16_t oracle_f32_to_bf16(float f) { return to_bf16(f); }
float oracle_bf16_to_f32(uint16_t h) { return from_bf16(h); }
#define oracle_f32_to_bf16 to_bf16
#define oracle_bf16_to_f32 from_bf16

void oracle_adam_scalars(double lr, double beta1, double beta2, double eps,
                         double weight_decay, int adamw, int step,
                         double grad_scale, oracle_adam_scalars_t* s) {
  const double bc1 = 1.0 - pow(beta1, (double)step);
  const double bc2 = 1.0 - pow(beta2, (double)step);
  s->gscale = (float)grad_scale;
  s->adamw = adamw;
  s->wd = adamw ? 0.0f : (float)weight_decay;
  s->decay = adamw ? (float)(1.0 - lr * weight_decay) : 1.0f;
  s->w1 = (float)(1.0 - beta1);
  s->b2 = (float)beta2;
  s->w2 = (float)(1.0 - beta2);
  s->eps = (float)eps;
  s->neg_step_size = (float)(-(lr / bc1));
  s->bc2_sqrt = (float)sqrt(bc2);
}

/* The per-element rule, shared by both grad precisions. */
static inline float adam_elem(const oracle_adam_scalars_t* s, float g, float* p,
                              float* m, float* v) {
  float pv = *p;
  if (s->wd != 0.0f) g = g + s->wd * pv;
  if (s->adamw) pv = pv * s->decay;
  float mv = *m;
  mv = mv + s->w1 * (g - mv);
  float vv = *v;
  vv = vv * s->b2 + s->w2 * (g * g);
  const float d = sqrtf(vv) / s->bc2_sqrt + s->eps;
  pv = pv + s->neg_step_size * (mv / d);
  *m = mv;
  *v = vv;
  *p = pv;
  return pv;
}

/* Blocks of 64 Ki elements per OpenMP iteration: the fp64 statistics loop
 * and the (vectorisable, reduction-free) update loop run per block. */
#define ORACLE_BLOCK ((int64_t)1 << 16)

void oracle_adam_step(const oracle_adam_scalars_t* s, float* master, float* m,
                      float* v, const uint16_t* grad, uint16_t* param_out,
                      int64_t n, double* sumsq, int64_t* nonfinite) {
  double sq = 0.0;
  int64_t bad = 0;
  const int64_t blocks = (n + ORACLE_BLOCK - 1) / ORACLE_BLOCK;
#pragma omp parallel for schedule(static) reduction(+ : sq, bad)
  for (int64_t b = 0; b < blocks; ++b) {
    const int64_t lo = b * ORACLE_BLOCK;
    const int64_t hi = lo + ORACLE_BLOCK < n ? lo + ORACLE_BLOCK : n;
    for (int64_t i = lo; i < hi; ++i) {
      const float g = oracle_bf16_to_f32(grad[i]) * s->gscale;
      sq += (double)g * (double)g;
      bad += isfinite(g) ? 0 : 1;
    }
    const oracle_adam_scalars_t sc = *s; /* local copy: provably not aliased by the stores */
    if (param_out) {
      for (int64_t i = lo; i < hi; ++i)
        param_out[i] = oracle_f32_to_bf16(
            adam_elem(&sc, oracle_bf16_to_f32(grad[i]) * sc.gscale, &master[i], &m[i], &v[i]));
    } else {
      for (int64_t i = lo; i < hi; ++i)
        adam_elem(&sc, oracle_bf16_to_f32(grad[i]) * sc.gscale, &master[i], &m[i], &v[i]);
    }
  }
  if (sumsq) *sumsq = sq;
  if (nonfinite) *nonfinite = bad;
}

void oracle_adam_step_f32grad(const oracle_adam_scalars_t* s, float* master,
                              float* m, float* v, const float* grad,
                              uint16_t* param_out, int64_t n, double* sumsq,
                              int64_t* nonfinite) {
  double sq = 0.0;
  int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : sq, bad)
  for (int64_t i = 0; i < n; ++i) {
    const float g = grad[i] * s->gscale;
    sq += (double)g * (double)g;
    bad += isfinite(g) ? 0 : 1;
    const float p = adam_elem(s, g, &master[i], &m[i], &v[i]);
    if (param_out) param_out[i] = oracle_f32_to_bf16(p);
  }
  if (sumsq) *sumsq = sq;
  if (nonfinite) *nonfinite = bad;
}

int64_t oracle_shard_elems(int64_t n, int world) {
  const int64_t q = (int64_t)world * 8;
  const int64_t n_pad = (n + q - 1) / q * q;
  return n_pad / world;
}

void oracle_allgather_bf16(const uint16_t* const* shards, int world,
                           int64_t shard, uint16_t* full) {
  for (int r = 0; r < world; ++r)
    memcpy(full + (int64_t)r * shard, shards[r], (size_t)shard * sizeof(uint16_t));
}

void oracle_reduce_scatter_f32(const uint16_t* const* grads, int world,
                               int rank, int64_t shard, float* out) {
  const int64_t off = (int64_t)rank * shard;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < shard; ++i) {
    float acc = oracle_bf16_to_f32(grads[0][off + i]);
    for (int r = 1; r < world; ++r) acc = acc + oracle_bf16_to_f32(grads[r][off + i]);
    out[i] = acc;
  }
}

void oracle_reduce_scatter_bf16(const uint16_t* const* grads, int world,
                                int rank, int64_t shard, uint16_t* out) {
  const int64_t off = (int64_t)rank * shard;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < shard; ++i) {
    float acc = oracle_bf16_to_f32(grads[0][off + i]);
    for (int r = 1; r < world; ++r) acc = acc + oracle_bf16_to_f32(grads[r][off + i]);
    out[i] = oracle_f32_to_bf16(acc);
  }
}

static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline float uniform_pm1(uint64_t seed, uint64_t i) {
  const uint32_t top = (uint32_t)(splitmix64(seed ^ i) >> 40); /* 24 bits */
  return ((float)top * 0x1p-24f) * 2.0f - 1.0f;
}

void oracle_fill_uniform_f32(float* out, int64_t n, uint64_t seed, int64_t index0, float scale) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = scale * uniform_pm1(seed, (uint64_t)(index0 + i));
}

void oracle_fill_uniform_bf16(uint16_t* out, int64_t n, uint64_t seed, int64_t index0,
                              float scale) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    out[i] = oracle_f32_to_bf16(scale * uniform_pm1(seed, (uint64_t)(index0 + i)));
}
