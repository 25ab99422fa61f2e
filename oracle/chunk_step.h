/* CPU ORACLE for the chunk data plane — TEST INFRASTRUCTURE, NOT PRODUCT.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference arm may load this library.
 *
 * What it restates. The reference (memplan) never executes the data plane:
 * it models it as times — all-gather `gather_time` (proj/src/hardware.cpp:29-34),
 * reduce-scatter `reduce_time` (hardware.cpp:36-38), GPU/CPU Adam
 * `persist_params / gpu_optim_rate` (proj/src/cost.cpp:206-219) — and SPEC.md:514
 * makes optimizer numerics a non-goal. The data-plane numerics are therefore
 * PARITY UNPINNED by the reference. The paper names apex FusedAdam /
 * DeepSpeed CPU Adam; neither is present or pinned here, so the
 * update rule below follows torch 2.11 `torch.optim.Adam` single-tensor order
 * (torch/optim/adam.py:414-540: lerp_ first moment, mul_+addcmul_ second
 * moment, sqrt/bias_correction2_sqrt + eps denominator, addcdiv_ with
 * -step_size) and tests/test_oracle_adam.py cross-checks it against torch.
 *
 * Per element, fp32, no FMA contraction (built with -ffp-contract=off):
 *   g  = f32(grad_bf16) * gscale
 *   L2:    g = g + wd * p          AdamW:  p = p * (1 - lr*wd)
 *   m  = m + (1-b1) * (g - m)
 *   v  = v * b2 + (1-b2) * (g * g)
 *   d  = sqrt(v) / sqrt(1-b2^t) + eps
 *   p  = p + (-lr/(1-b1^t)) * (m / d)
 *   param_bf16 = RNE(p)   (NaN -> 0x7FFF)
 * Scalars are derived in double on the host and rounded once to float
 * (oracle_adam_scalars), the same derivation the CUDA path uses, so the GPU
 * kernel and this oracle agree BIT-EXACTLY on master/m/v/param.
 *
 * Simulated ranks: all-gather = memcpy of w shards; reduce-scatter = fp32
 * sum over ranks in rank order 0..w-1, rounded once to bf16 (or kept fp32).
 * Shard mapping: a chunk of n elements is padded to n_pad = roundup(n, w*8)
 * and rank r owns [r*n_pad/w, (r+1)*n_pad/w). The reference's modeled shard
 * is floor(used/w) bytes (proj/src/cost.cpp:20-22); padding is physical only.
 */
#ifndef ORACLE_CHUNK_STEP_H
#define ORACLE_CHUNK_STEP_H
#include <stdint.h>
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  float gscale, wd, decay, w1, b2, w2, eps, neg_step_size, bc2_sqrt;
  int adamw;
} oracle_adam_scalars_t;

void oracle_adam_scalars(double lr, double beta1, double beta2, double eps,
                         double weight_decay, int adamw, int step,
                         double grad_scale, oracle_adam_scalars_t* out);

/* One Adam step over n elements; sumsq/nonfinite (nullable) get the grad
 * statistics of g (after gscale, before weight decay). Threads: OpenMP. */
void oracle_adam_step(const oracle_adam_scalars_t* s, float* master, float* m,
                      float* v, const uint16_t* grad, uint16_t* param_out,
                      int64_t n, double* sumsq, int64_t* nonfinite);

/* Same, grads given as fp32 (used after an fp32 reduce-scatter). */
void oracle_adam_step_f32grad(const oracle_adam_scalars_t* s, float* master,
                              float* m, float* v, const float* grad,
                              uint16_t* param_out, int64_t n, double* sumsq,
                              int64_t* nonfinite);

int64_t oracle_shard_elems(int64_t n, int world);

/* full[w*shard] <- concat(shards[r]) */
void oracle_allgather_bf16(const uint16_t* const* shards, int world,
                           int64_t shard, uint16_t* full);
/* out <- RNE(sum_r grads[r][rank*shard : (rank+1)*shard]) */
void oracle_reduce_scatter_bf16(const uint16_t* const* grads, int world,
                                int rank, int64_t shard, uint16_t* out);
void oracle_reduce_scatter_f32(const uint16_t* const* grads, int world,
                               int rank, int64_t shard, float* out);

uint16_t oracle_f32_to_bf16(float f);
float oracle_bf16_to_f32(uint16_t h);
/* counter-based input generator: u in [-1,1), exact in fp32 */
void oracle_fill_uniform_f32(float* out, int64_t n, uint64_t seed, int64_t index0, float scale);
void oracle_fill_uniform_bf16(uint16_t* out, int64_t n, uint64_t seed, int64_t index0,
                              float scale);
int oracle_num_threads(void);
void oracle_set_num_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
