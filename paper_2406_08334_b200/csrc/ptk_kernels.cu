// libptk device kernels for sm_100a: the chunk data plane of ProTrain.
//
//   K1+K2  chunk_adam_kernel     fused grad cast/scale + grad-norm/overflow
//                                statistics + Adam/AdamW over a flat chunk
//                                shard (28 B/param of HBM traffic, bf16 grad)
//   K2     grad_stats_kernel     standalone statistics (+ fp32 scaled copy)
//   K1+K3+K4 fused_peer_kernel   reduce-scatter (fp32 sum over NVLink peer
//                                loads) -> Adam -> all-gather (peer stores)
//   aux    fill kernels (counter-based synthetic inputs), clip coefficient,
//          peer barrier (system-scope release/acquire flags)
//
// The modeled counterparts in the reference are listed in include/ptk.h.
// Design notes: every kernel is HBM-streaming integer/fp32
// element work — no data reuse, so no tensor cores and no shared-memory
// tiling; the levers are 128-bit coalesced accesses, enough bytes in flight
// per SM (UNROLL independent 8-element units per thread, all loads issued
// before any math), a persistent grid sized to the SM count × occupancy,
// streaming cache hints (.cs) so the once-touched chunk bytes do not thrash
// L2, and deterministic warp-shuffle → CTA → last-CTA reductions for the
// statistics. The update arithmetic uses explicit round-to-nearest
// intrinsics (no FMA contraction) so it matches oracle/chunk_step.c bit for
// bit.
#include <cuda_runtime.h>

#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "ptk_common.h"

namespace ptk {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxGrid = 4096;

struct StatsWorkspace {
  double sq[kMaxGrid];
  unsigned long long bad[kMaxGrid];
  unsigned int arrived;
  unsigned int pad[3];
};

// ---------------------------------------------------------------- helpers --

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  f[0] = bf_lo(u.x); f[1] = bf_hi(u.x);
  f[2] = bf_lo(u.y); f[3] = bf_hi(u.y);
  f[4] = bf_lo(u.z); f[5] = bf_hi(u.z);
  f[6] = bf_lo(u.w); f[7] = bf_hi(u.w);
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  return make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                    pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
}

__device__ __forceinline__ void ld8f(const float* p, float (&f)[8]) {
  const float4 a = __ldcs(reinterpret_cast<const float4*>(p));
  const float4 b = __ldcs(reinterpret_cast<const float4*>(p) + 1);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

__device__ __forceinline__ void st8f(float* p, const float (&f)[8]) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(f[0], f[1], f[2], f[3]));
  __stcs(reinterpret_cast<float4*>(p) + 1, make_float4(f[4], f[5], f[6], f[7]));
}

// Gradient loaders: 8 consecutive elements as fp32.
struct GradBf16 {
  using T = uint16_t;
  __device__ __forceinline__ static void load8(const uint16_t* g, float (&f)[8]) {
    const uint4 u = __ldcs(reinterpret_cast<const uint4*>(g));
    unpack8(u, f);
  }
  __device__ __forceinline__ static float load1(const uint16_t* g) {
    return __uint_as_float(static_cast<uint32_t>(*g) << 16);
  }
};
struct GradF32 {
  using T = float;
  __device__ __forceinline__ static void load8(const float* g, float (&f)[8]) { ld8f(g, f); }
  __device__ __forceinline__ static float load1(const float* g) { return *g; }
};

// The per-element update rule (see oracle/chunk_step.h for the statement).
__device__ __forceinline__ float adam_elem(const ptk_adam_scalars& s, float g, float& p,
                                           float& m, float& v) {
  if (s.wd != 0.0f) g = __fadd_rn(g, __fmul_rn(s.wd, p));
  if (s.adamw) p = __fmul_rn(p, s.decay);
  m = __fadd_rn(m, __fmul_rn(s.w1, __fsub_rn(g, m)));
  v = __fadd_rn(__fmul_rn(v, s.b2), __fmul_rn(s.w2, __fmul_rn(g, g)));
  const float d = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), s.bc2_sqrt), s.eps);
  p = __fadd_rn(p, __fmul_rn(s.neg_step_size, __fdiv_rn(m, d)));
  return p;
}

// Statistics: squares are summed in fp32 over one 8-element unit, the unit
// sums in fp64 per thread (keeps the full-chunk sum within ~1e-7 relative).
__device__ __forceinline__ void accum_stats(float g, float& sq, unsigned& bad) {
  sq = __fmaf_rn(g, g, sq);
  bad += isfinite(g) ? 0u : 1u;
}

// Deterministic grid reduction: warp shuffle -> CTA (fixed order) -> the last
// CTA to arrive sums the per-CTA partials in index order and ADDS the result
// to *stats. Safe across back-to-back launches on one stream (the arrival
// counter is re-armed by the last CTA).
__device__ __forceinline__ void reduce_stats(double sq, unsigned bad, StatsWorkspace* ws,
                                             ptk_grad_stats_t* stats) {
  __shared__ double s_sq[32];
  __shared__ unsigned long long s_bad[32];
  __shared__ bool s_last;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sq += __shfl_xor_sync(0xffffffffu, sq, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_sq[warp] = sq;
    s_bad[warp] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bsq = 0.0;
    unsigned long long bbad = 0;
    for (unsigned w = 0; w < blockDim.x / 32; ++w) {
      bsq += s_sq[w];
      bbad += s_bad[w];
    }
    ws->sq[blockIdx.x] = bsq;
    ws->bad[blockIdx.x] = bbad;
    __threadfence();
    const unsigned prev = atomicAdd(&ws->arrived, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // one warp: lane l sums partials l, l+32, ... then a fixed xor tree, so the
  // total is the same every run (and not a 148-long serial chain of L2 loads)
  if (threadIdx.x < 32) {
    double tsq = 0.0;
    unsigned long long tbad = 0;
    const volatile double* vsq = ws->sq;
    const volatile unsigned long long* vbad = ws->bad;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) {
      tsq += vsq[b];
      tbad += vbad[b];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tsq += __shfl_xor_sync(0xffffffffu, tsq, o);
      tbad += __shfl_xor_sync(0xffffffffu, tbad, o);
    }
    if (threadIdx.x == 0) {
      stats->sumsq += tsq;
      stats->nonfinite += tbad;
      ws->arrived = 0;
    }
  }
}

// ------------------------------------------------------------ K1 + K2 ----

template <class G, int U, bool kStats>
__device__ __forceinline__ void adam_body(ptk_adam_scalars s, float* __restrict__ master,
                                          float* __restrict__ exp_avg,
                                          float* __restrict__ exp_avg_sq,
                                          const typename G::T* __restrict__ grad,
                                          uint16_t* __restrict__ param_out, int64_t n,
                                          StatsWorkspace* ws, ptk_grad_stats_t* stats,
                                          const float* gscale_dev, const int32_t* skip_dev) {
  if (skip_dev != nullptr && *skip_dev != 0) return;  // grid-uniform
  float gs = s.gscale;
  if (gscale_dev != nullptr) gs = __fmul_rn(gs, *gscale_dev);
  double sq = 0.0;
  unsigned bad = 0;

  const int64_t nvec = n >> 3;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
  int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;

  // Main loop: U independent 8-element units per thread, loads first.
  for (; i + (U - 1) * stride < nvec; i += U * stride) {
    float p[U][8], m[U][8], v[U][8], g[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = (i + u * stride) << 3;
      G::load8(grad + e, g[u]);
      ld8f(master + e, p[u]);
      ld8f(exp_avg + e, m[u]);
      ld8f(exp_avg_sq + e, v[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = (i + u * stride) << 3;
      float usq = 0.0f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float gk = __fmul_rn(g[u][k], gs);
        if (kStats) accum_stats(gk, usq, bad);
        adam_elem(s, gk, p[u][k], m[u][k], v[u][k]);
      }
      if (kStats) sq += usq;
      st8f(master + e, p[u]);
      st8f(exp_avg + e, m[u]);
      st8f(exp_avg_sq + e, v[u]);
      if (param_out != nullptr) __stcs(reinterpret_cast<uint4*>(param_out + e), pack8(p[u]));
    }
  }
  // Remainder units.
  for (; i < nvec; i += stride) {
    const int64_t e = i << 3;
    float p[8], m[8], v[8], g[8];
    G::load8(grad + e, g);
    ld8f(master + e, p);
    ld8f(exp_avg + e, m);
    ld8f(exp_avg_sq + e, v);
    float usq = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float gk = __fmul_rn(g[k], gs);
      if (kStats) accum_stats(gk, usq, bad);
      adam_elem(s, gk, p[k], m[k], v[k]);
    }
    if (kStats) sq += usq;
    st8f(master + e, p);
    st8f(exp_avg + e, m);
    st8f(exp_avg_sq + e, v);
    if (param_out != nullptr) __stcs(reinterpret_cast<uint4*>(param_out + e), pack8(p));
  }
  // Scalar tail (< 8 elements) on CTA 0.
  const int64_t t0 = nvec << 3;
  if (blockIdx.x == 0 && threadIdx.x < n - t0) {
    const int64_t e = t0 + threadIdx.x;
    const float gk = __fmul_rn(G::load1(grad + e), gs);
    float usq = 0.0f;
    if (kStats) accum_stats(gk, usq, bad);
    sq += usq;
    float p = master[e], m = exp_avg[e], v = exp_avg_sq[e];
    adam_elem(s, gk, p, m, v);
    master[e] = p;
    exp_avg[e] = m;
    exp_avg_sq[e] = v;
    if (param_out != nullptr) param_out[e] = static_cast<uint16_t>(pack_bf16x2(p, 0.0f) & 0xffffu);
  }
  if (kStats) reduce_stats(sq, bad, ws, stats);
}

template <class G, int U, bool kStats>
__global__ void __launch_bounds__(kThreads)
chunk_adam_kernel(ptk_adam_scalars s, float* __restrict__ master, float* __restrict__ exp_avg,
                  float* __restrict__ exp_avg_sq, const typename G::T* __restrict__ grad,
                  uint16_t* __restrict__ param_out, int64_t n, StatsWorkspace* ws,
                  ptk_grad_stats_t* stats, const float* gscale_dev, const int32_t* skip_dev) {
  adam_body<G, U, kStats>(s, master, exp_avg, exp_avg_sq, grad, param_out, n, ws, stats,
                          gscale_dev, skip_dev);
}

// Same body, higher occupancy (launch bounds force <= 64 registers).
template <class G, int U, bool kStats, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
chunk_adam_occ_kernel(ptk_adam_scalars s, float* __restrict__ master, float* __restrict__ exp_avg,
                      float* __restrict__ exp_avg_sq, const typename G::T* __restrict__ grad,
                      uint16_t* __restrict__ param_out, int64_t n, StatsWorkspace* ws,
                      ptk_grad_stats_t* stats, const float* gscale_dev, const int32_t* skip_dev) {
  adam_body<G, U, kStats>(s, master, exp_avg, exp_avg_sq, grad, param_out, n, ws, stats,
                          gscale_dev, skip_dev);
}

// ------------------------------------------- K1 + K2, TMA bulk pipeline --
//
// Persistent CTAs walk whole tiles of kTile elements. One elected thread
// moves every tile with 1-D bulk copies (cp.async.bulk, the TMA engine):
// master/m/v/grad global -> shared, completion counted on an mbarrier
// (complete_tx), and after the update master/m/v/param shared -> global as a
// bulk_group. kStages tiles of shared memory form a ring; the producer runs
// kStages-2 tiles ahead of the consumers, and a stage is refilled only after
// the bulk store that last read it has finished reading shared memory
// (cp.async.bulk.wait_group.read 1). Register pressure no longer limits the
// bytes in flight: they live in shared memory.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Variants with an L2 eviction-priority hint (createpolicy evict_first): the
// chunk bytes are touched once per step, so they need not compete for L2.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, uint32_t bytes,
                                               uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void bulk_store_hint(void* dst, const void* src, uint32_t bytes,
                                                uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::
                   "l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(policy)
               : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int kTile>
struct TmaStage {
  float master[kTile];
  float m[kTile];
  float v[kTile];
  uint16_t grad[kTile];
  uint16_t param[kTile];
};

template <int kTile, int kStages, int kThr, bool kStats, bool kHint>
__global__ void __launch_bounds__(kThr, 1)
chunk_adam_tma_kernel(ptk_adam_scalars s, float* __restrict__ master, float* __restrict__ exp_avg,
                      float* __restrict__ exp_avg_sq, const uint16_t* __restrict__ grad,
                      uint16_t* __restrict__ param_out, int64_t n, StatsWorkspace* ws,
                      ptk_grad_stats_t* stats, const float* gscale_dev, const int32_t* skip_dev) {
  static_assert(kTile % (kThr * 4) == 0, "tile must be a multiple of 4 elements per thread");
  static_assert(kStages >= 3, "ring needs >= 3 stages");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto* stage = reinterpret_cast<TmaStage<kTile>*>(smem_raw);
  __shared__ __align__(8) uint64_t full[kStages];

  if (skip_dev != nullptr && *skip_dev != 0) return;
  float gs = s.gscale;
  if (gscale_dev != nullptr) gs = __fmul_rn(gs, *gscale_dev);

  const int tid = threadIdx.x;
  // Ring items of this CTA: its full tiles blockIdx.x, blockIdx.x + gridDim.x,
  // ...; the last CTA (which has no more full tiles than any other) also
  // carries the partial tile -- its multiple-of-8 part as one more, shorter
  // ring item (TMA sizes stay 16-byte multiples), so no CTA finishes with
  // un-pipelined plain loads. The < 8 trailing elements (n % 8, never the
  // case for padded shards) are updated with plain loads at the end.
  const int64_t n_full = n / kTile;
  const int64_t my_full =
      n_full > blockIdx.x ? (n_full - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const bool has_part = blockIdx.x == gridDim.x - 1;
  const int64_t rem = n - n_full * kTile;
  const int rem8 = has_part ? static_cast<int>(rem & ~int64_t{7}) : 0;
  const int64_t my_items = my_full + (rem8 > 0 ? 1 : 0);
  const bool has_param = param_out != nullptr;

  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();  // the inits are visible to the async proxy (complete_tx)
  }
  __syncthreads();

  const uint64_t policy = kHint ? evict_first_policy() : 0;
  auto load = [&](void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    if (kHint) bulk_load_hint(dst, src, bytes, bar, policy);
    else bulk_load(dst, src, bytes, bar);
  };
  auto store = [&](void* dst, const void* src, uint32_t bytes) {
    if (kHint) bulk_store_hint(dst, src, bytes, policy);
    else bulk_store(dst, src, bytes);
  };
  // item k -> (first element, length)
  auto item = [&](int64_t k, int64_t& e, int& len) {
    if (k < my_full) {
      e = (blockIdx.x + k * gridDim.x) * static_cast<int64_t>(kTile);
      len = kTile;
    } else {
      e = n_full * kTile;
      len = rem8;
    }
  };
  // Ring positions are carried as (stage, phase) counters -- the pipeline
  // state of CUTLASS -- rather than k % kStages: no 64-bit division per tile,
  // and every mbarrier access is a plain [base + 8*stage] address.
  int load_st = 0;
  auto issue_load = [&](int64_t k) {  // k-th item of this CTA, into stage load_st
    const int st = load_st;
    load_st = load_st + 1 == kStages ? 0 : load_st + 1;
    int64_t e;
    int len;
    item(k, e, len);
    TmaStage<kTile>& S = stage[st];
    mbar_expect_tx(&full[st], static_cast<uint32_t>(len) * (3 * sizeof(float) + sizeof(uint16_t)));
    load(S.master, master + e, len * 4, &full[st]);
    load(S.m, exp_avg + e, len * 4, &full[st]);
    load(S.v, exp_avg_sq + e, len * 4, &full[st]);
    load(S.grad, grad + e, len * 2, &full[st]);
  };

  constexpr int kAhead = kStages - 2;
  if (tid == 0)
    for (int64_t k = 0; k < kAhead && k < my_items; ++k) issue_load(k);

  double sq = 0.0;
  unsigned bad = 0;
  int st = 0;
  uint32_t phase = 0;
  for (int64_t k = 0; k < my_items; ++k) {
    if (tid == 0 && k + kAhead < my_items) {
      bulk_wait_read<1>();  // the store of item k-2 (same stage) has read its smem
      issue_load(k + kAhead);
    }
    int64_t ge;
    int len;
    item(k, ge, len);
    mbar_wait(&full[st], phase);
    TmaStage<kTile>& S = stage[st];
    float usq = 0.0f;
#pragma unroll
    for (int j = 0; j < kTile / (kThr * 4); ++j) {
      const int e = (j * kThr + tid) * 4;
      if (e >= len) break;  // only in the partial item (len is a multiple of 8)
      float4 p = *reinterpret_cast<float4*>(&S.master[e]);
      float4 m = *reinterpret_cast<float4*>(&S.m[e]);
      float4 v = *reinterpret_cast<float4*>(&S.v[e]);
      const uint2 g2 = *reinterpret_cast<const uint2*>(&S.grad[e]);
      float g[4] = {bf_lo(g2.x), bf_hi(g2.x), bf_lo(g2.y), bf_hi(g2.y)};
      float* pp = &p.x;
      float* mm = &m.x;
      float* vv = &v.x;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float gk = __fmul_rn(g[q], gs);
        if (kStats) accum_stats(gk, usq, bad);
        adam_elem(s, gk, pp[q], mm[q], vv[q]);
      }
      *reinterpret_cast<float4*>(&S.master[e]) = p;
      *reinterpret_cast<float4*>(&S.m[e]) = m;
      *reinterpret_cast<float4*>(&S.v[e]) = v;
      *reinterpret_cast<uint2*>(&S.param[e]) =
          make_uint2(pack_bf16x2(p.x, p.y), pack_bf16x2(p.z, p.w));
    }
    if (kStats) sq += usq;
    fence_async_smem();  // generic-proxy smem writes -> visible to the bulk store
    __syncthreads();
    if (tid == 0) {
      store(master + ge, S.master, len * 4);
      store(exp_avg + ge, S.m, len * 4);
      store(exp_avg_sq + ge, S.v, len * 4);
      if (has_param) store(param_out + ge, S.param, len * 2);
      bulk_commit();
    }
    if (++st == kStages) {
      st = 0;
      phase ^= 1u;
    }
  }
  if (tid == 0) bulk_wait_all();
  // the < 8 trailing elements of a chunk whose length is not a multiple of 8
  if (has_part) {
    const int64_t e = n_full * kTile + rem8 + tid;
    if (e < n) {
      float usq = 0.0f;
      const float gk = __fmul_rn(GradBf16::load1(grad + e), gs);
      if (kStats) accum_stats(gk, usq, bad);
      float p = master[e], mm = exp_avg[e], vv = exp_avg_sq[e];
      adam_elem(s, gk, p, mm, vv);
      master[e] = p;
      exp_avg[e] = mm;
      exp_avg_sq[e] = vv;
      if (has_param) param_out[e] = static_cast<uint16_t>(pack_bf16x2(p, 0.0f) & 0xffffu);
      if (kStats) sq += usq;
    }
  }
  if (kStats) reduce_stats(sq, bad, ws, stats);
}

// -------------------------------------------------------------- K2 -------

template <bool kWrite>
__global__ void __launch_bounds__(kThreads)
grad_stats_kernel(const uint16_t* __restrict__ grad, int64_t n, float scale,
                  float* __restrict__ out, StatsWorkspace* ws, ptk_grad_stats_t* stats) {
  double sq = 0.0;
  unsigned bad = 0;
  const int64_t nvec = n >> 3;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < nvec;
       i += stride) {
    float g[8];
    GradBf16::load8(grad + (i << 3), g);
    float usq = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      g[k] = __fmul_rn(g[k], scale);
      accum_stats(g[k], usq, bad);
    }
    sq += usq;
    if (kWrite) st8f(out + (i << 3), g);
  }
  const int64_t t0 = nvec << 3;
  if (blockIdx.x == 0 && threadIdx.x < n - t0) {
    const int64_t e = t0 + threadIdx.x;
    const float gk = __fmul_rn(GradBf16::load1(grad + e), scale);
    float usq = 0.0f;
    accum_stats(gk, usq, bad);
    sq += usq;
    if (kWrite) out[e] = gk;
  }
  reduce_stats(sq, bad, ws, stats);
}

__global__ void stats_reset_kernel(ptk_grad_stats_t* stats) {
  stats->sumsq = 0.0;
  stats->nonfinite = 0;
}

__global__ void clip_coef_kernel(const ptk_grad_stats_t* stats, double max_norm, float* coef,
                                 int32_t* skip) {
  const double norm = sqrt(stats->sumsq);
  double c = 1.0;
  if (max_norm > 0.0) {
    c = max_norm / (norm + 1e-6);
    if (c > 1.0) c = 1.0;
  }
  *coef = static_cast<float>(c);
  if (skip != nullptr) *skip = stats->nonfinite != 0 ? 1 : 0;
}

// ------------------------------------------------ K1+K3+K4 over NVLink ----

struct PeerTable {
  const uint16_t* grad[PTK_MAX_PEERS];
  uint16_t* param[PTK_MAX_PEERS];
};

template <int W>
__global__ void __launch_bounds__(kThreads)
fused_peer_kernel(ptk_adam_scalars s, PeerTable peers, int64_t offset, int64_t shard,
                  float* __restrict__ master, float* __restrict__ exp_avg,
                  float* __restrict__ exp_avg_sq, StatsWorkspace* ws, ptk_grad_stats_t* stats) {
  double sq = 0.0;
  unsigned bad = 0;
  const int64_t nvec = shard >> 3;  // shards are multiples of 8 elements
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < nvec;
       i += stride) {
    const int64_t e = i << 3;
    uint4 raw[W];
#pragma unroll
    for (int r = 0; r < W; ++r)
      raw[r] = __ldcs(reinterpret_cast<const uint4*>(peers.grad[r] + offset + e));
    float p[8], m[8], v[8], g[8], t[8];
    ld8f(master + e, p);
    ld8f(exp_avg + e, m);
    ld8f(exp_avg_sq + e, v);
    unpack8(raw[0], g);
#pragma unroll
    for (int r = 1; r < W; ++r) {  // fp32 sum in rank order (deterministic)
      unpack8(raw[r], t);
#pragma unroll
      for (int k = 0; k < 8; ++k) g[k] = __fadd_rn(g[k], t[k]);
    }
    float usq = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float gk = __fmul_rn(g[k], s.gscale);
      accum_stats(gk, usq, bad);
      adam_elem(s, gk, p[k], m[k], v[k]);
    }
    sq += usq;
    st8f(master + e, p);
    st8f(exp_avg + e, m);
    st8f(exp_avg_sq + e, v);
    const uint4 out = pack8(p);
#pragma unroll
    for (int r = 0; r < W; ++r)  // all-gather by push
      __stcs(reinterpret_cast<uint4*>(peers.param[r] + offset + e), out);
  }
  if (stats != nullptr) reduce_stats(sq, bad, ws, stats);
}

// The same K1+K3+K4 step through the TMA ring of chunk_adam_tma_kernel: per
// tile of kFusedTile owned elements one elected thread bulk-loads the local
// fp32 master/m/v tiles and the owned tile of EVERY rank's gradient chunk
// (peer memory, NVLink on a node) into one stage, the CTA sums the W
// gradients in fp32 in rank order (bit-identical to fused_peer_kernel and
// the oracle), applies Adam, and the elected thread bulk-stores the state
// locally and the bf16 tile into every rank's parameter chunk (push
// all-gather). Bytes in flight live in shared memory, not registers.
// Tile shape per W (elements; threads = tile / 4), measured with virtual
// ranks (profiles/README.md): W = 2 -> 2048, W = 1, 3, 4 -> 1536, W >= 5 -> 1024.
// Smaller W means smaller stages; the wider tile keeps ~140-150 KB of loads
// in flight per SM (tile 1024 at W = 2 reached only 0.66 of HBM).
constexpr int kFusedSmemBudget = 220 * 1024;
template <int W>
__host__ __device__ constexpr int fused_tile() { return W == 1 ? 1536 : W == 2 ? 2048 : W <= 4 ? 1536 : 1024; }
template <int W>
__host__ __device__ constexpr int fused_threads() { return fused_tile<W>() / 4; }

template <int W>
struct FusedStage {
  static constexpr int kTile = fused_tile<W>();
  float master[kTile];
  float m[kTile];
  float v[kTile];
  uint16_t grad[W][kTile];
  uint16_t param[kTile];
};

template <int W>
constexpr int fused_stages() {
  constexpr int s = kFusedSmemBudget / static_cast<int>(sizeof(FusedStage<W>));
  return s > 9 ? 9 : s;
}

template <int W, int kStages>
__global__ void __launch_bounds__(fused_threads<W>(), 1)
fused_peer_tma_kernel(ptk_adam_scalars s, PeerTable peers, int64_t offset, int64_t shard,
                      float* __restrict__ master, float* __restrict__ exp_avg,
                      float* __restrict__ exp_avg_sq, StatsWorkspace* ws,
                      ptk_grad_stats_t* stats) {
  constexpr int kFusedTile = fused_tile<W>();
  static_assert(kStages >= 3, "ring needs >= 3 stages");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto* stage = reinterpret_cast<FusedStage<W>*>(smem_raw);
  __shared__ __align__(8) uint64_t full[kStages];
  const int tid = threadIdx.x;
  // ring items: this CTA's full tiles, plus -- on the last CTA -- the partial
  // tile (shards are multiples of 8 elements, so its TMA sizes are 16-byte
  // multiples) as one shorter item: no un-pipelined tail
  const int64_t n_tiles = shard / kFusedTile;
  const int64_t my_full = n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int rem = blockIdx.x == gridDim.x - 1 ? static_cast<int>(shard - n_tiles * kFusedTile) : 0;
  const int64_t my_items = my_full + (rem > 0 ? 1 : 0);
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto item = [&](int64_t k, int64_t& e, int& len) {
    if (k < my_full) {
      e = (blockIdx.x + k * gridDim.x) * static_cast<int64_t>(kFusedTile);
      len = kFusedTile;
    } else {
      e = n_tiles * kFusedTile;
      len = rem;
    }
  };
  int load_st = 0;
  auto issue_load = [&](int64_t k) {
    const int st = load_st;
    load_st = load_st + 1 == kStages ? 0 : load_st + 1;
    int64_t e;
    int len;
    item(k, e, len);
    FusedStage<W>& S = stage[st];
    mbar_expect_tx(&full[st], static_cast<uint32_t>(len) * (3 * sizeof(float) + W * sizeof(uint16_t)));
    bulk_load(S.master, master + e, len * 4, &full[st]);
    bulk_load(S.m, exp_avg + e, len * 4, &full[st]);
    bulk_load(S.v, exp_avg_sq + e, len * 4, &full[st]);
#pragma unroll
    for (int r = 0; r < W; ++r)
      bulk_load(S.grad[r], peers.grad[r] + offset + e, len * 2, &full[st]);
  };
  constexpr int kAhead = kStages - 2;
  if (tid == 0)
    for (int64_t k = 0; k < kAhead && k < my_items; ++k) issue_load(k);

  double sq = 0.0;
  unsigned bad = 0;
  int st = 0;
  uint32_t phase = 0;
  for (int64_t k = 0; k < my_items; ++k) {
    if (tid == 0 && k + kAhead < my_items) {
      bulk_wait_read<1>();
      issue_load(k + kAhead);
    }
    int64_t ge;
    int len;
    item(k, ge, len);
    mbar_wait(&full[st], phase);
    FusedStage<W>& S = stage[st];
    const int e = tid * 4;
    if (e < len) {  // always, except in the partial item
      float4 p = *reinterpret_cast<float4*>(&S.master[e]);
      float4 m = *reinterpret_cast<float4*>(&S.m[e]);
      float4 v = *reinterpret_cast<float4*>(&S.v[e]);
      uint2 g2 = *reinterpret_cast<const uint2*>(&S.grad[0][e]);
      float g[4] = {bf_lo(g2.x), bf_hi(g2.x), bf_lo(g2.y), bf_hi(g2.y)};
#pragma unroll
      for (int r = 1; r < W; ++r) {  // fp32 sum in rank order (deterministic)
        g2 = *reinterpret_cast<const uint2*>(&S.grad[r][e]);
        g[0] = __fadd_rn(g[0], bf_lo(g2.x));
        g[1] = __fadd_rn(g[1], bf_hi(g2.x));
        g[2] = __fadd_rn(g[2], bf_lo(g2.y));
        g[3] = __fadd_rn(g[3], bf_hi(g2.y));
      }
      float* pp = &p.x;
      float* mm = &m.x;
      float* vv = &v.x;
      float usq = 0.0f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float gk = __fmul_rn(g[q], s.gscale);
        accum_stats(gk, usq, bad);
        adam_elem(s, gk, pp[q], mm[q], vv[q]);
      }
      sq += usq;
      *reinterpret_cast<float4*>(&S.master[e]) = p;
      *reinterpret_cast<float4*>(&S.m[e]) = m;
      *reinterpret_cast<float4*>(&S.v[e]) = v;
      *reinterpret_cast<uint2*>(&S.param[e]) =
          make_uint2(pack_bf16x2(p.x, p.y), pack_bf16x2(p.z, p.w));
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      bulk_store(master + ge, S.master, len * 4);
      bulk_store(exp_avg + ge, S.m, len * 4);
      bulk_store(exp_avg_sq + ge, S.v, len * 4);
#pragma unroll
      for (int r = 0; r < W; ++r) bulk_store(peers.param[r] + offset + ge, S.param, len * 2);
      bulk_commit();
    }
    if (++st == kStages) {
      st = 0;
      phase ^= 1u;
    }
  }
  if (tid == 0) bulk_wait_all();
  if (stats != nullptr) reduce_stats(sq, bad, ws, stats);
}

struct SignalTable {
  int32_t* slot[PTK_MAX_PEERS];
};

// A peer that never arrives (crashed rank, mismatched epochs) must not hang
// the device: after timeout_ns of device time the barrier traps, which fails
// the launch (and every later call of this context) loudly instead.
__global__ void peer_barrier_kernel(SignalTable sig, int world, int rank, int epoch,
                                    int64_t timeout_ns) {
  const int t = threadIdx.x;
  if (t >= world) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(sig.slot[t] + rank), "r"(epoch)
               : "memory");
  const int32_t* mine = sig.slot[rank] + t;
  int32_t seen;
  uint64_t t0, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(seen) : "l"(mine) : "memory");
    if (seen >= epoch) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (static_cast<int64_t>(now - t0) > timeout_ns) {
      printf("ptk_peer_barrier: rank %d timed out waiting for rank %d (epoch %d, seen %d)\n",
             rank, t, epoch, seen);
      __trap();
    }
    __nanosleep(64);
  }
}

// Occupies the stream for `ns` nanoseconds of device time (global timer).
// Stand-in for an operator's compute when the executor replays a trace
// without the model (the real model's kernels replace it in training).
__global__ void busy_wait_kernel(int64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (static_cast<int64_t>(t - t0) < ns);
}

// ----------------------------------------------------------- synthetic ----

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float uniform_pm1(uint64_t seed, uint64_t i) {
  const uint32_t top = static_cast<uint32_t>(splitmix64(seed ^ i) >> 40);
  return __fsub_rn(__fmul_rn(__fmul_rn(static_cast<float>(top), 0x1p-24f), 2.0f), 1.0f);
}

__global__ void fill_f32_kernel(float* out, int64_t n, uint64_t seed, int64_t index0, float scale) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = __fmul_rn(scale, uniform_pm1(seed, static_cast<uint64_t>(index0 + i)));
}

__global__ void fill_bf16_kernel(uint16_t* out, int64_t n, uint64_t seed, int64_t index0, float scale) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float f = __fmul_rn(scale, uniform_pm1(seed, static_cast<uint64_t>(index0 + i)));
    out[i] = static_cast<uint16_t>(pack_bf16x2(f, 0.0f) & 0xffffu);
  }
}

// --------------------------------------------------------- launch sizing --

int sm_count() {
  static int count = [] {
    int dev = 0, c = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    return c > 0 ? c : 148;
  }();
  return count;
}

template <typename K>
int grid_for(K kernel, int64_t work_items) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  int64_t g = static_cast<int64_t>(sm_count()) * per_sm;
  const int64_t need = (work_items + kThreads - 1) / kThreads;
  if (g > need) g = need;
  if (g > kMaxGrid) g = kMaxGrid;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

constexpr int kUnroll = 2;

// Kernel variant of the bf16-gradient chunk Adam. Selected once per process
// from PTK_ADAM_VARIANT (benchmarking aid); the default is the measured best.
// TMA pipeline shapes: (name, tile elements, ring stages, CTAs per SM,
// threads, L2 evict-first hint).
#define PTK_TMA_VARIANTS(X)                     \
  X(Tma1536x8t384, 1536, 8, 1, 384, false)      \
  X(Tma1536x8t384h, 1536, 8, 1, 384, true)      \
  X(Tma1536x9t384, 1536, 9, 1, 384, false)      \
  X(Tma1536x9t384h, 1536, 9, 1, 384, true)      \
  X(Tma1536x4x2t384, 1536, 4, 2, 384, false)    \
  X(Tma2048x6, 2048, 6, 1, 256, false)          \
  X(Tma2048x6h, 2048, 6, 1, 256, true)          \
  X(Tma3072x4t384, 3072, 4, 1, 384, false)      \
  X(Tma1792x7t448, 1792, 7, 1, 448, false)

#define PTK_ENUM_ENTRY(V, T, S, P, THR, H) V,
enum class AdamVariant { Ldg, LdgOcc, PTK_TMA_VARIANTS(PTK_ENUM_ENTRY) };
#undef PTK_ENUM_ENTRY

// Default: the fastest shape measured on B200 (profiles/README.md).
AdamVariant adam_variant() {
  static AdamVariant v = [] {
    const char* e = std::getenv("PTK_ADAM_VARIANT");
    std::string name = e ? e : "";
    for (auto& ch : name) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    if (name == "ldg") return AdamVariant::Ldg;
    if (name == "ldg_occ") return AdamVariant::LdgOcc;
#define PTK_NAME_ENTRY(V, T, S, P, THR, H)                                \
    {                                                                     \
      std::string tag = #V;                                               \
      for (auto& ch : tag) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch))); \
      if (name == tag) return AdamVariant::V;                             \
    }
    PTK_TMA_VARIANTS(PTK_NAME_ENTRY)
#undef PTK_NAME_ENTRY
    return AdamVariant::Tma1536x9t384;  // profiles/README.md, interleaved sweep
  }();
  return v;
}

template <class G, int U, bool kStats, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
chunk_adam_occ_kernel(ptk_adam_scalars s, float* __restrict__ master, float* __restrict__ exp_avg,
                      float* __restrict__ exp_avg_sq, const typename G::T* __restrict__ grad,
                      uint16_t* __restrict__ param_out, int64_t n, StatsWorkspace* ws,
                      ptk_grad_stats_t* stats, const float* gscale_dev, const int32_t* skip_dev);

template <class G, bool kStats>
void launch_ldg(const ptk_adam_scalars& s, float* master, float* m, float* v,
                const typename G::T* grad, uint16_t* param_out, int64_t n, StatsWorkspace* ws,
                ptk_grad_stats_t* stats, const float* gscale_dev, const int32_t* skip_dev,
                cudaStream_t st) {
  const int64_t units = (n >> 3) > 0 ? (n >> 3) : 1;
  auto k = chunk_adam_kernel<G, kUnroll, kStats>;
  k<<<grid_for(k, units), kThreads, 0, st>>>(s, master, m, v, grad, param_out, n, ws, stats,
                                             gscale_dev, skip_dev);
  launch_counter()++;
}

template <int kTile, int kStages, int kPerSm, int kThr, bool kStats, bool kHint>
int launch_tma(const ptk_adam_scalars& s, float* master, float* m, float* v,
               const uint16_t* grad, uint16_t* param_out, int64_t n, StatsWorkspace* ws,
               ptk_grad_stats_t* stats, const float* gscale_dev, const int32_t* skip_dev,
               cudaStream_t st) {
  auto k = chunk_adam_tma_kernel<kTile, kStages, kThr, kStats, kHint>;
  constexpr int kSmem = kStages * static_cast<int>(sizeof(TmaStage<kTile>));
  static bool configured = false;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return check_cuda(e, "chunk_adam_tma_kernel smem attribute");
    configured = true;
  }
  int64_t grid = static_cast<int64_t>(sm_count()) * kPerSm;
  if (grid > n / kTile) grid = n / kTile;
  if (grid < 1) grid = 1;  // partial tile only
  k<<<static_cast<int>(grid), kThr, kSmem, st>>>(s, master, m, v, grad, param_out, n, ws, stats,
                                                 gscale_dev, skip_dev);
  launch_counter()++;
  return PTK_OK;
}

// One launch per chunk: full tiles through the TMA ring, the partial tile by
// the last CTA.
template <int kTile, int kStages, int kPerSm, int kThr, bool kHint>
int adam_tma_then_tail(const ptk_adam_scalars& s, float* master, float* m, float* v,
                       const uint16_t* grad, uint16_t* param_out, int64_t n, StatsWorkspace* ws,
                       ptk_grad_stats_t* stats, const float* gscale_dev, const int32_t* skip_dev,
                       cudaStream_t st) {
  return stats ? launch_tma<kTile, kStages, kPerSm, kThr, true, kHint>(
                     s, master, m, v, grad, param_out, n, ws, stats, gscale_dev, skip_dev, st)
               : launch_tma<kTile, kStages, kPerSm, kThr, false, kHint>(
                     s, master, m, v, grad, param_out, n, ws, stats, gscale_dev, skip_dev, st);
}

template <class G>
int launch_adam(const ptk_adam_config* cfg, float* master, float* m, float* v,
                const typename G::T* grad, uint16_t* param_out, int64_t n,
                ptk_grad_stats_t* stats, void* workspace, const float* gscale_dev,
                const int32_t* skip_dev, void* stream) {
  if (!cfg || !master || !m || !v || !grad) return fail(PTK_EINVAL, "ptk_chunk_adam: null buffer");
  if (n < 0) return fail(PTK_EINVAL, "ptk_chunk_adam: negative n");
  if (cfg->step < 1) return fail(PTK_EINVAL, "ptk_chunk_adam: step must be >= 1");
  if (!aligned16(master) || !aligned16(m) || !aligned16(v) || !aligned16(grad) ||
      (param_out && !aligned16(param_out)))
    return fail(PTK_EINVAL, "ptk_chunk_adam: buffers must be 16-byte aligned");
  if (stats && !workspace) return fail(PTK_EINVAL, "ptk_chunk_adam: stats requires workspace");
  if (n == 0) return PTK_OK;
  const ptk_adam_scalars s = derive_scalars(*cfg);
  auto* ws = static_cast<StatsWorkspace*>(workspace);
  cudaStream_t st = as_stream(stream);
  int rc = PTK_OK;
  if constexpr (std::is_same_v<G, GradBf16>) {
    switch (adam_variant()) {
#define PTK_TMA_CASE(V, T, S, P, THR, H)                                                    \
  case AdamVariant::V:                                                                       \
    rc = adam_tma_then_tail<T, S, P, THR, H>(s, master, m, v, grad, param_out, n, ws, stats, \
                                             gscale_dev, skip_dev, st);                      \
    return rc != PTK_OK ? rc : check_cuda(cudaGetLastError(), "chunk_adam_tma launch");
      PTK_TMA_VARIANTS(PTK_TMA_CASE)
#undef PTK_TMA_CASE
      case AdamVariant::LdgOcc: {
        const int64_t units = (n >> 3) > 0 ? (n >> 3) : 1;
        if (stats) {
          auto k = chunk_adam_occ_kernel<G, 1, true, 4>;
          k<<<grid_for(k, units), kThreads, 0, st>>>(s, master, m, v, grad, param_out, n, ws,
                                                     stats, gscale_dev, skip_dev);
        } else {
          auto k = chunk_adam_occ_kernel<G, 1, false, 4>;
          k<<<grid_for(k, units), kThreads, 0, st>>>(s, master, m, v, grad, param_out, n, ws,
                                                     stats, gscale_dev, skip_dev);
        }
        launch_counter()++;
        return check_cuda(cudaGetLastError(), "chunk_adam_occ_kernel launch");
      }
      default:
        break;
    }
  }
  if (stats)
    launch_ldg<G, true>(s, master, m, v, grad, param_out, n, ws, stats, gscale_dev, skip_dev, st);
  else
    launch_ldg<G, false>(s, master, m, v, grad, param_out, n, ws, stats, gscale_dev, skip_dev, st);
  return check_cuda(cudaGetLastError(), "chunk_adam_kernel launch");
}

// Fused-kernel variant, once per process from PTK_FUSED_KERNEL ("tma", the
// default, or "ldg" = the register-staged fused_peer_kernel).
// 0 = auto (TMA ring when every peer buffer lives on this device -- virtual
// ranks, cudaIpc mappings of the same GPU, which is what is tested here --
// and the register-staged LDG kernel, the plain peer load / store pattern,
// when a buffer is on another GPU), 1 = always TMA, 2 = always LDG.
int fused_mode() {
  static const int mode = [] {
    const char* e = std::getenv("PTK_FUSED_KERNEL");
    if (e && std::string(e) == "tma") return 1;
    if (e && std::string(e) == "ldg") return 2;
    return 0;
  }();
  return mode;
}

bool same_device(const void* p, int dev) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice && a.device == dev;
}

template <int W>
int launch_fused(const ptk_adam_scalars& s, const PeerTable& t, int64_t off, int64_t shard,
                 float* p, float* m, float* v, StatsWorkspace* ws, ptk_grad_stats_t* stats,
                 cudaStream_t st, bool tma) {
  if (!tma) {
    auto k = fused_peer_kernel<W>;
    const int grid = grid_for(k, (shard >> 3) > 0 ? (shard >> 3) : 1);
    k<<<grid, kThreads, 0, st>>>(s, t, off, shard, p, m, v, ws, stats);
    return PTK_OK;
  }
  constexpr int kSt = fused_stages<W>();
  constexpr int kSmem = kSt * static_cast<int>(sizeof(FusedStage<W>));
  auto k = fused_peer_tma_kernel<W, kSt>;
  static bool configured = false;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return check_cuda(e, "fused_peer_tma_kernel smem attribute");
    configured = true;
  }
  int64_t grid = sm_count();
  if (grid > shard / fused_tile<W>()) grid = shard / fused_tile<W>();
  if (grid < 1) grid = 1;
  k<<<static_cast<int>(grid), fused_threads<W>(), kSmem, st>>>(s, t, off, shard, p, m, v, ws,
                                                                stats);
  return PTK_OK;
}

}  // namespace
}  // namespace ptk

using namespace ptk;

extern "C" {

int64_t ptk_stats_workspace_bytes(void) { return static_cast<int64_t>(sizeof(StatsWorkspace)); }

const char* ptk_adam_kernel_name(void) {
  switch (adam_variant()) {
    case AdamVariant::Ldg: return "ldg";
    case AdamVariant::LdgOcc: return "ldg_occ";
#define PTK_NAME_CASE(V, T, S, P, THR, H) \
  case AdamVariant::V:                    \
    return "tma tile=" #T " stages=" #S " ctas/sm=" #P " threads=" #THR " l2_evict_first=" #H;
    PTK_TMA_VARIANTS(PTK_NAME_CASE)
#undef PTK_NAME_CASE
  }
  return "?";
}

const char* ptk_fused_kernel_name(void) {
  switch (fused_mode()) {
    case 1:
      return "fused_peer_tma_kernel (tile 2048 for W=2, 1536 for W=1,3,4, 1024 for W>=5; "
             "threads = tile/4; stages = min(9, 220 KB / stage))";
    case 2:
      return "fused_peer_kernel (ldg)";
    default:
      return "fused RS->Adam->AG, auto: fused_peer_tma_kernel (tile 2048 for W=2, 1536 for "
             "W=1,3,4, 1024 for W>=5) when every peer buffer is on this device, "
             "fused_peer_kernel (ldg) across devices";
  }
}

int ptk_chunk_adam(const ptk_adam_config* cfg, float* master, float* exp_avg, float* exp_avg_sq,
                   const uint16_t* grad, uint16_t* param_out, int64_t n, ptk_grad_stats_t* stats,
                   void* workspace, const float* gscale_dev, const int32_t* skip_dev,
                   void* stream) {
  return launch_adam<GradBf16>(cfg, master, exp_avg, exp_avg_sq, grad, param_out, n, stats,
                               workspace, gscale_dev, skip_dev, stream);
}

int ptk_chunk_adam_f32grad(const ptk_adam_config* cfg, float* master, float* exp_avg,
                           float* exp_avg_sq, const float* grad, uint16_t* param_out, int64_t n,
                           ptk_grad_stats_t* stats, void* workspace, const float* gscale_dev,
                           const int32_t* skip_dev, void* stream) {
  return launch_adam<GradF32>(cfg, master, exp_avg, exp_avg_sq, grad, param_out, n, stats,
                              workspace, gscale_dev, skip_dev, stream);
}

int ptk_grad_stats(const uint16_t* grad, int64_t n, float scale, float* out_f32,
                   ptk_grad_stats_t* stats, void* workspace, void* stream) {
  if (!grad || !stats || !workspace) return fail(PTK_EINVAL, "ptk_grad_stats: null argument");
  if (!aligned16(grad) || (out_f32 && !aligned16(out_f32)))
    return fail(PTK_EINVAL, "ptk_grad_stats: buffers must be 16-byte aligned");
  if (n <= 0) return n == 0 ? PTK_OK : fail(PTK_EINVAL, "ptk_grad_stats: negative n");
  auto* ws = static_cast<StatsWorkspace*>(workspace);
  const int64_t units = (n >> 3) > 0 ? (n >> 3) : 1;
  if (out_f32) {
    auto k = grad_stats_kernel<true>;
    k<<<grid_for(k, units), kThreads, 0, as_stream(stream)>>>(grad, n, scale, out_f32, ws, stats);
  } else {
    auto k = grad_stats_kernel<false>;
    k<<<grid_for(k, units), kThreads, 0, as_stream(stream)>>>(grad, n, scale, out_f32, ws, stats);
  }
  launch_counter()++;
  return check_cuda(cudaGetLastError(), "grad_stats_kernel launch");
}

int ptk_grad_prep(const uint16_t* grad, int64_t n, float scale, float* out_f32,
                  ptk_grad_stats_t* stats, void* workspace, void* stream) {
  if (!out_f32) return fail(PTK_EINVAL, "ptk_grad_prep: null fp32 output");
  return ptk_grad_stats(grad, n, scale, out_f32, stats, workspace, stream);
}

int ptk_stats_reset(ptk_grad_stats_t* stats, void* stream) {
  if (!stats) return fail(PTK_EINVAL, "ptk_stats_reset: null stats");
  stats_reset_kernel<<<1, 1, 0, as_stream(stream)>>>(stats);
  launch_counter()++;
  return check_cuda(cudaGetLastError(), "stats_reset_kernel launch");
}

int ptk_clip_coef(const ptk_grad_stats_t* stats, double max_norm, float* coef_out,
                  int32_t* skip_out, void* stream) {
  if (!stats || !coef_out) return fail(PTK_EINVAL, "ptk_clip_coef: null argument");
  clip_coef_kernel<<<1, 1, 0, as_stream(stream)>>>(stats, max_norm, coef_out, skip_out);
  launch_counter()++;
  return check_cuda(cudaGetLastError(), "clip_coef_kernel launch");
}

int ptk_fused_rs_adam_ag(const ptk_adam_config* cfg, const uint16_t* const* grad_peers,
                         uint16_t* const* param_peers, int32_t world, int32_t rank, int64_t shard,
                         float* master, float* exp_avg, float* exp_avg_sq,
                         ptk_grad_stats_t* stats, void* workspace, void* stream) {
  if (!cfg || !grad_peers || !param_peers || !master || !exp_avg || !exp_avg_sq)
    return fail(PTK_EINVAL, "ptk_fused_rs_adam_ag: null argument");
  if (world < 1 || world > PTK_MAX_PEERS || rank < 0 || rank >= world)
    return fail(PTK_EINVAL, "ptk_fused_rs_adam_ag: bad world/rank");
  if (shard < 0 || (shard & 7) != 0)
    return fail(PTK_EINVAL, "ptk_fused_rs_adam_ag: shard must be a multiple of 8 elements");
  if (cfg->step < 1) return fail(PTK_EINVAL, "ptk_fused_rs_adam_ag: step must be >= 1");
  if (stats && !workspace) return fail(PTK_EINVAL, "ptk_fused_rs_adam_ag: stats requires workspace");
  PeerTable t{};
  for (int r = 0; r < world; ++r) {
    if (!grad_peers[r] || !param_peers[r] || !aligned16(grad_peers[r]) || !aligned16(param_peers[r]))
      return fail(PTK_EINVAL, "ptk_fused_rs_adam_ag: peer buffers must be non-null and 16-byte aligned");
    t.grad[r] = grad_peers[r];
    t.param[r] = param_peers[r];
  }
  if (!aligned16(master) || !aligned16(exp_avg) || !aligned16(exp_avg_sq))
    return fail(PTK_EINVAL, "ptk_fused_rs_adam_ag: state buffers must be 16-byte aligned");
  if (shard == 0) return PTK_OK;
  const ptk_adam_scalars s = derive_scalars(*cfg);
  const int64_t off = static_cast<int64_t>(rank) * shard;
  auto* ws = static_cast<StatsWorkspace*>(workspace);
  cudaStream_t st = as_stream(stream);
  bool tma = fused_mode() != 2;
  if (fused_mode() == 0) {
    int dev = 0;
    PTK_TRY_CUDA(cudaGetDevice(&dev));
    for (int r = 0; r < world && tma; ++r)
      tma = same_device(grad_peers[r], dev) && same_device(param_peers[r], dev);
  }
  int rc = PTK_OK;
  switch (world) {
    case 1: rc = launch_fused<1>(s, t, off, shard, master, exp_avg, exp_avg_sq, ws, stats, st, tma); break;
    case 2: rc = launch_fused<2>(s, t, off, shard, master, exp_avg, exp_avg_sq, ws, stats, st, tma); break;
    case 3: rc = launch_fused<3>(s, t, off, shard, master, exp_avg, exp_avg_sq, ws, stats, st, tma); break;
    case 4: rc = launch_fused<4>(s, t, off, shard, master, exp_avg, exp_avg_sq, ws, stats, st, tma); break;
    case 5: rc = launch_fused<5>(s, t, off, shard, master, exp_avg, exp_avg_sq, ws, stats, st, tma); break;
    case 6: rc = launch_fused<6>(s, t, off, shard, master, exp_avg, exp_avg_sq, ws, stats, st, tma); break;
    case 7: rc = launch_fused<7>(s, t, off, shard, master, exp_avg, exp_avg_sq, ws, stats, st, tma); break;
    default: rc = launch_fused<8>(s, t, off, shard, master, exp_avg, exp_avg_sq, ws, stats, st, tma); break;
  }
  if (rc != PTK_OK) return rc;
  launch_counter()++;
  return check_cuda(cudaGetLastError(), "fused_peer_kernel launch");
}

int ptk_peer_barrier(int32_t* const* signal_peers, int32_t world, int32_t rank, int32_t epoch,
                     void* stream) {
  if (!signal_peers || world < 1 || world > PTK_MAX_PEERS || rank < 0 || rank >= world)
    return fail(PTK_EINVAL, "ptk_peer_barrier: bad arguments");
  SignalTable t{};
  for (int r = 0; r < world; ++r) {
    if (!signal_peers[r]) return fail(PTK_EINVAL, "ptk_peer_barrier: null signal slot");
    t.slot[r] = signal_peers[r];
  }
  static const int64_t timeout_ns = [] {
    const char* e = std::getenv("PTK_PEER_BARRIER_TIMEOUT_MS");
    const long long ms = e ? std::atoll(e) : 60000;
    return static_cast<int64_t>(ms > 0 ? ms : 60000) * 1000000;
  }();
  peer_barrier_kernel<<<1, 32, 0, as_stream(stream)>>>(t, world, rank, epoch, timeout_ns);
  launch_counter()++;
  return check_cuda(cudaGetLastError(), "peer_barrier_kernel launch");
}

int ptk_busy_wait(int64_t ns, void* stream) {
  if (ns < 0) return fail(PTK_EINVAL, "ptk_busy_wait: negative duration");
  if (ns == 0) return PTK_OK;
  busy_wait_kernel<<<1, 1, 0, as_stream(stream)>>>(ns);
  launch_counter()++;
  return check_cuda(cudaGetLastError(), "busy_wait_kernel launch");
}

int ptk_fill_uniform_f32(float* out, int64_t n, uint64_t seed, int64_t index0, float scale,
                         void* stream) {
  if (!out || n < 0) return fail(PTK_EINVAL, "ptk_fill_uniform_f32: bad arguments");
  if (n == 0) return PTK_OK;
  const int64_t blocks = (n + 255) / 256;
  const int grid = static_cast<int>(blocks < 8 * 148 * 4 ? blocks : 8 * 148 * 4);
  fill_f32_kernel<<<grid, 256, 0, as_stream(stream)>>>(out, n, seed, index0, scale);
  launch_counter()++;
  return check_cuda(cudaGetLastError(), "fill_f32_kernel launch");
}

int ptk_fill_uniform_bf16(uint16_t* out, int64_t n, uint64_t seed, int64_t index0, float scale,
                          void* stream) {
  if (!out || n < 0) return fail(PTK_EINVAL, "ptk_fill_uniform_bf16: bad arguments");
  if (n == 0) return PTK_OK;
  const int64_t blocks = (n + 255) / 256;
  const int grid = static_cast<int>(blocks < 8 * 148 * 4 ? blocks : 8 * 148 * 4);
  fill_bf16_kernel<<<grid, 256, 0, as_stream(stream)>>>(out, n, seed, index0, scale);
  launch_counter()++;
  return check_cuda(cudaGetLastError(), "fill_bf16_kernel launch");
}

}  // extern "C"
