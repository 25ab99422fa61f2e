// libptk device kernels for sm_100a: the chunk data plane of ProTrain.
//
//   K1+K2    chunk_adam_tma_kernel  fused grad cast/scale + grad-norm/overflow
//                                   statistics + Adam/AdamW over a TABLE of flat
//                                   chunk shards in ONE launch (28 B/param of
//                                   HBM traffic, bf16 grad): a TMA bulk ring
//   K1+K2    chunk_adam_kernel      register-staged variant (fp32 grads, "ldg")
//   K2       grad_stats_kernel      standalone statistics (+ fp32 scaled copy)
//   K1+K3+K4 fused_peer_tma_kernel  reduce-scatter (fp32 rank-order sum of every
//            fused_peer_kernel      rank's gradient tile read over NVLink) ->
//                                   Adam -> all-gather (push of the bf16 tile
//                                   into every rank), over a chunk table
//   K2'      fused_stats_kernel     phase 1 of a clipped fused step: statistics
//                                   of the reduced gradient, no update
//   aux      stats mailbox (publish / collect of per-rank statistics over peer
//            memory), clip coefficient, peer barrier, fill kernels
//
// The modeled counterparts in the reference are listed in include/ptk.h.
// Design notes: every kernel is HBM-streaming element work —
// no data reuse, so no tensor cores; the levers are 128-bit / TMA bulk
// accesses, enough bytes in flight per SM (a shared-memory ring, not
// registers), a persistent grid of one CTA per SM that walks every chunk of
// the step (the ring stays full across chunk boundaries: one fill and one
// drain per step, not per chunk), and deterministic warp-shuffle → CTA →
// last-CTA reductions for the statistics. The update arithmetic uses explicit
// round-to-nearest intrinsics (no FMA contraction) so it matches
// oracle/chunk_step.c bit for bit.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "ptk_common.h"

namespace ptk {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxGrid = 4096;
constexpr int kMaxDevices = 64;

struct StatsWorkspace {
  unsigned long long sq[3][kMaxGrid];  // per-CTA fixed-point partial sums (SumSq words)
  unsigned long long bad[kMaxGrid];
  unsigned int arrived;
  unsigned int exited;             // tile scheduler: CTAs done taking tiles this launch
  unsigned long long next_tile;    // tile scheduler: next unclaimed tile of this launch
};

// Dynamic tile scheduler of the persistent TMA kernels: the producer of every
// CTA claims the next tile of the step with one atomic, so SMs that stream
// faster (ncu: SM active cycles min/avg/max 0.85/1.00/1.14 under a static
// round-robin split) take more tiles and all finish together. A CTA's claims
// are increasing, so its chunk cursor still only moves forward. The last CTA
// to finish claiming re-arms the counter for the next launch on the stream
// (one workspace per stream at a time, as for the statistics).
__device__ __forceinline__ int64_t claim_tile(StatsWorkspace* ws) {
  return static_cast<int64_t>(atomicAdd(&ws->next_tile, 1ull));
}
__device__ __forceinline__ void release_scheduler(StatsWorkspace* ws) {
  __threadfence();
  if (atomicAdd(&ws->exited, 1u) == gridDim.x - 1) {
    ws->next_tile = 0;
    ws->exited = 0;
    __threadfence();
  }
}

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

// Statistics: squares are summed in fp32 over one 4- or 8-element unit; the
// unit sums are accumulated EXACTLY in a 192-bit fixed-point integer (units of
// 2^-64, range 2^128) per thread, then per warp, CTA and grid. Integer sums do
// not depend on the order of the terms, so the statistics (and the clip
// coefficient derived from them) are bit-identical from run to run whichever
// CTA processed which tile -- the dynamic tile scheduler's order varies. Unit
// sums below 2^-64 (|g| < 2^-33) are dropped and sums above 2^90 saturate at
// 2^90 (a norm >= 3.5e13; 2^32 such units still fit in the range).
__device__ __forceinline__ void accum_stats(float g, float& sq, unsigned& bad) {
  sq = __fmaf_rn(g, g, sq);
  bad += isfinite(g) ? 0u : 1u;
}

struct SumSq {
  unsigned long long w0 = 0, w1 = 0, w2 = 0;  // value = (w2:w1:w0) * 2^-64

  __device__ __forceinline__ void add(unsigned long long a0, unsigned long long a1,
                                      unsigned long long a2) {
    asm("add.cc.u64 %0, %0, %3;\n\taddc.cc.u64 %1, %1, %4;\n\taddc.u64 %2, %2, %5;"
        : "+l"(w0), "+l"(w1), "+l"(w2)
        : "l"(a0), "l"(a1), "l"(a2));
  }
  __device__ __forceinline__ void add(const SumSq& o) { add(o.w0, o.w1, o.w2); }
  // x >= 0 (a sum of squares); NaN / inf are counted by `bad` and skipped here
  __device__ __forceinline__ void add(float x) {
    const uint32_t b = __float_as_uint(x);
    int ef = static_cast<int>((b >> 23) & 0xffu);
    if (ef == 0 || ef == 255 || (b >> 31)) return;
    unsigned long long m = (b & 0x7fffffu) | 0x800000u;
    if (ef > 127 + 90) {  // saturate at 2^90
      ef = 127 + 90;
      m = 0x800000u;
    }
    int sh = ef - 150 + 64;  // x = m * 2^(ef-150); units of 2^-64
    if (sh < 0) {
      if (sh <= -24) return;
      m >>= -sh;
      sh = 0;
    }
    const int word = sh >> 6, bit = sh & 63;
    const unsigned long long lo = m << bit;
    const unsigned long long hi = bit ? m >> (64 - bit) : 0ull;
    if (word == 0) add(lo, hi, 0ull);
    else add(0ull, lo, hi);  // sh < 128 + 24: word <= 1 after saturation
  }
  __device__ __forceinline__ void shfl_add(int o) {
    add(__shfl_xor_sync(0xffffffffu, w0, o), __shfl_xor_sync(0xffffffffu, w1, o),
        __shfl_xor_sync(0xffffffffu, w2, o));
  }
  __device__ __forceinline__ double to_double() const {
    return static_cast<double>(w2) * 0x1p64 + static_cast<double>(w1) +
           static_cast<double>(w0) * 0x1p-64;
  }
};

// Effective gradient scale of a launch: the host scalar times the optional
// device multiplier (a clip coefficient); skip_dev != 0 makes it a no-op.
__device__ __forceinline__ float launch_gscale(const ptk_adam_scalars& s, const float* gscale_dev) {
  return gscale_dev != nullptr ? __fmul_rn(s.gscale, *gscale_dev) : s.gscale;
}

// Grid reduction of the statistics: warp shuffle -> CTA -> the last CTA to
// arrive sums the per-CTA partials, converts the exact sum to fp64 once and
// ADDS it to *stats (launch order across launches: deterministic). Safe
// across back-to-back launches on one stream (the arrival counter is re-armed
// by the last CTA).
__device__ __forceinline__ void reduce_stats(SumSq sq, unsigned bad, StatsWorkspace* ws,
                                             ptk_grad_stats_t* stats) {
  __shared__ SumSq s_sq[32];
  __shared__ unsigned long long s_bad[32];
  __shared__ bool s_last;
  unsigned long long wbad = bad;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sq.shfl_add(o);
    wbad += __shfl_xor_sync(0xffffffffu, wbad, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_sq[warp] = sq;
    s_bad[warp] = wbad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    SumSq bsq;
    unsigned long long bbad = 0;
    for (unsigned w = 0; w < blockDim.x / 32; ++w) {
      bsq.add(s_sq[w]);
      bbad += s_bad[w];
    }
    ws->sq[0][blockIdx.x] = bsq.w0;
    ws->sq[1][blockIdx.x] = bsq.w1;
    ws->sq[2][blockIdx.x] = bsq.w2;
    ws->bad[blockIdx.x] = bbad;
    __threadfence();
    const unsigned prev = atomicAdd(&ws->arrived, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    SumSq tsq;
    unsigned long long tbad = 0;
    const volatile unsigned long long* v0 = ws->sq[0];
    const volatile unsigned long long* v1 = ws->sq[1];
    const volatile unsigned long long* v2 = ws->sq[2];
    const volatile unsigned long long* vbad = ws->bad;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) {
      tsq.add(v0[b], v1[b], v2[b]);
      tbad += vbad[b];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tsq.shfl_add(o);
      tbad += __shfl_xor_sync(0xffffffffu, tbad, o);
    }
    if (threadIdx.x == 0) {
      stats->sumsq += tbad != 0 ? __longlong_as_double(0x7ff0000000000000ll) : tsq.to_double();
      stats->nonfinite += tbad;
      ws->arrived = 0;
    }
  }
}

// ------------------------------------------------------------ K1 + K2 ----
// Register-staged chunk Adam (one chunk per launch): U independent 8-element
// units per thread with every load issued before any math. Used for fp32
// gradients (ptk_chunk_adam_f32grad) and as the "ldg" variant.

template <class G, int U, bool kStats>
__global__ void __launch_bounds__(kThreads)
chunk_adam_kernel(ptk_adam_scalars s, float* __restrict__ master, float* __restrict__ exp_avg,
                  float* __restrict__ exp_avg_sq, const typename G::T* __restrict__ grad,
                  uint16_t* __restrict__ param_out, int64_t n, StatsWorkspace* ws,
                  ptk_grad_stats_t* stats, const float* gscale_dev, const int32_t* skip_dev) {
  if (skip_dev != nullptr && *skip_dev != 0) return;  // grid-uniform
  const float gs = launch_gscale(s, gscale_dev);
  SumSq sq;
  unsigned bad = 0;

  const int64_t nvec = n >> 3;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
  int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;

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
      if (kStats) sq.add(usq);
      st8f(master + e, p[u]);
      st8f(exp_avg + e, m[u]);
      st8f(exp_avg_sq + e, v[u]);
      if (param_out != nullptr) __stcs(reinterpret_cast<uint4*>(param_out + e), pack8(p[u]));
    }
  }
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
    if (kStats) sq.add(usq);
    st8f(master + e, p);
    st8f(exp_avg + e, m);
    st8f(exp_avg_sq + e, v);
    if (param_out != nullptr) __stcs(reinterpret_cast<uint4*>(param_out + e), pack8(p));
  }
  const int64_t t0 = nvec << 3;  // scalar tail (< 8 elements) on CTA 0
  if (blockIdx.x == 0 && threadIdx.x < n - t0) {
    const int64_t e = t0 + threadIdx.x;
    const float gk = __fmul_rn(G::load1(grad + e), gs);
    float usq = 0.0f;
    if (kStats) accum_stats(gk, usq, bad);
    sq.add(usq);
    float p = master[e], m = exp_avg[e], v = exp_avg_sq[e];
    adam_elem(s, gk, p, m, v);
    master[e] = p;
    exp_avg[e] = m;
    exp_avg_sq[e] = v;
    if (param_out != nullptr) param_out[e] = static_cast<uint16_t>(pack_bf16x2(p, 0.0f) & 0xffffu);
  }
  if (kStats) reduce_stats(sq, bad, ws, stats);
}

// ---------------------------------------------------- TMA bulk primitives --

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

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

// ------------------------------------------------------------ chunk tables --
//
// A step's chunks are described by a table (device memory, built once by
// ptk_chunk_table_create / ptk_fused_table_create) or, for the single-chunk
// entry points, by one descriptor passed in the launch parameters. Every
// chunk's multiple-of-8 prefix is cut into tiles of the kernel's tile size;
// tile0 = index of the chunk's first tile in the step's global tile order.
// CTA b walks global tiles b, b + G, b + 2G, ... across chunk boundaries, so
// the TMA ring is filled once per step. The < 8 trailing elements of a chunk
// whose length is not a multiple of 8 (never the case for padded shards) are
// updated with plain loads by CTA (chunk % G) after the ring drains.

struct ChunkDesc {
  float* master;
  float* m;
  float* v;
  const uint16_t* grad;
  uint16_t* param;  // nullable
  int64_t n;
  int64_t tile0;
};

struct FusedDesc {
  const uint16_t* grad[PTK_MAX_PEERS];  // rank r's full gradient chunk
  uint16_t* param[PTK_MAX_PEERS];       // rank r's full parameter chunk
  float* master;                        // this rank's shard state
  float* m;
  float* v;
  int64_t shard;  // elements per rank (multiple of 8)
  int64_t tile0;
};

struct FusedList {
  const FusedDesc* table;
  FusedDesc one;
  int64_t total_tiles;
  int32_t n_chunks;
  int32_t rank;
};

__device__ __forceinline__ const FusedDesc& fused_at(const FusedList& l, int c) {
  return l.table != nullptr ? l.table[c] : l.one;
}

// tid 0's cursor over the global tile order (monotone per CTA) with the
// current chunk's descriptor cached in registers: descriptors are read from
// the table once per chunk, not once per tile (the elected thread's per-tile
// latency is on every CTA's critical path).
template <class D>
struct TileCursor {
  int c = -1;
  int64_t end = 0;  // first global tile of chunk c + 1
  D d;
};

__device__ __forceinline__ const FusedDesc& desc_at(const FusedList& l, int c) { return fused_at(l, c); }

template <class L, class D>
__device__ __forceinline__ void cursor_seek(const L& l, TileCursor<D>& cur, int64_t t) {
  if (t < cur.end) return;
  do {  // skips chunks without tiles (tile0 equal to the next one)
    ++cur.c;
    cur.end = cur.c + 1 < l.n_chunks ? desc_at(l, cur.c + 1).tile0 : l.total_tiles;
  } while (t >= cur.end);
  cur.d = desc_at(l, cur.c);
}

// The store side follows the same chunks in the same order.
template <class L, class D>
__device__ __forceinline__ const D& cursor_at(const L& l, TileCursor<D>& cur, int c) {
  if (c != cur.c) {
    cur.c = c;
    cur.d = desc_at(l, c);
  }
  return cur.d;
}

struct ItemMeta {
  int64_t e;  // first element of the tile within its chunk (shard)
  int32_t c;  // chunk
  int32_t len;
};

// Warp-specialized rings: stage / phase position of a role.

struct RingPos {
  int st = 0;
  uint32_t ph = 0;
  template <int kStages>
  __device__ __forceinline__ void next() {
    if (++st == kStages) {
      st = 0;
      ph ^= 1u;
    }
  }
};

constexpr int kRoleThreads = 64;  // producer warp + storer warp

// ------------------------------------------- K1 + K2, TMA bulk pipeline --
//
// Persistent CTAs (one per SM) stream the step's tiles through a ring of
// kStages shared-memory stages, with the roles split by warp:
//   * producer warp (one elected lane): claims the next tile (dynamic
//     scheduler) and moves master/m/v/grad global -> shared with 1-D bulk
//     copies (cp.async.bulk, the TMA engine), completion counted on the
//     stage's `full` mbarrier (complete_tx);
//   * consumer warps (kThr threads, one 4-element unit each per tile): Adam
//     + statistics in shared memory, then arrive on the stage's `done`;
//   * storer warp (one elected lane): bulk-stores master/m/v/param shared ->
//     global as a bulk_group and frees the stage (`empty`) once the store has
//     read it (wait_group.read).
// No CTA-wide barrier sits on the per-tile path, so the producer's claim /
// descriptor latency and the stores overlap the math of other stages.
//
// The chunk table travels in the KERNEL PARAMETERS (__grid_constant__, the
// constant bank): the descriptor fields load into uniform registers and the
// elected lanes' bulk-copy addresses need no per-thread -> uniform
// conversion. Tables larger than kCap chunks are launched in batches of kCap.

template <int kTile>
struct TmaStage {
  float master[kTile];
  float m[kTile];
  float v[kTile];
  uint16_t grad[kTile];
  uint16_t param[kTile];
};

template <int kCap>
struct ChunkBatch {
  ChunkDesc d[kCap];  // tile0 counted from this batch's first chunk
  int64_t total_tiles;
  int32_t n_chunks;
};

// Uniform cursor over a batch's tiles (every thread keeps its own copy).
template <int kCap>
struct BatchCursor {
  int c = 0;
  int64_t end;
  __device__ __forceinline__ explicit BatchCursor(const ChunkBatch<kCap>& b)
      : end(b.n_chunks > 1 ? b.d[1].tile0 : b.total_tiles) {}
  __device__ __forceinline__ int seek(const ChunkBatch<kCap>& b, int64_t t) {
    while (t >= end) {  // skips chunks without tiles
      ++c;
      end = c + 1 < b.n_chunks ? b.d[c + 1].tile0 : b.total_tiles;
    }
    return c;
  }
};

template <int kTile, int kStages, int kThr, bool kStats, bool kHint, int kCap, bool kDynamic>
__global__ void __launch_bounds__(kThr + kRoleThreads, 1)
chunk_adam_tma_kernel(ptk_adam_scalars s, const __grid_constant__ ChunkBatch<kCap> b,
                      StatsWorkspace* ws, ptk_grad_stats_t* stats, const float* gscale_dev,
                      const int32_t* skip_dev) {
  static_assert(kTile == kThr * 4, "one 4-element unit per consumer thread per tile");
  static_assert(kStages >= 2, "ring needs >= 2 stages");
  constexpr int kConsumerWarps = kThr / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto* stage = reinterpret_cast<TmaStage<kTile>*>(smem_raw);
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ __align__(8) uint64_t done[kStages];
  __shared__ __align__(8) uint64_t empty[kStages];
  __shared__ ItemMeta meta[kStages];

  if (skip_dev != nullptr && *skip_dev != 0) return;
  const float gs = launch_gscale(s, gscale_dev);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t T = b.total_tiles;
  const int64_t my_items = T > blockIdx.x ? (T - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&done[i], kConsumerWarps);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();  // the inits are visible to the async proxy (complete_tx)
  }
  __syncthreads();

  SumSq sq;
  unsigned bad = 0;
  if (warp == kConsumerWarps) {
    // ------------------------- producer: master/m/v/grad tiles -> stage --
    if (lane == 0) {
      const uint64_t policy = kHint ? evict_first_policy() : 0;
      BatchCursor<kCap> cur(b);
      RingPos pos;
      int64_t claimed = kDynamic ? claim_tile(ws) : 0;  // one claim in flight ahead
      for (int64_t k = 0; kDynamic || k < my_items; ++k) {
        if (k >= kStages) mbar_wait(&empty[pos.st], pos.ph ^ 1u);
        int64_t t = blockIdx.x + k * gridDim.x;
        if (kDynamic) {
          t = claimed;
          if (t >= T) {  // end of the step: a tile-less stage tells the others
            meta[pos.st] = ItemMeta{0, -1, 0};
            mbar_arrive(&full[pos.st]);
            release_scheduler(ws);
            break;
          }
          claimed = claim_tile(ws);
        }
        const int c = cur.seek(b, t);
        const ChunkDesc& d = b.d[c];
        const int64_t e = (t - d.tile0) * kTile;
        const int64_t left = (d.n & ~int64_t{7}) - e;
        const int len = left < kTile ? static_cast<int>(left) : kTile;
        meta[pos.st] = ItemMeta{e, c, len};
        TmaStage<kTile>& S = stage[pos.st];
        uint64_t* bar = &full[pos.st];
        mbar_expect_tx(bar, static_cast<uint32_t>(len) * (3 * sizeof(float) + sizeof(uint16_t)));
        if (kHint) {
          bulk_load_hint(S.master, d.master + e, len * 4, bar, policy);
          bulk_load_hint(S.m, d.m + e, len * 4, bar, policy);
          bulk_load_hint(S.v, d.v + e, len * 4, bar, policy);
          bulk_load_hint(S.grad, d.grad + e, len * 2, bar, policy);
        } else {
          bulk_load(S.master, d.master + e, len * 4, bar);
          bulk_load(S.m, d.m + e, len * 4, bar);
          bulk_load(S.v, d.v + e, len * 4, bar);
          bulk_load(S.grad, d.grad + e, len * 2, bar);
        }
        pos.next<kStages>();
      }
    }
  } else if (warp == kConsumerWarps + 1) {
    // ---------------------------- storer: stage -> master/m/v/param -----
    if (lane == 0) {
      const uint64_t policy = kHint ? evict_first_policy() : 0;
      RingPos pos;
      int prev = -1;
      for (int64_t k = 0; kDynamic || k < my_items; ++k) {
        mbar_wait(&done[pos.st], pos.ph);
        const ItemMeta it = meta[pos.st];
        if (kDynamic && it.c < 0) break;
        const ChunkDesc& d = b.d[it.c];
        TmaStage<kTile>& S = stage[pos.st];
        if (kHint) {
          bulk_store_hint(d.master + it.e, S.master, it.len * 4, policy);
          bulk_store_hint(d.m + it.e, S.m, it.len * 4, policy);
          bulk_store_hint(d.v + it.e, S.v, it.len * 4, policy);
          if (d.param != nullptr) bulk_store_hint(d.param + it.e, S.param, it.len * 2, policy);
        } else {
          bulk_store(d.master + it.e, S.master, it.len * 4);
          bulk_store(d.m + it.e, S.m, it.len * 4);
          bulk_store(d.v + it.e, S.v, it.len * 4);
          if (d.param != nullptr) bulk_store(d.param + it.e, S.param, it.len * 2);
        }
        bulk_commit();
        if (prev >= 0) {
          bulk_wait_read<1>();  // the previous stage's store has read its smem
          mbar_arrive(&empty[prev]);
        }
        prev = pos.st;
        pos.next<kStages>();
      }
      bulk_wait_all();
    }
  } else {
    // ------------------------------------------------------ consumers --
    RingPos pos;
    for (int64_t k = 0; kDynamic || k < my_items; ++k) {
      mbar_wait(&full[pos.st], pos.ph);
      if (kDynamic && meta[pos.st].c < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[pos.st]);  // lets the storer see the end
        break;
      }
      const int len = meta[pos.st].len;
      TmaStage<kTile>& S = stage[pos.st];
      const int e = tid * 4;
      if (e < len) {  // always, except in a chunk's last tile
        float4 p = *reinterpret_cast<float4*>(&S.master[e]);
        float4 m = *reinterpret_cast<float4*>(&S.m[e]);
        float4 v = *reinterpret_cast<float4*>(&S.v[e]);
        const uint2 g2 = *reinterpret_cast<const uint2*>(&S.grad[e]);
        const float g[4] = {bf_lo(g2.x), bf_hi(g2.x), bf_lo(g2.y), bf_hi(g2.y)};
        float* pp = &p.x;
        float* mm = &m.x;
        float* vv = &v.x;
        float usq = 0.0f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float gk = __fmul_rn(g[q], gs);
          if (kStats) accum_stats(gk, usq, bad);
          adam_elem(s, gk, pp[q], mm[q], vv[q]);
        }
        if (kStats) sq.add(usq);
        *reinterpret_cast<float4*>(&S.master[e]) = p;
        *reinterpret_cast<float4*>(&S.m[e]) = m;
        *reinterpret_cast<float4*>(&S.v[e]) = v;
        *reinterpret_cast<uint2*>(&S.param[e]) =
            make_uint2(pack_bf16x2(p.x, p.y), pack_bf16x2(p.z, p.w));
      }
      fence_async_smem();  // generic-proxy smem writes -> visible to the bulk store
      __syncwarp();
      if (lane == 0) mbar_arrive(&done[pos.st]);
      pos.next<kStages>();
    }
  }
  // the < 8 trailing elements of chunks whose length is not a multiple of 8
  for (int c = blockIdx.x; c < b.n_chunks; c += gridDim.x) {
    const ChunkDesc& d = b.d[c];
    const int64_t e = (d.n & ~int64_t{7}) + tid;
    if (e < d.n) {
      float usq = 0.0f;
      const float gk = __fmul_rn(GradBf16::load1(d.grad + e), gs);
      if (kStats) accum_stats(gk, usq, bad);
      float p = d.master[e], mm = d.m[e], vv = d.v[e];
      adam_elem(s, gk, p, mm, vv);
      d.master[e] = p;
      d.m[e] = mm;
      d.v[e] = vv;
      if (d.param != nullptr) d.param[e] = static_cast<uint16_t>(pack_bf16x2(p, 0.0f) & 0xffffu);
      if (kStats) sq.add(usq);
    }
  }
  __syncthreads();
  if (kStats) reduce_stats(sq, bad, ws, stats);
}

// -------------------------------------------------------------- K2 -------

template <bool kWrite>
__global__ void __launch_bounds__(kThreads)
grad_stats_kernel(const uint16_t* __restrict__ grad, int64_t n, float scale,
                  float* __restrict__ out, StatsWorkspace* ws, ptk_grad_stats_t* stats) {
  SumSq sq;
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
    sq.add(usq);
    if (kWrite) st8f(out + (i << 3), g);
  }
  const int64_t t0 = nvec << 3;
  if (blockIdx.x == 0 && threadIdx.x < n - t0) {
    const int64_t e = t0 + threadIdx.x;
    const float gk = __fmul_rn(GradBf16::load1(grad + e), scale);
    float usq = 0.0f;
    accum_stats(gk, usq, bad);
    sq.add(usq);
    if (kWrite) out[e] = gk;
  }
  reduce_stats(sq, bad, ws, stats);
}

__global__ void stats_reset_kernel(ptk_grad_stats_t* stats) {
  stats->sumsq = 0.0;
  stats->nonfinite = 0;
}

__device__ __forceinline__ void clip_from_stats(double sumsq, unsigned long long nonfinite,
                                                double max_norm, float* coef, int32_t* skip) {
  const double norm = sqrt(sumsq);
  double c = 1.0;
  if (max_norm > 0.0) {
    c = max_norm / (norm + 1e-6);
    if (c > 1.0) c = 1.0;
  }
  if (coef != nullptr) *coef = static_cast<float>(c);
  if (skip != nullptr) *skip = nonfinite != 0 ? 1 : 0;
}

__global__ void clip_coef_kernel(const ptk_grad_stats_t* stats, double max_norm, float* coef,
                                 int32_t* skip) {
  clip_from_stats(stats->sumsq, stats->nonfinite, max_norm, coef, skip);
}

// ------------------------------------------------ K1+K3+K4 over NVLink ----

// Register-staged fused step: per 8-element unit, W 128-bit gradient loads
// (peer memory), fp32 rank-order sum, Adam on the local state, W 128-bit
// stores of the bf16 result (push all-gather). Chunks in table order.
template <int W>
__global__ void __launch_bounds__(kThreads)
fused_peer_kernel(ptk_adam_scalars s, const __grid_constant__ FusedList list, StatsWorkspace* ws,
                  ptk_grad_stats_t* stats, const float* gscale_dev, const int32_t* skip_dev) {
  if (skip_dev != nullptr && *skip_dev != 0) return;
  const float gs = launch_gscale(s, gscale_dev);
  SumSq sq;
  unsigned bad = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
  for (int c = 0; c < list.n_chunks; ++c) {
    const FusedDesc& d = fused_at(list, c);
    const int64_t off = static_cast<int64_t>(list.rank) * d.shard;
    const int64_t nvec = d.shard >> 3;  // shards are multiples of 8 elements
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < nvec;
         i += stride) {
      const int64_t e = i << 3;
      uint4 raw[W];
#pragma unroll
      for (int r = 0; r < W; ++r)
        raw[r] = __ldcs(reinterpret_cast<const uint4*>(d.grad[r] + off + e));
      float p[8], m[8], v[8], g[8], t[8];
      ld8f(d.master + e, p);
      ld8f(d.m + e, m);
      ld8f(d.v + e, v);
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
        const float gk = __fmul_rn(g[k], gs);
        accum_stats(gk, usq, bad);
        adam_elem(s, gk, p[k], m[k], v[k]);
      }
      sq.add(usq);
      st8f(d.master + e, p);
      st8f(d.m + e, m);
      st8f(d.v + e, v);
      const uint4 out = pack8(p);
#pragma unroll
      for (int r = 0; r < W; ++r)  // all-gather by push
        __stcs(reinterpret_cast<uint4*>(d.param[r] + off + e), out);
    }
  }
  if (stats != nullptr) reduce_stats(sq, bad, ws, stats);
}

// Phase 1 of a clipped / overflow-checked fused step: the statistics of the
// reduced, scaled gradient of this rank's shards (the same fp32 rank-order
// sum and the same per-element values the update kernel then uses), no
// update. 2 B per chunk parameter of gradient reads per rank.
template <int W>
__global__ void __launch_bounds__(kThreads)
fused_stats_kernel(ptk_adam_scalars s, const __grid_constant__ FusedList list, StatsWorkspace* ws,
                   ptk_grad_stats_t* stats) {
  constexpr int U = W <= 2 ? 4 : W <= 4 ? 2 : 1;  // >= 4 x 16 B loads in flight per thread
  SumSq sq;
  unsigned bad = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
  for (int c = 0; c < list.n_chunks; ++c) {
    const FusedDesc& d = fused_at(list, c);
    const int64_t off = static_cast<int64_t>(list.rank) * d.shard;
    const int64_t nvec = d.shard >> 3;
    int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    for (; i < nvec; i += U * stride) {
      uint4 raw[U][W];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < W; ++r)
          if (i + u * stride < nvec)
            raw[u][r] = __ldcs(reinterpret_cast<const uint4*>(d.grad[r] + off +
                                                              ((i + u * stride) << 3)));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i + u * stride >= nvec) break;
        float g[8], t[8];
        unpack8(raw[u][0], g);
#pragma unroll
        for (int r = 1; r < W; ++r) {
          unpack8(raw[u][r], t);
#pragma unroll
          for (int k = 0; k < 8; ++k) g[k] = __fadd_rn(g[k], t[k]);
        }
        // the update kernels sum squares per 4 elements (TMA tile) or per 8
        // (LDG): statistics are reproducible per kernel, within 1e-6 across
        float usq = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) accum_stats(__fmul_rn(g[k], s.gscale), usq, bad);
        sq.add(usq);
      }
    }
  }
  reduce_stats(sq, bad, ws, stats);
}

// The same K1+K3+K4 step through a TMA ring: per tile of owned elements one
// elected thread bulk-loads the local fp32 master/m/v tiles and the owned tile
// of EVERY rank's gradient chunk (peer memory, NVLink on a node) into one
// stage, the CTA sums the W gradients in fp32 in rank order (bit-identical to
// fused_peer_kernel and the oracle), applies Adam, and the elected thread
// bulk-stores the state locally and the bf16 tile into every rank's parameter
// chunk (push all-gather). Tile shape per W (elements; threads = tile / 4),
// measured with virtual ranks (profiles/README.md): W = 2 -> 2048,
// W = 1, 3, 4 -> 1536, W >= 5 -> 1024.
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

template <int W, int kStages, bool kDynamic>
__global__ void __launch_bounds__(fused_threads<W>() + kRoleThreads, 1)
fused_peer_tma_kernel(ptk_adam_scalars s, const __grid_constant__ FusedList list,
                      StatsWorkspace* ws, ptk_grad_stats_t* stats, const float* gscale_dev,
                      const int32_t* skip_dev) {
  constexpr int kFusedTile = fused_tile<W>();
  constexpr int kThr = fused_threads<W>();
  constexpr int kConsumerWarps = kThr / 32;
  static_assert(kStages >= 2, "ring needs >= 2 stages");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto* stage = reinterpret_cast<FusedStage<W>*>(smem_raw);
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ __align__(8) uint64_t done[kStages];
  __shared__ __align__(8) uint64_t empty[kStages];
  __shared__ ItemMeta meta[kStages];
  if (skip_dev != nullptr && *skip_dev != 0) return;
  const float gs = launch_gscale(s, gscale_dev);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t T = list.total_tiles;
  const int64_t my_items = T > blockIdx.x ? (T - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&done[i], kConsumerWarps);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  SumSq sq;
  unsigned bad = 0;
  if (warp == kConsumerWarps) {
    // ---------------- producer: local state + every rank's gradient tile --
    if (lane == 0) {
      TileCursor<FusedDesc> cur;
      RingPos pos;
      int64_t claimed = kDynamic ? claim_tile(ws) : 0;  // one claim in flight ahead
      for (int64_t k = 0; kDynamic || k < my_items; ++k) {
        if (k >= kStages) mbar_wait(&empty[pos.st], pos.ph ^ 1u);
        int64_t t = blockIdx.x + k * gridDim.x;
        if (kDynamic) {
          t = claimed;
          if (t >= T) {  // end of the step: a tile-less stage tells the others
            meta[pos.st] = ItemMeta{0, -1, 0};
            mbar_arrive(&full[pos.st]);
            release_scheduler(ws);
            break;
          }
          claimed = claim_tile(ws);
        }
        cursor_seek(list, cur, t);
        const FusedDesc& d = cur.d;
        const int64_t e = (t - d.tile0) * kFusedTile;
        const int64_t left = d.shard - e;
        const int len = left < kFusedTile ? static_cast<int>(left) : kFusedTile;
        const int64_t off = static_cast<int64_t>(list.rank) * d.shard + e;
        meta[pos.st] = ItemMeta{e, cur.c, len};
        FusedStage<W>& S = stage[pos.st];
        uint64_t* bar = &full[pos.st];
        mbar_expect_tx(bar, static_cast<uint32_t>(len) * (3 * sizeof(float) + W * sizeof(uint16_t)));
        bulk_load(S.master, d.master + e, len * 4, bar);
        bulk_load(S.m, d.m + e, len * 4, bar);
        bulk_load(S.v, d.v + e, len * 4, bar);
#pragma unroll
        for (int r = 0; r < W; ++r) bulk_load(S.grad[r], d.grad[r] + off, len * 2, bar);
        pos.next<kStages>();
      }
    }
  } else if (warp == kConsumerWarps + 1) {
    // ------------- storer: local state + the bf16 tile into every rank --
    if (lane == 0) {
      TileCursor<FusedDesc> scur;
      RingPos pos;
      int prev = -1;
      for (int64_t k = 0; kDynamic || k < my_items; ++k) {
        mbar_wait(&done[pos.st], pos.ph);
        const ItemMeta it = meta[pos.st];
        if (kDynamic && it.c < 0) break;
        const FusedDesc& d = cursor_at(list, scur, it.c);
        const int64_t off = static_cast<int64_t>(list.rank) * d.shard + it.e;
        FusedStage<W>& S = stage[pos.st];
        bulk_store(d.master + it.e, S.master, it.len * 4);
        bulk_store(d.m + it.e, S.m, it.len * 4);
        bulk_store(d.v + it.e, S.v, it.len * 4);
#pragma unroll
        for (int r = 0; r < W; ++r) bulk_store(d.param[r] + off, S.param, it.len * 2);
        bulk_commit();
        if (prev >= 0) {
          bulk_wait_read<1>();
          mbar_arrive(&empty[prev]);
        }
        prev = pos.st;
        pos.next<kStages>();
      }
      bulk_wait_all();
    }
  } else {
    // ------------------------------------------------------ consumers --
    RingPos pos;
    for (int64_t k = 0; kDynamic || k < my_items; ++k) {
      mbar_wait(&full[pos.st], pos.ph);
      if (kDynamic && meta[pos.st].c < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[pos.st]);  // lets the storer see the end
        break;
      }
      const int len = meta[pos.st].len;
      FusedStage<W>& S = stage[pos.st];
      const int e = tid * 4;
      if (e < len) {  // always, except in a chunk's last tile
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
          const float gk = __fmul_rn(g[q], gs);
          accum_stats(gk, usq, bad);
          adam_elem(s, gk, pp[q], mm[q], vv[q]);
        }
        sq.add(usq);
        *reinterpret_cast<float4*>(&S.master[e]) = p;
        *reinterpret_cast<float4*>(&S.m[e]) = m;
        *reinterpret_cast<float4*>(&S.v[e]) = v;
        *reinterpret_cast<uint2*>(&S.param[e]) =
            make_uint2(pack_bf16x2(p.x, p.y), pack_bf16x2(p.z, p.w));
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&done[pos.st]);
      pos.next<kStages>();
    }
  }
  __syncthreads();
  if (stats != nullptr) reduce_stats(sq, bad, ws, stats);
}

// ------------------------------------------------- peer synchronisation ----

struct SignalTable {
  int32_t* slot[PTK_MAX_PEERS];
};

__device__ __forceinline__ void spin_until(const int32_t* flag, int32_t epoch, int64_t timeout_ns,
                                           const char* what, int rank, int peer) {
  int32_t seen;
  uint64_t t0, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(seen) : "l"(flag) : "memory");
    if (seen >= epoch) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (static_cast<int64_t>(now - t0) > timeout_ns) {
      printf("%s: rank %d timed out waiting for rank %d (epoch %d, seen %d)\n", what, rank, peer,
             epoch, seen);
      __trap();
    }
    __nanosleep(64);
  }
}

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
  spin_until(sig.slot[rank] + t, epoch, timeout_ns, "ptk_peer_barrier", rank, t);
}

// Statistics mailbox: slot r of every rank's mailbox receives rank r's
// partial statistics; a release-stored epoch publishes them.
struct alignas(32) MailSlot {
  double sumsq;
  unsigned long long nonfinite;
  int32_t epoch;
  int32_t pad[3];
};
static_assert(sizeof(MailSlot) == 32, "mailbox slot is 32 bytes");

struct MailTable {
  MailSlot* box[PTK_MAX_PEERS];
};

__global__ void stats_publish_kernel(const ptk_grad_stats_t* stats, MailTable peers, int world,
                                     int rank, int epoch) {
  const int t = threadIdx.x;
  if (t >= world) return;
  MailSlot* slot = peers.box[t] + rank;
  slot->sumsq = stats->sumsq;
  slot->nonfinite = stats->nonfinite;
  __threadfence_system();
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(&slot->epoch), "r"(epoch) : "memory");
}

// Sums the world's slots in rank order 0..W-1 (the same bits on every rank),
// writes the global statistics, the clip coefficient and the skip flag.
__global__ void stats_collect_kernel(const MailSlot* box, int world, int epoch, double max_norm,
                                     int64_t timeout_ns, ptk_grad_stats_t* global_out, float* coef,
                                     int32_t* skip) {
  if (threadIdx.x != 0) return;
  double sq = 0.0;
  unsigned long long bad = 0;
  for (int r = 0; r < world; ++r) {
    spin_until(&box[r].epoch, epoch, timeout_ns, "ptk_stats_collect", -1, r);
    const volatile MailSlot* v = box + r;
    sq += v->sumsq;
    bad += v->nonfinite;
  }
  if (global_out != nullptr) {
    global_out->sumsq = sq;
    global_out->nonfinite = bad;
  }
  clip_from_stats(sq, bad, max_norm, coef, skip);
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

// ------------------------------------------- K4 for non-persistent chunks --
// Reduce-scatter over peer memory for a chunk that leaves the device after its
// backward (the offload path): the owned shard of every rank's bf16 gradient
// chunk, summed in fp32 in rank order 0..W-1 -- the same sum the fused
// persistent step feeds its Adam -- written as fp32 (the host Adam consumes
// it unrounded, so an offloaded chunk's update is bit-identical to a
// persistent one's). Pure streaming over NVLink: register-staged 128-bit
// loads, every peer's 8-element unit issued before any add.
struct PeerGrads {
  const uint16_t* g[PTK_MAX_PEERS];  // rank r's gradient chunk + this rank's shard offset
};

// U units per thread per iteration keep >= 8 independent 16-byte loads in
// flight per thread whatever W is (W = 2: 4 units).
template <int W>
__host__ __device__ constexpr int peer_reduce_units() { return W >= 8 ? 1 : 8 / W; }

template <int W>
__global__ void __launch_bounds__(kThreads)
peer_reduce_f32_kernel(PeerGrads p, int64_t n, float* __restrict__ out) {
  constexpr int U = peer_reduce_units<W>();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t nvec = n >> 3;
  for (int64_t u0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u0 < nvec;
       u0 += stride * U) {
    uint4 raw[U][W];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t u = u0 + j * stride;
#pragma unroll
      for (int r = 0; r < W; ++r)
        raw[j][r] = u < nvec ? __ldcs(reinterpret_cast<const uint4*>(p.g[r]) + u) : uint4{};
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t u = u0 + j * stride;
      if (u >= nvec) break;
      float acc[8], f[8];
      unpack8(raw[j][0], acc);
#pragma unroll
      for (int r = 1; r < W; ++r) {
        unpack8(raw[j][r], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = __fadd_rn(acc[k], f[k]);
      }
      st8f(out + 8 * u, acc);
    }
  }
  // n % 8 trailing elements (unpadded shards only)
  for (int64_t i = 8 * nvec + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    float acc = GradBf16::load1(p.g[0] + i);
#pragma unroll
    for (int r = 1; r < W; ++r) acc = __fadd_rn(acc, GradBf16::load1(p.g[r] + i));
    out[i] = acc;
  }
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
// Per-device caches: a process may launch on several devices (single-process
// multi-GPU harnesses, the executor), and both the SM count and the opt-in
// dynamic shared-memory attribute are properties of a device context.

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}

int sm_count() {
  static std::atomic<int> cache[kMaxDevices];
  const int dev = current_device();
  int c = cache[dev].load(std::memory_order_relaxed);
  if (c == 0) {
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    if (c <= 0) c = 148;
    cache[dev].store(c, std::memory_order_relaxed);
  }
  return c;
}

// Opt-in dynamic shared memory for kernel `k` on the current device, once per
// (kernel instantiation, device): `done` is the caller's per-kernel static.
template <typename K>
int ensure_smem(K k, int bytes, std::atomic<bool> (&done)[kMaxDevices], const char* what) {
  const int dev = current_device();
  if (done[dev].load(std::memory_order_acquire)) return PTK_OK;
  const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return check_cuda(e, what);
  done[dev].store(true, std::memory_order_release);
  return PTK_OK;
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

// PTK_TILE_SCHEDULE=static forces the round-robin tile split (A/B runs).
bool static_schedule() {
  static const bool v = [] {
    const char* e = std::getenv("PTK_TILE_SCHEDULE");
    return e != nullptr && std::string(e) == "static";
  }();
  return v;
}

constexpr int kUnroll = 2;

// TMA ring shapes of the chunk Adam: (name, tile elements, ring stages, CTAs
// per SM, threads, L2 evict-first hint). The product build has the measured
// best only (profiles/README.md, interleaved sweep); the shape sweep is
// compiled in with -DPTK_BENCH_VARIANTS and selected by PTK_ADAM_VARIANT.
#ifdef PTK_BENCH_VARIANTS
#define PTK_TMA_VARIANTS(X)                     \
  X(Tma1536x9t384, 1536, 9, 1, 384, false)      \
  X(Tma2048x6t512, 2048, 6, 1, 512, false)      \
  X(Tma2048x6t512h, 2048, 6, 1, 512, true)      \
  X(Tma2560x5t640, 2560, 5, 1, 640, false)      \
  X(Tma3072x4t768, 3072, 4, 1, 768, false)      \
  X(Tma1024x13t256, 1024, 13, 1, 256, false)    \
  X(Tma1792x7t448, 1792, 7, 1, 448, false)      \
  X(Tma1024x6x2t256, 1024, 6, 2, 256, false)
#else
#define PTK_TMA_VARIANTS(X) X(Tma2048x6t512, 2048, 6, 1, 512, false)
#endif

#define PTK_ENUM_ENTRY(V, T, S, P, THR, H) V,
enum class AdamVariant { Ldg, PTK_TMA_VARIANTS(PTK_ENUM_ENTRY) };
#undef PTK_ENUM_ENTRY

// Default: the fastest shape measured on B200; "ldg" selects the register-
// staged kernel (per-chunk launches) in any build.
AdamVariant adam_variant() {
  static const AdamVariant v = [] {
    const char* e = std::getenv("PTK_ADAM_VARIANT");
    std::string name = e ? e : "";
    for (auto& ch : name) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    if (name == "ldg") return AdamVariant::Ldg;
#define PTK_NAME_ENTRY(V, T, S, P, THR, H)                                \
    {                                                                     \
      std::string tag = #V;                                               \
      for (auto& ch : tag) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch))); \
      if (name == tag) return AdamVariant::V;                             \
    }
    PTK_TMA_VARIANTS(PTK_NAME_ENTRY)
#undef PTK_NAME_ENTRY
    return AdamVariant::Tma2048x6t512;
  }();
  return v;
}

int adam_tile() {
  switch (adam_variant()) {
#define PTK_TILE_CASE(V, T, S, P, THR, H) \
  case AdamVariant::V:                    \
    return T;
    PTK_TMA_VARIANTS(PTK_TILE_CASE)
#undef PTK_TILE_CASE
    default:
      return 2048;
  }
}

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

template <int kTile, int kStages, int kPerSm, int kThr, bool kStats, bool kHint, int kCap>
int launch_tma(const ptk_adam_scalars& s, const ChunkBatch<kCap>& b, StatsWorkspace* ws,
               ptk_grad_stats_t* stats, const float* gscale_dev, const int32_t* skip_dev,
               cudaStream_t st) {
  const bool dynamic = ws != nullptr && !static_schedule();
  auto k = dynamic ? chunk_adam_tma_kernel<kTile, kStages, kThr, kStats, kHint, kCap, true>
                   : chunk_adam_tma_kernel<kTile, kStages, kThr, kStats, kHint, kCap, false>;
  constexpr int kSmem = kStages * static_cast<int>(sizeof(TmaStage<kTile>));
  static std::atomic<bool> configured[2][kMaxDevices];
  const int rc = ensure_smem(k, kSmem, configured[dynamic], "chunk_adam_tma_kernel smem attribute");
  if (rc != PTK_OK) return rc;
  int64_t grid = static_cast<int64_t>(sm_count()) * kPerSm;
  if (grid > b.total_tiles) grid = b.total_tiles;
  if (grid < 1) grid = 1;  // tails only
  k<<<static_cast<int>(grid), kThr + kRoleThreads, kSmem, st>>>(s, b, ws, stats, gscale_dev,
                                                                skip_dev);
  launch_counter()++;
  return PTK_OK;
}

template <int kTile, int kStages, int kPerSm, int kThr, bool kHint, int kCap>
int launch_tma_any(const ptk_adam_scalars& s, const ChunkBatch<kCap>& b, StatsWorkspace* ws,
                   ptk_grad_stats_t* stats, const float* gscale_dev, const int32_t* skip_dev,
                   cudaStream_t st) {
  return stats ? launch_tma<kTile, kStages, kPerSm, kThr, true, kHint, kCap>(
                     s, b, ws, stats, gscale_dev, skip_dev, st)
               : launch_tma<kTile, kStages, kPerSm, kThr, false, kHint, kCap>(
                     s, b, ws, stats, gscale_dev, skip_dev, st);
}

int64_t tiles_of(int64_t n, int tile) { return ((n & ~int64_t{7}) + tile - 1) / tile; }

// One TMA launch over a batch (tile0 computed for adam_tile()).
template <int kCap>
int launch_tma_batch(const ptk_adam_scalars& s, const ChunkBatch<kCap>& b, StatsWorkspace* ws,
                     ptk_grad_stats_t* stats, const float* gscale_dev, const int32_t* skip_dev,
                     cudaStream_t st) {
  switch (adam_variant()) {
#define PTK_TMA_CASE(V, T, S, P, THR, H) \
  case AdamVariant::V:                   \
    return launch_tma_any<T, S, P, THR, H, kCap>(s, b, ws, stats, gscale_dev, skip_dev, st);
    PTK_TMA_VARIANTS(PTK_TMA_CASE)
#undef PTK_TMA_CASE
    default:
      return fail(PTK_EINVAL, "launch_tma_batch: not a TMA variant");
  }
}

// Batch capacities: one chunk (ptk_chunk_adam), small tables (a model's
// handful of 512 MiB - 1 GiB chunks) and large tables (up to 128 chunks per
// launch: 7 KB of kernel parameters).
constexpr int kSmallCap = 16;
constexpr int kLargeCap = 128;

template <int kCap>
void fill_batch(ChunkBatch<kCap>& b, const ChunkDesc* descs, int n, int tile) {
  b = ChunkBatch<kCap>{};
  int64_t tile0 = 0;
  for (int c = 0; c < n; ++c) {
    b.d[c] = descs[c];
    b.d[c].tile0 = tile0;
    tile0 += tiles_of(descs[c].n, tile);
  }
  b.n_chunks = n;
  b.total_tiles = tile0;
}

int validate_adam_buffers(const float* master, const float* m, const float* v, const void* grad,
                          const uint16_t* param_out, int64_t n, const char* what) {
  if (n == 0) return PTK_OK;  // an empty chunk touches no buffer
  if (!master || !m || !v || !grad) return fail(PTK_EINVAL, std::string(what) + ": null buffer");
  if (n < 0) return fail(PTK_EINVAL, std::string(what) + ": negative n");
  if (!aligned16(master) || !aligned16(m) || !aligned16(v) || !aligned16(grad) ||
      (param_out && !aligned16(param_out)))
    return fail(PTK_EINVAL, std::string(what) + ": buffers must be 16-byte aligned");
  return PTK_OK;
}

template <class G>
int launch_adam(const ptk_adam_config* cfg, float* master, float* m, float* v,
                const typename G::T* grad, uint16_t* param_out, int64_t n,
                ptk_grad_stats_t* stats, void* workspace, const float* gscale_dev,
                const int32_t* skip_dev, void* stream) {
  if (!cfg) return fail(PTK_EINVAL, "ptk_chunk_adam: null config");
  int rc = validate_adam_buffers(master, m, v, grad, param_out, n, "ptk_chunk_adam");
  if (rc != PTK_OK) return rc;
  if (cfg->step < 1) return fail(PTK_EINVAL, "ptk_chunk_adam: step must be >= 1");
  if (stats && !workspace) return fail(PTK_EINVAL, "ptk_chunk_adam: stats requires workspace");
  if (n == 0) return PTK_OK;
  const ptk_adam_scalars s = derive_scalars(*cfg);
  auto* ws = static_cast<StatsWorkspace*>(workspace);
  cudaStream_t st = as_stream(stream);
  if constexpr (std::is_same_v<G, GradBf16>) {
    if (adam_variant() != AdamVariant::Ldg) {
      const ChunkDesc one{master, m, v, grad, param_out, n, 0};
      ChunkBatch<1> b;
      fill_batch(b, &one, 1, adam_tile());
      rc = launch_tma_batch(s, b, ws, stats, gscale_dev, skip_dev, st);
      return rc != PTK_OK ? rc : check_cuda(cudaGetLastError(), "chunk_adam_tma launch");
    }
  }
  if (stats)
    launch_ldg<G, true>(s, master, m, v, grad, param_out, n, ws, stats, gscale_dev, skip_dev, st);
  else
    launch_ldg<G, false>(s, master, m, v, grad, param_out, n, ws, stats, gscale_dev, skip_dev, st);
  return check_cuda(cudaGetLastError(), "chunk_adam_kernel launch");
}

// Fused-kernel override from PTK_FUSED_KERNEL ("tma" / "ldg"), read once; the
// per-table choice (ptk_fused_table_create's `kernel`) applies otherwise.
int fused_env_override() {
  static const int mode = [] {
    const char* e = std::getenv("PTK_FUSED_KERNEL");
    if (e && std::string(e) == "tma") return PTK_FUSED_TMA;
    if (e && std::string(e) == "ldg") return PTK_FUSED_LDG;
    return PTK_FUSED_AUTO;
  }();
  return mode;
}


int fused_tile_for(int world) {
  switch (world) {
    case 1: return fused_tile<1>();
    case 2: return fused_tile<2>();
    case 3: return fused_tile<3>();
    case 4: return fused_tile<4>();
    case 5: return fused_tile<5>();
    case 6: return fused_tile<6>();
    case 7: return fused_tile<7>();
    default: return fused_tile<8>();
  }
}

enum class FusedOp { Step, Stats };

template <int W>
int launch_fused(FusedOp op, const ptk_adam_scalars& s, const FusedList& list, int64_t max_shard,
                 StatsWorkspace* ws, ptk_grad_stats_t* stats, const float* gscale_dev,
                 const int32_t* skip_dev, cudaStream_t st, bool tma) {
  const int64_t units = (max_shard >> 3) > 0 ? (max_shard >> 3) : 1;
  if (op == FusedOp::Stats) {
    auto k = fused_stats_kernel<W>;
    k<<<grid_for(k, units), kThreads, 0, st>>>(s, list, ws, stats);
    return PTK_OK;
  }
  if (!tma) {
    auto k = fused_peer_kernel<W>;
    k<<<grid_for(k, units), kThreads, 0, st>>>(s, list, ws, stats, gscale_dev, skip_dev);
    return PTK_OK;
  }
  constexpr int kSt = fused_stages<W>();
  constexpr int kSmem = kSt * static_cast<int>(sizeof(FusedStage<W>));
  int64_t grid = sm_count();
  if (grid > list.total_tiles) grid = list.total_tiles;
  if (grid < 1) grid = 1;
  // the dynamic tile scheduler keeps its counter in the workspace
  const bool dynamic = ws != nullptr && !static_schedule();
  auto k = dynamic ? fused_peer_tma_kernel<W, kSt, true> : fused_peer_tma_kernel<W, kSt, false>;
  static std::atomic<bool> configured[2][kMaxDevices];
  const int rc = ensure_smem(k, kSmem, configured[dynamic], "fused_peer_tma_kernel smem attribute");
  if (rc != PTK_OK) return rc;
  k<<<static_cast<int>(grid), fused_threads<W>() + kRoleThreads, kSmem, st>>>(s, list, ws, stats, gscale_dev,
                                                                skip_dev);
  return PTK_OK;
}

int dispatch_fused(int world, FusedOp op, const ptk_adam_scalars& s, const FusedList& list,
                   int64_t max_shard, StatsWorkspace* ws, ptk_grad_stats_t* stats,
                   const float* gscale_dev, const int32_t* skip_dev, cudaStream_t st, bool tma) {
  switch (world) {
    case 1: return launch_fused<1>(op, s, list, max_shard, ws, stats, gscale_dev, skip_dev, st, tma);
    case 2: return launch_fused<2>(op, s, list, max_shard, ws, stats, gscale_dev, skip_dev, st, tma);
    case 3: return launch_fused<3>(op, s, list, max_shard, ws, stats, gscale_dev, skip_dev, st, tma);
    case 4: return launch_fused<4>(op, s, list, max_shard, ws, stats, gscale_dev, skip_dev, st, tma);
    case 5: return launch_fused<5>(op, s, list, max_shard, ws, stats, gscale_dev, skip_dev, st, tma);
    case 6: return launch_fused<6>(op, s, list, max_shard, ws, stats, gscale_dev, skip_dev, st, tma);
    case 7: return launch_fused<7>(op, s, list, max_shard, ws, stats, gscale_dev, skip_dev, st, tma);
    default: return launch_fused<8>(op, s, list, max_shard, ws, stats, gscale_dev, skip_dev, st, tma);
  }
}

int64_t peer_timeout_ns() {
  static const int64_t ns = [] {
    const char* e = std::getenv("PTK_PEER_BARRIER_TIMEOUT_MS");
    const long long ms = e ? std::atoll(e) : 60000;
    return static_cast<int64_t>(ms > 0 ? ms : 60000) * 1000000;
  }();
  return ns;
}

}  // namespace
}  // namespace ptk

using namespace ptk;

// Opaque table handles of the C-ABI (include/ptk.h).
struct ptk_chunk_table {
  std::vector<ChunkDesc> host;                    // the caller's chunks
  ChunkBatch<kSmallCap> small{};                  // n <= kSmallCap: one launch
  std::vector<ChunkBatch<kLargeCap>> large;       // else batches of kLargeCap
  int tile = 0;                                   // tile size the batches were cut for
};

struct ptk_fused_table {
  std::vector<FusedDesc> host;
  FusedDesc* dev = nullptr;
  int64_t total_tiles = 0;
  int64_t max_shard = 0;
  int32_t world = 1;
  int32_t rank = 0;
  int32_t kernel = PTK_FUSED_TMA;  // resolved: PTK_FUSED_TMA or PTK_FUSED_LDG
  int device = 0;
};

extern "C" {

int64_t ptk_stats_workspace_bytes(void) { return static_cast<int64_t>(sizeof(StatsWorkspace)); }

const char* ptk_adam_kernel_name(void) {
  switch (adam_variant()) {
    case AdamVariant::Ldg: return "ldg";
#define PTK_NAME_CASE(V, T, S, P, THR, H) \
  case AdamVariant::V:                    \
    return "tma tile=" #T " stages=" #S " ctas/sm=" #P " threads=" #THR " l2_evict_first=" #H;
    PTK_TMA_VARIANTS(PTK_NAME_CASE)
#undef PTK_NAME_CASE
  }
  return "?";
}

const char* ptk_fused_kernel_name(void) {
  switch (fused_env_override()) {
    case PTK_FUSED_TMA:
      return "fused_peer_tma_kernel (forced by PTK_FUSED_KERNEL=tma)";
    case PTK_FUSED_LDG:
      return "fused_peer_kernel (ldg, forced by PTK_FUSED_KERNEL=ldg)";
    default:
      return "fused_peer_tma_kernel (tile 2048 for W=2, 1536 for W=1,3,4, 1024 for W>=5; "
             "threads = tile/4 + producer/storer warps; stages = min(9, 220 KB / stage); dynamic "
             "tile schedule)";
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

// ---- chunk tables: one launch per step over every chunk ----

int ptk_chunk_table_create(const ptk_chunk_desc* descs, int32_t n_chunks, ptk_chunk_table** out) {
  if (!out || (!descs && n_chunks > 0) || n_chunks < 0)
    return fail(PTK_EINVAL, "ptk_chunk_table_create: bad arguments");
  *out = nullptr;
  auto* t = new ptk_chunk_table;
  for (int32_t c = 0; c < n_chunks; ++c) {
    const ptk_chunk_desc& d = descs[c];
    const int rc = validate_adam_buffers(d.master, d.exp_avg, d.exp_avg_sq, d.grad, d.param_out,
                                         d.n, "ptk_chunk_table_create");
    if (rc != PTK_OK) {
      delete t;
      return rc;
    }
    t->host.push_back(ChunkDesc{d.master, d.exp_avg, d.exp_avg_sq, d.grad, d.param_out, d.n, 0});
  }
  // the table lives in host memory and travels in the kernel parameters
  t->tile = adam_tile();
  const int n = static_cast<int>(t->host.size());
  if (n <= kSmallCap) {
    fill_batch(t->small, t->host.data(), n, t->tile);
  } else {
    for (int lo = 0; lo < n; lo += kLargeCap) {
      t->large.emplace_back();
      fill_batch(t->large.back(), t->host.data() + lo, n - lo < kLargeCap ? n - lo : kLargeCap,
                 t->tile);
    }
  }
  *out = t;
  return PTK_OK;
}

int ptk_chunk_table_destroy(ptk_chunk_table* t) {
  delete t;
  return PTK_OK;
}

int64_t ptk_chunk_table_params(const ptk_chunk_table* t) {
  int64_t n = 0;
  if (t)
    for (const auto& d : t->host) n += d.n;
  return n;
}

int ptk_chunk_adam_table(const ptk_adam_config* cfg, const ptk_chunk_table* t,
                         ptk_grad_stats_t* stats, void* workspace, const float* gscale_dev,
                         const int32_t* skip_dev, void* stream) {
  if (!cfg || !t) return fail(PTK_EINVAL, "ptk_chunk_adam_table: null argument");
  if (cfg->step < 1) return fail(PTK_EINVAL, "ptk_chunk_adam_table: step must be >= 1");
  if (stats && !workspace) return fail(PTK_EINVAL, "ptk_chunk_adam_table: stats requires workspace");
  if (t->host.empty()) return PTK_OK;
  if (adam_variant() == AdamVariant::Ldg || t->tile != adam_tile()) {
    // per-chunk launches (the "ldg" variant)
    for (const auto& d : t->host) {
      const int rc = ptk_chunk_adam(cfg, d.master, d.m, d.v, d.grad, d.param, d.n, stats, workspace,
                                    gscale_dev, skip_dev, stream);
      if (rc != PTK_OK) return rc;
    }
    return PTK_OK;
  }
  const ptk_adam_scalars s = derive_scalars(*cfg);
  auto* ws = static_cast<StatsWorkspace*>(workspace);
  cudaStream_t st = as_stream(stream);
  int rc = PTK_OK;
  if (t->large.empty()) {
    rc = launch_tma_batch(s, t->small, ws, stats, gscale_dev, skip_dev, st);
  } else {
    for (const auto& b : t->large) {
      rc = launch_tma_batch(s, b, ws, stats, gscale_dev, skip_dev, st);
      if (rc != PTK_OK) break;
    }
  }
  return rc != PTK_OK ? rc : check_cuda(cudaGetLastError(), "chunk_adam_tma (table) launch");
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

// ---- fused RS -> Adam -> AG ----

int ptk_fused_table_create(const ptk_fused_desc* descs, int32_t n_chunks, int32_t world,
                           int32_t rank, int32_t kernel, ptk_fused_table** out) {
  if (!out || (!descs && n_chunks > 0) || n_chunks < 0)
    return fail(PTK_EINVAL, "ptk_fused_table_create: bad arguments");
  *out = nullptr;
  if (world < 1 || world > PTK_MAX_PEERS || rank < 0 || rank >= world)
    return fail(PTK_EINVAL, "ptk_fused_table_create: bad world/rank");
  if (kernel != PTK_FUSED_AUTO && kernel != PTK_FUSED_TMA && kernel != PTK_FUSED_LDG)
    return fail(PTK_EINVAL, "ptk_fused_table_create: unknown kernel selector");
  auto* t = new ptk_fused_table;
  t->world = world;
  t->rank = rank;
  t->device = current_device();
  const int tile = fused_tile_for(world);
  int64_t tile0 = 0;
  for (int32_t c = 0; c < n_chunks; ++c) {
    const ptk_fused_desc& d = descs[c];
    const char* bad = nullptr;
    if (d.shard < 0 || (d.shard & 7) != 0) bad = "shard must be a non-negative multiple of 8 elements";
    if (!d.master || !d.exp_avg || !d.exp_avg_sq || !aligned16(d.master) || !aligned16(d.exp_avg) ||
        !aligned16(d.exp_avg_sq))
      bad = "state buffers must be non-null and 16-byte aligned";
    FusedDesc f{};
    for (int r = 0; r < world && !bad; ++r) {
      if (!d.grad_peers[r] || !d.param_peers[r] || !aligned16(d.grad_peers[r]) ||
          !aligned16(d.param_peers[r]))
        bad = "peer buffers must be non-null and 16-byte aligned";
      f.grad[r] = d.grad_peers[r];
      f.param[r] = d.param_peers[r];
    }
    if (bad) {
      delete t;
      return fail(PTK_EINVAL, std::string("ptk_fused_table_create: ") + bad);
    }
    f.master = d.master;
    f.m = d.exp_avg;
    f.v = d.exp_avg_sq;
    f.shard = d.shard;
    f.tile0 = tile0;
    tile0 += (d.shard + tile - 1) / tile;
    if (d.shard > t->max_shard) t->max_shard = d.shard;
    t->host.push_back(f);
  }
  t->total_tiles = tile0;
  // Kernel choice, once per table: the caller's, else PTK_FUSED_KERNEL, else
  // the TMA ring. Bulk copies address peer memory like any global memory (a
  // cudaIpc / peer mapping is a global address), as TMA loads from peer GPUs
  // do in distributed GEMMs; the register-staged kernel stays selectable.
  int k = kernel;
  if (k == PTK_FUSED_AUTO) k = fused_env_override();
  if (k == PTK_FUSED_AUTO) k = PTK_FUSED_TMA;
  t->kernel = k;
  if (n_chunks > 0) {
    const size_t bytes = sizeof(FusedDesc) * t->host.size();
    cudaError_t e = cudaMalloc(&t->dev, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(t->dev, t->host.data(), bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      if (t->dev) cudaFree(t->dev);
      delete t;
      return check_cuda(e, "ptk_fused_table_create: device table");
    }
  }
  *out = t;
  return PTK_OK;
}

int ptk_fused_table_destroy(ptk_fused_table* t) {
  if (!t) return PTK_OK;
  const cudaError_t e = t->dev ? cudaFree(t->dev) : cudaSuccess;
  delete t;
  return check_cuda(e, "ptk_fused_table_destroy");
}

int32_t ptk_fused_table_kernel(const ptk_fused_table* t) { return t ? t->kernel : -1; }

namespace {
int fused_table_launch(FusedOp op, const ptk_adam_config* cfg, const ptk_fused_table* t,
                       ptk_grad_stats_t* stats, void* workspace, const float* gscale_dev,
                       const int32_t* skip_dev, void* stream, const char* what) {
  if (!cfg || !t) return fail(PTK_EINVAL, std::string(what) + ": null argument");
  if (cfg->step < 1) return fail(PTK_EINVAL, std::string(what) + ": step must be >= 1");
  if (stats && !workspace) return fail(PTK_EINVAL, std::string(what) + ": stats requires workspace");
  if (op == FusedOp::Stats && !stats) return fail(PTK_EINVAL, std::string(what) + ": null stats");
  if (t->host.empty()) return PTK_OK;
  if (t->device != current_device())
    return fail(PTK_EINVAL, std::string(what) + ": table was created on another device");
  FusedList list{};
  list.table = t->dev;
  list.one = t->host[0];
  list.n_chunks = static_cast<int32_t>(t->host.size());
  list.total_tiles = t->total_tiles;
  list.rank = t->rank;
  const ptk_adam_scalars s = derive_scalars(*cfg);
  const int rc = dispatch_fused(t->world, op, s, list, t->max_shard,
                                static_cast<StatsWorkspace*>(workspace), stats, gscale_dev,
                                skip_dev, as_stream(stream), t->kernel == PTK_FUSED_TMA);
  if (rc != PTK_OK) return rc;
  launch_counter()++;
  return check_cuda(cudaGetLastError(), what);
}
}  // namespace

int ptk_fused_step_table(const ptk_adam_config* cfg, const ptk_fused_table* t,
                         ptk_grad_stats_t* stats, void* workspace, const float* gscale_dev,
                         const int32_t* skip_dev, void* stream) {
  return fused_table_launch(FusedOp::Step, cfg, t, stats, workspace, gscale_dev, skip_dev, stream,
                            "ptk_fused_step_table");
}

int ptk_fused_grad_stats_table(const ptk_adam_config* cfg, const ptk_fused_table* t,
                               ptk_grad_stats_t* stats, void* workspace, void* stream) {
  return fused_table_launch(FusedOp::Stats, cfg, t, stats, workspace, nullptr, nullptr, stream,
                            "ptk_fused_grad_stats_table");
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
  FusedList list{};
  for (int r = 0; r < world; ++r) {
    if (!grad_peers[r] || !param_peers[r] || !aligned16(grad_peers[r]) || !aligned16(param_peers[r]))
      return fail(PTK_EINVAL, "ptk_fused_rs_adam_ag: peer buffers must be non-null and 16-byte aligned");
    list.one.grad[r] = grad_peers[r];
    list.one.param[r] = param_peers[r];
  }
  if (!aligned16(master) || !aligned16(exp_avg) || !aligned16(exp_avg_sq))
    return fail(PTK_EINVAL, "ptk_fused_rs_adam_ag: state buffers must be 16-byte aligned");
  if (shard == 0) return PTK_OK;
  int k = fused_env_override();
  if (k == PTK_FUSED_AUTO) k = PTK_FUSED_TMA;
  list.table = nullptr;
  list.one.master = master;
  list.one.m = exp_avg;
  list.one.v = exp_avg_sq;
  list.one.shard = shard;
  list.one.tile0 = 0;
  list.n_chunks = 1;
  list.rank = rank;
  const int tile = fused_tile_for(world);
  list.total_tiles = (shard + tile - 1) / tile;
  const ptk_adam_scalars s = derive_scalars(*cfg);
  const int rc = dispatch_fused(world, FusedOp::Step, s, list, shard,
                                static_cast<StatsWorkspace*>(workspace), stats, nullptr, nullptr,
                                as_stream(stream), k == PTK_FUSED_TMA);
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
  peer_barrier_kernel<<<1, 32, 0, as_stream(stream)>>>(t, world, rank, epoch, peer_timeout_ns());
  launch_counter()++;
  return check_cuda(cudaGetLastError(), "peer_barrier_kernel launch");
}

int64_t ptk_stats_mailbox_bytes(void) {
  return static_cast<int64_t>(sizeof(MailSlot)) * PTK_MAX_PEERS;
}

int ptk_stats_publish(const ptk_grad_stats_t* stats, void* const* mailbox_peers, int32_t world,
                      int32_t rank, int32_t epoch, void* stream) {
  if (!stats || !mailbox_peers || world < 1 || world > PTK_MAX_PEERS || rank < 0 || rank >= world)
    return fail(PTK_EINVAL, "ptk_stats_publish: bad arguments");
  MailTable t{};
  for (int r = 0; r < world; ++r) {
    if (!mailbox_peers[r] || (reinterpret_cast<uintptr_t>(mailbox_peers[r]) & 31u) != 0)
      return fail(PTK_EINVAL, "ptk_stats_publish: mailboxes must be non-null and 32-byte aligned");
    t.box[r] = static_cast<MailSlot*>(mailbox_peers[r]);
  }
  stats_publish_kernel<<<1, 32, 0, as_stream(stream)>>>(stats, t, world, rank, epoch);
  launch_counter()++;
  return check_cuda(cudaGetLastError(), "stats_publish_kernel launch");
}

int ptk_stats_collect(const void* mailbox, int32_t world, int32_t epoch, double max_norm,
                      ptk_grad_stats_t* global_out, float* coef_out, int32_t* skip_out,
                      void* stream) {
  if (!mailbox || world < 1 || world > PTK_MAX_PEERS)
    return fail(PTK_EINVAL, "ptk_stats_collect: bad arguments");
  stats_collect_kernel<<<1, 32, 0, as_stream(stream)>>>(static_cast<const MailSlot*>(mailbox), world,
                                                        epoch, max_norm, peer_timeout_ns(),
                                                        global_out, coef_out, skip_out);
  launch_counter()++;
  return check_cuda(cudaGetLastError(), "stats_collect_kernel launch");
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

int ptk_peer_reduce_scatter_f32(const uint16_t* const* grad_peers, int32_t world, int32_t rank,
                                int64_t shard, float* out, void* stream) {
  if (!grad_peers || !out || world < 1 || world > PTK_MAX_PEERS || rank < 0 || rank >= world ||
      shard < 0)
    return fail(PTK_EINVAL, "ptk_peer_reduce_scatter_f32: bad arguments");
  if (shard == 0) return PTK_OK;
  PeerGrads p{};
  for (int r = 0; r < world; ++r) {
    if (!grad_peers[r]) return fail(PTK_EINVAL, "ptk_peer_reduce_scatter_f32: null peer");
    p.g[r] = grad_peers[r] + static_cast<int64_t>(rank) * shard;
    if ((reinterpret_cast<uintptr_t>(p.g[r]) & 15u) != 0)
      return fail(PTK_EINVAL, "ptk_peer_reduce_scatter_f32: shards must be 16-byte aligned");
  }
  if ((reinterpret_cast<uintptr_t>(out) & 15u) != 0)
    return fail(PTK_EINVAL, "ptk_peer_reduce_scatter_f32: out must be 16-byte aligned");
  cudaStream_t st = as_stream(stream);
  int grid = 1;
  switch (world) {
#define PTK_RS_CASE(W)                                                             \
  case W:                                                                          \
    grid = grid_for(peer_reduce_f32_kernel<W>,                                     \
                    (shard / 8 + peer_reduce_units<W>() - 1) / peer_reduce_units<W>()); \
    peer_reduce_f32_kernel<W><<<grid, kThreads, 0, st>>>(p, shard, out);           \
    break;
    PTK_RS_CASE(1) PTK_RS_CASE(2) PTK_RS_CASE(3) PTK_RS_CASE(4)
    PTK_RS_CASE(5) PTK_RS_CASE(6) PTK_RS_CASE(7) PTK_RS_CASE(8)
#undef PTK_RS_CASE
    default:
      return fail(PTK_EINVAL, "ptk_peer_reduce_scatter_f32: world > 8");
  }
  launch_counter()++;
  return check_cuda(cudaGetLastError(), "peer_reduce_f32_kernel launch");
}

// Side streams of the peer all-gather: the W-1 pulls run as concurrent
// copy-engine transfers (one stream per pull, forked from and joined back into
// the caller's stream by events), created once per device.
struct PullStreams {
  std::mutex mu;
  cudaStream_t s[PTK_MAX_PEERS] = {};
  cudaEvent_t fork = nullptr, join[PTK_MAX_PEERS] = {};
  bool ready = false;
};

PullStreams& pull_streams() {
  static PullStreams per_dev[kMaxDevices];
  return per_dev[current_device()];
}

int ptk_peer_allgather(void* const* buf_peers, int32_t world, int32_t rank, int64_t shard_bytes,
                       void* stream) {
  if (!buf_peers || world < 1 || world > PTK_MAX_PEERS || rank < 0 || rank >= world ||
      shard_bytes < 0)
    return fail(PTK_EINVAL, "ptk_peer_allgather: bad arguments");
  char* local = static_cast<char*>(buf_peers[rank]);
  if (!local) return fail(PTK_EINVAL, "ptk_peer_allgather: null local buffer");
  for (int q = 0; q < world; ++q)
    if (!buf_peers[q]) return fail(PTK_EINVAL, "ptk_peer_allgather: null peer buffer");
  if (world == 1 || shard_bytes == 0) return PTK_OK;
  cudaStream_t st = as_stream(stream);
  PullStreams& ps = pull_streams();
  std::lock_guard<std::mutex> lock(ps.mu);
  if (!ps.ready) {
    for (int k = 0; k < PTK_MAX_PEERS; ++k) {
      PTK_TRY_CUDA(cudaStreamCreateWithFlags(&ps.s[k], cudaStreamNonBlocking));
      PTK_TRY_CUDA(cudaEventCreateWithFlags(&ps.join[k], cudaEventDisableTiming));
    }
    PTK_TRY_CUDA(cudaEventCreateWithFlags(&ps.fork, cudaEventDisableTiming));
    ps.ready = true;
  }
  // pull every peer's own shard, starting from the next rank (spreads the
  // W-1 readers of one rank), each on its own copy engine stream; no SMs
  PTK_TRY_CUDA(cudaEventRecord(ps.fork, st));
  for (int k = 1; k < world; ++k) {
    const int q = (rank + k) % world;
    const int64_t off = static_cast<int64_t>(q) * shard_bytes;
    PTK_TRY_CUDA(cudaStreamWaitEvent(ps.s[k], ps.fork, 0));
    PTK_TRY_CUDA(cudaMemcpyAsync(local + off, static_cast<const char*>(buf_peers[q]) + off,
                                 static_cast<size_t>(shard_bytes), cudaMemcpyDeviceToDevice,
                                 ps.s[k]));
    PTK_TRY_CUDA(cudaEventRecord(ps.join[k], ps.s[k]));
    PTK_TRY_CUDA(cudaStreamWaitEvent(st, ps.join[k], 0));
  }
  return PTK_OK;
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
