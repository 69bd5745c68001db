// Shared device-side pieces of the stencil-reduce engine (sm_100a).
//
// Every sweep kernel in this library has the same epilogue: per-thread
// delta/reduce accumulation -> warp shuffle -> CTA partial -> a
// last-CTA-done "finalize" that folds the CTA partials per partition, folds
// the partitions in ascending order from the combinator identity (the
// reference's host combine, partition.py:642-646), evaluates the loop
// condition on the device (loop.py:209-218) and publishes the value.  That is
// what lets the whole repeat-until loop stay on the GPU (one kernel launch
// per iteration, or one CUDA-graph launch for the whole loop).
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#else
// Compiled by NVRTC as part of a user elemental kernel (sk_jit.cu): no host
// headers.  Device graphs are never used by JIT kernels.
typedef unsigned long long cudaGraphConditionalHandle;
#ifndef INFINITY
#define INFINITY __int_as_float(0x7f800000)
#endif
#endif

#include "../../include/stencilkit_b200.h"

namespace sk {

constexpr int kRing = 64;  // host-visible per-iteration value ring

// Device-resident loop status.  Written only by the finalizing CTA of each
// iteration; read by every CTA of the next launch (kernel boundary orders it).
struct Status {
  long long iter;       // completed iterations
  int stop;             // 1 once the loop is over (cond true or cap hit)
  int exhausted;        // cap hit without cond
  int cond_true;        // the device condition said stop
  int pad;
  double value;         // combined reduce value of iteration `iter` (this run's partitions)
  unsigned int ticket;  // last-CTA-done counter
  unsigned int work;    // dynamic work-chunk counter
  double gvalue;        // value combined across ranks (sk_run_combine), multi-GPU runs
  long long gdecided;   // iterations the cross-rank combine has evaluated
  unsigned int gen;     // grid-barrier generation (persistent loops)
  unsigned int pad3;
  // first elemental failure of the run (JIT kernels): ~((index << 8) | code),
  // 0 = none; atomicMax keeps the lowest row-major index
  unsigned long long err;
  long long err_iter;   // iteration whose fold first saw `err` (0 = none)
  int fix;              // two-iteration launches: the loop stopped at the first
                        // of the pair; its grid must be recomputed (sk_run_loop)
  int pad4;
};

constexpr int kMaxParts = 64;
constexpr int kMaxPeers = 8;  // SK_MAX_PEERS

struct CondDev {
  int kind;             // SK_COND_*
  double a;             // threshold
  double n;             // divisor (RMS/MEAN) or iteration count (ITER_GE)
  long long max_it;
};

// Everything the shared epilogue needs; embedded in each kernel's params.
struct LoopCtl {
  Status* st;
  double* partials;         // one slot per work chunk
  int nparts;
  int part_chunk[kMaxParts + 1];  // chunk ranges per partition (ascending rows)
  const int* part_chunk_dev;      // if set: device-resident chunk ranges (restore)
  const int* flagged_dev;         // if set: the run's flagged count (MEAN_FLAGGED_LT)
  int reduce;               // SK_REDUCE_SUM / SK_REDUCE_MAX
  double identity;
  volatile double* ring;    // host-mapped per-iteration values (may be null)
  CondDev cond;
  cudaGraphConditionalHandle gh;
  int use_graph;
  int persistent;  // whole loop inside one cooperative launch (loop_barrier)
  // multi-GPU peer transport (sk_run_set_peers; world 0 = off): every launch
  // publishes this rank's value into each rank's mailbox, then its sequence
  // number into each rank's flag word
  struct {
    int rank, world;
    unsigned seq;
    double* mail[kMaxPeers];
    unsigned* flag[kMaxPeers];
  } peer;
};

// Publish launch L.peer.seq: value -> mail[p][(seq & 1) * world + rank] for
// every rank p, a system-scope fence (the caller fenced this launch's halo
// rows already), then seq -> flag[p][rank].  One thread.
__device__ __forceinline__ void peer_publish(const LoopCtl& L, double v) {
  const int w = L.peer.world, me = L.peer.rank;
  const unsigned q = L.peer.seq;
  for (int p = 0; p < w; ++p) L.peer.mail[p][(q & 1u) * w + me] = v;
  __threadfence_system();
  for (int p = 0; p < w; ++p) *reinterpret_cast<volatile unsigned*>(L.peer.flag[p] + me) = q;
}

// ---------------------------------------------------------------- exact math
// The reference evaluates numpy/Python expressions op by op: no fused
// multiply-add, IEEE division and sqrt.  These wrappers pin that down
// regardless of -fmad (the library is also built with -fmad=false).
__device__ __forceinline__ float xmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float xadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float xsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float xdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double xsqrt(double a) { return __dsqrt_rn(a); }

// Correctly rounded x / b for a run-constant b, in 3 ops instead of the
// ~10-op IEEE division sequence: q0 = RN(x*r) with r = RN(1/b) is within one
// ulp of x/b, and one FMA residual step then yields RN(x/b) (Markstein's
// theorem; the residual fma(-q0, b, x) is exact).  Valid while nothing
// over/underflows: callers take this path only for 2^-100 <= |x| < 2^100 and
// 2^-60 <= |b| <= 2^60 (checked on the host) and use the IEEE division
// otherwise.  The fp32 form is verified exhaustively on the GPU
// (tests/test_gpu_division.py).
__device__ __forceinline__ float div_const(float x, float b, float r) {
  const float q0 = __fmul_rn(x, r);
  const float e = __fmaf_rn(-q0, b, x);
  return __fmaf_rn(e, r, q0);
}
__device__ __forceinline__ double div_const(double x, double b, double r) {
  const double q0 = __dmul_rn(x, r);
  const double e = __fma_rn(-q0, b, x);
  return __fma_rn(e, r, q0);
}
__device__ __forceinline__ bool div_safe(float x) {
  const float a = fabsf(x);
  return a >= 0x1p-60f && a < 0x1p60f;
}
__device__ __forceinline__ bool div_safe(double x) {
  const double a = fabs(x);
  return a >= 0x1p-500 && a < 0x1p500;
}
#ifndef __CUDACC_RTC__
// host: is b inside the range where div_const is valid for div_safe(x)?
inline bool div_b_ok(double b, bool f32) {
  const double a = b < 0 ? -b : b;
  return f32 ? (a >= 0x1p-30 && a <= 0x1p30) : (a >= 0x1p-200 && a <= 0x1p200);
}
#endif

__device__ __forceinline__ float tabs(float x) { return fabsf(x); }
__device__ __forceinline__ double tabs(double x) { return fabs(x); }

// NaN-propagating max (np.max semantics) in the element type.
__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ double max_nan(double a, double b) {
  return (a != a || b != b) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(a, b);
}

// ---------------------------------------------------------------- reduce ops
// MAX follows np.max: NaN propagates.
__device__ __forceinline__ double rmax(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return b > a ? b : a;
}
__device__ __forceinline__ double rcombine(int op, double a, double b) {
  return op == SK_REDUCE_MAX ? rmax(a, b) : a + b;
}
__device__ __forceinline__ double rneutral(int op) {
  return op == SK_REDUCE_MAX ? -INFINITY : 0.0;
}

template <int BLOCK>
__device__ __forceinline__ double block_reduce(int op, double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = rcombine(op, v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = rneutral(op);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < BLOCK / 32; ++w) r = rcombine(op, r, sh[w]);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

// Device-side loop condition (the recognised threshold forms of the
// reference's conditions; loop.py:43-57, apps/helmholtz.py:128-131,
// apps/denoise.py:282-283, loop.py:70-74).  Same fp64 expression as the
// Python predicate, so the decision is bit-identical.
__device__ __forceinline__ int eval_cond(const CondDev& c, double v, long long it,
                                         const int* flagged = nullptr) {
  switch (c.kind) {
    case SK_COND_MEAN_FLAGGED_LT: {
      const int f = flagged ? *flagged : 0;
      return xdiv(v, (double)(f > 1 ? f : 1)) < c.a;
    }
    case SK_COND_LT: return v < c.a;
    case SK_COND_RMS_LT: return xsqrt(xdiv(v, c.n)) < c.a;
    case SK_COND_MEAN_LT: return xdiv(v, c.n) < c.a;
    case SK_COND_ITER_GE: return (double)it >= c.n;
    default: return 0;  // SK_COND_HOST: the host decides
  }
}

// Loop-entry check shared by all sweep kernels.  Returns the iteration
// number this launch computes, or 0 if the loop is already over (an
// over-launched iteration: every CTA returns without touching memory).
__device__ __forceinline__ long long loop_enter(const LoopCtl& L) {
  volatile Status* st = L.st;
  if (st->stop) {
    // a graph WHILE body entered after the loop ended must still clear the
    // condition, or the graph would spin
#ifndef __CUDACC_RTC__
    if (L.use_graph && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(L.gh, 0u);
#endif
    // launches after the decided stop still publish their sequence number:
    // the peers' stream waits for it
    if (L.peer.world > 1 && blockIdx.x == 0 && threadIdx.x == 0) peer_publish(L, 0.0);
    return 0;
  }
  return st->iter + 1;
}

// Dynamic work distribution: CTAs pull chunk ids until exhausted.  Every
// chunk writes its own partial (partials[chunk]), so the reduce tree depends
// only on the chunk geometry -- never on which CTA ran which chunk.
__device__ __forceinline__ int next_chunk(const LoopCtl& L, int* s_chunk) {
  __syncthreads();
  if (threadIdx.x == 0) *s_chunk = (int)atomicAdd(&L.st->work, 1u);
  __syncthreads();
  return *s_chunk;
}

// The same from a stream's self-resetting counter (stream_counter): each CTA
// fetches exactly once past `total`, so fetch total + gridDim.x - 1 is the
// launch's last use of the counter and puts it back to 0.
__device__ __forceinline__ int next_chunk_stream(unsigned* work, int total, int* s_chunk) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int c = (int)atomicAdd(work, 1u);
    if (c == total + (int)gridDim.x - 1) *work = 0u;
    *s_chunk = c;
  }
  __syncthreads();
  return *s_chunk;
}

// The engine's own reduce ops (SUM / MAX, patterns.py:195-211).  JIT
// kernels pass their user combinator instead (same interface).
struct OpCombine {
  int op;
  __device__ __forceinline__ double operator()(double a, double b) const { return rcombine(op, a, b); }
  // fold of the partition values from the identity (the reference's host
  // combine: `acc + v` / `a if b < a else b`, partition.py:642-646)
  __device__ __forceinline__ double fold(double acc, double v) const {
    return op == SK_REDUCE_SUM ? acc + v : ((v < acc) ? acc : v);
  }
  __device__ __forceinline__ double neutral(double) const { return rneutral(op); }
};

template <int BLOCK, class Comb>
__device__ __forceinline__ double block_reduce_c(const Comb& comb, double neutral, double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = comb(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = neutral;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < BLOCK / 32; ++w) r = comb(r, sh[w]);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

// Fold + decide, run by all threads of the last CTA to finish an iteration:
// chunk partials per partition (fixed strided split + fixed tree), then
// partitions in ascending order from the identity (partition.py:642-646),
// then the loop condition (loop.py:209-218).  Publishes the iteration;
// returns the stop decision (valid in every thread).  A recorded elemental
// failure (Status::err) stops the loop as well.
template <int BLOCK, class Comb>
__device__ __noinline__ int fold_and_decide(const LoopCtl& L, long long it, double* sh, const Comb comb) {
  __shared__ int s_stop;
  double acc = L.identity;
  const double neutral = comb.neutral(L.identity);
  for (int p = 0; p < L.nparts; ++p) {
    const int c0 = L.part_chunk_dev ? L.part_chunk_dev[p] : L.part_chunk[p];
    const int c1 = L.part_chunk_dev ? L.part_chunk_dev[p + 1] : L.part_chunk[p + 1];
    double t = neutral;
    // 8 partials in flight per thread, combined in the same (strided) order
    // as one at a time: a MAX combine's NaN branches otherwise serialise one
    // L2 round trip per partial (~45 us per fold at 16k chunks)
    int c = c0 + (int)threadIdx.x;
    for (; c + 7 * BLOCK < c1; c += 8 * BLOCK) {
      double v8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v8[k] = __ldcg(&L.partials[c + k * BLOCK]);
#pragma unroll
      for (int k = 0; k < 8; ++k) t = comb(t, v8[k]);
    }
    for (; c < c1; c += BLOCK) t = comb(t, __ldcg(&L.partials[c]));
    const double v = block_reduce_c<BLOCK>(comb, neutral, t, sh);
    if (threadIdx.x == 0) acc = comb.fold(acc, v);
  }
  if (threadIdx.x == 0) {
    Status* st = L.st;
    const int failed = *(volatile unsigned long long*)&st->err != 0ull;
    const int c = failed ? 0 : eval_cond(L.cond, acc, it, L.flagged_dev);
    const int capped = (it >= L.cond.max_it);
    st->value = acc;
    st->cond_true = c;
    st->exhausted = (!c && capped && !failed);
    st->stop = c || capped || failed;
    st->iter = it;
    st->ticket = 0;
    st->work = 0;
    if (failed && st->err_iter == 0) st->err_iter = it;
    // a failed iteration publishes NaN: the host then asks sk_run_error
    if (L.ring) L.ring[it % kRing] = failed ? __longlong_as_double(0x7ff8000000000000ll) : acc;
    s_stop = c || capped || failed;
  }
  __syncthreads();
  return s_stop;
}

template <int BLOCK>
__device__ __forceinline__ int fold_and_decide(const LoopCtl& L, long long it, double* sh) {
  return fold_and_decide<BLOCK>(L, it, sh, OpCombine{L.reduce});
}

// OpCombine defaults carry no op: take the run's reduce op from the LoopCtl.
__device__ __forceinline__ OpCombine pick_comb(const LoopCtl& L, const OpCombine&) { return OpCombine{L.reduce}; }
template <class Comb>
__device__ __forceinline__ const Comb& pick_comb(const LoopCtl&, const Comb& c) { return c; }

// End of a launched iteration (one launch per iteration, or a graph WHILE
// body): every CTA arrives; the last one folds, decides and -- in graph
// mode -- clears the WHILE condition.
template <int BLOCK, class Comb = OpCombine>
__device__ void loop_finalize(const LoopCtl& L, long long it, double* sh, const Comb comb = Comb{0}) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    // peer transport: this CTA's halo-row stores to the neighbours must be
    // visible system-wide before the finalizer raises the flags
    if (L.peer.world > 1) __threadfence_system();
    else __threadfence();
    unsigned prev = atomicAdd(&L.st->ticket, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int stop = fold_and_decide<BLOCK>(L, it, sh, pick_comb(L, comb));
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (L.peer.world > 1) peer_publish(L, ((volatile Status*)L.st)->value);
#ifndef __CUDACC_RTC__
    if (L.use_graph) cudaGraphSetConditional(L.gh, stop ? 0u : 1u);
#endif
  }
}

// Persistent mode (one cooperative launch runs the whole loop): a grid
// barrier per iteration whose last arriver folds and decides before it
// releases the others -- one barrier carries both the data dependency (the
// next sweep reads what every CTA just wrote) and the loop test.  The
// gpu-scope fences on both sides also invalidate L1, so the next sweep's
// read-only loads see the fresh buffer.  Returns the next iteration or 0.
template <int BLOCK, class Comb = OpCombine>
__device__ long long loop_barrier(const LoopCtl& L, long long it, double* sh, const Comb comb = Comb{0}) {
  __shared__ int s_last;
  __shared__ unsigned s_gen;
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* genp = &L.st->gen;
    s_gen = *genp;
    __threadfence();
    const unsigned prev = atomicAdd(&L.st->ticket, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    fold_and_decide<BLOCK>(L, it, sh, pick_comb(L, comb));
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&L.st->gen, 1u);  // release
    }
  } else if (threadIdx.x == 0) {
    volatile unsigned* genp = &L.st->gen;
    while (*genp == s_gen) __nanosleep(64);
  }
  __syncthreads();
  __threadfence();
  volatile Status* st = L.st;
  return st->stop ? 0 : it + 1;
}

// Compile-time variant: PERSIST = false lets the compiler drop the
// iteration loop entirely (the one-launch-per-iteration kernels keep their
// register budget).
template <int BLOCK, bool PERSIST>
__device__ __forceinline__ long long loop_next_t(const LoopCtl& L, long long it, double* sh) {
  if (!PERSIST) {
    loop_finalize<BLOCK>(L, it, sh);
    return 0;
  }
  return loop_barrier<BLOCK>(L, it, sh);
}

// Iteration driver used by every sweep kernel:
//   for (long long it = loop_enter(L); it; it = loop_next<BLOCK>(L, it, sh)) { sweep it }
template <int BLOCK>
__device__ __forceinline__ long long loop_next(const LoopCtl& L, long long it, double* sh) {
  if (!L.persistent) {
    loop_finalize<BLOCK>(L, it, sh);
    return 0;
  }
  return loop_barrier<BLOCK>(L, it, sh);
}

}  // namespace sk
