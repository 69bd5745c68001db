// Fused Helmholtz/Jacobi sweep: 5-point relaxed stencil + per-element delta
// + reduce + loop control, one launch per iteration.
//
// Reference: the block kernel apps/helmholtz.py:85-92 (point form :72-83),
// constants :55-65, delta/sum :98-105; the per-partition reduce in
// _step_block (partition.py:302-316); the host combine partition.py:642-646.
//
// HBM-bound: 12 B/cell (fp32: read u 4 + read f 4 + write u' 4), 24 B/cell
// fp64.  Each thread owns 4 contiguous elements of a row (one float4 / two
// double2 loads)
// and marches down a chunk of rows keeping the up/centre/down rows in
// registers, so every u row is read from DRAM once per chunk (+2 halo rows
// per chunk); horizontal neighbours come from warp shuffles plus one scalar
// load at each warp edge.  Loads for U rows are issued before any of them
// is consumed (memory-level parallelism).  Work is pulled in chunks from an
// atomic counter (balanced tail); each chunk writes its own reduce partial so
// the reduce tree is independent of scheduling.
//
// Exactness: the update is evaluated op by op in the reference's expression
// order with round-to-nearest intrinsics (no FMA contraction, IEEE
// division): keep*c + ((relax*((f + ax*(l+r)) + ay*(u+d))) / b), constants
// rounded to the grid dtype first (numpy NEP 50).  Results are bit-identical
// to the reference block route in fp32 and fp64.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "sk_internal.h"
#include "sk_sweep.cuh"

#ifndef SK_F64_UNROLL
#define SK_F64_UNROLL 1
#endif
#ifndef SK_F32_MINB
#define SK_F32_MINB 5
#endif
#ifndef SK_F64_MINB
#define SK_F64_MINB 8
#endif

namespace sk {

template <typename T>
struct HelmArgs {
  Sweep2D g;
  LoopCtl L;
  T ax, ay, b, keep, relax;
  int fast_div;  // b inside div_b_ok and verified: use div_const for safe numerators
  long long xpitch;  // resident loop: row stride of the edge-row exchange buffer
  // peer transport (sk_run_set_peers): the neighbours' halo rows in their
  // buf0 / buf1, written with this rank's first / last owned row
  T* peer_up[2];
  T* peer_dn[2];
};

__device__ __forceinline__ float rcp_rn(float b) { return __frcp_rn(b); }
__device__ __forceinline__ double rcp_rn(double b) { return __drcp_rn(b); }

template <typename T, int BLOCK, int U, int DELTA, int REDUCE, bool PERSIST, bool PEER = false>
__global__ void __launch_bounds__(BLOCK, (sizeof(T) == 8 ? (PERSIST ? 4 : SK_F64_MINB) : SK_F32_MINB))
    helmholtz_sweep(const __grid_constant__ HelmArgs<T> a) {
  constexpr int VEC = 4;
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ double sh[BLOCK / 32];
  __shared__ int s_chunk;

  const Sweep2D& g = a.g;
  long long it = loop_enter(a.L);
  if (it == 0) return;
  for (;;) {
  const T* front;
  long long fp;
  if (it == 1) {
    front = static_cast<const T*>(g.src);
    fp = g.src_pitch;
  } else {
    front = static_cast<const T*>(g.buf[(it - 1) & 1]);
    fp = g.pitch;
  }
  T* back = static_cast<T*>(g.buf[it & 1]) + (long long)g.halo_top * g.pitch;
  front += (long long)g.halo_top * fp;
  const T* env = static_cast<const T*>(g.env) + (long long)g.halo_top * g.env_pitch;
  const int lane = threadIdx.x & 31;
  const int cols = g.cols, rows = g.rows;
  // PEER (peer transport on): the neighbours' halo rows for this iteration
  T* const peer_up = PEER ? a.peer_up[it & 1] : nullptr;
  T* const peer_dn = PEER ? a.peer_dn[it & 1] : nullptr;
  const T ax = a.ax, ay = a.ay, b = a.b, keep = a.keep, relax = a.relax;
  const T rb = rcp_rn(b);
  const bool fast = a.fast_div != 0;
  const int total = a.L.part_chunk[a.L.nparts];

  for (int c = next_chunk(a.L, &s_chunk); c < total; c = next_chunk(a.L, &s_chunk)) {
    int cb, r0, r1;
    chunk_geom(a.L, g, c, &cb, &r0, &r1);
    const int col = cb * (BLOCK * VEC) + (int)threadIdx.x * VEC;
    const int nvalid = cols - col;  // >= VEC: whole vector inside the row
    const bool active = nvalid > 0;
    const bool has_l = (lane == 0) && col > 0 && active;
    const bool has_r = (lane == 31) && nvalid > VEC;
    const bool top_zero = !g.halo_top, bot_zero = !g.halo_bottom;

    auto ldrow = [&](int r) -> Vec4<T> {
      if (!active || (r < 0 && top_zero) || (r >= rows && bot_zero)) return zero4<T>();
      return ldg4(front + (long long)r * fp + col);
    };

    T accm = -INFINITY;  // MAX accumulator (exact in T)
    double accs = 0.0;   // SUM accumulator
    Vec4<T> up = ldrow(r0 - 1);
    Vec4<T> cen = ldrow(r0);
    const T* pc = front + (long long)r0 * fp + col;  // centre row r
    const T* pe = env + (long long)r0 * g.env_pitch + col;
    T* po = back + (long long)r0 * g.pitch + col;
    for (int r = r0; r < r1; r += U) {
      Vec4<T> dn[U], fv[U];
      T ls[U], rs[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int rr = r + u;
        if (rr < r1) {
          dn[u] = ldrow(rr + 1);
          fv[u] = active ? ldg4(pe + u * g.env_pitch) : zero4<T>();
          ls[u] = has_l ? __ldg(pc + u * fp - 1) : T(0);
          rs[u] = has_r ? __ldg(pc + u * fp + VEC) : T(0);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int rr = r + u;
        if (rr < r1) {
          T lv = __shfl_up_sync(FULL, cen.v[VEC - 1], 1);
          T rv = __shfl_down_sync(FULL, cen.v[0], 1);
          if (lane == 0) lv = ls[u];
          if (lane == 31) rv = rs[u];
          T num[VEC];
          bool ok = fast;
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const T l = e == 0 ? lv : cen.v[e - 1];
            T rt = e == VEC - 1 ? rv : cen.v[e + 1];
            if (e + 1 >= nvalid) rt = T(0);  // Dirichlet-0 right border
            // reference order: relax * ((f + ax*(l+r)) + ay*(up+dn))
            const T t3 = xadd(fv[u].v[e], xmul(ax, xadd(l, rt)));
            num[e] = xmul(relax, xadd(t3, xmul(ay, xadd(up.v[e], dn[u].v[e]))));
            ok = ok && div_safe(num[e]);
          }
          T q[VEC];
          if (ok) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) q[e] = div_const(num[e], b, rb);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) q[e] = xdiv(num[e], b);
          }
          Vec4<T> o;
          T dd[VEC];
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const T cc = cen.v[e];
            const T out = xadd(xmul(keep, cc), q[e]);
            const bool in = e < nvalid;
            o.v[e] = in ? out : T(0);  // keep row padding zero
            T d;
            if (DELTA == SK_DELTA_ABS) {
              d = tabs(xsub(out, cc));
            } else if (DELTA == SK_DELTA_SQUARE) {
              const T t = xsub(out, cc);
              d = xmul(t, t);
            } else {
              d = out;
            }
            if (REDUCE == SK_REDUCE_MAX) {
              if (in) accm = max_nan(accm, d);
            } else {
              dd[e] = in ? d : T(0);
            }
          }
          if (REDUCE == SK_REDUCE_SUM) {
            T s4;
            s4 = xadd(xadd(dd[0], dd[1]), xadd(dd[2], dd[3]));
            accs += (double)s4;
          }
          if (active) {
            st4(po, o);
            // boundary rows also land in the neighbours' halo rows (peer
            // stores, overlapped with the rest of the sweep)
            if constexpr (PEER) {
              if (rr == 0 && peer_up) st4(peer_up + col, o);
              if (rr == rows - 1 && peer_dn) st4(peer_dn + col, o);
            }
          }
          up = cen;
          cen = dn[u];
          pc += fp;
          pe += g.env_pitch;
          po += g.pitch;
        }
      }
    }
    const double mine = REDUCE == SK_REDUCE_MAX ? (double)accm : accs;
    const double v = block_reduce<BLOCK>(REDUCE, mine, sh);
    if (threadIdx.x == 0) a.L.partials[c] = v;
  }
  if (!PERSIST) {  // one launch per iteration: no loop back edge at all
    loop_finalize<BLOCK>(a.L, it, sh);
    return;
  }
  it = loop_barrier<BLOCK>(a.L, it, sh);
  if (it == 0) return;
  }  // iterations
}

// ---------------------------------------------------------------- two iterations per pass
// Temporal blocking: one launch computes iterations t and t+1 of the loop
// while every grid element crosses HBM once (read u(t-1), f; write
// u(t+1)) -- u(t) lives only in registers.  A thread keeps, per output row
// r, the window u(t-1) rows r..r+2, u(t) rows r-1..r+1 and f rows r, r+1;
// per row it loads u(t-1) row r+2 and f row r+1, computes u(t) row r+1
// (delta_t accumulated for owned rows), then u(t+1) row r (delta_{t+1}),
// and stores it.  Horizontal neighbours come from warp shuffles; at warp
// edges lanes 0 / 31 also compute u(t) one column beyond the warp (from two
// extra scalar columns of u(t-1)).  Every value is computed with
// helmholtz_sweep's exact expression, so u(t+1), both deltas and both
// chunk partials are bit-identical to two single sweeps (same chunks, same
// accumulation order).  The loop test runs for t, then t+1: if the loop
// stops at t, u(t) is recomputed by one single sweep from u(t-1), which
// this launch did not overwrite (sk_run_loop does that fix-up).
// Buffers: launch L (iterations 2L+1, 2L+2) reads src / buf[(L-1)&1] and
// writes buf[L&1].
template <typename T>
__device__ __forceinline__ T helm_at(const T* p, long long off, bool ok) {
  return ok ? __ldg(p + off) : T(0);
}

template <typename T, int BLOCK, int U, int DELTA, int REDUCE>
__global__ void __launch_bounds__(BLOCK, (sizeof(T) == 8 ? 3 : 4))
    helmholtz_sweep2(const __grid_constant__ HelmArgs<T> a) {
  constexpr int VEC = 4;
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ double sh[BLOCK / 32];
  __shared__ int s_chunk;
  const Sweep2D& g = a.g;
  const long long t = loop_enter(a.L);  // first of the two iterations (odd)
  if (t == 0) return;
  const long long L2 = (t - 1) >> 1;
  const T* front = static_cast<const T*>(L2 == 0 ? g.src : g.buf[(L2 - 1) & 1]);
  const long long fp = L2 == 0 ? g.src_pitch : g.pitch;
  T* back = static_cast<T*>(g.buf[L2 & 1]);
  const T* env = static_cast<const T*>(g.env);
  const long long ep = g.env_pitch;
  const int lane = threadIdx.x & 31;
  const int cols = g.cols, rows = g.rows;
  const T rb = rcp_rn(a.b);
  const bool fast = a.fast_div != 0;
  const int total = a.L.part_chunk[a.L.nparts];
  double* part2 = a.L.partials + total;  // partials of iteration t+1

  for (int c = next_chunk(a.L, &s_chunk); c < total; c = next_chunk(a.L, &s_chunk)) {
    int cb, r0, r1;
    chunk_geom(a.L, g, c, &cb, &r0, &r1);
    const int col = cb * (BLOCK * VEC) + (int)threadIdx.x * VEC;
    const int nvalid = cols - col;
    const bool active = nvalid > 0;
    const bool L0 = lane == 0, L31 = lane == 31;
    const bool okl = L0 && col >= 1 && active, okl2 = L0 && col >= 2 && active;
    const bool okr = L31 && nvalid > VEC, okr2 = L31 && nvalid > VEC + 1;
    const bool el_in = okl, er_in = okr;  // the extra u(t) column lies on the grid

    auto rowok = [&](long long r) { return r >= 0 && r < rows; };
    auto ld4 = [&](const T* base, long long pitch, long long r) -> Vec4<T> {
      return (active && rowok(r)) ? ldg4(base + r * pitch + col) : zero4<T>();
    };
    // one updated value (the reference's expression; see helm_update)
    auto upd = [&](T cc, T l, T rt, T up, T dn, T fv) -> T {
      return helm_update(cc, l, rt, up, dn, fv, a, rb, fast);
    };
    // u at time (level) of a full 4-vector row: centre / up / down rows, the
    // lanes' left / right neighbours (lv for lane 0, rv for lane 31), f row
    auto upd4 = [&](const Vec4<T>& cen, const Vec4<T>& up, const Vec4<T>& dn, T lv_edge,
                    T rv_edge, const Vec4<T>& fv) -> Vec4<T> {
      T lv = __shfl_up_sync(FULL, cen.v[VEC - 1], 1);
      T rv = __shfl_down_sync(FULL, cen.v[0], 1);
      if (L0) lv = lv_edge;
      if (L31) rv = rv_edge;
      Vec4<T> o;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const T l = e == 0 ? lv : cen.v[e - 1];
        T rt = e == VEC - 1 ? rv : cen.v[e + 1];
        if (e + 1 >= nvalid) rt = T(0);
        const T out = upd(cen.v[e], l, rt, up.v[e], dn.v[e], fv.v[e]);
        o.v[e] = e < nvalid ? out : T(0);
      }
      return o;
    };
    T accm1 = -INFINITY, accm2 = -INFINITY;
    double accs1 = 0.0, accs2 = 0.0;
    auto acc_delta = [&](const Vec4<T>& nw, const Vec4<T>& old, T& accm, double& accs) {
      T dd[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        T d;
        if (DELTA == SK_DELTA_ABS) {
          d = tabs(xsub(nw.v[e], old.v[e]));
        } else if (DELTA == SK_DELTA_SQUARE) {
          const T tt = xsub(nw.v[e], old.v[e]);
          d = xmul(tt, tt);
        } else {
          d = nw.v[e];
        }
        const bool in = e < nvalid;
        if (REDUCE == SK_REDUCE_MAX) {
          if (in) accm = max_nan(accm, d);
        } else {
          dd[e] = in ? d : T(0);
        }
      }
      if (REDUCE == SK_REDUCE_SUM) accs += (double)xadd(xadd(dd[0], dd[1]), xadd(dd[2], dd[3]));
    };

    // ---- prologue: u(t-1) rows r0-2 .. r0+1, f rows r0-1, r0; u(t) rows r0-1, r0
    Vec4<T> pm2 = ld4(front, fp, r0 - 2), pm1 = ld4(front, fp, r0 - 1);
    Vec4<T> P1 = ld4(front, fp, r0), P2 = ld4(front, fp, r0 + 1);
    Vec4<T> fm1 = ld4(env, ep, r0 - 1), F1 = ld4(env, ep, r0);
    // edge columns of u(t-1): c-1, c-2 (lane 0), c+4, c+5 (lane 31)
    auto el = [&](long long r, int dc, bool ok) { return helm_at(front, r * fp + col + dc, ok && rowok(r)); };
    auto fe = [&](long long r, int dc, bool ok) { return helm_at(env, r * ep + col + dc, ok && rowok(r)); };
    T lm2 = el(r0 - 2, -1, okl), lm1 = el(r0 - 1, -1, okl), l1 = el(r0, -1, okl), l2 = el(r0 + 1, -1, okl);
    T llm1 = el(r0 - 1, -2, okl2), ll1 = el(r0, -2, okl2);
    T rm2 = el(r0 - 2, VEC, okr), rm1 = el(r0 - 1, VEC, okr), rr1 = el(r0, VEC, okr), rr2 = el(r0 + 1, VEC, okr);
    T rrm1 = el(r0 - 1, VEC + 1, okr2), rrr1 = el(r0, VEC + 1, okr2);
    // u(t) rows r0-1 (halo, not reduced) and r0, own columns + edge columns
    Vec4<T> Q0 = rowok(r0 - 1) ? upd4(pm1, pm2, P1, lm1, rm1, fm1) : zero4<T>();
    T e0l = (el_in && rowok(r0 - 1)) ? upd(lm1, llm1, pm1.v[0], lm2, l1, fe(r0 - 1, -1, okl)) : T(0);
    T e0r = (er_in && rowok(r0 - 1)) ? upd(rm1, pm1.v[VEC - 1], rrm1, rm2, rr1, fe(r0 - 1, VEC, okr)) : T(0);
    Vec4<T> Q1 = upd4(P1, pm1, P2, l1, rr1, F1);
    acc_delta(Q1, P1, accm1, accs1);
    T e1l = el_in ? upd(l1, ll1, P1.v[0], lm1, l2, fe(r0, -1, okl)) : T(0);
    T e1r = er_in ? upd(rr1, P1.v[VEC - 1], rrr1, rm1, rr2, fe(r0, VEC, okr)) : T(0);
    T ll2 = el(r0 + 1, -2, okl2), rrr2 = el(r0 + 1, VEC + 1, okr2);

    T* po = back + (long long)r0 * g.pitch + col;
    for (int r = r0; r < r1; r += U) {
      // prefetch u(t-1) rows r+2.., f rows r+1.. (+ edge columns)
      Vec4<T> pu[U], pfv[U];
      T pl[U], pll[U], pr[U], prr[U], pfl[U], pfr[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (r + u < r1) {
          const long long rr = r + u + 2, rf = r + u + 1;
          pu[u] = ld4(front, fp, rr);
          pfv[u] = ld4(env, ep, rf);
          pl[u] = el(rr, -1, okl);
          pll[u] = el(rr, -2, okl2);
          pr[u] = el(rr, VEC, okr);
          prr[u] = el(rr, VEC + 1, okr2);
          pfl[u] = fe(rf, -1, okl);
          pfr[u] = fe(rf, VEC, okr);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int rw = r + u;
        if (rw < r1) {
          const Vec4<T> P3 = pu[u];
          // u(t) row rw+1 (0 below the grid); reduced when owned
          Vec4<T> Q2;
          T e2l = T(0), e2r = T(0);
          if (rw + 1 < rows) {
            Q2 = upd4(P2, P1, P3, l2, rr2, pfv[u]);
            if (el_in) e2l = upd(l2, ll2, P2.v[0], l1, pl[u], pfl[u]);
            if (er_in) e2r = upd(rr2, P2.v[VEC - 1], rrr2, rr1, pr[u], pfr[u]);
            if (rw + 1 < r1) acc_delta(Q2, P2, accm1, accs1);
          } else {
            Q2 = zero4<T>();
          }
          // u(t+1) row rw
          const Vec4<T> O = upd4(Q1, Q0, Q2, e1l, e1r, F1);
          acc_delta(O, Q1, accm2, accs2);
          if (active) st4(po, O);
          po += g.pitch;
          // rotate the windows
          P1 = P2;
          P2 = P3;
          l1 = l2;
          l2 = pl[u];
          ll2 = pll[u];
          rr1 = rr2;
          rr2 = pr[u];
          rrr2 = prr[u];
          Q0 = Q1;
          Q1 = Q2;
          e1l = e2l;
          e1r = e2r;
          F1 = pfv[u];
        }
      }
    }
    const double mine1 = REDUCE == SK_REDUCE_MAX ? (double)accm1 : accs1;
    const double v1 = block_reduce<BLOCK>(REDUCE, mine1, sh);
    const double mine2 = REDUCE == SK_REDUCE_MAX ? (double)accm2 : accs2;
    const double v2 = block_reduce<BLOCK>(REDUCE, mine2, sh);
    if (threadIdx.x == 0) {
      a.L.partials[c] = v1;
      part2[c] = v2;
    }
  }
  // ---- finish: iteration t, then (unless the loop stops at t) t+1
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&a.L.st->ticket, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  int stop = fold_and_decide<BLOCK>(a.L, t, sh);
  if (stop) {
    if (threadIdx.x == 0) a.L.st->fix = 1;  // the result is u(t): recompute it
  } else {
    LoopCtl L2c = a.L;
    L2c.partials = part2;
    stop = fold_and_decide<BLOCK>(L2c, t + 1, sh);
  }
  if (threadIdx.x == 0) {
    __threadfence_system();
#ifndef __CUDACC_RTC__
    if (a.L.use_graph) cudaGraphSetConditional(a.L.gh, stop ? 0u : 1u);
#endif
  }
}

// ---------------------------------------------------------------- resident loop
// Small grids (BASELINE C1: 1024^2, 36 sweeps) are latency-bound: a sweep
// moves 12.6 MB that sit in L2, so what costs is the per-iteration round
// trip, not bandwidth.  This variant keeps the whole grid ON CHIP for the
// whole loop: one cooperative launch, one CTA per row band (<= RMAX rows x
// the full width; 4 columns per thread), u in registers, f in shared memory.
// Per iteration a CTA reads nothing from memory but its two halo rows (the
// neighbouring bands' edge rows, exchanged through a small global buffer),
// and writes only its two edge rows and its reduce partial; the grid barrier
// that follows also folds the partials and decides the loop (sk_common.cuh).
// The final iteration's values are written to buf[it & 1] once, at the end.
// Bands are the chunks of chunk_geom with one column block, so they never
// span a partition and the reduce tree is the engine's usual one.
// Arithmetic is helmholtz_sweep's, op for op (bit-identical results).
template <typename T>
__device__ __forceinline__ T helm_update(T c, T l, T rt, T up, T dn, T fv, const HelmArgs<T>& a,
                                         T rb, bool fast) {
  const T t3 = xadd(fv, xmul(a.ax, xadd(l, rt)));
  const T num = xmul(a.relax, xadd(t3, xmul(a.ay, xadd(up, dn))));
  T q;
  if (fast && div_safe(num)) {
    q = div_const(num, a.b, rb);
  } else {
    q = xdiv(num, a.b);
  }
  return xadd(xmul(a.keep, c), q);
}

// Grid-wide step of the resident loop: every CTA publishes its partial
// (double-buffered by iteration parity), arrives on a monotonic counter with
// release semantics and waits for all nb arrivals with acquire semantics;
// then EVERY CTA folds the nb partials itself -- per partition in the
// engine's fixed tree, partitions ascending from the identity, as
// fold_and_decide -- and evaluates the loop test on identical data, so all
// reach the same decision without a second round trip.  CTA 0 publishes the
// status for the host at the end.  Returns the stop decision.
template <int BLOCK, bool AMAX, class Pre>
__device__ __forceinline__ int res_step(const LoopCtl& L, long long it, double mine, unsigned* cnt, double* parts,
                        int nb, double* sh, const Pre& prefetch) {
  __shared__ int s_stop;
  const double v = block_reduce<BLOCK>(L.reduce, mine, sh);
  double* slot = parts + (it & 1) * nb;
  // AMAX (one partition, MAX of a non-negative delta): the partials meet in
  // one atomicMax on the value bits (order-free; non-negative doubles and
  // NaN order like their bit patterns), three slots by iteration mod 3
  unsigned long long* amax = reinterpret_cast<unsigned long long*>(parts + 2 * nb);
  if (threadIdx.x == 0) {
    if (AMAX) {
      atomicMax(&amax[it % 3], (unsigned long long)__double_as_longlong(v));
      if (blockIdx.x == 0) amax[(it + 1) % 3] = 0ull;  // next iteration's slot
    } else {
      slot[blockIdx.x] = v;
    }
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    const unsigned want = (unsigned)(nb * it);
    unsigned seen;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
    } while ((int)(seen - want) < 0);
  }
  __syncthreads();
  // every band has published: start the next iteration's halo loads now, so
  // they are in flight while the decision is read and made
  prefetch();
  const OpCombine comb{L.reduce};
  double acc = L.identity;
  if (AMAX) {
    if (threadIdx.x == 0)
      acc = comb.fold(acc, __longlong_as_double((long long)__ldcg(&amax[it % 3])));
  } else {
    const double neutral = comb.neutral(L.identity);
    for (int p = 0; p < L.nparts; ++p) {
      double t = neutral;
      for (int c = L.part_chunk[p] + (int)threadIdx.x; c < L.part_chunk[p + 1]; c += BLOCK)
        t = comb(t, __ldcg(&slot[c]));
      const double pv = block_reduce_c<BLOCK>(comb, neutral, t, sh);
      if (threadIdx.x == 0) acc = comb.fold(acc, pv);
    }
  }

  if (threadIdx.x == 0) {
    const int c = eval_cond(L.cond, acc, it, L.flagged_dev);
    const int capped = it >= L.cond.max_it;
    const int stop = c || capped;
    if (stop && blockIdx.x == 0) {
      Status* st = L.st;
      st->value = acc;
      st->cond_true = c;
      st->exhausted = !c && capped;
      st->iter = it;
      st->stop = 1;
      __threadfence();
    }
    s_stop = stop;
  }
  __syncthreads();
  return s_stop;
}

// VEC contiguous elements per thread for the resident loop (VEC = 4: one
// 16-byte vector for float, two for double; 1 or 2: scalar accesses)
template <typename T, int V>
struct alignas(sizeof(T) * V <= 16 ? sizeof(T) * V : 16) VecN {
  T v[V];
};
template <typename T, int V>
__device__ __forceinline__ VecN<T, V> ldgN(const T* p) {
  VecN<T, V> r;
  if constexpr (V == 4) {
    const Vec4<T> q = ldg4(p);
#pragma unroll
    for (int e = 0; e < 4; ++e) r.v[e] = q.v[e];
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e) r.v[e] = __ldg(p + e);
  }
  return r;
}
template <typename T, int V>
__device__ __forceinline__ void stN(T* p, const VecN<T, V>& x) {
  if constexpr (V == 4) {
    Vec4<T> q;
#pragma unroll
    for (int e = 0; e < 4; ++e) q.v[e] = x.v[e];
    st4(p, q);
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e) p[e] = x.v[e];
  }
}
template <typename T, int V>
__device__ __forceinline__ VecN<T, V> zeroN() {
  VecN<T, V> r;
#pragma unroll
  for (int e = 0; e < V; ++e) r.v[e] = T(0);
  return r;
}
template <typename T, int V>
__device__ __forceinline__ T sumN(const T* d) {  // helmholtz_sweep's order for V = 4
  if constexpr (V == 4) return xadd(xadd(d[0], d[1]), xadd(d[2], d[3]));
  else if constexpr (V == 2) return xadd(d[0], d[1]);
  else return d[0];
}

template <typename T, int BLOCK, int VEC, int RMAX, int DELTA, int REDUCE>
__global__ void __launch_bounds__(BLOCK, 1) helm_resident(const __grid_constant__ HelmArgs<T> a,
                                                          T* xbuf, unsigned* cnt, double* parts) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NW = BLOCK / 32;
  __shared__ double sh[NW];
  __shared__ T s_edge[RMAX][2][NW];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  T* s_f = reinterpret_cast<T*>(s_dyn);  // f of this band, RMAX rows x cols
  const Sweep2D& g = a.g;
  long long it = loop_enter(a.L);
  if (it == 0) return;
  const int cols = g.cols, rows = g.rows;
  int cb, r0, r1;
  chunk_geom(a.L, g, blockIdx.x, &cb, &r0, &r1);
  const int R = r1 - r0;
  const int nb = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = threadIdx.x * VEC;
  const int nvalid = cols - col;
  const bool active = nvalid > 0;
  const T rb = rcp_rn(a.b);
  const bool fast = a.fast_div != 0;
  const bool top_zero = !g.halo_top, bot_zero = !g.halo_bottom;

  // iteration-1 input and f, straight from memory (the only full reads)
  VecN<T, VEC> u[RMAX];
  const T* src = static_cast<const T*>(g.src) + (long long)g.halo_top * g.src_pitch;
  const T* env = static_cast<const T*>(g.env) + (long long)g.halo_top * g.env_pitch;
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    u[r] = (active && r < R) ? ldgN<T, VEC>(src + (long long)(r0 + r) * g.src_pitch + col) : zeroN<T, VEC>();
    if (active && r < R) {
      const VecN<T, VEC> fv = ldgN<T, VEC>(env + (long long)(r0 + r) * g.env_pitch + col);
      // only the row's own columns: s_f rows are `cols` long, so a lane's
      // vector tail past the last column would land on the next row's head
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (e < nvalid) s_f[r * cols + col + e] = fv.v[e];
    }
  }
  VecN<T, VEC> up = (active && !(r0 == 0 && top_zero)) ? ldgN<T, VEC>(src + (long long)(r0 - 1) * g.src_pitch + col)
                                                   : zeroN<T, VEC>();
  VecN<T, VEC> dn = (active && !(r1 == rows && bot_zero)) ? ldgN<T, VEC>(src + (long long)r1 * g.src_pitch + col)
                                                      : zeroN<T, VEC>();
  for (;;) {
    // warp-edge columns for the horizontal neighbours of lanes 0 / 31
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      if (r < R) {
        if (lane == 0) s_edge[r][0][warp] = u[r].v[0];
        if (lane == 31) s_edge[r][1][warp] = u[r].v[VEC - 1];
      }
    }
    __syncthreads();
    T accm = -INFINITY;
    double accs = 0.0;
    // one row's update: centre row r (old values), the rows above / below
    auto update = [&](int r, const VecN<T, VEC>& cen, const VecN<T, VEC>& above,
                      const VecN<T, VEC>& below) {
      T lv = __shfl_up_sync(FULL, cen.v[VEC - 1], 1);
      T rv = __shfl_down_sync(FULL, cen.v[0], 1);
      if (lane == 0) lv = warp > 0 ? s_edge[r][1][warp - 1] : T(0);
      if (lane == 31) rv = warp + 1 < NW ? s_edge[r][0][warp + 1] : T(0);
      VecN<T, VEC> o;
      T dd[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const T l = e == 0 ? lv : cen.v[e - 1];
        T rt = e == VEC - 1 ? rv : cen.v[e + 1];
        if (e + 1 >= nvalid) rt = T(0);  // Dirichlet-0 right border
        const T fv = active && e < nvalid ? s_f[r * cols + col + e] : T(0);
        const T out = helm_update(cen.v[e], l, rt, above.v[e], below.v[e], fv, a, rb, fast);
        const bool in = e < nvalid;
        o.v[e] = in ? out : T(0);
        T d;
        if (DELTA == SK_DELTA_ABS) {
          d = tabs(xsub(out, cen.v[e]));
        } else if (DELTA == SK_DELTA_SQUARE) {
          const T t = xsub(out, cen.v[e]);
          d = xmul(t, t);
        } else {
          d = out;
        }
        if (REDUCE == SK_REDUCE_MAX) {
          if (in) accm = max_nan(accm, d);
        } else {
          dd[e] = in ? d : T(0);
        }
      }
      if (REDUCE == SK_REDUCE_SUM) accs += (double)sumN<T, VEC>(dd);
      return o;
    };
    if constexpr (REDUCE == SK_REDUCE_MAX) {
      // MAX is order-free: rows 1 .. R-1 first (the last one with the halo
      // row below), row 0 (the halo row above) last, so the halo loads
      // issued at the previous grid step have the longest time to land
      const VecN<T, VEC> old0 = u[0];
      const VecN<T, VEC> old1 = R > 1 ? u[RMAX > 1 ? 1 : 0] : dn;
      VecN<T, VEC> prev = old0;  // old value of the row above the current one
#pragma unroll
      for (int r = 1; r < RMAX; ++r) {
        if (r < R) {
          const VecN<T, VEC> cen = u[r];
          const VecN<T, VEC> below = (r + 1 < R) ? u[r + 1 < RMAX ? r + 1 : r] : dn;
          u[r] = update(r, cen, prev, below);
          prev = cen;
        }
      }
      u[0] = update(0, old0, up, old1);
    } else {  // SUM: row order fixed (the partial's summation order)
      VecN<T, VEC> prev = up;
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
        if (r < R) {
          const VecN<T, VEC> cen = u[r];
          const VecN<T, VEC> below = (r + 1 < R) ? u[r + 1 < RMAX ? r + 1 : r] : dn;
          u[r] = update(r, cen, prev, below);
          prev = cen;
        }
      }
    }
    // this band's edge rows for the neighbouring bands (iteration parity slot)
    if (active) {
      T* x = xbuf + ((long long)((it & 1) * nb + blockIdx.x) * 2) * a.xpitch;
      stN<T, VEC>(x + col, u[0]);
#pragma unroll
      for (int r = 0; r < RMAX; ++r)
        if (r == R - 1) stN<T, VEC>(x + a.xpitch + col, u[r]);
    }
    const double mine = REDUCE == SK_REDUCE_MAX ? (double)accm : accs;
    constexpr bool kAmaxOk = REDUCE == SK_REDUCE_MAX && DELTA != SK_DELTA_NONE;
    // halo rows of the next iteration: the neighbours' edge rows (loaded as
    // soon as the grid step shows every band has published them)
    const long long cur = it;
    auto prefetch = [&]() {
      if (!active) return;
      const T* xb = xbuf + (long long)((cur & 1) * nb) * 2 * a.xpitch;
      if (blockIdx.x > 0 && !(r0 == 0)) {
        const T* p = xb + ((long long)(blockIdx.x - 1) * 2 + 1) * a.xpitch + col;
#pragma unroll
        for (int e = 0; e < VEC; ++e) up.v[e] = __ldcg(p + e);
      } else {
        up = zeroN<T, VEC>();
      }
      if (r1 < rows) {
        const T* p = xb + ((long long)(blockIdx.x + 1) * 2) * a.xpitch + col;
#pragma unroll
        for (int e = 0; e < VEC; ++e) dn.v[e] = __ldcg(p + e);
      } else {
        dn = zeroN<T, VEC>();
      }
    };
    const long long nxt =
        ((kAmaxOk && a.L.nparts == 1)
             ? res_step<BLOCK, kAmaxOk>(a.L, it, mine, cnt, parts, nb, sh, prefetch)
             : res_step<BLOCK, false>(a.L, it, mine, cnt, parts, nb, sh, prefetch))
            ? 0 : it + 1;
    if (nxt == 0) {
      // the loop is over: iteration `it` is the result
      if (active) {
        T* out = static_cast<T*>(g.buf[it & 1]) + (long long)g.halo_top * g.pitch;
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
          if (r < R) stN<T, VEC>(out + (long long)(r0 + r) * g.pitch + col, u[r]);
      }
      return;
    }
    it = nxt;
  }
}

// ---- split-phase resident loop (MAX reduces; SK_RES_SPLIT=0 turns it off)
// helm_resident with the grid step split into arrive and wait: after a band
// publishes its edge rows and its partial for iteration t and arrives, it
// computes the INTERIOR rows of t+1 -- they need only its own rows of t --
// while the other bands arrive, then waits, loads the halo rows, decides,
// and finishes t+1 with its first and last rows.  The grid step's latency
// hides behind most of the next iteration's update.  If the loop stops at
// t, the speculative rows are dropped and u(t) is written.  MAX reduces
// only (order-free: the interior rows' deltas fold before the edge rows'),
// every value op for op as helm_resident: bit-identical.
template <int BLOCK, bool AMAX>
__device__ __forceinline__ void res_arrive(const LoopCtl& L, long long it, double mine,
                                           unsigned* cnt, double* parts, int nb, double* sh) {
  const double v = block_reduce<BLOCK>(L.reduce, mine, sh);
  double* slot = parts + (it & 1) * nb;
  unsigned long long* amax = reinterpret_cast<unsigned long long*>(parts + 2 * nb);
  if (threadIdx.x == 0) {
    if (AMAX) {
      atomicMax(&amax[it % 3], (unsigned long long)__double_as_longlong(v));
      if (blockIdx.x == 0) amax[(it + 1) % 3] = 0ull;
    } else {
      slot[blockIdx.x] = v;
    }
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
  }
}

template <int BLOCK, bool AMAX, class Pre>
__device__ __forceinline__ int res_wait(const LoopCtl& L, long long it, unsigned* cnt,
                                        double* parts, int nb, double* sh, const Pre& prefetch) {
  __shared__ int s_stop;
  if (threadIdx.x == 0) {
    const unsigned want = (unsigned)(nb * it);
    unsigned seen;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
    } while ((int)(seen - want) < 0);
  }
  __syncthreads();
  prefetch();
  const OpCombine comb{L.reduce};
  double acc = L.identity;
  double* slot = parts + (it & 1) * nb;
  unsigned long long* amax = reinterpret_cast<unsigned long long*>(parts + 2 * nb);
  if (AMAX) {
    if (threadIdx.x == 0)
      acc = comb.fold(acc, __longlong_as_double((long long)__ldcg(&amax[it % 3])));
  } else {
    const double neutral = comb.neutral(L.identity);
    for (int p = 0; p < L.nparts; ++p) {
      double t = neutral;
      for (int c = L.part_chunk[p] + (int)threadIdx.x; c < L.part_chunk[p + 1]; c += BLOCK)
        t = comb(t, __ldcg(&slot[c]));
      const double pv = block_reduce_c<BLOCK>(comb, neutral, t, sh);
      if (threadIdx.x == 0) acc = comb.fold(acc, pv);
    }
  }
  if (threadIdx.x == 0) {
    const int c = eval_cond(L.cond, acc, it, L.flagged_dev);
    const int capped = it >= L.cond.max_it;
    const int stop = c || capped;
    if (stop && blockIdx.x == 0) {
      Status* st = L.st;
      st->value = acc;
      st->cond_true = c;
      st->exhausted = !c && capped;
      st->iter = it;
      st->stop = 1;
      __threadfence();
    }
    s_stop = stop;
  }
  __syncthreads();
  return s_stop;
}

template <typename T, int BLOCK, int VEC, int RMAX, int DELTA>
__global__ void __launch_bounds__(BLOCK, 1) helm_resident_split(const __grid_constant__ HelmArgs<T> a,
                                                                T* xbuf, unsigned* cnt, double* parts) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NW = BLOCK / 32;
  __shared__ double sh[NW];
  // warp-edge columns, double-buffered by iteration parity: a band's warps
  // read parity t while the fastest may already write parity t+1
  __shared__ T s_edge[2][RMAX][2][NW];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  T* s_f = reinterpret_cast<T*>(s_dyn);  // f of this band, RMAX rows x kFP
  constexpr int kFP = BLOCK * VEC;
  const Sweep2D& g = a.g;
  long long it = loop_enter(a.L);
  if (it == 0) return;
  const int cols = g.cols, rows = g.rows;
  int cb, r0, r1;
  chunk_geom(a.L, g, blockIdx.x, &cb, &r0, &r1);
  const int R = r1 - r0;
  const int nb = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = threadIdx.x * VEC;
  const int nvalid = cols - col;
  const bool active = nvalid > 0;
  const T rb = rcp_rn(a.b);
  const bool fast = a.fast_div != 0;
  const bool top_zero = !g.halo_top, bot_zero = !g.halo_bottom;
  constexpr bool kAmax = DELTA != SK_DELTA_NONE;  // MAX of a non-negative delta

  VecN<T, VEC> u[RMAX], w[RMAX];
  const T* src = static_cast<const T*>(g.src) + (long long)g.halo_top * g.src_pitch;
  const T* env = static_cast<const T*>(g.env) + (long long)g.halo_top * g.env_pitch;
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    u[r] = (active && r < R) ? ldgN<T, VEC>(src + (long long)(r0 + r) * g.src_pitch + col) : zeroN<T, VEC>();
    w[r] = u[r];
    if (r < R) {  // s_f rows are BLOCK*VEC long: every thread owns a whole vector
      VecN<T, VEC> fv = active ? ldgN<T, VEC>(env + (long long)(r0 + r) * g.env_pitch + col) : zeroN<T, VEC>();
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (e >= nvalid) fv.v[e] = T(0);
      *reinterpret_cast<VecN<T, VEC>*>(s_f + r * kFP + col) = fv;
    }
  }
  VecN<T, VEC> up = (active && !(r0 == 0 && top_zero)) ? ldgN<T, VEC>(src + (long long)(r0 - 1) * g.src_pitch + col)
                                                   : zeroN<T, VEC>();
  VecN<T, VEC> dn = (active && !(r1 == rows && bot_zero)) ? ldgN<T, VEC>(src + (long long)r1 * g.src_pitch + col)
                                                      : zeroN<T, VEC>();
  T accm = -INFINITY;
  int sp = (int)((it - 1) & 1);  // s_edge slot of the state being updated: u(t) -> t & 1
  // one row's update, the VEC elements as one vector: a single exact-division
  // check per row (helmholtz_sweep's form; bit-identical), f as one shared
  // vector load, the run constants in registers
  const T ax = a.ax, ay = a.ay, bb = a.b, keep = a.keep, relax = a.relax;
  const bool has_lw = warp > 0, has_rw = warp + 1 < NW;
  auto update = [&](int r, const VecN<T, VEC>& cen, const VecN<T, VEC>& above,
                    const VecN<T, VEC>& below) {
    T lv = __shfl_up_sync(FULL, cen.v[VEC - 1], 1);
    T rv = __shfl_down_sync(FULL, cen.v[0], 1);
    if (lane == 0) lv = has_lw ? s_edge[sp][r][1][warp - 1] : T(0);
    if (lane == 31) rv = has_rw ? s_edge[sp][r][0][warp + 1] : T(0);
    const VecN<T, VEC> fv = *reinterpret_cast<const VecN<T, VEC>*>(s_f + r * kFP + col);
    T num[VEC];
    bool ok = fast;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const T l = e == 0 ? lv : cen.v[e - 1];
      T rt = e == VEC - 1 ? rv : cen.v[e + 1];
      if (e + 1 >= nvalid) rt = T(0);
      const T t3 = xadd(fv.v[e], xmul(ax, xadd(l, rt)));
      num[e] = xmul(relax, xadd(t3, xmul(ay, xadd(above.v[e], below.v[e]))));
      ok = ok && div_safe(num[e]);
    }
    T q[VEC];
    if (ok) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) q[e] = div_const(num[e], bb, rb);
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) q[e] = xdiv(num[e], bb);
    }
    VecN<T, VEC> o;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const T out = xadd(xmul(keep, cen.v[e]), q[e]);
      const bool in = e < nvalid;
      o.v[e] = in ? out : T(0);
      T d;
      if (DELTA == SK_DELTA_ABS) {
        d = tabs(xsub(out, cen.v[e]));
      } else if (DELTA == SK_DELTA_SQUARE) {
        const T t = xsub(out, cen.v[e]);
        d = xmul(t, t);
      } else {
        d = out;
      }
      if (in) accm = max_nan(accm, d);
    }
    return o;
  };
  auto sedge = [&]() {  // warp-edge columns of u for the horizontal neighbours
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      if (r < R) {
        if (lane == 0) s_edge[sp][r][0][warp] = u[r].v[0];
        if (lane == 31) s_edge[sp][r][1][warp] = u[r].v[VEC - 1];
      }
    }
  };
  // interior rows 1 .. R-2 of the next iteration into w (own rows only)
  auto interior = [&]() {
#pragma unroll
    for (int r = 1; r < RMAX - 1; ++r)
      if (r < R - 1) w[r] = update(r, u[r], u[r - 1], u[r + 1]);
  };
  // first and last rows (the halo rows up / dn), then w becomes u
  auto edges = [&]() {
    w[0] = update(0, u[0], up, R > 1 ? u[RMAX > 1 ? 1 : 0] : dn);
#pragma unroll
    for (int r = 1; r < RMAX; ++r)
      if (r == R - 1) w[r] = update(r, u[r], u[r - 1], dn);
#pragma unroll
    for (int r = 0; r < RMAX; ++r) u[r] = w[r];
  };
  // iteration `it` (normally 1) in full
  sedge();
  __syncthreads();
  interior();
  edges();
  for (;;) {
    sp = (int)(it & 1);  // u holds u(it)
    if (active) {  // this band's edge rows of `it` for the neighbours
      T* x = xbuf + ((long long)((it & 1) * nb + blockIdx.x) * 2) * a.xpitch;
      stN<T, VEC>(x + col, u[0]);
#pragma unroll
      for (int r = 0; r < RMAX; ++r)
        if (r == R - 1) stN<T, VEC>(x + a.xpitch + col, u[r]);
    }
    sedge();  // made visible by the block reduce's barriers
    const bool amax = kAmax && a.L.nparts == 1;
    if (amax) res_arrive<BLOCK, true>(a.L, it, (double)accm, cnt, parts, nb, sh);
    else res_arrive<BLOCK, false>(a.L, it, (double)accm, cnt, parts, nb, sh);
    accm = -INFINITY;
    interior();  // speculative: iteration it+1's own rows, while the grid arrives
    const long long cur = it;
    auto prefetch = [&]() {
      if (!active) return;
      const T* xb = xbuf + (long long)((cur & 1) * nb) * 2 * a.xpitch;
      if (blockIdx.x > 0 && !(r0 == 0)) {
        const T* p = xb + ((long long)(blockIdx.x - 1) * 2 + 1) * a.xpitch + col;
#pragma unroll
        for (int e = 0; e < VEC; ++e) up.v[e] = __ldcg(p + e);
      } else {
        up = zeroN<T, VEC>();
      }
      if (r1 < rows) {
        const T* p = xb + ((long long)(blockIdx.x + 1) * 2) * a.xpitch + col;
#pragma unroll
        for (int e = 0; e < VEC; ++e) dn.v[e] = __ldcg(p + e);
      } else {
        dn = zeroN<T, VEC>();
      }
    };
    const int stop = amax ? res_wait<BLOCK, true>(a.L, it, cnt, parts, nb, sh, prefetch)
                          : res_wait<BLOCK, false>(a.L, it, cnt, parts, nb, sh, prefetch);
    if (stop) {  // iteration `it` is the result (the speculative rows are dropped)
      if (active) {
        T* out = static_cast<T*>(g.buf[it & 1]) + (long long)g.halo_top * g.pitch;
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
          if (r < R) stN<T, VEC>(out + (long long)(r0 + r) * g.pitch + col, u[r]);
      }
      return;
    }
    edges();
    ++it;
  }
}

// ---- barrier-free resident loop (fp32, one partition, MAX or SUM of |delta| or delta^2)
// helm_resident_split without the grid barrier.  Every value a band sends
// carries its iteration in the same 8-byte word ("LL" words: tag << 32 |
// fp32 bits), stored with one relaxed 8-byte store and polled with relaxed
// loads until the tag matches -- no fence, no counter, one L2 round trip:
//  * halo rows: the band's first / last row of iteration t go to an
//    exchange slot (t & 1); the neighbours poll them to compute t+1;
//  * reduce partials: the band's MAX of iteration t goes to parts[t % 4][band].
// The loop decision for iteration t is taken while computing t+1 (one
// iteration of lag): warp 0 issues the loads of all partials of t at the
// start of t+1, checks their tags after the update and folds them, and the
// CTA barrier that ends t+1 hands the decision to every warp (spreading
// the fold over warps 0..7 measured slower: 168 vs 154 us per C1 solve --
// eight warps then wait on late partials instead of one; deciding two
// iterations late with u(t-1) kept in registers: 156 vs 154 us).  The neighbours'
// halo words are loaded before the interior update and polled after it.  If the loop
// stops at t, the speculative u(t+1) is dropped and u(t) written.  Safety
// of the reused slots: a band publishes into halo slot t & 1 only after it
// read its neighbours' rows of t-1, which they sent after consuming its rows
// of t-2; partial slot t % 4 is rewritten at t+4, after every band has
// published t+2, i.e. after every band folded t (read at t+1).  Tags are
// run-unique (tag_base advances by max_it + 8 per launch), so no buffer
// needs clearing between launches.  Every value is helm_resident_split's op
// for op and the MAX is order-free (non-negative floats order as their bits,
// NaN above +inf): bit-identical, same iteration count.
__device__ __forceinline__ unsigned long long ll_pack(unsigned tag, float v) {
  return ((unsigned long long)tag << 32) | __float_as_uint(v);
}
__device__ __forceinline__ void ll_st2(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ll_st1(unsigned long long* p, unsigned long long a) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
}
__device__ __forceinline__ unsigned long long ll_ld1(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <int VEC>
__device__ __forceinline__ void ll_store_row(unsigned long long* p, unsigned tag, const VecN<float, VEC>& x) {
  if constexpr (VEC == 1) {
    ll_st1(p, ll_pack(tag, x.v[0]));
  } else {
#pragma unroll
    for (int e = 0; e < VEC; e += 2) ll_st2(p + e, ll_pack(tag, x.v[e]), ll_pack(tag, x.v[e + 1]));
  }
}

// poll until every element of this thread's slice carries `tag`
template <int VEC>
__device__ __forceinline__ VecN<float, VEC> ll_load_row(const unsigned long long* p, unsigned tag) {
  VecN<float, VEC> r;
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    unsigned long long v = ll_ld1(p + e);
    while ((unsigned)(v >> 32) != tag) v = ll_ld1(p + e);
    r.v[e] = __uint_as_float((unsigned)v);
  }
  return r;
}

template <int BLOCK, int VEC, int RMAX, int DELTA, int REDUCE>
__global__ void __launch_bounds__(BLOCK, 1) helm_resident_ll(const __grid_constant__ HelmArgs<float> a,
                                                             unsigned long long* xbuf, unsigned long long* parts,
                                                             unsigned tag_base) {
  using T = float;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NW = BLOCK / 32;
  constexpr int kPS = 4;  // partial slots
  __shared__ T s_edge[2][RMAX][2][NW];
  constexpr bool SUM = REDUCE == SK_REDUCE_SUM;
  __shared__ unsigned s_max[3];
  __shared__ double s_sum[3][NW];  // SUM: the warps' partial sums of t, by t % 3
  __shared__ int s_dec[2];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  T* s_f = reinterpret_cast<T*>(s_dyn);  // f of this band, RMAX rows x kFP
  constexpr int kFP = BLOCK * VEC;
  const Sweep2D& g = a.g;
  long long it = loop_enter(a.L);
  if (it == 0) return;
  const int cols = g.cols, rows = g.rows;
  int cb, r0, r1;
  chunk_geom(a.L, g, blockIdx.x, &cb, &r0, &r1);
  const int R = r1 - r0;
  const int nb = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = threadIdx.x * VEC;
  const int nvalid = cols - col;
  const bool active = nvalid > 0;
  const T rb = rcp_rn(a.b);
  const bool fast = a.fast_div != 0;
  const bool top_zero = !g.halo_top, bot_zero = !g.halo_bottom;
  const bool has_up = !(r0 == 0 && top_zero), has_dn = !(r1 == rows && bot_zero);
  const long long xp = a.xpitch;
  if (threadIdx.x < 3) s_max[threadIdx.x] = 0u;

  // RMAX is the band height: every band but the last has exactly RMAX rows,
  // the last band's rows >= R are held at zero (the Dirichlet rows below
  // the grid), so every row index below is static -- no local-memory arrays
  VecN<T, VEC> u[RMAX], w[RMAX];
  const T* src = static_cast<const T*>(g.src) + (long long)g.halo_top * g.src_pitch;
  const T* env = static_cast<const T*>(g.env) + (long long)g.halo_top * g.env_pitch;
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    u[r] = (active && r < R) ? ldgN<T, VEC>(src + (long long)(r0 + r) * g.src_pitch + col) : zeroN<T, VEC>();
    w[r] = u[r];
    {
      VecN<T, VEC> fv = (active && r < R) ? ldgN<T, VEC>(env + (long long)(r0 + r) * g.env_pitch + col) : zeroN<T, VEC>();
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (e >= nvalid) fv.v[e] = T(0);
      *reinterpret_cast<VecN<T, VEC>*>(s_f + r * kFP + col) = fv;
    }
  }
  VecN<T, VEC> up = (active && has_up) ? ldgN<T, VEC>(src + (long long)(r0 - 1) * g.src_pitch + col) : zeroN<T, VEC>();
  VecN<T, VEC> dn = (active && has_dn) ? ldgN<T, VEC>(src + (long long)r1 * g.src_pitch + col) : zeroN<T, VEC>();
  T accm = -INFINITY;
  double rsum[RMAX];  // SUM: each row's delta sum (added in row order at publish)
#pragma unroll
  for (int r = 0; r < RMAX; ++r) rsum[r] = 0.0;
  int sp = (int)((it - 1) & 1);
  const T ax = a.ax, ay = a.ay, bb = a.b, keep = a.keep, relax = a.relax;
  const bool has_lw = warp > 0, has_rw = warp + 1 < NW;
  auto update = [&](int r, const VecN<T, VEC>& cen, const VecN<T, VEC>& above,
                    const VecN<T, VEC>& below) {
    const bool vr = r < R;  // a real row (else a zero row of the last band)
    T lv = __shfl_up_sync(FULL, cen.v[VEC - 1], 1);
    T rv = __shfl_down_sync(FULL, cen.v[0], 1);
    if (lane == 0) lv = has_lw ? s_edge[sp][r][1][warp - 1] : T(0);
    if (lane == 31) rv = has_rw ? s_edge[sp][r][0][warp + 1] : T(0);
    const VecN<T, VEC> fv = *reinterpret_cast<const VecN<T, VEC>*>(s_f + r * kFP + col);
    T num[VEC];
    bool ok = fast;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const T l = e == 0 ? lv : cen.v[e - 1];
      T rt = e == VEC - 1 ? rv : cen.v[e + 1];
      if (e + 1 >= nvalid) rt = T(0);
      const T t3 = xadd(fv.v[e], xmul(ax, xadd(l, rt)));
      num[e] = xmul(relax, xadd(t3, xmul(ay, xadd(above.v[e], below.v[e]))));
      ok = ok && div_safe(num[e]);
    }
    T q[VEC];
    if (ok) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) q[e] = div_const(num[e], bb, rb);
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) q[e] = xdiv(num[e], bb);
    }
    VecN<T, VEC> o;
    T dd[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const T out = xadd(xmul(keep, cen.v[e]), q[e]);
      const bool in = e < nvalid && vr;
      o.v[e] = in ? out : T(0);
      T d;
      if (DELTA == SK_DELTA_ABS) {
        d = tabs(xsub(out, cen.v[e]));
      } else if (DELTA == SK_DELTA_SQUARE) {
        const T t = xsub(out, cen.v[e]);
        d = xmul(t, t);
      } else {
        d = out;
      }
      if constexpr (SUM) dd[e] = in ? d : T(0);
      else if (in) accm = max_nan(accm, d);
    }
    if constexpr (SUM) rsum[r] = (double)sumN<T, VEC>(dd);  // helm_resident's row term
    return o;
  };
  auto sedge = [&](int slot, const VecN<T, VEC>* x) {
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      if (lane == 0) s_edge[slot][r][0][warp] = x[r].v[0];
      if (lane == 31) s_edge[slot][r][1][warp] = x[r].v[VEC - 1];
    }
  };
  auto interior = [&]() {
#pragma unroll
    for (int r = 1; r < RMAX - 1; ++r) w[r] = update(r, u[r], u[r - 1], u[r + 1]);
  };
  auto edges = [&]() {
    if constexpr (RMAX == 1) {
      w[0] = update(0, u[0], up, dn);
    } else {
      w[0] = update(0, u[0], up, u[1]);
      w[RMAX - 1] = update(RMAX - 1, u[RMAX - 1], u[RMAX - 2], dn);
    }
  };
  // publish w = u(t): halo rows to the exchange slot, warp-edge columns to
  // s_edge, and the warp maxima into s_max[t % 3]
  auto publish = [&](long long t) {
    const unsigned tag = tag_base + (unsigned)t;
    if (active) {
      unsigned long long* x = xbuf + ((long long)((t & 1) * nb + blockIdx.x) * 2) * xp + col;
      ll_store_row<VEC>(x, tag, w[0]);
      // (the last band's row RMAX-1 may be a zero row: nobody reads it)
      ll_store_row<VEC>(x + xp, tag, w[RMAX - 1]);
    }
    sedge((int)(t & 1), w);
    if constexpr (SUM) {
      // block_reduce's order: rows in order per thread, xor tree per warp,
      // warps in order (send_partial)
      double v = 0.0;
#pragma unroll
      for (int r = 0; r < RMAX; ++r)
        if (r < R) v += rsum[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(FULL, v, o);
      if (lane == 0) s_sum[t % 3][warp] = v;
    } else {
      T m = accm;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max_nan(m, __shfl_xor_sync(FULL, m, o));
      // no valid element: -inf -> 0, the identity of a non-negative max
      if (lane == 0 && !(m < T(0))) atomicMax(&s_max[t % 3], __float_as_uint(m));
      accm = -INFINITY;
    }
  };
  // the CTA's partial of t (after the barrier that completed s_max[t % 3])
  auto send_partial = [&](long long t) {
    if (threadIdx.x == 0) {
      const unsigned tg = tag_base + (unsigned)t;
      if constexpr (SUM) {
        double v = 0.0;
        for (int w2 = 0; w2 < NW; ++w2) v = v + s_sum[t % 3][w2];
        const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
        ll_st2(parts + ((long long)(t % kPS) * nb + blockIdx.x) * 2,
               ((unsigned long long)tg << 32) | (bits & 0xffffffffull), ((unsigned long long)tg << 32) | (bits >> 32));
      } else {
        ll_st1(parts + (long long)(t % kPS) * nb + blockIdx.x, ll_pack(tg, __uint_as_float(s_max[t % 3])));
        s_max[(t + 2) % 3] = 0u;  // slot of t+2 (t-1's partial went out last iteration)
      }
    }
  };
  // iteration `it` in full (its halo rows come straight from the input)
  sedge(sp, u);
  __syncthreads();
  interior();
  edges();
  publish(it);
  __syncthreads();
  send_partial(it);
  for (;;) {
    // u <- u(it); compute u(it + 1) while deciding iteration `it`
#pragma unroll
    for (int r = 0; r < RMAX; ++r) u[r] = w[r];
    sp = (int)(it & 1);
    const unsigned tag = tag_base + (unsigned)it;
    // warp 0: the partials of `it` (published one CTA barrier ago by this
    // band, a little earlier or later by the others)
    constexpr int kPL = 5;  // up to 160 bands (one per SM)
    constexpr int kPW = SUM ? 2 : 1;  // tagged words per partial
    unsigned long long pv[kPL][kPW];
    const unsigned long long* ps = parts + (long long)(it % kPS) * nb * kPW;
    if (warp == 0) {
#pragma unroll
      for (int k = 0; k < kPL; ++k) {
        const int c = lane + 32 * k;
#pragma unroll
        for (int q = 0; q < kPW; ++q) pv[k][q] = c < nb ? ll_ld1(ps + (long long)c * kPW + q) : 0ull;
      }
    }
    // the neighbours' rows of `it`: first loads issued before the interior
    // update (usually already tagged `it` when they land), polled after it
    const unsigned long long* xb = xbuf + (long long)((it & 1) * nb) * 2 * xp + col;
    // (only formed for existing neighbours: no pointer past either end)
    const unsigned long long* pu = has_up ? xb + ((long long)(blockIdx.x - 1) * 2 + 1) * xp : xb;
    const unsigned long long* pd = has_dn ? xb + ((long long)(blockIdx.x + 1) * 2) * xp : xb;
    const bool lu = active && has_up, ld = active && has_dn;
    unsigned long long wu[VEC], wd[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      wu[e] = lu ? ll_ld1(pu + e) : 0ull;
      wd[e] = ld ? ll_ld1(pd + e) : 0ull;
    }
    interior();
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      if (lu)
        while ((unsigned)(wu[e] >> 32) != tag) wu[e] = ll_ld1(pu + e);
      if (ld)
        while ((unsigned)(wd[e] >> 32) != tag) wd[e] = ll_ld1(pd + e);
      up.v[e] = lu ? __uint_as_float((unsigned)wu[e]) : T(0);
      dn.v[e] = ld ? __uint_as_float((unsigned)wd[e]) : T(0);
    }
    edges();
    publish(it + 1);
    if (warp == 0) {
#pragma unroll
      for (int k = 0; k < kPL; ++k) {
        const int c = lane + 32 * k;
        if (c < nb) {
#pragma unroll
          for (int q = 0; q < kPW; ++q)
            while ((unsigned)(pv[k][q] >> 32) != tag) pv[k][q] = ll_ld1(ps + (long long)c * kPW + q);
        }
      }
      double acc;
      if constexpr (SUM) {
        // fold_and_decide's tree emulated over the CTA's NW warps: thread
        // c holds 0.0 + partial[c] (or the neutral 0.0), xor tree per warp,
        // warps summed in order, then identity + sum
        double r = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < NW; ++w2) {
          double x = 0.0;
          if (w2 < kPL) {
            const int c = lane + 32 * w2;
            if (c < nb)
              x = 0.0 + __longlong_as_double((long long)(((pv[w2][1] & 0xffffffffull) << 32) |
                                                           (pv[w2][0] & 0xffffffffull)));
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) x = x + __shfl_xor_sync(FULL, x, o);
          r = r + x;
        }
        const OpCombine comb{SK_REDUCE_SUM};
        acc = comb.fold(a.L.identity, r);
      } else {
        unsigned m = 0u;
#pragma unroll
        for (int k = 0; k < kPL; ++k) {
          const int c = lane + 32 * k;
          if (c < nb) {
            const unsigned b = (unsigned)pv[k][0];
            m = b > m ? b : m;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned x = __shfl_xor_sync(FULL, m, o);
          m = x > m ? x : m;
        }
        const OpCombine comb{SK_REDUCE_MAX};
        acc = comb.fold(a.L.identity, (double)__uint_as_float(m));
      }
      if (lane == 0) {
        const int c = eval_cond(a.L.cond, acc, it, a.L.flagged_dev);
        const int capped = it >= a.L.cond.max_it;
        s_dec[it & 1] = c || capped;
        if ((c || capped) && blockIdx.x == 0) {
          Status* st = a.L.st;
          st->value = acc;
          st->cond_true = c;
          st->exhausted = !c && capped;
          st->iter = it;
          st->stop = 1;
          __threadfence();
        }
      }
    }
    __syncthreads();
    if (s_dec[it & 1]) {  // iteration `it` is the result (u(it+1) is dropped)
      if (active) {
        T* out = static_cast<T*>(g.buf[it & 1]) + (long long)g.halo_top * g.pitch;
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
          if (r < R) stN<T, VEC>(out + (long long)(r0 + r) * g.pitch + col, u[r]);
      }
      return;
    }
    send_partial(it + 1);
    ++it;
  }
}

#include "sk_helm_tma.cuh"

// ---------------------------------------------------------------- host side

namespace {

constexpr int kBlock = 128;
// Above this size a sweep is long enough that per-iteration graph launches
// cost nothing; below it the whole loop runs as one persistent launch.
constexpr long long kPersistMaxCells = 1ll << 24;
constexpr int kUnroll = 4;  // rows prefetched per group (fp32)
template <typename T>
constexpr int unroll_for() { return sizeof(T) == 8 ? SK_F64_UNROLL : kUnroll; }

template <typename T>
using KernelFn = void (*)(const HelmArgs<T>);

template <typename T>
KernelFn<T> pick(int delta, int reduce, bool persist = false, bool peer = false) {
#define SK_H(D, R)                                                                            \
  if (delta == D && reduce == R)                                                              \
    return persist ? helmholtz_sweep<T, kBlock, unroll_for<T>(), D, R, true>                  \
                   : peer ? helmholtz_sweep<T, kBlock, unroll_for<T>(), D, R, false, true>    \
                          : helmholtz_sweep<T, kBlock, unroll_for<T>(), D, R, false>;
  SK_H(SK_DELTA_NONE, SK_REDUCE_SUM)
  SK_H(SK_DELTA_NONE, SK_REDUCE_MAX)
  SK_H(SK_DELTA_ABS, SK_REDUCE_SUM)
  SK_H(SK_DELTA_ABS, SK_REDUCE_MAX)
  SK_H(SK_DELTA_SQUARE, SK_REDUCE_SUM)
  SK_H(SK_DELTA_SQUARE, SK_REDUCE_MAX)
#undef SK_H
  return nullptr;
}

template <typename T>
int setup_t(sk_run* r) {
  const sk_plan& p = r->plan;
  constexpr int VEC = 4;
  KernelFn<T> fn = pick<T>(p.delta_op, p.reduce_op);
  if (!fn) {
    set_error("helmholtz: unsupported delta/reduce combination");
    return SK_ERR_UNSUPPORTED;
  }
  const int per_sm = occupancy(reinterpret_cast<const void*>(fn), kBlock);
  const int sms = device_sms(r->device);
  const long long cells = (long long)p.rows * p.cols;
  r->block = kBlock;
  r->colblocks = (int)((p.cols + kBlock * VEC - 1) / (kBlock * VEC));
  // Chunk height: tall enough that the 2 extra halo-row reads per chunk are
  // noise (>= 64 rows when the grid is large), short enough that every SM
  // gets several chunks (dynamic balance) on small grids.
  const long long slots = (long long)sms * per_sm;
  // ~4 chunks per resident CTA; small (L2-resident, latency-bound) grids
  // get short chunks so every SM has several warps in flight.
  long long want_chunks = slots * 4;
  long long ch = (p.rows * (long long)r->colblocks + want_chunks - 1) / want_chunks;
  if (cells >= (1ll << 24)) ch = ch < 64 ? 64 : ch;
  ch = ch < 4 ? 4 : (ch > 256 ? 256 : ch);
  // Large fp64 grids: one row-at-a-time march per thread (U = 1) gives each
  // chunk a long single-row dependency chain, so tall chunks leave a long
  // tail of half-empty SMs at the end of the sweep.  64-row chunks (~14 per
  // CTA at 23168^2) measured 1.91 vs 2.00 ms per sweep against 225-row ones.
  if (sizeof(T) == 8 && cells >= (1ll << 24)) ch = 64;
  if (const char* e = getenv("SK_HELM_CHUNK_ROWS")) {  // A/B knob
    const int v = atoi(e);
    if (v >= 4 && v <= 1024) ch = v;
  }
  r->chunk_rows = (int)ch;
  int nchunks = 0;
  r->part_chunk[0] = 0;
  for (int i = 0; i < r->nparts; ++i) {
    const int pr = r->part_row[i + 1] - r->part_row[i];
    nchunks += ((pr + r->chunk_rows - 1) / r->chunk_rows) * r->colblocks;
    r->part_chunk[i + 1] = nchunks;
  }
  r->nchunks = nchunks;
  r->grid = (int)(slots < nchunks ? slots : nchunks);
  if (r->grid < 1) r->grid = 1;
  // division by the run constant b: 3-op exact path when b is in range and
  // (fp32) verified exhaustively against IEEE division on this device
  const T bt = (T)p.params[2];
  bool fast = div_b_ok((double)bt, sizeof(T) == 4);
  if (fast && sizeof(T) == 4) fast = verify_div_f32((float)bt, r->stream) == 0;
  r->aux_n[0] = fast ? 1 : 0;
  return SK_OK;
}

constexpr int kResRows = 8;  // RMAX: rows per band (registers)

template <typename T>
using ResFn = void (*)(const HelmArgs<T>, T*, unsigned*, double*);

bool res_split() {
  static const bool v = [] {
    const char* e = getenv("SK_RES_SPLIT");
    return !(e && e[0] == '0');
  }();
  return v;
}

template <typename T, int BLOCK, int VEC>
ResFn<T> pick_res_b(int delta, int reduce) {
  // (1024-thread bands would spill the doubled row state at 64 registers)
  if constexpr (BLOCK <= 512) {
    if (reduce == SK_REDUCE_MAX && res_split()) {
      if (delta == SK_DELTA_NONE) return helm_resident_split<T, BLOCK, VEC, kResRows, SK_DELTA_NONE>;
      if (delta == SK_DELTA_ABS) return helm_resident_split<T, BLOCK, VEC, kResRows, SK_DELTA_ABS>;
      if (delta == SK_DELTA_SQUARE)
        return helm_resident_split<T, BLOCK, VEC, kResRows, SK_DELTA_SQUARE>;
    }
  }
#define SK_R(D, R) \
  if (delta == D && reduce == R) return helm_resident<T, BLOCK, VEC, kResRows, D, R>;
  SK_R(SK_DELTA_NONE, SK_REDUCE_SUM)
  SK_R(SK_DELTA_NONE, SK_REDUCE_MAX)
  SK_R(SK_DELTA_ABS, SK_REDUCE_SUM)
  SK_R(SK_DELTA_ABS, SK_REDUCE_MAX)
  SK_R(SK_DELTA_SQUARE, SK_REDUCE_SUM)
  SK_R(SK_DELTA_SQUARE, SK_REDUCE_MAX)
#undef SK_R
  return nullptr;
}

using ResLLFn = void (*)(const HelmArgs<float>, unsigned long long*, unsigned long long*, unsigned);

template <int RMAX>
ResLLFn pick_res_ll(int delta, int reduce) {
  if (reduce == SK_REDUCE_MAX) {  // (MAX of a non-negative delta: partials order as bits)
    if (delta == SK_DELTA_ABS) return helm_resident_ll<512, 2, RMAX, SK_DELTA_ABS, SK_REDUCE_MAX>;
    if (delta == SK_DELTA_SQUARE) return helm_resident_ll<512, 2, RMAX, SK_DELTA_SQUARE, SK_REDUCE_MAX>;
  } else if (reduce == SK_REDUCE_SUM) {
    if (delta == SK_DELTA_ABS) return helm_resident_ll<512, 2, RMAX, SK_DELTA_ABS, SK_REDUCE_SUM>;
    if (delta == SK_DELTA_SQUARE) return helm_resident_ll<512, 2, RMAX, SK_DELTA_SQUARE, SK_REDUCE_SUM>;
  }
  return nullptr;
}

ResLLFn pick_res_ll_band(int band, int delta, int reduce) {
  switch (band) {
    case 1: return pick_res_ll<1>(delta, reduce);
    case 2: return pick_res_ll<2>(delta, reduce);
    case 3: return pick_res_ll<3>(delta, reduce);
    case 4: return pick_res_ll<4>(delta, reduce);
    case 5: return pick_res_ll<5>(delta, reduce);
    case 6: return pick_res_ll<6>(delta, reduce);
    case 7: return pick_res_ll<7>(delta, reduce);
    case 8: return pick_res_ll<8>(delta, reduce);
    default: return nullptr;
  }
}

// helm_resident_ll: same bands as launch_resident; scratch = 4 partial
// slots x bands | halo exchange (2 parities x bands x 2 rows x cols) of
// 8-byte tagged words.  The scratch belongs to the stream, not the run: runs
// on one stream execute in order, so every run on it reuses one buffer that
// is never cleared -- tags are unique over its lifetime (tag_base + it, the
// base advancing by max_it + 8 per launch) -- and a C1 solve costs no
// allocation, memset or occupancy query.
struct LLScratch {
  void* p = nullptr;
  size_t bytes = 0;
  long long epoch = 0;
};

int launch_resident_ll(sk_run* r, const LoopCtl& L, cudaStream_t s, const HelmArgs<float>& base, int block) {
  const sk_plan& p = r->plan;
  if (block != 512) return SK_ERR_UNSUPPORTED;  // (1024 threads would spill)
  const int sms = device_sms(r->device);
  int band = (int)((p.rows + sms - 1) / sms);
  if (band < 1) band = 1;
  ResLLFn fn = pick_res_ll_band(band, p.delta_op, p.reduce_op);
  if (!fn) return SK_ERR_UNSUPPORTED;
  const int nb = (p.rows + band - 1) / band;
  if (nb > 160) return SK_ERR_UNSUPPORTED;  // warp 0 folds <= 5 partials per lane
  const size_t dyn = (size_t)band * block * 2 * sizeof(float);
  static std::mutex mu;
  static std::map<std::pair<const void*, size_t>, int> occ_cache;
  static std::map<std::pair<int, cudaStream_t>, LLScratch> scratch;
  std::lock_guard<std::mutex> lk(mu);
  const auto okey = std::make_pair(reinterpret_cast<const void*>(fn), dyn);
  auto oit = occ_cache.find(okey);
  if (oit == occ_cache.end()) {
    SK_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dyn));
    int occ = 0;
    SK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(fn), block, dyn));
    oit = occ_cache.emplace(okey, occ).first;
  }
  if (oit->second < 1 || nb > oit->second * sms) return SK_ERR_UNSUPPORTED;
  const long long cpad = (p.cols + 3) / 4 * 4;
  const size_t pbytes = (size_t)4 * nb * 16;  // 4 slots x bands x (up to) 2 tagged words
  const size_t bytes = pbytes + (size_t)2 * nb * 2 * cpad * 8;
  const long long span = L.cond.max_it + 8;
  const auto skey = std::make_pair(r->device, s);
  if (scratch.size() >= 32 && scratch.find(skey) == scratch.end()) {
    // many streams seen (e.g. a new stream per call): drop the cache rather
    // than keep a buffer per stream forever (cudaFree waits for the device)
    for (auto& kv : scratch)
      if (kv.second.p) cudaFree(kv.second.p);
    scratch.clear();
  }
  LLScratch& sc = scratch[skey];
  bool clear = false;
  if (!sc.p || sc.bytes < bytes) {
    if (sc.p) SK_CUDA(cudaFreeAsync(sc.p, s));
    sc.p = nullptr;
    SK_CUDA(cudaMallocAsync(&sc.p, bytes, s));
    sc.bytes = bytes;
    clear = true;
  }
  if (sc.epoch < 1 || sc.epoch + span >= (1ll << 32)) clear = true;
  if (clear) {
    SK_CUDA(cudaMemsetAsync(sc.p, 0, sc.bytes, s));
    sc.epoch = 1;
  }
  const unsigned tag_base = (unsigned)sc.epoch;
  sc.epoch += span;
  HelmArgs<float> a = base;
  a.g.colblocks = 1;
  a.g.chunk_rows = band;
  a.xpitch = cpad;
  a.L = L;
  a.L.part_chunk[0] = 0;
  a.L.part_chunk[1] = nb;
  a.L.ring = nullptr;
  unsigned long long* parts = static_cast<unsigned long long*>(sc.p);
  unsigned long long* xbuf = reinterpret_cast<unsigned long long*>(static_cast<char*>(sc.p) + pbytes);
  unsigned tb = tag_base;
  void* params[] = {&a, &xbuf, &parts, &tb};
  SK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), nb, block, params, dyn, s));
  return SK_OK;
}

// Register-resident whole-loop launch (see helm_resident) when the grid fits
// on chip: one band of <= kResRows rows per co-resident CTA, f in shared
// memory.  Returns SK_ERR_UNSUPPORTED (nothing launched) otherwise.
template <typename T>
int launch_resident(sk_run* r, const LoopCtl& L, cudaStream_t s, const HelmArgs<T>& base) {
  const sk_plan& p = r->plan;
  if (p.halo_top || p.halo_bottom) return SK_ERR_UNSUPPORTED;
  const char* off = getenv("SK_NO_RESIDENT");
  if (off && off[0] == '1') return SK_ERR_UNSUPPORTED;
  // two columns per thread: 512 threads up to 1024 columns (C1: 7% faster
  // per iteration than 1024 x 1 -- cheaper block barriers and reduces, the
  // loop is barrier-latency-bound), 1024 threads up to 2048
  int block = p.cols <= 1024 ? 512 : 1024;
  int vec = p.cols <= 2048 ? 2 : 0;
  if (!vec) return SK_ERR_UNSUPPORTED;
  // SK_RES_VEC=1 / 4 for grids up to 1024 columns: 1024 x 1 or 256 x 4
  // threads (measurement knob)
  const char* ev = getenv("SK_RES_VEC");
  const int want = ev ? atoi(ev) : 0;
  if (p.cols <= 1024 && (want == 1 || want == 4)) {
    vec = want;
    block = 1024 / want;
  }
  // barrier-free form (helm_resident_ll): fp32, one partition, MAX or SUM
  // of |delta| or delta^2, 2 columns per thread; SK_RES_LL=0 turns it off
  const char* ll_env = getenv("SK_RES_LL");
  if constexpr (sizeof(T) == 4) {
    if (!(ll_env && ll_env[0] == '0') && vec == 2 && r->nparts == 1 &&
        (p.reduce_op == SK_REDUCE_MAX || p.reduce_op == SK_REDUCE_SUM) &&
        (p.delta_op == SK_DELTA_ABS || p.delta_op == SK_DELTA_SQUARE) && L.cond.max_it < (1ll << 30)) {
      const int rc = launch_resident_ll(r, L, s, base, block);
      if (rc != SK_ERR_UNSUPPORTED) return rc;
    }
  }
  ResFn<T> fn = block == 256   ? pick_res_b<T, 256, 4>(p.delta_op, p.reduce_op)
                : block == 512 ? pick_res_b<T, 512, 2>(p.delta_op, p.reduce_op)
                : vec == 1     ? pick_res_b<T, 1024, 1>(p.delta_op, p.reduce_op)
                               : pick_res_b<T, 1024, 2>(p.delta_op, p.reduce_op);
  if (!fn) return SK_ERR_UNSUPPORTED;
  const int sms = device_sms(r->device);
  // band height: the smallest that gives at most one band per SM
  int band = (int)((p.rows + sms - 1) / sms);
  if (band < 1) band = 1;
  if (band > kResRows) return SK_ERR_UNSUPPORTED;
  LoopCtl L2 = L;
  int nb = 0;
  L2.part_chunk[0] = 0;
  for (int i = 0; i < r->nparts; ++i) {
    const int pr = r->part_row[i + 1] - r->part_row[i];
    nb += (pr + band - 1) / band;
    L2.part_chunk[i + 1] = nb;
  }
  // f rows padded to the CTA's width (the split kernel reads whole vectors)
  const size_t dyn = (size_t)band * block * vec * sizeof(T);
  if (dyn > 200 * 1024) return SK_ERR_UNSUPPORTED;
  SK_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  int occ = 0;
  SK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(fn),
                                                        block, dyn));
  if (occ < 1 || nb > occ * sms) return SK_ERR_UNSUPPORTED;
  // scratch: arrival counter | partials (2 x bands) | edge-row exchange
  // buffer (2 iteration parities x bands x 2 rows x cols)
  const size_t pbytes = (16 + (size_t)(2 * nb + 3) * sizeof(double) + 255) / 256 * 256;
  const long long cpad = (p.cols + 3) / 4 * 4;  // aligned rows
  const size_t xbytes = pbytes + (size_t)2 * nb * 2 * cpad * sizeof(T);
  if (!r->aux[7] || (size_t)r->aux_n[7] < xbytes) {
    if (r->aux[7]) SK_CUDA(cudaFreeAsync(r->aux[7], s));
    SK_CUDA(cudaMallocAsync(&r->aux[7], xbytes, s));
    r->aux_n[7] = (long long)xbytes;
  }
  SK_CUDA(cudaMemsetAsync(r->aux[7], 0, pbytes, s));
  HelmArgs<T> a = base;
  a.g.colblocks = 1;
  a.g.chunk_rows = band;
  a.xpitch = cpad;
  a.L = L2;
  a.L.ring = nullptr;
  unsigned* cnt = static_cast<unsigned*>(r->aux[7]);
  double* parts = reinterpret_cast<double*>(static_cast<char*>(r->aux[7]) + 16);
  T* xbuf = reinterpret_cast<T*>(static_cast<char*>(r->aux[7]) + pbytes);
  void* params[] = {&a, &xbuf, &cnt, &parts};
  SK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), nb, block, params, dyn, s));
  return SK_OK;
}

template <typename T>
using Kernel2Fn = void (*)(const HelmArgs<T>);

template <typename T>
Kernel2Fn<T> pick2(int delta, int reduce) {
#define SK_H2(D, R) \
  if (delta == D && reduce == R) return helmholtz_sweep2<T, kBlock, (sizeof(T) == 8 ? 2 : 4), D, R>;
  SK_H2(SK_DELTA_NONE, SK_REDUCE_SUM)
  SK_H2(SK_DELTA_NONE, SK_REDUCE_MAX)
  SK_H2(SK_DELTA_ABS, SK_REDUCE_SUM)
  SK_H2(SK_DELTA_ABS, SK_REDUCE_MAX)
  SK_H2(SK_DELTA_SQUARE, SK_REDUCE_SUM)
  SK_H2(SK_DELTA_SQUARE, SK_REDUCE_MAX)
#undef SK_H2
  return nullptr;
}

// Two iterations per launch for device-decided loops over one whole grid,
// opt-in (SK_TWOSTEP=1): measured on B200 at 32768^2 fp32 it is slower --
// 6.2 ms per launch (2 iterations) against 2 x 1.99 ms -- because the exact
// update costs ~25 instructions per cell, so halving the HBM traffic leaves
// the kernel issue- and latency-bound (47% issue-active at 16 warps/SM);
// see DESIGN.md.
bool twostep_ok(const sk_run* r, const LoopCtl& L) {
  const char* on = getenv("SK_TWOSTEP");
  if (!(on && on[0] == '1')) return false;
  return !L.persistent && L.cond.kind != SK_COND_HOST && r->plan.halo_top == 0 &&
         r->plan.halo_bottom == 0 && r->env != nullptr;
}

template <typename T>
HelmArgs<T> helm_args(const sk_run* r, const LoopCtl& L) {
  const sk_plan& p = r->plan;
  HelmArgs<T> a;
  Sweep2D& g = a.g;
  g.src = r->src;
  g.src_pitch = r->src_pitch;
  g.buf[0] = r->buf[0];
  g.buf[1] = r->buf[1];
  g.pitch = r->pitch;
  g.env = r->env;
  g.env_pitch = r->env_pitch;
  g.rows = (int)p.rows;
  g.cols = (int)p.cols;
  g.halo_top = p.halo_top;
  g.halo_bottom = p.halo_bottom;
  g.colblocks = r->colblocks;
  g.chunk_rows = r->chunk_rows;
  for (int i = 0; i <= r->nparts; ++i) g.part_row[i] = r->part_row[i];
  a.L = L;
  // Python-float constants meet the grid dtype: rounded once (NEP 50).
  a.ax = (T)p.params[0];
  a.ay = (T)p.params[1];
  a.b = (T)p.params[2];
  a.keep = (T)p.params[3];
  a.relax = (T)p.params[4];
  a.fast_div = r->aux_n[0] ? 1 : 0;
  a.xpitch = 0;
  for (int j = 0; j < 2; ++j) {
    a.peer_up[j] = r->has_peers ? static_cast<T*>(r->peers.up_rows[j]) : nullptr;
    a.peer_dn[j] = r->has_peers ? static_cast<T*>(r->peers.down_rows[j]) : nullptr;
  }
  return a;
}

// The loop stopped at the first iteration `it` of a two-iteration launch:
// recompute u(it) from u(it-1) (the launch's front, untouched) into the
// launch's back buffer with one single sweep under a scratch status.
template <typename T>
int fixup_t(sk_run* r, long long it, cudaStream_t s) {
  const long long L2 = (it - 1) >> 1;
  if (!r->aux[6]) SK_CUDA(cudaMallocAsync(&r->aux[6], sizeof(Status), s));
  SK_CUDA(cudaMemsetAsync(r->aux[6], 0, sizeof(Status), s));
  LoopCtl L;
  memset(&L, 0, sizeof(L));
  L.st = static_cast<Status*>(r->aux[6]);
  L.partials = r->d_partials;
  L.nparts = r->nparts;
  for (int i = 0; i <= r->nparts; ++i) L.part_chunk[i] = r->part_chunk[i];
  L.reduce = r->plan.reduce_op;
  L.identity = r->plan.identity;
  L.cond.kind = SK_COND_ITER_GE;
  L.cond.n = 1.0;
  L.cond.max_it = 1;
  HelmArgs<T> a = helm_args<T>(r, L);
  a.g.src = L2 == 0 ? r->src : r->buf[(L2 - 1) & 1];
  a.g.src_pitch = L2 == 0 ? r->src_pitch : r->pitch;
  a.g.buf[0] = a.g.buf[1] = r->buf[L2 & 1];
  KernelFn<T> fn = pick<T>(r->plan.delta_op, r->plan.reduce_op, false);
  SK_CUDA(launch_kernel(fn, r->grid, r->block, a, s, false));
  return SK_OK;
}

// ---- TMA row-ring sweep (sk_helm_tma.cuh), opt-in: SK_HELM_TMA=1 for fp64
// grids, =2 for fp32 too.  Measured on B200 (23170^2 fp64, 36 sweeps):
// 2.16-2.17 ms per sweep, level with the register march below (2.16-2.17,
// run to run) -- the ring keeps the bytes in flight, but with 8 consumer
// warps per CTA the dependent fp64 update chain per row bounds the
// consumers (the register march hides it with 32 warps per SM).  Ring
// shapes tried (rows per stage x stages x CTAs per SM, elements per
// thread): 6x2x2 v2 2.16-2.17, 4x3x2 v2 2.26, 4x2x3 v2 2.32, 6x2x2 v4 2.31,
// 2x4x3 v2 2.31, 4x3x2 v4 2.29 ms.  Parity-tested (SK_HELM_TMA=2 runs the
// Helmholtz / production / fuzz / odd-width suites through it).
constexpr int kTmaSR = 6, kTmaStages = 2, kTmaMinB = 2, kTmaVec = 2;

template <typename T>
using TmaFn = void (*)(const helm_tma::Args<T>);

template <typename T>
TmaFn<T> pick_tma(int delta, int reduce) {
#define SK_HT(D, R)                                                                         \
  if (delta == D && reduce == R)                                                            \
    return helm_tma::helm_tma_sweep<T, kTmaSR, kTmaStages, kTmaMinB, kTmaVec, D, R>;
  SK_HT(SK_DELTA_NONE, SK_REDUCE_SUM)
  SK_HT(SK_DELTA_NONE, SK_REDUCE_MAX)
  SK_HT(SK_DELTA_ABS, SK_REDUCE_SUM)
  SK_HT(SK_DELTA_ABS, SK_REDUCE_MAX)
  SK_HT(SK_DELTA_SQUARE, SK_REDUCE_SUM)
  SK_HT(SK_DELTA_SQUARE, SK_REDUCE_MAX)
#undef SK_HT
  return nullptr;
}

template <typename T>
size_t tma_stage_bytes(int sr) {
  const size_t hb = 16 / sizeof(T);
  return 4 * (size_t)sr * helm_tma::HALF * sizeof(T) + 2 * ((sr * hb * sizeof(T) + 127) & ~(size_t)127);
}

int tma_mode() {
  static const int v = [] {
    const char* e = getenv("SK_HELM_TMA");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// the run's tensor maps (host memory in aux[5]; built on first use)
struct HelmMaps {
  CUtensorMap um[3], uh[3], fm;
};

template <typename T>
int launch_tma(sk_run* r, const LoopCtl& L, cudaStream_t s, const HelmArgs<T>& a) {
  const sk_plan& p = r->plan;
  const int mode = tma_mode();
  if (mode == 0 || (sizeof(T) == 4 && mode < 2)) return SK_ERR_UNSUPPORTED;
  const int SR = kTmaSR;
  const size_t esz = sizeof(T);
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (L.persistent || r->has_peers || p.halo_top || p.halo_bottom || !r->env || p.cols < 512 ||
      p.rows < SR || (r->pitch * esz) % 16 || (r->src_pitch * esz) % 16 ||
      (r->env_pitch * esz) % 16 || !al16(r->src) || !al16(r->env) || !al16(r->buf[0]) ||
      !al16(r->buf[1]))
    return SK_ERR_UNSUPPORTED;
  TmaFn<T> fn = pick_tma<T>(p.delta_op, p.reduce_op);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tma_encoder());
  if (!fn || !enc) return SK_ERR_UNSUPPORTED;
  HelmMaps* mp = static_cast<HelmMaps*>(r->aux[5]);
  if (!mp) {
    mp = static_cast<HelmMaps*>(malloc(sizeof(HelmMaps)));
    if (!mp) return SK_ERR_UNSUPPORTED;
    const CUtensorMapDataType dt =
        sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    auto make = [&](CUtensorMap* m, const void* ptr, long long pitch, int boxw) {
      cuuint64_t dims[2] = {(cuuint64_t)p.cols, (cuuint64_t)p.rows};
      cuuint64_t strides[1] = {(cuuint64_t)(pitch * esz)};
      cuuint32_t box[2] = {(cuuint32_t)boxw, (cuuint32_t)SR};
      cuuint32_t estr[2] = {1, 1};
      return enc(m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
             CUDA_SUCCESS;
    };
    const void* us[3] = {r->src, r->buf[0], r->buf[1]};
    const long long ps[3] = {r->src_pitch, r->pitch, r->pitch};
    bool ok = make(&mp->fm, r->env, r->env_pitch, helm_tma::HALF);
    for (int i = 0; i < 3 && ok; ++i)
      ok = make(&mp->um[i], us[i], ps[i], helm_tma::HALF) &&
           make(&mp->uh[i], us[i], ps[i], (int)(16 / sizeof(T)));
    if (!ok) {
      free(mp);
      return SK_ERR_UNSUPPORTED;
    }
    r->aux[5] = mp;
  }
  helm_tma::Args<T> A;
  for (int i = 0; i < 3; ++i) {
    A.um[i] = mp->um[i];
    A.uh[i] = mp->uh[i];
  }
  A.fm = mp->fm;
  A.h = a;
  const size_t smem = 128 + (size_t)kTmaStages * tma_stage_bytes<T>(SR) + 16 * kTmaStages;
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, bool> attr;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(r->device, reinterpret_cast<const void*>(fn));
    if (!attr[key]) {
      SK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr[key] = true;
    }
  }
  int per_sm = 0;
  const int nt = helm_tma::nthreads<kTmaVec>();
  SK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nt, smem));
  if (per_sm < 1) return SK_ERR_UNSUPPORTED;
  const int nch = r->part_chunk[r->nparts];
  int grid = device_sms(r->device) * per_sm;
  if (grid > nch) grid = nch;
  fn<<<grid, nt, smem, s>>>(A);
  SK_CUDA(cudaGetLastError());
  return SK_OK;
}

template <typename T>
int launch_t(sk_run* r, const LoopCtl& L, cudaStream_t s) {
  const sk_plan& p = r->plan;
  HelmArgs<T> a = helm_args<T>(r, L);
  if (r->has_peers && L.persistent) {
    set_error("helmholtz: the peer transport drives one launch per iteration");
    return SK_ERR_UNSUPPORTED;
  }
  if (!r->has_peers && twostep_ok(r, L)) {
    Kernel2Fn<T> fn2 = pick2<T>(p.delta_op, p.reduce_op);
    if (fn2) {
      r->steps_per_launch = 2;
      const int occ2 = occupancy(reinterpret_cast<const void*>(fn2), r->block);
      const int slots = device_sms(r->device) * occ2;
      SK_CUDA(launch_kernel(fn2, r->grid < slots ? r->grid : slots, r->block, a, s, false));
      return SK_OK;
    }
  }
  const bool persist = L.persistent != 0;
  if (persist && (long long)p.rows * p.cols > kPersistMaxCells) {
    set_error("helmholtz: persistent loop reserved for small grids");
    return SK_ERR_UNSUPPORTED;  // caller falls back to the graph loop
  }
  if (persist) {
    const int rc = launch_resident<T>(r, L, s, a);
    if (rc == SK_OK) return SK_OK;
    if (rc != SK_ERR_UNSUPPORTED) return rc;
  }
  if (!persist) {
    const int rc = launch_tma<T>(r, L, s, a);
    if (rc == SK_OK) return SK_OK;
    if (rc != SK_ERR_UNSUPPORTED) return rc;
  }
  KernelFn<T> fn = pick<T>(p.delta_op, p.reduce_op, persist, r->has_peers);
  if (persist) {
    // the persistent variant has its own register budget: size the grid to
    // what is co-resident
    const int slots = device_sms(r->device) * occupancy(reinterpret_cast<const void*>(fn), r->block);
    SK_CUDA(launch_kernel(fn, r->grid < slots ? r->grid : slots, r->block, a, s, true));
  } else {
    SK_CUDA(launch_kernel(fn, r->grid, r->block, a, s, false));
  }
  return SK_OK;
}

int setup(sk_run* r) {
  if (r->plan.dtype == SK_F32) return setup_t<float>(r);
  if (r->plan.dtype == SK_F64) return setup_t<double>(r);
  set_error("helmholtz: dtype must be f32 or f64");
  return SK_ERR_UNSUPPORTED;
}

int launch(sk_run* r, const LoopCtl& L, cudaStream_t s) {
  if (r->plan.dtype == SK_F32) return launch_t<float>(r, L, s);
  return launch_t<double>(r, L, s);
}

int fixup(sk_run* r, long long it, cudaStream_t s) {
  if (r->plan.dtype == SK_F32) return fixup_t<float>(r, it, s);
  return fixup_t<double>(r, it, s);
}

void teardown(sk_run* r) {
  if (r->aux[5]) {  // tensor maps (host memory)
    free(r->aux[5]);
    r->aux[5] = nullptr;
  }
  for (int i : {6, 7})  // 6: fix-up status, 7: resident scratch
    if (r->aux[i]) {
      cudaFreeAsync(r->aux[i], r->stream);
      r->aux[i] = nullptr;
    }
}

const KernelOps kOps = {setup, launch, teardown, fixup};

}  // namespace

const KernelOps* helmholtz_ops() { return &kOps; }

}  // namespace sk
