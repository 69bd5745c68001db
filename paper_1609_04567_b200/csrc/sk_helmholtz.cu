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
};

__device__ __forceinline__ float rcp_rn(float b) { return __frcp_rn(b); }
__device__ __forceinline__ double rcp_rn(double b) { return __drcp_rn(b); }

template <typename T, int BLOCK, int U, int DELTA, int REDUCE, bool PERSIST>
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
          if (active) st4(po, o);
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
KernelFn<T> pick(int delta, int reduce, bool persist = false) {
#define SK_H(D, R)                                                                            \
  if (delta == D && reduce == R)                                                              \
    return persist ? helmholtz_sweep<T, kBlock, unroll_for<T>(), D, R, true>                  \
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

template <typename T>
int launch_t(sk_run* r, const LoopCtl& L, cudaStream_t s) {
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
  const bool persist = L.persistent != 0;
  if (persist && (long long)p.rows * p.cols > kPersistMaxCells) {
    set_error("helmholtz: persistent loop reserved for small grids");
    return SK_ERR_UNSUPPORTED;  // caller falls back to the graph loop
  }
  KernelFn<T> fn = pick<T>(p.delta_op, p.reduce_op, persist);
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

void teardown(sk_run*) {}

const KernelOps kOps = {setup, launch, teardown};

}  // namespace

const KernelOps* helmholtz_ops() { return &kOps; }

}  // namespace sk
