// Helmholtz sweep with the rows streamed into shared memory by the Tensor
// Memory Accelerator (included by sk_helmholtz.cu; uses HelmArgs and the
// sweep's exact arithmetic).
//
// Reference: the block kernel apps/helmholtz.py:85-92, delta/reduce :98-105,
// per-partition reduce partition.py:302-316 -- the arithmetic, chunk
// geometry and reduce tree are helmholtz_sweep's, op for op, so grids,
// deltas and partials are bit-identical to it.  What changes is how the
// bytes arrive: in helmholtz_sweep each thread's register march keeps at
// most one row of loads in flight per warp, which leaves fp64 (24 B/cell)
// latency-bound at ~0.91 of HBM.  Here a producer warp streams each chunk's
// rows (the chunk's column block of 512 elements, rows r0-1 .. r1) with
// cp.async.bulk.tensor into a ring of STAGES stages of SR rows -- u as two
// 256-element boxes plus a 16-byte box either side for the horizontal
// neighbours, f as two boxes -- so the bytes in flight are set by the ring,
// not by registers.  Cells outside the grid arrive zero-filled, which is
// the reference's Dirichlet-0 border.  Four consumer warps (4 elements per
// thread, the sweep's layout) march down the rows from shared memory; each
// input row is read once (its u, f and edge neighbours together), so a
// stage is released as soon as its rows are taken.  Chunks are assigned
// statically (c = CTA, CTA + grid, ...): every chunk still writes its own
// partial, so the reduce tree is the sweep's.  One launch per iteration
// (graph WHILE or batched launches), single-GPU runs.

namespace helm_tma {

constexpr int HALF = 256;  // elements per main box (the TMA box limit)
// consumer warps for VEC elements per thread over a 512-element column block
template <int VEC>
__host__ __device__ constexpr int ncw() { return 2 * HALF / (32 * VEC); }
template <int VEC>
__host__ __device__ constexpr int nthreads() { return (ncw<VEC>() + 1) * 32; }  // + the producer warp

template <typename T>
struct Args {
  CUtensorMap um[3];  // u main boxes {256, SR}: src, buf0, buf1
  CUtensorMap uh[3];  // u halo boxes {16 B, SR}
  CUtensorMap fm;     // f main boxes
  HelmArgs<T> h;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned a, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned parity) {
  unsigned done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive(unsigned a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned a, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_2d(unsigned dst, const CUtensorMap* tm, int x, int y,
                                       unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
// consumer-warp barrier (named barrier 1, the consumer threads)
template <int N>
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory");
}
// VEC elements of a row from shared memory (16-byte vector loads)
template <typename T, int VEC>
__device__ __forceinline__ VecN<T, VEC> lds_vec(unsigned a) {
  VecN<T, VEC> r;
  if constexpr (sizeof(T) == 8) {
#pragma unroll
    for (int v = 0; v < VEC / 2; ++v)
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                   : "=d"(r.v[2 * v]), "=d"(r.v[2 * v + 1]) : "r"(a + 16 * v) : "memory");
  } else if constexpr (VEC == 4) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]) : "r"(a) : "memory");
  } else {
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(r.v[0]), "=f"(r.v[1]) : "r"(a) : "memory");
  }
  return r;
}

// stage layout (bytes): u main half 0 | u main half 1 | f half 0 | f half 1 |
// u halo left | u halo right (halos padded to 128-byte TMA destinations)
template <typename T, int SR>
struct Layout {
  static constexpr int kHB = 16 / (int)sizeof(T);  // halo box width (elements)
  static constexpr unsigned kMain = SR * HALF * sizeof(T);
  static constexpr unsigned kHalo = (SR * kHB * sizeof(T) + 127u) & ~127u;
  static constexpr unsigned kStage = 4 * kMain + 2 * kHalo;
  static constexpr unsigned kTx = 4 * kMain + 2 * SR * kHB * sizeof(T);  // TMA bytes per stage
};

template <typename T, int SR, int STAGES, int MINB, int VEC, int DELTA, int REDUCE>
__global__ void __launch_bounds__(nthreads<VEC>(), MINB)
    helm_tma_sweep(const __grid_constant__ Args<T> A) {
  using LY = Layout<T, SR>;
  constexpr int HB = LY::kHB;
  constexpr int NCW = ncw<VEC>();
  constexpr int NT = nthreads<VEC>();
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(128) unsigned char dyn[];
  __shared__ double sh[NT / 32];
  const HelmArgs<T>& a = A.h;
  const Sweep2D& g = a.g;
  const long long it = loop_enter(a.L);
  if (it == 0) return;

  const unsigned base = (smem_u32(dyn) + 127u) & ~127u;
  const unsigned bars = base + STAGES * LY::kStage;  // full[STAGES], empty[STAGES]
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 8u * (STAGES + s); };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int total = a.L.part_chunk[a.L.nparts];
  const int rows = g.rows, cols = g.cols;
  const int sel = it == 1 ? 0 : 1 + (int)((it - 1) & 1);  // the front's tensor map

  if (warp == NCW) {  // --------------------------------------------- producer
    if (lane == 0) {
      unsigned q = 0;
      for (int c = blockIdx.x; c < total; c += gridDim.x) {
        int cb, r0, r1;
        chunk_geom(a.L, g, c, &cb, &r0, &r1);
        const int c0 = cb * (2 * HALF);
        const int nst = (r1 - r0 + 2 + SR - 1) / SR;
        for (int k = 0; k < nst; ++k, ++q) {
          const int s = (int)(q % STAGES);
          if (q >= (unsigned)STAGES) mbar_wait(empty(s), ((q / STAGES) - 1) & 1);
          const unsigned sb = base + s * LY::kStage;
          const int y = r0 - 1 + SR * k;
          mbar_expect_tx(full(s), LY::kTx);
          tma_2d(sb, &A.um[sel], c0, y, full(s));
          tma_2d(sb + LY::kMain, &A.um[sel], c0 + HALF, y, full(s));
          tma_2d(sb + 2 * LY::kMain, &A.fm, c0, y, full(s));
          tma_2d(sb + 3 * LY::kMain, &A.fm, c0 + HALF, y, full(s));
          tma_2d(sb + 4 * LY::kMain, &A.uh[sel], c0 - HB, y, full(s));
          tma_2d(sb + 4 * LY::kMain + LY::kHalo, &A.uh[sel], c0 + 2 * HALF, y, full(s));
        }
      }
    }
  } else {  // ------------------------------------------------------ consumers
    T* const back = static_cast<T*>(g.buf[it & 1]);
    const T ax = a.ax, ay = a.ay, b = a.b, keep = a.keep, relax = a.relax;
    const T rb = rcp_rn(b);
    const bool fast = a.fast_div != 0;
    const int t = threadIdx.x;          // 0 .. 32 NCW - 1
    const int e0 = t * VEC;             // element offset in the column block
    const int hf = e0 / HALF;           // which main box
    const unsigned eoff = (unsigned)((e0 - hf * HALF) * sizeof(T));
    // the warp-edge neighbours: element 128w - 1 (lane 0) and 128w + 128 (lane 31)
    const int el = warp * 32 * VEC - 1, er = warp * 32 * VEC + 32 * VEC;
    unsigned q = 0;
    for (int c = blockIdx.x; c < total; c += gridDim.x) {
      int cb, r0, r1;
      chunk_geom(a.L, g, c, &cb, &r0, &r1);
      const int col = cb * (2 * HALF) + e0;
      const int nvalid = cols - col;
      const bool active = nvalid > 0;
      const int n_in = r1 - r0 + 2;
      const int nst = (n_in + SR - 1) / SR;
      T accm = -INFINITY;
      double accs = 0.0;
      VecN<T, VEC> up, cen, fc;
      T lc = T(0), rc = T(0);  // centre row's warp-edge neighbours (lanes 0 / 31)
      T* po = back + (long long)r0 * g.pitch + col;
      // take input row i (image row r0 - 1 + i) from stage buffer sb, row j:
      // its u, f and edge neighbours; from i = 2 on, emit output row r0 + i - 2
      auto row = [&](auto hot_t, unsigned sb, int j, int i) {
        constexpr bool HOT = decltype(hot_t)::value;  // i >= 2 for sure
        // take input row i: u, f, and the edge neighbours, all from the stage
        const unsigned ru = sb + hf * LY::kMain + (unsigned)(j * HALF * sizeof(T)) + eoff;
        const VecN<T, VEC> un = lds_vec<T, VEC>(ru);
        const VecN<T, VEC> fn = lds_vec<T, VEC>(ru + 2 * LY::kMain);
        T ln = T(0), rn = T(0);
        if (lane == 0 || lane == 31) {
          unsigned pa;
          if (lane == 0)
            pa = el < 0 ? sb + 4 * LY::kMain + (unsigned)((j * HB + HB - 1) * sizeof(T))
                        : sb + (el / HALF) * LY::kMain +
                              (unsigned)((j * HALF + el % HALF) * sizeof(T));
          else
            pa = er >= 2 * HALF ? sb + 4 * LY::kMain + LY::kHalo + (unsigned)(j * HB * sizeof(T))
                                : sb + (er / HALF) * LY::kMain +
                                      (unsigned)((j * HALF + er % HALF) * sizeof(T));
          T x;
          if constexpr (sizeof(T) == 8)
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(pa) : "memory");
          else
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(pa) : "memory");
          if (lane == 0) ln = x;
          else rn = x;
        }
        if (!HOT && i == 0) {
          up = un;
          return;
        }
        if (!HOT && i == 1) {
          cen = un;
          fc = fn;
          lc = ln;
          rc = rn;
          return;
        }
        // output row r0 + i - 2 from up / cen / dn = un (helmholtz_sweep's arithmetic)
        T lv = __shfl_up_sync(FULL, cen.v[VEC - 1], 1);
        T rv = __shfl_down_sync(FULL, cen.v[0], 1);
        if (lane == 0) lv = lc;
        if (lane == 31) rv = rc;
        T num[VEC];
        bool ok = fast;
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const T l = e == 0 ? lv : cen.v[e - 1];
          T rt = e == VEC - 1 ? rv : cen.v[e + 1];
          if (e + 1 >= nvalid) rt = T(0);  // Dirichlet-0 right border
          const T t3 = xadd(fc.v[e], xmul(ax, xadd(l, rt)));
          num[e] = xmul(relax, xadd(t3, xmul(ay, xadd(up.v[e], un.v[e]))));
          ok = ok && div_safe(num[e]);
        }
        T qv[VEC];
        if (ok) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) qv[e] = div_const(num[e], b, rb);
        } else {
#pragma unroll
          for (int e = 0; e < VEC; ++e) qv[e] = xdiv(num[e], b);
        }
        VecN<T, VEC> o;
        T dd[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const T cc = cen.v[e];
          const T out = xadd(xmul(keep, cc), qv[e]);
          const bool in = e < nvalid;
          o.v[e] = in ? out : T(0);  // keep row padding zero
          T d;
          if (DELTA == SK_DELTA_ABS) {
            d = tabs(xsub(out, cc));
          } else if (DELTA == SK_DELTA_SQUARE) {
            const T tt = xsub(out, cc);
            d = xmul(tt, tt);
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
        if (active) stN<T, VEC>(po, o);
        po += g.pitch;
        up = cen;
        cen = un;
        fc = fn;
        lc = ln;
        rc = rn;
    
      };
      int cs = (int)(q % STAGES);
      unsigned cph = (q / STAGES) & 1;
      for (int k = 0; k < nst; ++k, ++q) {
        mbar_wait(full(cs), cph);
        const unsigned sb = base + cs * LY::kStage;
        if (k > 0 && SR * (k + 1) <= n_in) {
#pragma unroll
          for (int j = 0; j < SR; ++j) row(std::true_type{}, sb, j, SR * k + j);
        } else {
          const int jn = min(SR, n_in - SR * k);
          for (int j = 0; j < jn; ++j) row(std::false_type{}, sb, j, SR * k + j);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty(cs));
        if (++cs == STAGES) {
          cs = 0;
          cph ^= 1u;
        }
      }
      // the chunk's partial: consumer warps only (named barrier)
      double v = REDUCE == SK_REDUCE_MAX ? (double)accm : accs;
      const OpCombine comb{REDUCE};
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = comb(v, __shfl_xor_sync(FULL, v, o));
      if (lane == 0) sh[warp] = v;
      consumers_sync<NCW * 32>();
      if (t == 0) {  // block_reduce's order: from the neutral element, warps ascending
        double r = rneutral(REDUCE);
#pragma unroll
        for (int w = 0; w < NCW; ++w) r = comb(r, sh[w]);
        a.L.partials[c] = r;
      }
      consumers_sync<NCW * 32>();
    }
  }
  loop_finalize<NT>(a.L, it, sh);
}

}  // namespace helm_tma
