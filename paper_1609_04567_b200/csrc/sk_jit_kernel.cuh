// The fused sweep of a user elemental function (NVRTC; see sk_jit_prelude.cuh).
//
// One iteration = the reference's per-partition step (_step_block /
// _step_list_2d, partition.py:273-366): every element's window is presented
// to the elemental function, the result is written to the back buffer, the
// delta against the old value is folded with the combinator, and the
// iteration ends with the shared device-side fold + loop test
// (sk_common.cuh).  Work unit = a tile of SK_TH x SK_TW elements; its input
// window (tile + radius-k frame) is staged once in shared memory with
// coalesced loads, so each element is read from HBM once per sweep however
// wide the stencil.  Tiles never span a partition, and each tile writes its
// own reduce partial (deterministic fold, independent of scheduling).
//
// Required from the generated part: sk_in_t, sk_val_t, sk_delta_t, SK_K,
// SK_PAD_EDGE, SK_PAD_VALUE, sk_elemental_1/_n, sk_delta_1/_n, struct SkComb;
// optional SK_LOCAL_MAX (the combinator is the engine's max: each thread
// keeps its running max in sk_delta_t and converts it once).
#pragma once


#ifndef SK_BLOCK
#define SK_BLOCK 256
#endif
#ifndef SK_MINB
#define SK_MINB 1
#endif
#define SK_TW 128
#ifndef SK_TH
#define SK_TH 16  // rows per tile (jit.py may pick 8 for wide windows)
#endif

namespace sk {

// left/right frame of the staged tile: the radius rounded up to 4 elements,
// so tile rows start on 16-byte boundaries of the grid row (vector staging)
constexpr int kJitKA = (SK_K + 3) / 4 * 4;
constexpr int kJitTWP = SK_TW + 2 * kJitKA;
constexpr int kJitTileElems = (SK_TH + 2 * SK_K) * kJitTWP;
constexpr int kJitElemMax = sizeof(sk_in_t) > sizeof(sk_val_t) ? sizeof(sk_in_t) : sizeof(sk_val_t);

// A thread's running max starts at the type's lowest value and folds every
// element with one NaN-propagating max (max.NaN for float): the same value
// as folding from the first element with jit_lmax, NaN for NaN (the payload
// is not observable), without a per-element first-element flag.
template <class T>
__device__ __forceinline__ T jit_lowest() {
  if constexpr (sizeof(T) == 1) return T(0);  // bool
  else if constexpr (sizeof(T) == 8 && T(0.5) == T(0)) return (T)(-0x7fffffffffffffffll - 1);
  else return (T)(-INFINITY);
}
template <class T>
__device__ __forceinline__ T jit_max_fast(T a, T b) {
  if constexpr (sizeof(T) == 4) return max_nan(a, b);
  else if constexpr (sizeof(T) == 8 && T(0.5) != T(0)) return max_nan(a, b);
  else return b > a ? b : a;
}

template <class T>
__device__ __forceinline__ T jit_lmax(T a, T b) {  // NaN-propagating, as rmax
  return (a != a) ? a : ((b != b) ? b : (b > a ? b : a));
}

__device__ __forceinline__ void jit_fail(Status* st, long long index, int code) {
  atomicMax(&st->err, ~(((unsigned long long)index << 8) | (unsigned)code));
}

// Stage rows [r0 - K, r0 + nr + K) x columns [c0 - KA, c0 + TW + KA) of the
// front into the tile: off-grid slots take the pad value ("constant") or the
// nearest border element ("edge"), like the reference's context assembly
// (partition.py:278-288, 551-581).
// one element global -> shared: 4/8-byte elements with cp.async (no register
// round trip, every load of the tile in flight at once), others by value
template <class V>
__device__ __forceinline__ void stage_one(V* dst, const V* src) {
  if constexpr (sizeof(V) == 4 || sizeof(V) == 8) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(d), "l"(src), "n"((int)sizeof(V)));
  } else {
    *dst = *src;
  }
}

// Local rows [rlo, rhi) are readable: the owned rows plus the halo rows a
// row block carries (multi-rank runs); beyond them is off the global grid.
template <class V>
__device__ __forceinline__ void jit_stage(V* tile, const V* front, long long fp, int r0, int nr,
                                          int c0, int rlo, int rhi, int cols) {
  const int nrow = nr + 2 * SK_K;
  const bool rows_in = r0 - SK_K >= rlo && r0 + nr + SK_K <= rhi;
  const bool cols_in = c0 - kJitKA >= 0 && c0 + SK_TW + kJitKA <= cols;
  const V* p = front + (long long)(r0 - SK_K) * fp + (c0 - kJitKA);
  if constexpr (sizeof(V) == 4 || sizeof(V) == 8) {
    // interior tile on 16-byte aligned rows: 16-byte cp.async vectors
    const bool aligned = ((reinterpret_cast<unsigned long long>(front) | (fp * sizeof(V))) & 15) == 0;
    if (rows_in && cols_in && aligned) {
      constexpr int VE = 16 / sizeof(V);
      constexpr int NV = kJitTWP / VE;  // vectors per tile row
      constexpr int NW = SK_BLOCK / 32;
      // warp w copies rows w, w + NW, ...; its lanes cover the row's NV
      // vectors (no index division; addresses advance by whole rows)
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      const unsigned d0 = (unsigned)__cvta_generic_to_shared(tile + warp * kJitTWP);
      const V* s0 = p + (long long)warp * fp;
      for (int tr = warp; tr < nrow; tr += NW) {
#pragma unroll
        for (int cv = lane; cv < NV; cv += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                           d0 + (unsigned)(((tr - warp) * kJitTWP + cv * VE) * sizeof(V))),
                       "l"(s0 + (long long)(tr - warp) * fp + cv * VE));
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      return;
    }
  }
  const int tx = threadIdx.x % SK_TW, ty = threadIdx.x / SK_TW;
  if (rows_in && cols_in) {  // the whole window frame lies on the grid: plain copies
#pragma unroll 4
    for (int tr = ty; tr < nrow; tr += SK_BLOCK / SK_TW) {
      const V* rp = p + (long long)tr * fp;
      V* tp = tile + tr * kJitTWP;
#pragma unroll
      for (int tc = tx; tc < kJitTWP; tc += SK_TW) stage_one(tp + tc, rp + tc);
    }
  } else {
    for (int tr = ty; tr < nrow; tr += SK_BLOCK / SK_TW) {
      int gi = r0 - SK_K + tr;
      const bool rin = gi >= rlo && gi < rhi;
#if SK_PAD_EDGE
      gi = gi < rlo ? rlo : (gi >= rhi ? rhi - 1 : gi);
#endif
      const V* rp = front + (long long)gi * fp;
      V* tp = tile + tr * kJitTWP;
#pragma unroll
      for (int tc = tx; tc < kJitTWP; tc += SK_TW) {
        int gj = c0 - kJitKA + tc;
#if SK_PAD_EDGE
        gj = gj < 0 ? 0 : (gj >= cols ? cols - 1 : gj);
        stage_one(tp + tc, rp + gj);
#else
        if (rin && (unsigned)gj < (unsigned)cols) stage_one(tp + tc, rp + gj);
        else tp[tc] = (V)(SK_PAD_VALUE);
#endif
      }
    }
  }
  if constexpr (sizeof(V) == 4 || sizeof(V) == 8)
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// cp.async groups one staged tile commits: the grid tile (4 / 8-byte
// elements) and, when staged, env slot 0's tile
template <class V>
constexpr int kStageGroups = (sizeof(V) == 4 || sizeof(V) == 8 ? 1 : 0) + (SK_ENV0_STAGE ? 1 : 0);

// wait until at most `pending` staged tiles are still in flight
template <class V>
__device__ __forceinline__ void stage_wait_upto(int pending) {
  if constexpr (kStageGroups<V> == 2) {
    if (pending) asm volatile("cp.async.wait_group 2;\n" ::: "memory");
    else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  } else if constexpr (kStageGroups<V> == 1) {
    if (pending) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
}

#if SK_ENV0_STAGE
// env slot 0 of tile rows [t0, t0 + nr) x columns [c0, c0 + SK_TW) into a
// SK_TH x SK_TW shared buffer (columns past the grid are not copied: no
// thread reads them); one commit group
__device__ __forceinline__ void env0_stage(sk_env0_t* et, const JitArgs& a, int t0, int nr, int c0) {
  const sk_env0_t* p0 = static_cast<const sk_env0_t*>(a.env.p[0]) + (long long)t0 * a.env.pitch[0] + c0;
  const long long ep = a.env.pitch[0];
  constexpr int VE = 16 / sizeof(sk_env0_t);
  const bool vec = c0 + SK_TW <= a.g.cols &&
                   ((reinterpret_cast<unsigned long long>(a.env.p[0]) | (ep * sizeof(sk_env0_t))) & 15) == 0;
  if (vec) {
    constexpr int NV = SK_TW / VE;
    for (int v = threadIdx.x; v < nr * NV; v += SK_BLOCK) {
      const int r = v / NV, cv = v - r * NV;
      const unsigned d = (unsigned)__cvta_generic_to_shared(et + r * SK_TW + cv * VE);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(p0 + r * ep + cv * VE));
    }
  } else {
    const int cmax = a.g.cols - c0;
    for (int v = threadIdx.x; v < nr * SK_TW; v += SK_BLOCK) {
      const int r = v / SK_TW, c = v - r * SK_TW;
      if (c < cmax) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(et + r * SK_TW + c);
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(d), "l"(p0 + r * ep + c),
                     "n"((int)sizeof(sk_env0_t)));
      }
    }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
#endif

// env grids are read per element straight from global memory: a tile's env
// rows are pulled into L1 before the tile is computed, one prefetch per
// 128-byte line spread over the block (so the elemental's env loads hit
// instead of each waiting a DRAM round trip in turn)
__device__ __forceinline__ void env_prefetch(const JitArgs& a, int t0, int nr, int c0) {
#pragma unroll
  for (int s = 0; s < SK_NENV; ++s) {
    const char* e0 = static_cast<const char*>(sk_env_elem(a.env, s, 0));
    const int esize = (int)(static_cast<const char*>(sk_env_elem(a.env, s, 1)) - e0);
    const int lines = esize * SK_TW / 128;  // 128-byte lines per tile row
    const int cmax = a.g.cols - c0;         // columns of this block inside the grid
    for (int t = threadIdx.x; t < nr * lines; t += SK_BLOCK) {
      const int row = t / lines, ln = t - row * lines;
      if (ln * 128 / esize < cmax)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(
            e0 + ((long long)(t0 + row) * a.env.pitch[0] + c0) * esize + ln * 128));
    }
  }
}

// a thread's running reduce state across tiles
template <bool FIRST>
struct JitAcc {
  double acc;
#ifdef SK_LOCAL_MAX
  sk_delta_t lmax;
  bool lany;
#endif
};

// One tile's rows for this thread: elemental + delta + reduce per element.
// Per-element pointers advance by a fixed stride (no index arithmetic).
template <bool FIRST, class NB, class V>
__device__ __forceinline__ void jit_rows(const JitArgs& a, const V* tile, const sk_env0_t* etile,
                                         sk_val_t* back, int t0, int nr, int gj,
                                         const SkComb& comb, JitAcc<FIRST>& st) {
  constexpr int RS = SK_BLOCK / SK_TW;  // rows between a thread's elements
  const int tx = threadIdx.x % SK_TW, ty = threadIdx.x / SK_TW;
  const Sweep2D& g = a.g;
  const int cols = g.cols;
  NB nb;
  nb.c = tile + (ty + SK_K) * kJitTWP + tx + kJitKA;
  nb.stride = kJitTWP;
  nb.i = t0 + ty + a.env.row0;  // global row
  nb.j = gj;
  nb.rows = a.env.rows;
  nb.cols = cols;
  nb.k = SK_K;
  nb.eidx = (long long)(t0 + ty) * a.env.pitch[0] + gj;  // env element of the centre
  nb.ec = etile + ty * SK_TW + tx;  // (PRE) the staged env slot 0 element
  const long long estep = (long long)RS * a.env.pitch[0];
  sk_val_t* bp = back + (long long)(t0 + ty) * g.pitch + gj;
  const long long bstep = (long long)RS * g.pitch;
#ifdef SK_LOCAL_MAX
  if (ty < nr) st.lany = true;
#endif
  for (int lr = ty; lr < nr; lr += RS) {
    SkErr err;
    sk_val_t nw;
    sk_delta_t d;
    if constexpr (FIRST) {
      nw = sk_elemental_1(nb, a.env, err);
      d = sk_delta_1(nw, nb.center(), err);
    } else {
      nw = sk_elemental_n(nb, a.env, err);
      d = sk_delta_n(nw, nb.center(), err);
    }
    *bp = nw;
    if (err.code) jit_fail(a.L.st, (long long)nb.i * cols + gj, err.code);
#ifdef SK_LOCAL_MAX
    st.lmax = jit_max_fast(st.lmax, d);
#else
    st.acc = comb(st.acc, (double)d);
#endif
    nb.c += RS * kJitTWP;
    nb.i += RS;
    nb.eidx += estep;
    nb.ec += RS * SK_TW;
    bp += bstep;
  }
}

// A work chunk = one column block x chunk_rows rows = a run of SK_TH-row
// tiles.  Tiles are double-buffered: while tile t is computed, tile t+1 is
// already on its way into the other buffer (cp.async), so each CTA keeps
// its loads in flight.  One reduce partial per chunk.
template <class V, bool FIRST>
__device__ __forceinline__ void jit_sweep(const JitArgs& a, long long it, V* tiles, int* s_chunk,
                                          double* sh, const SkComb& comb) {
  const Sweep2D& g = a.g;
  const long long fp = FIRST ? g.src_pitch : g.pitch;
  // owned row 0 of the front / back buffers (row blocks carry halo rows)
  const V* front = static_cast<const V*>(FIRST ? g.src : g.buf[(it - 1) & 1]) +
                   (long long)g.halo_top * fp;
  sk_val_t* back = static_cast<sk_val_t*>(g.buf[it & 1]) + (long long)g.halo_top * g.pitch;
  const int rows = g.rows, cols = g.cols;
  const int rlo = -g.halo_top, rhi = rows + g.halo_bottom;
  const int row0 = a.env.row0, grows = a.env.rows;
  const int tx = threadIdx.x % SK_TW, ty = threadIdx.x / SK_TW;
  const double neutral = comb.neutral(a.L.identity);
  const int total = a.L.part_chunk[a.L.nparts];
  for (int c = next_chunk(a.L, s_chunk); c < total; c = next_chunk(a.L, s_chunk)) {
    int cb, r0, r1;
    chunk_geom(a.L, g, c, &cb, &r0, &r1);
    const int c0 = cb * SK_TW;
    double acc = neutral;
#ifdef SK_LOCAL_MAX
    sk_delta_t lmax = jit_lowest<sk_delta_t>();
    bool lany = false;
#endif
    const int gj = c0 + tx;
    int buf = 0;
    // env slot 0 tiles follow the two grid tile buffers
    sk_env0_t* etiles = reinterpret_cast<sk_env0_t*>(
        reinterpret_cast<unsigned char*>(tiles) + 2 * kJitTileElems * kJitElemMax);
#if SK_ENV0_STAGE
    env0_stage(etiles, a, r0, min(SK_TH, r1 - r0), c0);
#endif
    jit_stage<V>(tiles, front, fp, r0, min(SK_TH, r1 - r0), c0, rlo, rhi, cols);
    for (int t0 = r0; t0 < r1; t0 += SK_TH) {
      const int nr = min(SK_TH, r1 - t0);
      const bool more = t0 + SK_TH < r1;
      if (more) {
#if SK_ENV0_STAGE
        env0_stage(etiles + (buf ^ 1) * SK_TH * SK_TW, a, t0 + SK_TH, min(SK_TH, r1 - t0 - SK_TH), c0);
#endif
        jit_stage<V>(tiles + (buf ^ 1) * kJitTileElems, front, fp, t0 + SK_TH,
                     min(SK_TH, r1 - t0 - SK_TH), c0, rlo, rhi, cols);
      }
#if !SK_ENV0_STAGE
      env_prefetch(a, t0, nr, c0);  // this tile's env rows (not staged)
#endif
      stage_wait_upto<V>(more ? 1 : 0);
      __syncthreads();
      const V* tile = tiles + buf * kJitTileElems;
      const sk_env0_t* etile = etiles + buf * SK_TH * SK_TW;
      if (gj < cols) {
        // NB = SkNb<V, true> when all of this thread's windows in the tile
        // are on the grid: every ABSENT test compiles away
        const int gi0 = t0 + row0;  // global rows of the tile: [gi0, gi0 + nr)
        const bool inner = gi0 >= SK_K && gi0 + nr - 1 + SK_K < grows && gj >= SK_K &&
                           gj + SK_K < cols;
        JitAcc<FIRST> st{acc};
#ifdef SK_LOCAL_MAX
        st.lmax = lmax;
        st.lany = lany;
#endif
        constexpr bool PRE = SK_ENV0_STAGE != 0;
        if (inner)
          jit_rows<FIRST, SkNb<V, true, kJitTWP, sk_env0_t, PRE>>(a, tile, etile, back, t0, nr, gj,
                                                                  comb, st);
        else
          jit_rows<FIRST, SkNb<V, false, kJitTWP, sk_env0_t, PRE>>(a, tile, etile, back, t0, nr,
                                                                   gj, comb, st);
        acc = st.acc;
#ifdef SK_LOCAL_MAX
        lmax = st.lmax;
        lany = st.lany;
#endif
      }
      __syncthreads();  // tile `buf` is free for the tile after next
      buf ^= 1;
    }
#ifdef SK_LOCAL_MAX
    if (lany) acc = comb(acc, (double)lmax);
#endif
    const double v = block_reduce_c<SK_BLOCK>(comb, neutral, acc, sh);
    if (threadIdx.x == 0) a.L.partials[c] = v;
  }
}

#if SK_NDIM == 1
// ---------------------------------------------------------------- rank-1 grids
// A rank-1 grid is contiguous (pitch 1): a tile is SK_TH * SK_TW consecutive
// elements plus the radius on both sides, staged with cp.async; thread t
// computes elements t, t + SK_BLOCK, ... (coalesced).  Same window type,
// interior specialisation, reduce order and error reporting as the 2D sweep.
constexpr int kJit1Elems = SK_TH * SK_TW;
static_assert(kJit1Elems + 2 * kJitKA <= kJitTileElems, "1D tile fits the 2D tile buffer");

template <class V>
__device__ __forceinline__ void jit_stage1(V* tile, const V* front, long long fp, int t0, int ne,
                                           int rlo, int rhi) {
  // tile[kJitKA + e] = element t0 + e, e in [-SK_K, ne + SK_K)
  for (int x = threadIdx.x; x < ne + 2 * SK_K; x += SK_BLOCK) {
    int gi = t0 - SK_K + x;
    V* dst = tile + kJitKA - SK_K + x;
#if SK_PAD_EDGE
    gi = gi < rlo ? rlo : (gi >= rhi ? rhi - 1 : gi);
    stage_one(dst, front + (long long)gi * fp);
#else
    if (gi >= rlo && gi < rhi) stage_one(dst, front + (long long)gi * fp);
    else *dst = (V)(SK_PAD_VALUE);
#endif
  }
  if constexpr (sizeof(V) == 4 || sizeof(V) == 8)
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <bool FIRST, class NB, class V>
__device__ __forceinline__ void jit_elems1(const JitArgs& a, const V* tile, sk_val_t* back, int t0,
                                           int ne, const SkComb& comb, JitAcc<FIRST>& st) {
  const Sweep2D& g = a.g;
  for (int e = threadIdx.x; e < ne; e += SK_BLOCK) {
    NB nb;
    nb.c = tile + kJitKA + e;
    nb.stride = 1;
    nb.i = t0 + e + a.env.row0;  // global index
    nb.j = 0;
    nb.rows = a.env.rows;
    nb.cols = 1;
    nb.k = SK_K;
    nb.eidx = (long long)(t0 + e) * a.env.pitch[0];
    SkErr err;
    sk_val_t nw;
    sk_delta_t d;
    if constexpr (FIRST) {
      nw = sk_elemental_1(nb, a.env, err);
      d = sk_delta_1(nw, nb.center(), err);
    } else {
      nw = sk_elemental_n(nb, a.env, err);
      d = sk_delta_n(nw, nb.center(), err);
    }
    back[(long long)(t0 + e) * g.pitch] = nw;
    if (err.code) jit_fail(a.L.st, (long long)nb.i, err.code);
#ifdef SK_LOCAL_MAX
    st.lmax = st.lany ? jit_lmax(st.lmax, d) : d;
    st.lany = true;
#else
    st.acc = comb(st.acc, (double)d);
#endif
  }
}

template <class V, bool FIRST>
__device__ __forceinline__ void jit_sweep1(const JitArgs& a, long long it, V* tiles, int* s_chunk,
                                           double* sh, const SkComb& comb) {
  const Sweep2D& g = a.g;
  const long long fp = FIRST ? g.src_pitch : g.pitch;
  const V* front = static_cast<const V*>(FIRST ? g.src : g.buf[(it - 1) & 1]) +
                   (long long)g.halo_top * fp;
  sk_val_t* back = static_cast<sk_val_t*>(g.buf[it & 1]) + (long long)g.halo_top * g.pitch;
  const int n = g.rows;
  const int rlo = -g.halo_top, rhi = n + g.halo_bottom;
  const int row0 = a.env.row0, grows = a.env.rows;
  const double neutral = comb.neutral(a.L.identity);
  const int total = a.L.part_chunk[a.L.nparts];
  for (int c = next_chunk(a.L, s_chunk); c < total; c = next_chunk(a.L, s_chunk)) {
    int cb, r0, r1;
    chunk_geom(a.L, g, c, &cb, &r0, &r1);
    JitAcc<FIRST> st{neutral};
#ifdef SK_LOCAL_MAX
    st.lmax = 0;
    st.lany = false;
#endif
    int buf = 0;
    jit_stage1<V>(tiles, front, fp, r0, min(kJit1Elems, r1 - r0), rlo, rhi);
    for (int t0 = r0; t0 < r1; t0 += kJit1Elems) {
      const int ne = min(kJit1Elems, r1 - t0);
      const bool more = t0 + kJit1Elems < r1;
      if (more)
        jit_stage1<V>(tiles + (buf ^ 1) * kJitTileElems, front, fp, t0 + kJit1Elems,
                      min(kJit1Elems, r1 - t0 - kJit1Elems), rlo, rhi);
      stage_wait_upto<V>(more ? 1 : 0);
      __syncthreads();
      const V* tile = tiles + buf * kJitTileElems;
      const bool inner = t0 + row0 >= SK_K && t0 + ne - 1 + row0 + SK_K < grows;
      if (inner) jit_elems1<FIRST, SkNb<V, true, 1>>(a, tile, back, t0, ne, comb, st);
      else jit_elems1<FIRST, SkNb<V, false, 1>>(a, tile, back, t0, ne, comb, st);
      __syncthreads();  // tile `buf` is free for the tile after next
      buf ^= 1;
    }
    double acc = st.acc;
#ifdef SK_LOCAL_MAX
    if (st.lany) acc = comb(acc, (double)st.lmax);
#endif
    const double v = block_reduce_c<SK_BLOCK>(comb, neutral, acc, sh);
    if (threadIdx.x == 0) a.L.partials[c] = v;
  }
}
#endif  // SK_NDIM == 1

}  // namespace sk

// dynamic shared memory per launch (the host reads it at module load)
extern "C" __device__ const int sk_jit_smem_bytes =
    2 * sk::kJitTileElems * sk::kJitElemMax +
    (SK_ENV0_STAGE ? 2 * SK_TH * SK_TW * (int)sizeof(sk::sk_env0_t) : 0);

extern "C" __global__ void __launch_bounds__(SK_BLOCK, SK_MINB) sk_jit_sweep(const __grid_constant__ sk::JitArgs a) {
  using namespace sk;
  __shared__ double sh[SK_BLOCK / 32];
  __shared__ int s_chunk;
  extern __shared__ __align__(16) unsigned char s_tile[];  // 2 tile buffers (dynamic)
  const SkComb comb{};
  long long it = loop_enter(a.L);
  if (it == 0) return;
  for (;;) {
#if SK_NDIM == 1
    if (it == 1) jit_sweep1<sk_in_t, true>(a, it, reinterpret_cast<sk_in_t*>(s_tile), &s_chunk, sh, comb);
    else jit_sweep1<sk_val_t, false>(a, it, reinterpret_cast<sk_val_t*>(s_tile), &s_chunk, sh, comb);
#else
    if (it == 1) jit_sweep<sk_in_t, true>(a, it, reinterpret_cast<sk_in_t*>(s_tile), &s_chunk, sh, comb);
    else jit_sweep<sk_val_t, false>(a, it, reinterpret_cast<sk_val_t*>(s_tile), &s_chunk, sh, comb);
#endif
    if (!a.L.persistent) {
      loop_finalize<SK_BLOCK>(a.L, it, sh, comb);
      return;
    }
    it = loop_barrier<SK_BLOCK>(a.L, it, sh, comb);
    if (it == 0) return;
  }
}
