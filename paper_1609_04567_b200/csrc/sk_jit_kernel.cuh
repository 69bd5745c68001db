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
// Required from the generated part: sk_in_t, sk_val_t, SK_K, SK_PAD_EDGE,
// SK_PAD_VALUE, sk_elemental_1/_n, sk_delta_1/_n, struct SkComb.
#pragma once


#ifndef SK_BLOCK
#define SK_BLOCK 256
#endif
#define SK_TW 128
#define SK_TH 16

namespace sk {

constexpr int kJitTWP = SK_TW + 2 * SK_K;
constexpr int kJitTileElems = (SK_TH + 2 * SK_K) * kJitTWP;
constexpr int kJitElemMax = sizeof(sk_in_t) > sizeof(sk_val_t) ? sizeof(sk_in_t) : sizeof(sk_val_t);

__device__ __forceinline__ void jit_fail(Status* st, long long index, int code) {
  atomicMax(&st->err, ~(((unsigned long long)index << 8) | (unsigned)code));
}

// Stage rows [r0 - K, r0 + nr + K) x columns [c0 - K, c0 + TW + K) of the
// front into the tile: off-grid slots take the pad value ("constant") or the
// nearest border element ("edge"), like the reference's context assembly
// (partition.py:278-288, 551-581).
template <class V>
__device__ __forceinline__ void jit_stage(V* tile, const V* front, long long fp, int r0, int nr,
                                          int c0, int rows, int cols) {
  const int n = (nr + 2 * SK_K) * kJitTWP;
  for (int idx = threadIdx.x; idx < n; idx += SK_BLOCK) {
    const int tr = idx / kJitTWP, tc = idx - tr * kJitTWP;
    int gi = r0 - SK_K + tr, gj = c0 - SK_K + tc;
    V v;
#if SK_PAD_EDGE
    gi = gi < 0 ? 0 : (gi >= rows ? rows - 1 : gi);
    gj = gj < 0 ? 0 : (gj >= cols ? cols - 1 : gj);
    v = front[(long long)gi * fp + gj];
#else
    const bool in = (unsigned)gi < (unsigned)rows && (unsigned)gj < (unsigned)cols;
    v = in ? front[(long long)gi * fp + gj] : (V)(SK_PAD_VALUE);
#endif
    tile[idx] = v;
  }
}

template <class V, bool FIRST>
__device__ __forceinline__ double jit_sweep(const JitArgs& a, long long it, V* tile, int* s_chunk,
                                            double* sh, const SkComb& comb) {
  const Sweep2D& g = a.g;
  const V* front = static_cast<const V*>(FIRST ? g.src : g.buf[(it - 1) & 1]);
  const long long fp = FIRST ? g.src_pitch : g.pitch;
  sk_val_t* back = static_cast<sk_val_t*>(g.buf[it & 1]);
  const int rows = g.rows, cols = g.cols;
  const int tx = threadIdx.x % SK_TW, ty = threadIdx.x / SK_TW;
  const double neutral = comb.neutral(a.L.identity);
  const int total = a.L.part_chunk[a.L.nparts];
  for (int c = next_chunk(a.L, s_chunk); c < total; c = next_chunk(a.L, s_chunk)) {
    int cb, r0, r1;
    chunk_geom(a.L, g, c, &cb, &r0, &r1);
    const int c0 = cb * SK_TW, nr = r1 - r0;
    jit_stage<V>(tile, front, fp, r0, nr, c0, rows, cols);
    __syncthreads();
    double acc = neutral;
    const int gj = c0 + tx;
    if (gj < cols) {
      for (int lr = ty; lr < nr; lr += SK_BLOCK / SK_TW) {
        const int gi = r0 + lr;
        SkNb<V> nb;
        nb.c = tile + (lr + SK_K) * kJitTWP + tx + SK_K;
        nb.stride = kJitTWP;
        nb.i = gi;
        nb.j = gj;
        nb.rows = rows;
        nb.cols = cols;
        nb.k = SK_K;
        SkErr err;
        sk_val_t nw;
        double d;
        if (FIRST) {
          nw = sk_elemental_1(nb, a.env, err);
          d = sk_delta_1(nw, nb.center(), err);
        } else {
          nw = sk_elemental_n(nb, a.env, err);
          d = sk_delta_n(nw, nb.center(), err);
        }
        back[(long long)gi * g.pitch + gj] = nw;
        if (err.code) jit_fail(a.L.st, (long long)gi * cols + gj, err.code);
        acc = comb(acc, d);
      }
    }
    const double v = block_reduce_c<SK_BLOCK>(comb, neutral, acc, sh);
    if (threadIdx.x == 0) a.L.partials[c] = v;
  }
  return 0.0;
}

}  // namespace sk

extern "C" __global__ void __launch_bounds__(SK_BLOCK) sk_jit_sweep(const __grid_constant__ sk::JitArgs a) {
  using namespace sk;
  __shared__ double sh[SK_BLOCK / 32];
  __shared__ int s_chunk;
  __shared__ __align__(16) unsigned char s_tile[kJitTileElems * kJitElemMax];
  const SkComb comb{};
  long long it = loop_enter(a.L);
  if (it == 0) return;
  for (;;) {
    if (it == 1) jit_sweep<sk_in_t, true>(a, it, reinterpret_cast<sk_in_t*>(s_tile), &s_chunk, sh, comb);
    else jit_sweep<sk_val_t, false>(a, it, reinterpret_cast<sk_val_t*>(s_tile), &s_chunk, sh, comb);
    if (!a.L.persistent) {
      loop_finalize<SK_BLOCK>(a.L, it, sh, comb);
      return;
    }
    it = loop_barrier<SK_BLOCK>(a.L, it, sh, comb);
    if (it == 0) return;
  }
}
