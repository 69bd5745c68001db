// Variational restoration of flagged pixels (phase two of the denoiser).
//
// Reference: restore_kernel block route apps/denoise.py:209-246 (point route
// :178-207), ring order _RING :35, search constants :37-45, |new-old| delta
// and float sum :252-259, restore_regularize :262-288.
//
// For each flagged pixel (mask == 1), 18 ternary-search steps on [0, 255]
// minimise F(u) = beta * sum_ring w * sqrt((u - v)^2 + eps), with w = 1 for a
// flagged neighbour, 2 for a clean one, and off-image neighbours skipped (the
// block route's weight-0 terms add +0.0, which leaves the sum unchanged).
// Clean pixels never change.  Every value the reference computes is computed
// in fp64 in the reference's order with round-to-nearest intrinsics and IEEE
// sqrt; (hi - lo) / 3.0 uses the exact 3-op division by a constant.  Result:
// bit-identical grids.
//
// The reference's search costs ~1.5k fp64 flops + 288 sqrt per pixel-
// iteration; work is cut exactly, not approximately:
//  * comparison filter: most F(m1) <= F(m2) outcomes are certified by an
//    fp32 bracket of both sides (bound_decide); only the others are
//    evaluated in fp64, compacted per warp (restore_sweep, phase 2).
//  * flagged list: only flagged pixels are visited (built once per run by a
//    deterministic count/scan/scatter; in pixel order, so each partition's
//    pixels are a contiguous sub-range).
//  * exact active set: a pixel's output depends only on its 8 ring values
//    (the mask is static), so if none of them changed in the previous
//    iteration its output equals its previous output; it is copied, not
//    recomputed.  Change flags are ping-ponged per iteration.
//  * in-CTA compaction: active entries go to a shared-memory queue that all
//    threads drain, so a sparse active set still keeps every lane busy.
// The delta reduce is deterministic: each entry's |delta| lands at its fixed
// position in the chunk, positions are summed in a fixed order, chunk
// partials are folded per partition, partitions in ascending order.
#include "sk_internal.h"

namespace sk {

constexpr int kRB = 128;        // threads per CTA
constexpr int kPer = 4;         // list entries per thread per chunk
constexpr int kCh = kRB * kPer;  // entries per chunk
constexpr int kSteps = 18;      // ceil(log(1020) / log(1.5)), apps/denoise.py:39-45

struct RestoreArgs {
  const double* src;
  double* buf[2];
  const unsigned char* mask;
  long long pitch, src_pitch, mask_pitch;
  int rows, cols;
  const int* list;            // flagged pixels, row * cols + col, ascending
  unsigned char* chg[2];      // per-pixel change flags, ping-pong by iteration
  const int* part_off;        // device: list offsets per partition [nparts + 1]
  double beta, eps;
  LoopCtl L;
  // frame batches (SK_FLAG_FRAMES): partition p is an independent frame of
  // frame_rows rows with its own loop (stop test, iteration count, value)
  int frame_rows;             // 0: one image (partitions are row blocks of it)
  struct FrameStat* fstat;    // [nparts]
};

struct FrameStat {
  long long iter;   // iterations this frame completed
  int stop;         // its loop is over
  int exhausted;    // cap hit without the condition
  double value;     // last reduce value
};

// F(u) = beta * sum over the 8 ring terms, in ring order, of w * sqrt((u-v)^2 + eps).
// Off-image neighbours carry weight 0 exactly as in the block route
// (apps/denoise.py:230-233): they add +0.0, which leaves the sum unchanged.
// Each term w * sqrt((u - v)^2 + eps) is an independent fp64 product and the
// owner adds its pixel's 8 terms in ring order -- the reference's sum -- so
// the terms may be computed by any lane (restore_sweep, phase 2).

// ---- exact comparison filter.  The search only needs the OUTCOME of
// F(m1) <= F(m2) per step, F = fl(beta * S), S = sum_k w_k g(u - v_k),
// g(t) = sqrt(t^2 + eps).  Since |t| <= g(t) <= |t| + min(sqrt(eps),
// eps / (2|t|)), fp32 sums of w|t| bracket S with a provable slack; when the
// brackets of S(m1) and S(m2) do not overlap the outcome is known exactly
// (beta > 0, rounding is monotone, and the gap dwarfs fp64 rounding), and
// only overlapping (close) comparisons evaluate F in fp64.  Results stay
// bit-identical; SK_RESTORE_FILTER=0 at build time evaluates every step.
//
// Bracket, per pixel and side (a_k = |fl32(u32 - v32_k)|, u32 / v32_k the
// fp32 roundings of u / v_k):
//   | |t_k| - a_k | <= et = 2^-22 (256 + max_k |v32_k|)      (u in [0, 255])
//   L = sum w_k a_k (fp32, rel. error < 2^-20),  W = sum w_k
//   y_k = the fp32 with bits 0x7F000000 - bits(a_k) = 2^-E (1.5 - m/2) for
//       a_k = 2^E m, m in [1, 2): the chord of the convex 1/m, so
//       1/a_k <= y_k <= 1.125/a_k (one integer subtraction)
//   C = sum w_k min(sqrt_eps, eps/2 * y_k):  when a_k >= 64 et,
//       eps/(2|t_k|) <= eps/(2(a_k - et)) <= (64/63) eps/2 * y_k; below that
//       eps/2 * y_k > eps/(128 et) >= sqrt(eps) (the filter is on only when
//       128 et <= sqrt(eps)) and the min is sqrt_eps: (64/63) C bounds the
//       slack sum (fp32 rounding included: factor 1 + 2^-5 below).
//   L - W et - 2^-20 L  <=  S  <=  L + (1 + 2^-5) C + W et + 2^-20 L
// S1 < S2 is certain when fl(L1 + C1' + 3 W et + 2^-18 (L1 + C1' + L2)) < L2,
// C1' = (1 + 2^-5) C1 (the extra margin absorbs that expression's rounding).
#ifndef SK_RESTORE_FILTER
#define SK_RESTORE_FILTER 1
#endif
constexpr bool kFilter = SK_RESTORE_FILTER != 0;
// Warp-level compaction of the exact comparisons: a warp's 32 lanes run 32
// pixels' searches in lockstep; when k lanes of a warp are left undecided by
// the filter, their 16 k terms (k comparisons x 2 sides x 8 ring terms) are
// spread over the warp's 32 lanes (ceil(k / 2) terms per lane) and each
// owner adds up its own terms; only when many lanes are undecided (k >
// kDirect) does every undecided lane evaluate its own comparison.  Ring
// values, weights and terms live in shared memory so that any lane can
// compute any term; rows are padded to odd lengths (bank spread).
#ifndef SK_RESTORE_DIRECT
#define SK_RESTORE_DIRECT 12
#endif
constexpr int kDirect = SK_RESTORE_DIRECT;
static_assert(kDirect >= 1 && kDirect <= 32, "SK_RESTORE_DIRECT must be in [1, 32]");
constexpr int kRingPad = 9;  // doubles per ring row
constexpr int kTermPad = 17; // doubles per term row (2 x 8 + 1)
#ifndef SK_RESTORE_MINB
#define SK_RESTORE_MINB 8
#endif
constexpr int kMinBlocks = SK_RESTORE_MINB;  // resident CTAs per SM (register cap)

struct Ring {
  float v32[8], wf[8];
  float wet3;   // 3 W et, rounded up
  bool fil;     // the bound filter applies to this pixel
};

__device__ __forceinline__ void load_ring(const RestoreArgs& a, const double* front, long long fp,
                                          int i, int j, int rlo, int rhi, float sqrt_eps_dn,
                                          double (*ring)[kRingPad],
                                          unsigned short (*whi)[kRingPad], Ring& r) {
  float vmax = 0.0f, wsum = 0.0f;
  bool finite = true;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int di = k < 3 ? -1 : (k < 5 ? 0 : 1);  // _RING order
    const int dj = k < 3 ? k - 1 : (k < 5 ? (k == 3 ? -1 : 1) : k - 6);
    const int ni = i + di, nj = j + dj;
    const bool in = ni >= rlo && ni < rhi && nj >= 0 && nj < a.cols;
    const double v = in ? front[(long long)ni * fp + nj] : 0.0;
    ring[threadIdx.x][k] = v;
    const bool flagged = in && a.mask[(long long)ni * a.mask_pitch + nj] == 1;
    r.wf[k] = in ? (flagged ? 1.0f : 2.0f) : 0.0f;
    whi[threadIdx.x][k] = in ? (flagged ? 0x3FF0 : 0x4000) : 0;  // 1.0 / 2.0 / 0.0, bits 48-63
    r.v32[k] = __double2float_rn(v);
    finite = finite && isfinite(r.v32[k]);
    vmax = fmaxf(vmax, fabsf(r.v32[k]));
    wsum += r.wf[k];
  }
  const float et = __fmul_ru(__fadd_ru(256.0f, vmax), 1.0f / 4194304.0f);  // 2^-22
  r.wet3 = __fmul_ru(__fmul_ru(3.0f, wsum), et);
  r.fil = kFilter && finite && __fmul_ru(128.0f, et) <= sqrt_eps_dn;
}

// 1: F(m1) <= F(m2) certainly, 0: F(m1) > F(m2) certainly, -1: undecided.
// Only the side with the smaller L can be certified smaller, so the slack
// is summed for that side alone, as eps/2 * sum w min(kq, y) with
// kq >= sqrt_eps / (eps/2) (one min and one FMA per term).
__device__ __forceinline__ int bound_decide(float u1, float u2, const Ring& r, float kq,
                                            float eh) {
  // two partial sums per side halve the dependent FMA chains (any order of
  // the 8 non-negative terms keeps the 2^-20 bound)
  float l1a = 0.0f, l1b = 0.0f, l2a = 0.0f, l2b = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    l1a = fmaf(r.wf[k], fabsf(u1 - r.v32[k]), l1a);
    l2a = fmaf(r.wf[k], fabsf(u2 - r.v32[k]), l2a);
    l1b = fmaf(r.wf[k + 1], fabsf(u1 - r.v32[k + 1]), l1b);
    l2b = fmaf(r.wf[k + 1], fabsf(u2 - r.v32[k + 1]), l2b);
  }
  const float l1 = l1a + l1b, l2 = l2a + l2b;
  const bool one = l1 <= l2;
  const float us = one ? u1 : u2, ls = one ? l1 : l2, lb = one ? l2 : l1;
  float ca = 0.0f, cb = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const float ya = __int_as_float(0x7F000000 - __float_as_int(fabsf(us - r.v32[k])));  // >= 1/a
    const float yb = __int_as_float(0x7F000000 - __float_as_int(fabsf(us - r.v32[k + 1])));
    ca = fmaf(r.wf[k], fminf(kq, ya), ca);
    cb = fmaf(r.wf[k + 1], fminf(kq, yb), cb);
  }
  float c = ca + cb;
  c = __fmul_ru(c, eh);  // eh >= (1 + 2^-5) eps / 2
  constexpr float kRel = 1.0f / 262144.0f;  // 2^-18
  if (ls + c + r.wet3 + kRel * (ls + c + lb) < lb) return one ? 1 : 0;
  return -1;
}

// Cross-frame barrier for batched restores: the last CTA folds every active
// frame's chunk partials (same fixed order as a single-frame run), applies
// that frame's stop test, and releases the grid; the loop ends when every
// frame has stopped.
__device__ long long frames_barrier(const RestoreArgs& a, long long it, double* sh) {
  __shared__ int s_last;
  __shared__ unsigned s_gen;
  __shared__ int s_all;
  const LoopCtl& L = a.L;
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* genp = &L.st->gen;
    s_gen = *genp;
    __threadfence();
    const unsigned prev = atomicAdd(&L.st->ticket, 1u);
    s_last = (prev == gridDim.x - 1);
    s_all = 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    const int* pch = L.part_chunk_dev;
    for (int p = 0; p < L.nparts; ++p) {
      FrameStat* fs = &a.fstat[p];
      if (fs->stop) continue;  // uniform: every thread reads the same flag
      double t = 0.0;
      for (int c = pch[p] + (int)threadIdx.x; c < pch[p + 1]; c += kRB) t += __ldcg(&L.partials[c]);
      const double v = L.identity + block_reduce<kRB>(SK_REDUCE_SUM, t, sh);
      if (threadIdx.x == 0) {
        const int n = a.part_off[p + 1] - a.part_off[p];
        const int c = xdiv(v, (double)(n > 1 ? n : 1)) < L.cond.a;  // restore_regularize test
        const int capped = it >= L.cond.max_it;
        fs->iter = it;
        fs->value = v;
        fs->exhausted = !c && capped;
        fs->stop = c || capped;
        if (!(c || capped)) s_all = 0;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      Status* st = L.st;
      st->iter = it;
      st->stop = s_all;
      st->ticket = 0;
      st->work = 0;
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

template <bool FRAMES>
__global__ void __launch_bounds__(kRB, kMinBlocks) restore_sweep(const __grid_constant__ RestoreArgs a) {
  __shared__ double sh[kRB / 32];
  __shared__ double s_delta[kCh];
  __shared__ short s_queue[kCh];
  __shared__ int s_qlen;
  __shared__ int s_take;
  __shared__ double s_ring[kRB][kRingPad];  // ring values of the round's pixels
  __shared__ unsigned short s_whi[kRB][kRingPad];  // their weights (top 16 bits)
  __shared__ double s_m[kRB][2];            // m1, m2 of undecided comparisons
  __shared__ double s_T[kRB / 32 * kDirect][kTermPad];  // their terms, by rank
  __shared__ unsigned char s_xq[kRB];       // undecided lanes, per warp
  __shared__ int s_chunk;
  // bound-filter constants (see bound_decide); off unless beta > 0, eps >= 0
  const bool fil_ok = kFilter && a.beta > 0.0 && a.eps >= 0.0 && isfinite(a.beta) &&
                      isfinite(a.eps);
  const float sqrt_eps_dn = fil_ok ? __fsqrt_rd(__double2float_rd(a.eps)) : -1.0f;
  const float eps_half_up = __double2float_ru(xmul(a.eps, 0.5));
  const float kq = __fdiv_ru(__fsqrt_ru(__double2float_ru(a.eps)), eps_half_up);
  const float eh = __fmul_ru(eps_half_up, 1.03125f);
  const double r3 = __drcp_rn(3.0);
  for (long long it = loop_enter(a.L); it != 0;
       it = FRAMES ? frames_barrier(a, it, sh) : loop_next<kRB>(a.L, it, sh)) {
  const double* front = it == 1 ? a.src : a.buf[(it - 1) & 1];
  const long long fp = it == 1 ? a.src_pitch : a.pitch;
  double* back = a.buf[it & 1];
  const unsigned char* cprev = a.chg[(it - 1) & 1];
  unsigned char* ccur = a.chg[it & 1];
  // chunk geometry lives on the device (built by the setup kernels, so the
  // host never waits for the flagged count)
  const int* pch = a.L.part_chunk_dev;
  const int total = pch[a.L.nparts];
  for (int c = next_chunk(a.L, &s_chunk); c < total; c = next_chunk(a.L, &s_chunk)) {
    int p = 0;
    while (p + 1 < a.L.nparts && c >= pch[p + 1]) ++p;
    if (FRAMES && a.fstat[p].stop) continue;  // this frame's loop is over
    // ring reads stay inside the image (one image) or inside the frame (batch)
    const int rlo = FRAMES ? p * a.frame_rows : 0;
    const int rhi = FRAMES ? rlo + a.frame_rows : a.rows;
    const int e0 = a.part_off[p] + (c - pch[p]) * kCh;
    const int e1 = min(e0 + kCh, a.part_off[p + 1]);
    if (threadIdx.x == 0) {
      s_qlen = 0;
      s_take = 0;
    }
    __syncthreads();
    // phase 1: classify; inactive entries are settled immediately
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int pos = q * kRB + threadIdx.x;
      const int e = e0 + pos;
      s_delta[pos] = 0.0;
      if (e < e1) {
        const int pix = a.list[e];
        const int i = pix / a.cols, j = pix - i * a.cols;
        bool active = it == 1;
        if (!active) {
          for (int di = -1; di <= 1 && !active; ++di) {
            const int ni = i + di;
            if (ni < rlo || ni >= rhi) continue;
            for (int dj = -1; dj <= 1; ++dj) {
              const int nj = j + dj;
              if ((di | dj) == 0 || nj < 0 || nj >= a.cols) continue;
              if (cprev[(long long)ni * a.cols + nj]) {
                active = true;
                break;
              }
            }
          }
        }
        if (active) {
          const int slot = atomicAdd(&s_qlen, 1);
          s_queue[slot] = (short)pos;
        } else {
          back[(long long)i * a.pitch + j] = front[(long long)i * fp + j];
          ccur[pix] = 0;
        }
      }
    }
    __syncthreads();
    // phase 2: each warp drains the active queue 32 entries at a time, one
    // per lane, independently of the other warps (a result and its |delta|
    // go to the entry's own position)
    const int qlen = s_qlen;
    for (;;) {
      int base = 0;
      if ((threadIdx.x & 31) == 0) base = atomicAdd(&s_take, 32);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base >= qlen) break;
      const int q = base + (int)(threadIdx.x & 31);
      const bool has = q < qlen;
      int pos = 0, pix = 0;
      double lo = 0.0, hi = 255.0, old = 0.0;
      Ring r;
      r.fil = false;
      if (has) {
        pos = s_queue[q];
        pix = a.list[e0 + pos];
        const int i = pix / a.cols, j = pix - i * a.cols;
        old = front[(long long)i * fp + j];
        load_ring(a, front, fp, i, j, rlo, rhi, sqrt_eps_dn, s_ring, s_whi, r);
      }
#pragma unroll 1
      for (int step = 0; step < kSteps; ++step) {
        const double third = div_const(xsub(hi, lo), 3.0, r3);
        const double m1 = xadd(lo, third);
        const double m2 = xsub(hi, third);
        int d = 1;
        if (has) {
          d = r.fil ? bound_decide(__double2float_rn(m1), __double2float_rn(m2), r, kq, eh) : -1;
        }
        const bool und = d < 0;
        const unsigned bal = __ballot_sync(0xffffffffu, und);
        bool le = d != 0;
        if (bal) {
          const int k = __popc(bal);
          const unsigned lane = threadIdx.x & 31;
          const int wb = threadIdx.x & ~31;  // this warp's first slot
          if (k > kDirect) {
            if (und) {
              double s1 = 0.0, s2 = 0.0;
#pragma unroll 2
              for (int kk = 0; kk < 8; ++kk) {
                const double v = s_ring[threadIdx.x][kk];
                const double w = __hiloint2double((int)s_whi[threadIdx.x][kk] << 16, 0);
                const double t1 = xsub(m1, v), t2 = xsub(m2, v);
                s1 = xadd(s1, xmul(w, xsqrt(xadd(xmul(t1, t1), a.eps))));
                s2 = xadd(s2, xmul(w, xsqrt(xadd(xmul(t2, t2), a.eps))));
              }
              le = xmul(a.beta, s1) <= xmul(a.beta, s2);
            }
          } else {
            const int tb = (wb >> 5) * kDirect;  // this warp's term rows
            const int rank = __popc(bal & ((1u << lane) - 1u));
            if (und) {
              s_xq[wb + rank] = (unsigned char)threadIdx.x;
              s_m[threadIdx.x][0] = m1;
              s_m[threadIdx.x][1] = m2;
            }
            __syncwarp();
            for (int x = lane; x < 16 * k; x += 32) {
              const int p = s_xq[wb + (x >> 4)], side = (x >> 3) & 1, kk = x & 7;
              const double t = xsub(s_m[p][side], s_ring[p][kk]);
              s_T[tb + (x >> 4)][side * 8 + kk] =
                  xmul(__hiloint2double((int)s_whi[p][kk] << 16, 0), xsqrt(xadd(xmul(t, t), a.eps)));
            }
            __syncwarp();
            if (und) {
              double s1 = 0.0, s2 = 0.0;
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                s1 = xadd(s1, s_T[tb + rank][kk]);
                s2 = xadd(s2, s_T[tb + rank][8 + kk]);
              }
              le = xmul(a.beta, s1) <= xmul(a.beta, s2);
            }
            __syncwarp();  // s_xq / s_m / s_T reuse next step
          }
        }
        if (le) hi = m2;
        else lo = m1;
      }
      if (has) {
        const double nv = xmul(0.5, xadd(lo, hi));
        const int i = pix / a.cols, j = pix - i * a.cols;
        back[(long long)i * a.pitch + j] = nv;
        ccur[pix] = nv != old;
        s_delta[pos] = fabs(xsub(nv, old));
      }
      __syncwarp();  // the lanes' shared rows are reused by the next round
    }
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) t = xadd(t, s_delta[q * kRB + threadIdx.x]);
    const double v = block_reduce<kRB>(SK_REDUCE_SUM, t, sh);
    if (threadIdx.x == 0) a.L.partials[c] = v;
  }
  }  // iterations
}

// ---- flagged-list construction: count per segment, scan, scatter (ordered)

constexpr int kSeg = 4096;  // pixels per segment (one CTA of 256 threads x 16 pixels)

// Flags (mask byte == 1) of the 16 row-major pixels p .. p+15 as bits 0..15:
// one 16-byte load and four byte compares when the run lies inside one
// aligned row (the common case), byte by byte with row wrap otherwise.
__device__ __forceinline__ unsigned flag_bits16(const unsigned char* mask, long long mpitch, int cols,
                                                long long npix, long long p) {
  if (p >= npix) return 0u;
  const long long i = p / cols;
  int j = (int)(p - i * cols);
  const unsigned char* row = mask + i * mpitch;
  unsigned bits = 0u;
  if (j + 16 <= cols && p + 16 <= npix && (reinterpret_cast<unsigned long long>(row + j) & 15) == 0) {
    const uint4 v = *reinterpret_cast<const uint4*>(row + j);
    const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned eq = __vcmpeq4(w[q], 0x01010101u);  // 0xff per byte equal to 1
      bits |= ((eq & 1u) | ((eq >> 7) & 2u) | ((eq >> 14) & 4u) | ((eq >> 21) & 8u)) << (4 * q);
    }
  } else {
    for (int k = 0; k < 16 && p + k < npix; ++k) {
      bits |= (unsigned)(row[j] == 1) << k;
      if (++j == cols) {
        j = 0;
        row += mpitch;
      }
    }
  }
  return bits;
}

__global__ void __launch_bounds__(256) flag_count(const unsigned char* mask, long long mpitch, int rows,
                                                  int cols, int* seg_count) {
  const long long npix = (long long)rows * cols;
  const long long p = (long long)blockIdx.x * kSeg + 16 * threadIdx.x;
  int n = __popc(flag_bits16(mask, mpitch, cols, npix, p));
  n = __reduce_add_sync(0xffffffffu, n);
  __shared__ int ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += ws[w];
    seg_count[blockIdx.x] = t;
  }
}

__global__ void flag_scan(int* seg, int nseg) {  // exclusive, single CTA
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nseg; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = i < nseg ? seg[i] : 0;
    // inclusive warp scan then block scan
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    __shared__ int wsum[32];
    if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      int s = threadIdx.x < (blockDim.x >> 5) ? wsum[threadIdx.x] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, s, o);
        if (threadIdx.x >= o) s += y;
      }
      wsum[threadIdx.x] = s;
    }
    __syncthreads();
    const int w = threadIdx.x >> 5;
    const int incl = x + (w ? wsum[w - 1] : 0) + carry;
    if (i < nseg) seg[i] = incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = incl;
    __syncthreads();
  }
}

// Each thread owns 16 consecutive pixels of the segment: an exclusive scan of
// the threads' flag counts gives every thread its slot run, so the list
// comes out in pixel order with one barrier.
__global__ void __launch_bounds__(256) flag_scatter(const unsigned char* mask, long long mpitch, int rows,
                                                    int cols, const int* seg_off, int* list) {
  const long long npix = (long long)rows * cols;
  const long long p = (long long)blockIdx.x * kSeg + 16 * threadIdx.x;
  unsigned bits = flag_bits16(mask, mpitch, cols, npix, p);
  const int n = __popc(bits);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = n;  // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __shared__ int wsum[8];
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  int before = seg_off[blockIdx.x] + x - n;
  for (int k = 0; k < w; ++k) before += wsum[k];
  while (bits) {
    const int b = __ffs(bits) - 1;
    list[before++] = (int)(p + b);
    bits &= bits - 1;
  }
}

// partition p's flagged pixels start at lower_bound(list, part_row[p] * cols);
// then one thread turns the offsets into per-partition chunk ranges
__global__ void list_bounds(const int* list, const int* n_ptr, const int* part_row, int nparts,
                            int cols, int* off, int* pchunk, int pa, int pb) {
  const int p = threadIdx.x;
  const int n = *n_ptr;
  if (p < nparts) {
    const long long key = (long long)part_row[p] * cols;
    int lo = 0, hi = n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((long long)list[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    off[p] = lo;
  } else if (p == nparts) {
    off[p] = n;
  }
  __syncthreads();
  if (p == 0) {
    int acc = 0;
    pchunk[0] = 0;
    for (int i = 0; i < nparts; ++i) {
      // partitions outside [pa, pb) get no chunks: another run computes them
      // (a frame split across GPUs, sk_run_exchange_rows)
      if (i >= pa && i < pb) acc += (off[i + 1] - off[i] + kCh - 1) / kCh;
      pchunk[i + 1] = acc;
    }
  }
}

// ---------------------------------------------------------------- host side

namespace {

enum { AUX_LIST = 0, AUX_CHG = 1, AUX_SEG = 2, AUX_OFF = 3, AUX_FSTAT = 4 };

int setup(sk_run* r) {
  const sk_plan& p = r->plan;
  if (p.dtype != SK_F64 || p.reduce_op != SK_REDUCE_SUM || p.delta_op != SK_DELTA_ABS) {
    set_error("restore: f64 grid with the |new-old| SUM reduce (restore_regularize) required");
    return SK_ERR_UNSUPPORTED;
  }
  if (!r->env) {
    set_error("restore: the noise map (env) is required");
    return SK_ERR_ARG;
  }
  if ((long long)p.rows * p.cols >= (1ll << 31)) {
    set_error("restore: grid too large for 32-bit pixel indices");
    return SK_ERR_ARG;
  }
  // Entirely stream-ordered: no host synchronisation, so a farm of restore
  // runs never stalls its host thread here.
  cudaStream_t s = r->stream;
  const long long npix = p.rows * p.cols;
  const int nseg = (int)((npix + kSeg - 1) / kSeg);
  const unsigned char* mask = static_cast<const unsigned char*>(r->env);
  int* seg = nullptr;
  const size_t small = (size_t)nseg + 1 + 3 * (kMaxParts + 1);
  SK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&seg), sizeof(int) * small, s));
  r->aux[AUX_SEG] = seg;
  int* d_prow = seg + nseg + 1;
  int* d_off = d_prow + kMaxParts + 1;
  int* d_pch = d_off + kMaxParts + 1;
  SK_CUDA(cudaMemsetAsync(seg + nseg, 0, sizeof(int), s));
  flag_count<<<nseg, 256, 0, s>>>(mask, r->env_pitch, (int)p.rows, (int)p.cols, seg);
  flag_scan<<<1, 1024, 0, s>>>(seg, nseg + 1);  // seg[nseg] = total flagged
  int* list = nullptr;  // capacity: every pixel (the count is not read back)
  SK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&list), sizeof(int) * ((size_t)npix + 1), s));
  r->aux[AUX_LIST] = list;
  flag_scatter<<<nseg, 256, 0, s>>>(mask, r->env_pitch, (int)p.rows, (int)p.cols, seg, list);
  SK_CUDA(cudaMemcpyAsync(d_prow, r->part_row, sizeof(int) * (r->nparts + 1),
                          cudaMemcpyHostToDevice, s));
  // params[2], params[3]: this run computes partitions [pa, pb) only (pb = 0: all)
  int pa = 0, pb = r->nparts;
  if (p.params[3] > 0) {
    pa = (int)p.params[2];
    pb = (int)p.params[3];
    if (pa < 0 || pb > r->nparts || pa >= pb || (p.flags & SK_FLAG_FRAMES)) {
      set_error("restore: active partition range must satisfy 0 <= pa < pb <= partitions");
      return SK_ERR_ARG;
    }
  }
  list_bounds<<<1, kMaxParts + 1, 0, s>>>(list, seg + nseg, d_prow, r->nparts, (int)p.cols, d_off,
                                         d_pch, pa, pb);
  SK_CUDA(cudaGetLastError());
  unsigned char* chg = nullptr;
  SK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&chg), (size_t)npix * 2, s));
  r->aux[AUX_CHG] = chg;
  SK_CUDA(cudaMemsetAsync(chg, 0, (size_t)npix * 2, s));
  // both iteration buffers start as the input: clean pixels never change
  for (int b = 0; b < 2; ++b)
    SK_CUDA(cudaMemcpy2DAsync(r->buf[b], r->pitch * 8, r->src, r->src_pitch * 8, p.cols * 8,
                              p.rows, cudaMemcpyDeviceToDevice, s));
  r->aux[AUX_OFF] = d_off;
  if (p.flags & SK_FLAG_FRAMES) {
    if (p.rows % r->nparts) {
      set_error("restore: a frame batch must stack frames of equal height");
      return SK_ERR_ARG;
    }
    void* fs = nullptr;
    SK_CUDA(cudaMallocAsync(&fs, sizeof(FrameStat) * r->nparts, s));
    SK_CUDA(cudaMemsetAsync(fs, 0, sizeof(FrameStat) * r->nparts, s));
    r->aux[AUX_FSTAT] = fs;
  }
  r->part_chunk_dev = d_pch;
  r->flagged_dev = seg + nseg;
  // partial slots for the largest possible chunk count
  r->nchunks = (int)((npix + kCh - 1) / kCh) + r->nparts;
  const long long slots = (long long)device_sms(r->device) *
                          occupancy(reinterpret_cast<const void*>(restore_sweep<false>), kRB);
  const long long most = r->nchunks;
  r->grid = (int)(slots < most ? slots : most);
  if (r->grid < 1) r->grid = 1;
  r->block = kRB;
  return SK_OK;
}

int launch(sk_run* r, const LoopCtl& L, cudaStream_t s) {
  RestoreArgs a{};
  a.src = static_cast<const double*>(r->src);
  a.buf[0] = static_cast<double*>(r->buf[0]);
  a.buf[1] = static_cast<double*>(r->buf[1]);
  a.mask = static_cast<const unsigned char*>(r->env);
  a.pitch = r->pitch;
  a.src_pitch = r->src_pitch;
  a.mask_pitch = r->env_pitch;
  a.rows = (int)r->plan.rows;
  a.cols = (int)r->plan.cols;
  a.list = static_cast<const int*>(r->aux[AUX_LIST]);
  unsigned char* chg = static_cast<unsigned char*>(r->aux[AUX_CHG]);
  a.chg[0] = chg;
  a.chg[1] = chg + r->plan.rows * r->plan.cols;
  a.part_off = static_cast<const int*>(r->aux[AUX_OFF]);
  a.beta = r->plan.params[0];
  a.eps = r->plan.params[1];
  a.L = L;
  if (r->plan.flags & SK_FLAG_FRAMES) {
    // a batch of independent frames: always one persistent launch
    if (!L.persistent) {
      set_error("restore: frame batches run as one persistent loop");
      return SK_ERR_UNSUPPORTED;
    }
    a.frame_rows = (int)(r->plan.rows / r->nparts);
    a.fstat = static_cast<FrameStat*>(r->aux[AUX_FSTAT]);
    SK_CUDA(launch_kernel(restore_sweep<true>, r->grid, kRB, a, s, true));
    return SK_OK;
  }
  SK_CUDA(launch_kernel(restore_sweep<false>, r->grid, kRB, a, s, L.persistent != 0));
  return SK_OK;
}

void teardown(sk_run* r) {
  for (int k : {AUX_LIST, AUX_CHG, AUX_SEG, AUX_FSTAT})
    if (r->aux[k]) cudaFreeAsync(r->aux[k], r->stream);
  r->aux[AUX_OFF] = nullptr;  // lives inside the AUX_SEG block
}

const KernelOps kOps = {setup, launch, teardown};

}  // namespace

const KernelOps* restore_ops() { return &kOps; }

// Change-flag plane of iteration `it` (restore runs), for the row exchange.
unsigned char* restore_chg(sk_run* r, long long it) {
  if (r->ops != &kOps || !r->aux[AUX_CHG]) return nullptr;
  return static_cast<unsigned char*>(r->aux[AUX_CHG]) + (it & 1) * r->plan.rows * r->plan.cols;
}

int restore_frame_status(sk_run* r, long long* iters, double* values, int* exhausted) {
  if (!(r->plan.flags & SK_FLAG_FRAMES) || !r->aux[AUX_FSTAT]) {
    set_error("sk_run_frame_status: not a frame-batch run");
    return SK_ERR_STATE;
  }
  std::vector<FrameStat> fs(r->nparts);
  SK_CUDA(cudaMemcpyAsync(fs.data(), r->aux[AUX_FSTAT], sizeof(FrameStat) * r->nparts,
                          cudaMemcpyDeviceToHost, r->stream));
  SK_CUDA(cudaStreamSynchronize(r->stream));
  for (int i = 0; i < r->nparts; ++i) {
    iters[i] = fs[i].iter;
    values[i] = fs[i].value;
    exhausted[i] = fs[i].exhausted;
  }
  return SK_OK;
}

}  // namespace sk
