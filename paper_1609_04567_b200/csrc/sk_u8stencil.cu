// u8 3x3 stencils: Sobel edge magnitude and Conway's Game of Life.
//
// Reference: Sobel block kernel apps/sobel.py:47-66 (point :33-44; pixel-sum
// reduce :73-74); Life block kernel apps/life.py:35-43 (liveness :46-52).
//
// HBM-bound: 2 B/pixel (read 1 + write 1).  Each thread owns 8 contiguous
// pixels of a row (one 8-byte load) and marches down a chunk of rows.  Both
// stencils are separable, so each row is reduced once to per-pixel
// horizontal features and the output combines the features of rows r-1, r,
// r+1:
//   Sobel: D = x[c+1] - x[c-1],  S = x[c-1] + 2 x[c] + x[c+1]
//          gx = D(r-1) + 2 D(r) + D(r+1),  gy = S(r+1) - S(r-1)
//   Life : T = x[c-1] + x[c] + x[c+1];  n = T(r-1) + T(r) + T(r+1) - x
// Sobel's border rule (off-image neighbours read as the CENTRE pixel,
// apps/sobel.py:53-56) is not separable; border pixels take a generic 9-tap
// path.  Magnitude rounding: for every achievable n = gx^2 + gy^2,
// min(255, rint(sqrt(n))) needs sqrt only to ~1e-6 relative (n is an integer,
// so sqrt(n) is never within 4.9e-4 of a rounding boundary k+0.5 for k <= 255,
// and n >= 255.5^2 clips to 255), so the hardware sqrt.approx is exact here;
// tests compare every pixel against the reference.
#include <type_traits>

#include "sk_internal.h"
#include "sk_sweep.cuh"

namespace sk {

enum { U8_SOBEL = 0, U8_LIFE = 1 };

struct U8Args {
  Sweep2D g;
  LoopCtl L;
  // batched frames (BATCH mode): frame f at src/out + f * stride
  long long in_stride, out_stride;
  const unsigned char* bin;
  unsigned char* bout;
  long long* sums;
  int frames;
  int chunks_per_frame;
  const unsigned* magic;  // -> 0x4B000000 (Sobel lane extraction)
  unsigned* work;         // BATCH: the stream's chunk counter (0 between launches)
};

__device__ const unsigned kMagicWord = 0x4B000000u;

// device address of kMagicWord on the current device (cached per device)
inline const unsigned* magic_ptr() {
  static const unsigned* cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, kMagicWord) == cudaSuccess) cache[dev] = static_cast<const unsigned*>(p);
  }
  return cache[dev];
}

__device__ __forceinline__ int byte_of(unsigned w, int k) {
  return (int)__byte_perm(w, 0u, 0x4440u | (unsigned)k);
}

__device__ __forceinline__ int sobel_mag(int gx, int gy) {
  const int n = gx * gx + gy * gy;
  float s;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(s) : "f"((float)n));
  const int m = __float2int_rn(s);
  return m > 255 ? 255 : m;
}

// One image row as seen by a thread: 8 pixels plus the left/right neighbours.
struct Row8 {
  int x[10];  // x[0] = pixel col-1, x[1..8] = cols col..col+7, x[9] = col+8
};

struct RawRow {  // a row as loaded, before neighbour exchange
  uint2 w;
  int xl, xr;
};

__device__ __forceinline__ unsigned pack4(int a, int b, int c, int d) {
  const unsigned ab = __byte_perm((unsigned)a, (unsigned)b, 0x0040u);
  const unsigned cd = __byte_perm((unsigned)c, (unsigned)d, 0x0040u);
  return __byte_perm(ab, cd, 0x5410u);
}

// Warp-granular work: a chunk is one warp's 256-pixel-wide strip of rows, so
// no block barrier is ever needed inside the sweep; warps pull chunk ids from
// the run's atomic counter.  Rows are prefetched U at a time (memory-level
// parallelism), then turned into features and outputs.
template <int OP, int BLOCK, int REDUCE, bool BATCH>
__global__ void __launch_bounds__(BLOCK) u8_sweep(const __grid_constant__ U8Args a) {
  constexpr int VEC = 8;
  constexpr int U = 4;
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ double sh[BLOCK / 32];
  const Sweep2D& g = a.g;
  for (long long it = BATCH ? 1 : loop_enter(a.L); it != 0;
       it = BATCH ? 0 : loop_next<BLOCK>(a.L, it, sh)) {
  const int lane = threadIdx.x & 31;
  const int cols = g.cols, rows = g.rows;
  const int total = BATCH ? a.frames * a.chunks_per_frame : a.L.part_chunk[a.L.nparts];

  // chunks come from an atomic counter (loop mode: the run's; batched
  // frames: the stream's, which the last fetch resets to 0 -- every warp
  // makes exactly one fetch past the end, so fetch total + warps - 1 is the
  // last use of the counter in this launch)
  unsigned* const work = BATCH ? a.work : &a.L.st->work;
  for (;;) {
    int c = 0;
    if (lane == 0) {
      c = (int)atomicAdd(work, 1u);
      if (BATCH && c == total + (int)(gridDim.x * (BLOCK / 32)) - 1) *work = 0u;
    }
    c = __shfl_sync(FULL, c, 0);
    if (c >= total) break;
    int frame = 0, cb, r0, r1, cc = c;
    const unsigned char* front;
    unsigned char* back;
    long long fp, op;
    if (BATCH) {
      frame = c / a.chunks_per_frame;
      cc = c - frame * a.chunks_per_frame;
      front = a.bin + frame * a.in_stride;
      back = a.bout + frame * a.out_stride;
      fp = g.src_pitch;
      op = g.pitch;
    } else {
      front = static_cast<const unsigned char*>(it == 1 ? g.src : g.buf[(it - 1) & 1]);
      fp = it == 1 ? g.src_pitch : g.pitch;
      back = static_cast<unsigned char*>(g.buf[it & 1]);
      op = g.pitch;
    }
    chunk_geom(a.L, g, cc, &cb, &r0, &r1);
    const int col = cb * (32 * VEC) + lane * VEC;
    const int nvalid = cols - col;
    const bool active = nvalid > 0;
    const bool has_l = lane == 0 && col > 0 && active;
    const bool has_r = lane == 31 && nvalid > VEC;
    const bool edge_col = active && (col == 0 || nvalid <= VEC);

    auto fetch = [&](int r) -> RawRow {
      RawRow R;
      R.w = make_uint2(0u, 0u);
      R.xl = R.xr = 0;
      if (active && r >= 0 && r < rows) {
        const unsigned char* p = front + (long long)r * fp + col;
        R.w = __ldg(reinterpret_cast<const uint2*>(p));
        if (has_l) R.xl = __ldg(p - 1);
        if (has_r) R.xr = __ldg(p + VEC);
      }
      return R;
    };
    auto expand = [&](const RawRow& R, Row8& X) {
      const unsigned lo_prev = __shfl_up_sync(FULL, R.w.y, 1);
      const unsigned hi_next = __shfl_down_sync(FULL, R.w.x, 1);
      X.x[0] = lane != 0 ? byte_of(lo_prev, 3) : R.xl;
      X.x[9] = lane != 31 ? byte_of(hi_next, 0) : R.xr;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        X.x[1 + k] = byte_of(R.w.x, k);
        X.x[5 + k] = byte_of(R.w.y, k);
      }
      // off-image columns read 0 (Life: dead); Sobel border pixels are
      // recomputed by the generic path
      if (nvalid < VEC + 1) {
#pragma unroll
        for (int k = 1; k <= VEC + 1; ++k)
          if (k > nvalid) X.x[k] = 0;
      }
      if (col == 0) X.x[0] = 0;
    };

    int acc_i = 0;                                // SUM (fits: 255*8*256)
    int acc_m = REDUCE == SK_REDUCE_MAX ? -1 : 0;  // MAX
    Row8 up, cen, dn;
    expand(fetch(r0 - 1), up);
    expand(fetch(r0), cen);
    int hA[VEC], hB[VEC], hA2[VEC], hB2[VEC];  // Sobel: D, S of rows r-1, r; Life: T in hA
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      if (OP == U8_SOBEL) {
        hA[k] = up.x[k + 2] - up.x[k];
        hB[k] = up.x[k] + 2 * up.x[k + 1] + up.x[k + 2];
        hA2[k] = cen.x[k + 2] - cen.x[k];
        hB2[k] = cen.x[k] + 2 * cen.x[k + 1] + cen.x[k + 2];
      } else {
        hA[k] = up.x[k] + up.x[k + 1] + up.x[k + 2];
        hA2[k] = cen.x[k] + cen.x[k + 1] + cen.x[k + 2];
        hB[k] = hB2[k] = 0;
      }
    }
    for (int r = r0; r < r1; r += U) {
      RawRow pre[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (r + u < r1) pre[u] = fetch(r + u + 1);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int rr = r + u;
        if (rr < r1) {
          expand(pre[u], dn);
          int out[VEC];
#pragma unroll
          for (int k = 0; k < VEC; ++k) {
            if (OP == U8_SOBEL) {
              const int d3 = dn.x[k + 2] - dn.x[k];
              const int s3 = dn.x[k] + 2 * dn.x[k + 1] + dn.x[k + 2];
              out[k] = sobel_mag(hA[k] + 2 * hA2[k] + d3, s3 - hB[k]);
              hA[k] = hA2[k];
              hB[k] = hB2[k];
              hA2[k] = d3;
              hB2[k] = s3;
            } else {
              const int t3 = dn.x[k] + dn.x[k + 1] + dn.x[k + 2];
              const int x = cen.x[k + 1];
              const int n = hA[k] + hA2[k] + t3 - x;
              out[k] = (n == 3 || (x == 1 && n == 2)) ? 1 : 0;
              hA[k] = hA2[k];
              hA2[k] = t3;
            }
          }
          if (OP == U8_SOBEL && (rr == 0 || rr == rows - 1 || edge_col)) {
            // generic 9-tap: off-image reads are replaced by the centre pixel
            const bool uok = rr > 0, dok = rr < rows - 1;
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
              const int cc0 = col + k;
              const bool lok = cc0 > 0, rok = cc0 + 1 < cols;
              const int ctr = cen.x[k + 1];
              const int nw = (uok && lok) ? up.x[k] : ctr, n = uok ? up.x[k + 1] : ctr;
              const int ne = (uok && rok) ? up.x[k + 2] : ctr;
              const int w = lok ? cen.x[k] : ctr, e = rok ? cen.x[k + 2] : ctr;
              const int sw = (dok && lok) ? dn.x[k] : ctr, s = dok ? dn.x[k + 1] : ctr;
              const int se = (dok && rok) ? dn.x[k + 2] : ctr;
              out[k] = sobel_mag(-nw + ne - 2 * w + 2 * e - sw + se,
                                 -nw - 2 * n - ne + sw + 2 * s + se);
            }
          }
          if (nvalid < VEC) {
#pragma unroll
            for (int k = 0; k < VEC; ++k)
              if (k >= nvalid) out[k] = 0;  // row padding stays zero; not reduced
          }
#pragma unroll
          for (int k = 0; k < VEC; ++k) {
            if (REDUCE == SK_REDUCE_MAX) acc_m = k < nvalid ? max(acc_m, out[k]) : acc_m;
            else acc_i += out[k];
          }
          if (active)
            *reinterpret_cast<uint2*>(back + (long long)rr * op + col) = make_uint2(
                pack4(out[0], out[1], out[2], out[3]), pack4(out[4], out[5], out[6], out[7]));
          up = cen;
          cen = dn;
        }
      }
    }
    double v;
    if (REDUCE == SK_REDUCE_MAX) {
      int m = acc_m;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(FULL, m, o));
      v = m < 0 ? -INFINITY : (double)m;
    } else {
      v = (double)__reduce_add_sync(FULL, (unsigned)acc_i);
    }
    if (lane == 0) {
      if (BATCH) atomicAdd(reinterpret_cast<unsigned long long*>(&a.sums[frame]),
                           (unsigned long long)v);
      else a.L.partials[c] = v;
    }
  }
  }  // iterations
}

// ---------------------------------------------------------------- Sobel, SWAR
// Packed form of the separable Sobel: two pixels per 32-bit register in
// 16-bit lanes, biased so no lane ever borrows from its neighbour.
//   P_i = (x_{2i}, x_{2i+1}),  F_i = (x_{2i-1}, x_{2i})  (funnel shifts)
//   L_i = F_i, R_i = F_{i+1}
//   S_i = L_i + 2 P_i + R_i                 in [0, 1020]
//   D_i = R_i - L_i + 256                   in [1, 511]
//   gx' = D(r-1) + 2 D(r) + D(r+1)          = gx + 1024 in [4, 2044]
//   gy' = S(r+1) - S(r-1) + 1024            = gy + 1024 in [4, 2044]
// Each lane becomes an exact fp32 (2^23 + v, magic), n = gx^2 + gy^2 is exact
// in fp32 (< 2^24), and cvt.rni.sat.u8 rounds half-to-even and clips to 255
// in one instruction -- the reference's min(255, rint(sqrt(n))).
// K = 0x4B000000 (the exponent bits of 2^23).  A PRMT has one immediate
// slot; with both K and the selector constant, ptxas keeps K immediate and
// re-materialises the selector into a register before every use (2 extra
// moves per pixel).  K is therefore loaded from memory once (a device
// constant), which ptxas cannot fold: the selectors become immediates and K
// stays in one register.
__device__ __forceinline__ unsigned lane_lo(unsigned p, unsigned K) { return __byte_perm(p, K, 0x7610u); }
__device__ __forceinline__ unsigned lane_hi(unsigned p, unsigned K) { return __byte_perm(p, K, 0x7632u); }

#ifdef SK_SOBEL_MAGIC_ROUND
// fminf + one magic add (1.5 * 2^23 forces round-half-even to an integer in
// the low mantissa byte) instead of cvt.rni.sat.u8: keeps the conversion off
// the XU pipe, which MUFU.SQRT already loads with one op per pixel.
#define SK_SOBEL_ROUND(s) __float_as_uint(__fadd_rn(fminf((s), 255.0f), 12582912.0f))
#endif

__device__ __forceinline__ unsigned sobel_byte(unsigned gxm, unsigned gym) {
  const float gx = __fsub_rn(__uint_as_float(gxm), 8389632.0f);  // (2^23 + gx') - (2^23 + 1024)
  const float gy = __fsub_rn(__uint_as_float(gym), 8389632.0f);
  const float n = __fmaf_rn(gy, gy, __fmul_rn(gx, gx));  // exact: every term < 2^24
  float s;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(n));
#ifdef SK_SOBEL_ROUND
  return SK_SOBEL_ROUND(s);  // result in the low byte
#else
  unsigned b;
  asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(b) : "f"(s));
  return b;
#endif
}

// ------------------------------------------------- Sobel, paired fp32 (f32x2)
// Blackwell issues fp32 add/mul/fma on register PAIRS (FADD2/FMUL2/FFMA2):
// one instruction, two lanes.  A thread's 8 pixels x0..x7 are held as four
// pairs Q_k = (x_k, x_{k+4}), so the left/right neighbour pairs of Q_k are
// simply Q_{k-1} / Q_{k+1} (plus two edge pairs (x_-1, x_3), (x_4, x_8)).
// Each byte becomes the exact float 2^15 + x with ONE PRMT (the byte in
// mantissa bits 8..15 under the exponent word K2 = 0x47000000); the bias
// cancels in every feature (D = R - L, S = L + 2Q + R = 2^17 + s, exact: the
// ulp at 2^17 is 2^-6), so features and outputs are the integer Sobel
// quantities with no conversion instructions:
//   gx = Dm + 2 Dc + Dp,  gy = Sp - Sm,  n = gx^2 + gy^2 (exact, < 2^22),
//   rint: sqrt(n) + 1.5 * 2^23 in one FADD (round half-to-even), leaving
//   rint(sqrt(n)) <= 1443 in the low 16 bits; the clip to 255 is one
//   VIMNMX.U16x2 per two pixels after packing.
// the CUDA 12.8+ sm_100 builtins (FADD2 / FMUL2 / FFMA2 on register pairs)
using F2 = float2;
__device__ __forceinline__ F2 f2_pack(float lo, float hi) { return make_float2(lo, hi); }
__device__ __forceinline__ void f2_unpack(F2 a, float& lo, float& hi) {
  lo = a.x;
  hi = a.y;
}
__device__ __forceinline__ F2 f2_add(F2 a, F2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ F2 f2_sub(F2 a, F2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ F2 f2_mul(F2 a, F2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ F2 f2_fma(F2 a, F2 b, F2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ F2 f2_splat(float x) { return f2_pack(x, x); }

// byte k (0..3) of w -> float 2^15 + byte (K2 = 0x47000000)
template <int k>
__device__ __forceinline__ float byte_f(unsigned w, unsigned K) {
  return __uint_as_float(__byte_perm(w, K, 0x7604u | (k << 4)));
}

// rint(sqrt(n)) in the low 16 bits of each returned word
__device__ __forceinline__ void sobel_round2(F2 n, unsigned& lo, unsigned& hi) {
  float a, b;
  f2_unpack(n, a, b);
  asm("sqrt.approx.ftz.f32 %0, %0;" : "+f"(a));
  asm("sqrt.approx.ftz.f32 %0, %0;" : "+f"(b));
  F2 r = f2_add(f2_pack(a, b), f2_splat(12582912.0f));
  float x, y;
  f2_unpack(r, x, y);
  lo = __float_as_uint(x);
  hi = __float_as_uint(y);
}

#ifndef SK_SOBEL_MINB
#define SK_SOBEL_MINB 4
#endif
#ifndef SK_SOBEL_UNROLL
#define SK_SOBEL_UNROLL 2
#endif
constexpr int kSobelUnroll = SK_SOBEL_UNROLL;

// cp.async primitives (shared addresses are 32-bit)
__device__ __forceinline__ void cp_async8(unsigned dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4_if(bool p, unsigned dst, const void* src) {
  asm volatile(
      "{ .reg .pred q; setp.ne.b32 q, %0, 0; @q cp.async.ca.shared.global [%1], [%2], 4; }" ::"r"(
          (int)p),
      "r"(dst), "l"(src)
      : "memory");
}
__device__ __forceinline__ void st_global_if(bool p, void* q, unsigned v) {
  asm volatile("{ .reg .pred r; setp.ne.b32 r, %0, 0; @r st.global.u32 [%1], %2; }" ::"r"((int)p),
               "l"(q), "r"(v)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One border pixel with the reference's rule (off-image reads = centre),
// reading the three rows straight from memory.  Out of line: border work is
// rare, and inlining it would bloat the hot loop's instruction footprint.
__device__ __noinline__ unsigned sobel_border_px(const unsigned char* front, long long fp, int r,
                                                 int c, int rows, int cols) {
  const int ctr = front[(long long)r * fp + c];
  auto at = [&](int i, int j) -> int {
    return (i < 0 || i >= rows || j < 0 || j >= cols) ? ctr : (int)front[(long long)i * fp + j];
  };
  const int nw = at(r - 1, c - 1), n = at(r - 1, c), ne = at(r - 1, c + 1);
  const int w = at(r, c - 1), e = at(r, c + 1);
  const int sw = at(r + 1, c - 1), so = at(r + 1, c), se = at(r + 1, c + 1);
  return (unsigned)sobel_mag(-nw + ne - 2 * w + 2 * e - sw + se, -nw - 2 * n - ne + sw + 2 * so + se);
}

template <int BLOCK, int REDUCE, bool BATCH, bool PAIRED>
__global__ void __launch_bounds__(BLOCK, PAIRED ? SK_SOBEL_MINB : 1) sobel_sweep(const __grid_constant__ U8Args a) {
  constexpr int VEC = 8;
  constexpr int U = 6;  // multiple of the 3-row feature rotation: no register moves
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ double sh[BLOCK / 32];
  // PAIRED: per-warp ring of RING input-row slots
#ifndef SK_SOBEL_RING
#define SK_SOBEL_RING 8
#endif
  constexpr int RING = SK_SOBEL_RING, SLOT = 288;  // RING: a power of two
  __shared__ __align__(128) unsigned char ring_mem[PAIRED ? (BLOCK / 32) * RING * SLOT : 16];
  unsigned K;  // 0x4B000000, opaque to the compiler (see lane_lo)
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(K) : "l"(a.magic));
  const unsigned K2 = K - 0x04000000u;  // 0x47000000: exponent word of 2^15 (PAIRED)
  const Sweep2D& g = a.g;
  const unsigned ring = (unsigned)__cvta_generic_to_shared(ring_mem) +
                        (PAIRED ? (threadIdx.x >> 5) * RING * SLOT : 0u);
  for (long long it = BATCH ? 1 : loop_enter(a.L); it != 0;
       it = BATCH ? 0 : loop_next<BLOCK>(a.L, it, sh)) {
  const int lane = threadIdx.x & 31;
  const int cols = g.cols, rows = g.rows;
  const int total = BATCH ? a.frames * a.chunks_per_frame : a.L.part_chunk[a.L.nparts];

  // chunks come from an atomic counter (loop mode: the run's; batched
  // frames: the stream's, which the last fetch resets to 0 -- every warp
  // makes exactly one fetch past the end, so fetch total + warps - 1 is the
  // last use of the counter in this launch)
  unsigned* const work = BATCH ? a.work : &a.L.st->work;
  for (;;) {
    int c = 0;
    if (lane == 0) {
      c = (int)atomicAdd(work, 1u);
      if (BATCH && c == total + (int)(gridDim.x * (BLOCK / 32)) - 1) *work = 0u;
    }
    c = __shfl_sync(FULL, c, 0);
    if (c >= total) break;
    int frame = 0, cb, r0, r1, cc = c;
    const unsigned char* front;
    unsigned char* back;
    long long fp, op;
    if (BATCH) {
      frame = c / a.chunks_per_frame;
      cc = c - frame * a.chunks_per_frame;
      front = a.bin + frame * a.in_stride;
      back = a.bout + frame * a.out_stride;
      fp = g.src_pitch;
      op = g.pitch;
    } else {
      front = static_cast<const unsigned char*>(it == 1 ? g.src : g.buf[(it - 1) & 1]);
      fp = it == 1 ? g.src_pitch : g.pitch;
      back = static_cast<unsigned char*>(g.buf[it & 1]);
      op = g.pitch;
    }
    chunk_geom(a.L, g, cc, &cb, &r0, &r1);
    const int col = cb * (32 * VEC) + lane * VEC;
    const int nvalid = cols - col;
    const bool active = nvalid > 0;
    // Loads are never predicated: lanes past the image width read column 0
    // (their bytes are masked), and the rows above/below the image read row
    // 0 / rows-1 (those output rows are recomputed by the border pass).
    const int lcol = active ? col : 0;
    const int lsh = (lane == 0 && lcol > 0) ? -1 : 0;  // edge-lane scalar loads
    const int rsh = (lane == 31 && nvalid > VEC) ? VEC : 0;
    const bool ledge = lane == 0, redge = lane == 31;
    // bytes of this lane's 8 that lie inside the image (the rest store 0)
    const unsigned mlo = nvalid >= 4 ? 0xffffffffu : (nvalid <= 0 ? 0u : 0xffffffffu >> (32 - 8 * nvalid));
    const unsigned mhi = nvalid >= 8 ? 0xffffffffu : (nvalid <= 4 ? 0u : 0xffffffffu >> (64 - 8 * nvalid));
    const unsigned char* pbase = front + lcol;
    const unsigned char* plast = pbase + (long long)(rows - 1) * fp;

    auto fetch = [&](const unsigned char* p, uint2& w, unsigned& xl, unsigned& xr) {
      w = __ldg(reinterpret_cast<const uint2*>(p));
      xl = __ldg(p + lsh);  // lanes without a left neighbour load their own byte (unused)
      xr = __ldg(p + rsh);
    };
    auto features = [&](uint2 w, unsigned exl, unsigned exr, unsigned* S, unsigned* D) {
      const unsigned lo_prev = __shfl_up_sync(FULL, w.y, 1);
      const unsigned hi_next = __shfl_down_sync(FULL, w.x, 1);
      const unsigned xl = ledge ? exl : (lo_prev >> 24);
      const unsigned xr = redge ? exr : (hi_next & 0xffu);
      unsigned P[4], F[5];
      P[0] = __byte_perm(w.x, 0u, 0x4140u);
      P[1] = __byte_perm(w.x, 0u, 0x4342u);
      P[2] = __byte_perm(w.y, 0u, 0x4140u);
      P[3] = __byte_perm(w.y, 0u, 0x4342u);
      F[0] = __funnelshift_l(xl << 16, P[0], 16);
      F[1] = __funnelshift_l(P[0], P[1], 16);
      F[2] = __funnelshift_l(P[1], P[2], 16);
      F[3] = __funnelshift_l(P[2], P[3], 16);
      F[4] = __funnelshift_l(P[3], xr, 16);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        S[i] = F[i] + F[i + 1] + (P[i] << 1);
        D[i] = F[i + 1] - F[i] + 0x01000100u;
      }
    };
    auto emit = [&](const unsigned* Sm, const unsigned* Dm, const unsigned* Dc, const unsigned* Sp,
                    const unsigned* Dp, unsigned char* po, unsigned& acc, int& accm) {
      unsigned ob[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const unsigned gxp = Dm[i] + (Dc[i] << 1) + Dp[i];
        const unsigned gyp = Sp[i] - Sm[i] + 0x04000400u;
        ob[2 * i] = sobel_byte(lane_lo(gxp, K), lane_lo(gyp, K));
        ob[2 * i + 1] = sobel_byte(lane_hi(gxp, K), lane_hi(gyp, K));
      }
      const unsigned lo = pack4((int)ob[0], (int)ob[1], (int)ob[2], (int)ob[3]) & mlo;
      const unsigned hi = pack4((int)ob[4], (int)ob[5], (int)ob[6], (int)ob[7]) & mhi;
      if (REDUCE == SK_REDUCE_MAX) {
        const unsigned m = __vmaxu4(lo, hi);
        const unsigned m2 = __vmaxu4(m, m >> 16);
        accm = max(accm, (int)max(m2 & 0xffu, (m2 >> 8) & 0xffu));
      } else {
        acc = __dp4a(lo, 0x01010101u, acc);
        acc = __dp4a(hi, 0x01010101u, acc);
      }
      if (active) *reinterpret_cast<uint2*>(po) = make_uint2(lo, hi);
    };

    unsigned acc = 0;
    int accm = -1;
    auto finish = [&](unsigned lo, unsigned hi, unsigned char* q) {
      lo &= mlo;
      hi &= mhi;
      if (REDUCE == SK_REDUCE_MAX) {
        const unsigned m = __vmaxu4(lo, hi);
        const unsigned m2 = __vmaxu4(m, m >> 16);
        accm = max(accm, (int)max(m2 & 0xffu, (m2 >> 8) & 0xffu));
      } else {
        acc = __dp4a(lo, 0x01010101u, acc);
        acc = __dp4a(hi, 0x01010101u, acc);
      }
      if (active) *reinterpret_cast<uint2*>(q) = make_uint2(lo, hi);
    };
    if constexpr (PAIRED) {
    // Input rows stream through the warp's shared-memory ring by cp.async,
    // RING - 2 rows ahead of the row being consumed, so the bytes in flight
    // cost no registers.  Slot byte 16 + j holds column cb*256 + j: each lane
    // copies its own 8 bytes plus the 4-byte words either side of them (the
    // inner ones duplicate a neighbour lane's bytes; the outer ones are the
    // warp's left / right neighbour columns), so every lane runs the same
    // copy pattern with immediate offsets.  Bytes outside the image only
    // reach masked lanes or border pixels, which the border pass redoes.
    const int n_in = r1 - r0 + 2;  // input rows r0-1 .. r1, clamped to the image
    const unsigned dst = ring + 16 + lane * VEC;  // this lane's bytes in slot 0
    const bool cpl = lcol > 0, cpr = nvalid > VEC;  // neighbour words inside the row
    // copies past the chunk's last input row repeat that row (an L2 hit)
    const int rlim = r1 < rows - 1 ? r1 : rows - 1;
    const unsigned fp32 = (unsigned)fp;  // pitches < 2^31 (checked by the host)
    int ri = r0 - 1;  // image row of the next copy
    auto issue = [&](unsigned so) {  // one commit group per call
      const unsigned rc = (unsigned)min(max(ri, 0), rlim);
      const unsigned char* p;  // pbase + rc * pitch in one IMAD.WIDE.U32
      asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(rc), "r"(fp32), "l"(pbase));
      cp_async8(dst + so, p);
      cp_async4_if(cpl, dst + so - 4, p - 4);
      cp_async4_if(cpr, dst + so + VEC, p + VEC);
      cp_async_commit();
      ++ri;
    };
    // Compute layout (independent of the copy layout): lane j owns pixel
    // quads X = columns c0+4j .. +3 and Y = c0+128+4j .. +3, paired as
    // Q_t = (x_t, y_t); the neighbour pairs are (x_-1, y_-1) and (x_4, y_4),
    // all read from the slot, so no value sits in two register pairs.
    const int colx = cb * (32 * VEC) + lane * 4;
    const unsigned qx = ring + 16 + lane * 4;  // X quad in slot 0 (Y at +128)
    const int nx = cols - colx, ny = nx - 128;
    const unsigned mx = nx >= 4 ? 0xffffffffu : (nx <= 0 ? 0u : 0xffffffffu >> (32 - 8 * nx));
    const unsigned my = ny >= 4 ? 0xffffffffu : (ny <= 0 ? 0u : 0xffffffffu >> (32 - 8 * ny));
    // features of the input row in slot `so`; its slot is then refilled
    auto take = [&](unsigned so, F2* S, F2* D) {
      cp_async_wait<RING - 2>();
      __syncwarp();  // the slot holds bytes copied by other lanes
      const unsigned px = qx + so;
      unsigned wx, wy, xl, xr, yl, yr;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wx) : "r"(px) : "memory");
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wy) : "r"(px + 128) : "memory");
      asm volatile("ld.shared.u8 %0, [%1];" : "=r"(xl) : "r"(px - 1) : "memory");
      asm volatile("ld.shared.u8 %0, [%1];" : "=r"(xr) : "r"(px + 4) : "memory");
      asm volatile("ld.shared.u8 %0, [%1];" : "=r"(yl) : "r"(px + 127) : "memory");
      asm volatile("ld.shared.u8 %0, [%1];" : "=r"(yr) : "r"(px + 132) : "memory");
      // refill the slot read by the previous step (those reads are complete:
      // this step's __syncwarp follows them)
      issue(so == 0 ? (RING - 1) * SLOT : so - SLOT);
      const F2 Q0 = f2_pack(byte_f<0>(wx, K2), byte_f<0>(wy, K2));
      const F2 Q1 = f2_pack(byte_f<1>(wx, K2), byte_f<1>(wy, K2));
      const F2 Q2 = f2_pack(byte_f<2>(wx, K2), byte_f<2>(wy, K2));
      const F2 Q3 = f2_pack(byte_f<3>(wx, K2), byte_f<3>(wy, K2));
      const F2 L0 = f2_pack(byte_f<0>(xl, K2), byte_f<0>(yl, K2));
      const F2 R3 = f2_pack(byte_f<0>(xr, K2), byte_f<0>(yr, K2));
      const F2 two = f2_splat(2.0f);
      S[0] = f2_fma(Q0, two, f2_add(L0, Q1));
      S[1] = f2_fma(Q1, two, f2_add(Q0, Q2));
      S[2] = f2_fma(Q2, two, f2_add(Q1, Q3));
      S[3] = f2_fma(Q3, two, f2_add(Q2, R3));
      D[0] = f2_sub(Q1, L0);
      D[1] = f2_sub(Q2, Q0);
      D[2] = f2_sub(Q3, Q1);
      D[3] = f2_sub(R3, Q2);
    };
    // Running state at input row i: G = D(i-2) + 2 D(i-1) (gx of output row
    // i-1 before its lower neighbour), S(i-2), S(i-1), D(i-1).  Output row
    // i-1 = (G + D(i), S(i) - S(i-2)).  Two S and two D arrays alternate, so
    // a pair of steps needs no register moves.
    F2 G[4], SA[4], SB[4], DA[4], DB[4];
    unsigned char* po = back + (long long)r0 * op + colx;
    const F2 two_c = f2_splat(2.0f);
    // FULL (every column of the warp's strip inside the image -- all but the
    // last column block): no byte masks, unconditional stores
    auto step = [&](auto full, unsigned so, F2* Sold, F2* Dprev, F2* Dnew) {
      constexpr bool FULL = decltype(full)::value;
      F2 S[4];
      take(so, S, Dnew);
      unsigned o[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const F2 gx = f2_add(G[k], Dnew[k]);
        const F2 gy = f2_sub(S[k], Sold[k]);
        sobel_round2(f2_fma(gx, gx, f2_mul(gy, gy)), o[k], o[k + 4]);
        G[k] = f2_fma(Dnew[k], two_c, Dprev[k]);
        Sold[k] = S[k];
      }
      const unsigned x01 = __vminu2(__byte_perm(o[0], o[1], 0x5410u), 0x00ff00ffu);
      const unsigned x23 = __vminu2(__byte_perm(o[2], o[3], 0x5410u), 0x00ff00ffu);
      const unsigned y01 = __vminu2(__byte_perm(o[4], o[5], 0x5410u), 0x00ff00ffu);
      const unsigned y23 = __vminu2(__byte_perm(o[6], o[7], 0x5410u), 0x00ff00ffu);
      unsigned ox = __byte_perm(x01, x23, 0x6420u);
      unsigned oy = __byte_perm(y01, y23, 0x6420u);
      if constexpr (!FULL) {
        ox &= mx;
        oy &= my;
      }
      if (REDUCE == SK_REDUCE_MAX) {
        const unsigned m = __vmaxu4(ox, oy);
        const unsigned m2 = __vmaxu4(m, m >> 16);
        accm = max(accm, (int)max(m2 & 0xffu, (m2 >> 8) & 0xffu));
      } else {
        acc = __dp4a(ox, 0x01010101u, acc);
        acc = __dp4a(oy, 0x01010101u, acc);
      }
      if (FULL || nx > 0) *reinterpret_cast<unsigned*>(po) = ox;
      if (FULL || ny > 0) *reinterpret_cast<unsigned*>(po + 128) = oy;
      po += op;
    };
#pragma unroll
    for (int u = 0; u < RING - 1; ++u) issue(u * SLOT);
    take(0, SA, DA);  // input row 0 (r0-1): S in SA, D in DA
    take(SLOT, SB, DB);  // input row 1 (r0)
#pragma unroll
    for (int k = 0; k < 4; ++k) G[k] = f2_fma(DB[k], two_c, DA[k]);
    // step i: S(i-2) is in SA for even i, SB for odd i; D(i-1) in DB / DA
    auto rows_loop = [&](auto full) {
      int i = 2;
#pragma unroll (kSobelUnroll)
      for (; i + 2 <= n_in; i += 2) {
        step(full, (i & (RING - 1)) * SLOT, SA, DB, DA);
        step(full, ((i + 1) & (RING - 1)) * SLOT, SB, DA, DB);
      }
      if (i < n_in) step(full, (i & (RING - 1)) * SLOT, SA, DB, DA);
    };
    if (cols - cb * (32 * VEC) >= 32 * VEC) rows_loop(std::true_type{});
    else rows_loop(std::false_type{});
    } else {
    unsigned S0[4], D0[4], S1[4], D1[4], S2[4], D2[4];
    {
      uint2 w;
      unsigned xl, xr;
      fetch(r0 > 0 ? pbase + (long long)(r0 - 1) * fp : pbase, w, xl, xr);
      features(w, xl, xr, S0, D0);
      fetch(pbase + (long long)r0 * fp, w, xl, xr);
      features(w, xl, xr, S1, D1);
    }
    // next row to fetch is r0 + 1; only row r1 == rows (the chunk's last
    // fetch) can leave the image: clamped to rows - 1
    const unsigned char* pf = pbase + (long long)(r0 + 1) * fp;
    unsigned char* po = back + (long long)r0 * op + col;
    int r = r0;
    for (; r + U <= r1; r += U) {  // full groups: no per-row checks
      uint2 w[U];
      unsigned xl[U], xr[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned char* p = pf + u * fp;
        fetch(p > plast ? plast : p, w[u], xl[u], xr[u]);
      }
      pf += U * fp;
      // rows r..r+5 rotate the feature sets S0/S1/S2 by renaming
      features(w[0], xl[0], xr[0], S2, D2);
      emit(S0, D0, D1, S2, D2, po, acc, accm);
      po += op;
      features(w[1], xl[1], xr[1], S0, D0);
      emit(S1, D1, D2, S0, D0, po, acc, accm);
      po += op;
      features(w[2], xl[2], xr[2], S1, D1);
      emit(S2, D2, D0, S1, D1, po, acc, accm);
      po += op;
      features(w[3], xl[3], xr[3], S2, D2);
      emit(S0, D0, D1, S2, D2, po, acc, accm);
      po += op;
      features(w[4], xl[4], xr[4], S0, D0);
      emit(S1, D1, D2, S0, D0, po, acc, accm);
      po += op;
      features(w[5], xl[5], xr[5], S1, D1);
      emit(S2, D2, D0, S1, D1, po, acc, accm);
      po += op;
    }
#pragma unroll 1
    for (; r < r1; ++r) {  // tail rows
      uint2 w;
      unsigned xl, xr;
      fetch(pf > plast ? plast : pf, w, xl, xr);
      pf += fp;
      features(w, xl, xr, S2, D2);
      emit(S0, D0, D1, S2, D2, po, acc, accm);
      po += op;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        S0[i] = S1[i];
        D0[i] = D1[i];
        S1[i] = S2[i];
        D1[i] = D2[i];
      }
    }
    }  // SWAR
    // Border pass: pixels of image rows 0 / rows-1 and columns 0 / cols-1
    // follow the centre-substitution rule.  Border rows: each lane redoes its
    // own 8 pixels.  Border columns: the warp's lanes split the chunk's rows
    // (the column is owned by one lane, the work is spread over all 32).
    // Each redo corrects the lane's running sum by (new - old).
    const bool top = r0 == 0, bottom = r1 == rows;
    const int c_first = cb * (32 * VEC);
    const bool has_c0 = cb == 0;                                        // column 0 here
    const bool has_cl = cols - 1 >= c_first && cols - 1 < c_first + 32 * VEC;  // column cols-1
    if (top || bottom || has_c0 || has_cl) {
      __syncwarp();  // the owners' stores are visible to the lanes that redo them
      auto redo = [&](int rr, int cc2) {
        unsigned char* q = back + (long long)rr * op + cc2;
        const unsigned old = *q;
        const unsigned nv = sobel_border_px(front, fp, rr, cc2, rows, cols);
        *q = (unsigned char)nv;
        acc += nv - old;
      };
      if (active) {
        const int kmax = nvalid < VEC ? nvalid : VEC;
        if (top) for (int k = 0; k < kmax; ++k) redo(0, col + k);
        if (bottom && !(top && rows == 1)) for (int k = 0; k < kmax; ++k) redo(rows - 1, col + k);
      }
      const int ra = top ? 1 : r0, rb = bottom ? rows - 1 : r1;  // rows not yet redone
      for (int rr = ra + lane; rr < rb; rr += 32) {
        if (has_c0) redo(rr, 0);
        if (has_cl && cols > 1) redo(rr, cols - 1);
      }
      __syncwarp();
      if (REDUCE == SK_REDUCE_MAX) {  // rare: recompute this lane's max from what was stored
        __syncwarp();
        accm = -1;
        if (active)
          for (int rr = r0; rr < r1; ++rr)
            for (int k = 0; k < VEC && k < nvalid; ++k)
              accm = max(accm, (int)back[(long long)rr * op + col + k]);
      }
    }
    double v;
    if (REDUCE == SK_REDUCE_MAX) {
      int m = active ? accm : -1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(FULL, m, o));
      v = m < 0 ? -INFINITY : (double)m;
    } else {
      v = (double)__reduce_add_sync(FULL, acc);  // border redos may sit on any lane
    }
    if (lane == 0) {
      if (BATCH) atomicAdd(reinterpret_cast<unsigned long long*>(&a.sums[frame]),
                           (unsigned long long)v);
      else a.L.partials[c] = v;
    }
  }
  }  // iterations
}

// ---------------------------------------------------------------- host side

namespace {

constexpr int kBlock = 128;
constexpr int kVec = 8;
// Sobel feature form: f32x2 pairs (default) or the 16-bit SWAR kernel
// (SK_SOBEL_SWAR=1, kept for A/B measurement)
bool sobel_swar() {
  static const bool v = [] {
    const char* e = getenv("SK_SOBEL_SWAR");
    return e && e[0] == '1';
  }();
  return v;
}

using U8Fn = void (*)(const U8Args);

// aligned16: every row start the sweep reads is 16-byte aligned (the
// bulk-copy ring needs it); otherwise Sobel takes the SWAR kernel
U8Fn pick(int op, int reduce, bool batch, bool aligned16) {
  if (op == U8_SOBEL && (sobel_swar() || !aligned16)) {
    if (batch) return sobel_sweep<kBlock, SK_REDUCE_SUM, true, false>;
    return reduce == SK_REDUCE_MAX ? sobel_sweep<kBlock, SK_REDUCE_MAX, false, false>
                                   : sobel_sweep<kBlock, SK_REDUCE_SUM, false, false>;
  }
  if (batch) return op == U8_SOBEL ? sobel_sweep<kBlock, SK_REDUCE_SUM, true, true>
                                   : u8_sweep<U8_LIFE, kBlock, SK_REDUCE_SUM, true>;
  if (op == U8_SOBEL)
    return reduce == SK_REDUCE_MAX ? sobel_sweep<kBlock, SK_REDUCE_MAX, false, true>
                                   : sobel_sweep<kBlock, SK_REDUCE_SUM, false, true>;
  return reduce == SK_REDUCE_MAX ? u8_sweep<U8_LIFE, kBlock, SK_REDUCE_MAX, false>
                                 : u8_sweep<U8_LIFE, kBlock, SK_REDUCE_SUM, false>;
}

// chunk geometry shared by loop and batch mode; returns slots (grid cap)
int geometry(int device, U8Fn fn, long long rows, long long cols, int nparts, const int* part_row,
             long long frames, int* colblocks, int* chunk_rows, int* part_chunk, int* nchunks,
             int* grid) {
  const long long slots =
      (long long)device_sms(device) * occupancy(reinterpret_cast<const void*>(fn), kBlock);
  *colblocks = (int)((cols + 32 * kVec - 1) / (32 * kVec));  // one warp per chunk
#ifndef SK_U8_CHUNKS_PER_WARP
#define SK_U8_CHUNKS_PER_WARP 16
#endif
  const long long want = slots * (kBlock / 32) * SK_U8_CHUNKS_PER_WARP;
  long long ch = (rows * (long long)*colblocks * frames + want - 1) / want;
  ch = ch < 8 ? 8 : (ch > 256 ? 256 : ch);
  ch = (ch + 11) / 12 * 12;  // whole prefetch groups (Life: 4 rows, Sobel: 6)
  *chunk_rows = (int)ch;
  int n = 0;
  part_chunk[0] = 0;
  for (int i = 0; i < nparts; ++i) {
    const int pr = part_row[i + 1] - part_row[i];
    n += ((pr + *chunk_rows - 1) / *chunk_rows) * *colblocks;
    part_chunk[i + 1] = n;
  }
  *nchunks = n;
  const long long tot = (long long)n * frames;
  *grid = (int)(slots < tot ? slots : tot);
  if (*grid < 1) *grid = 1;
  return SK_OK;
}

int op_of(const sk_run* r) { return r->plan.kernel == SK_KERNEL_LIFE ? U8_LIFE : U8_SOBEL; }

bool aligned16(const sk_run* r) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return r->src_pitch % 16 == 0 && r->pitch % 16 == 0 && r->src_pitch < (1ll << 31) &&
         r->pitch < (1ll << 31) && al(r->src) && al(r->buf[0]) &&
         al(r->buf[1]);
}

int setup(sk_run* r) {
  if (r->plan.dtype != SK_U8) {
    set_error("sobel/life: grid must be u8");
    return SK_ERR_UNSUPPORTED;
  }
  if (r->plan.delta_op != SK_DELTA_NONE) {
    set_error("sobel/life: no delta reduce");
    return SK_ERR_UNSUPPORTED;
  }
  U8Fn fn = pick(op_of(r), r->plan.reduce_op, false, aligned16(r));
  return geometry(r->device, fn, r->plan.rows, r->plan.cols, r->nparts, r->part_row, 1,
                  &r->colblocks, &r->chunk_rows, r->part_chunk, &r->nchunks, &r->grid);
}

void fill_geom(const sk_run* r, Sweep2D& g) {
  g.src = r->src;
  g.src_pitch = r->src_pitch;
  g.buf[0] = r->buf[0];
  g.buf[1] = r->buf[1];
  g.pitch = r->pitch;
  g.env = nullptr;
  g.env_pitch = 0;
  g.rows = (int)r->plan.rows;
  g.cols = (int)r->plan.cols;
  g.halo_top = g.halo_bottom = 0;
  g.colblocks = r->colblocks;
  g.chunk_rows = r->chunk_rows;
  for (int i = 0; i <= r->nparts; ++i) g.part_row[i] = r->part_row[i];
}

int launch(sk_run* r, const LoopCtl& L, cudaStream_t s) {
  U8Args a{};
  a.magic = magic_ptr();
  fill_geom(r, a.g);
  a.L = L;
  U8Fn fn = pick(op_of(r), r->plan.reduce_op, false, aligned16(r));
  SK_CUDA(launch_kernel(fn, r->grid, kBlock, a, s, L.persistent != 0));
  return SK_OK;
}

void teardown(sk_run*) {}

const KernelOps kOps = {setup, launch, teardown};

}  // namespace

const KernelOps* u8_ops() { return &kOps; }

// Batched Sobel over frames (stream mode): one memset (the per-frame sums)
// and one launch per call.
int sobel_frames(const uint8_t* in, long long in_pitch, long long in_fs, uint8_t* out,
                 long long out_pitch, long long out_fs, int frames, long long rows, long long cols,
                 long long* sums, cudaStream_t s) {
  if (!in || !out || !sums || frames < 1 || rows < 1 || cols < 1 || in_pitch < cols ||
      out_pitch < cols || (in_pitch % 8) || (out_pitch % 8) || (in_fs % 8) || (out_fs % 8) ||
      (reinterpret_cast<uintptr_t>(in) % 8) || (reinterpret_cast<uintptr_t>(out) % 8)) {
    set_error("sk_sobel_frames: bad arguments (pitches/strides/pointers must be 8-byte aligned)");
    return SK_ERR_ARG;
  }
  {
    const int rc = sobel_frames_tma(in, in_pitch, in_fs, out, out_pitch, out_fs, frames, rows, cols,
                                    sums, s);
    if (rc != SK_ERR_UNSUPPORTED) return rc;
  }
  int dev = 0;
  SK_CUDA(cudaGetDevice(&dev));
  const bool al16 = in_pitch % 16 == 0 && in_fs % 16 == 0 && in_pitch < (1ll << 31) &&
                    (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  U8Fn fn = pick(U8_SOBEL, SK_REDUCE_SUM, true, al16);
  U8Args a{};
  a.magic = magic_ptr();
  int part_row[2] = {0, (int)rows};
  int nch = 0, grid = 0;
  int rc = geometry(dev, fn, rows, cols, 1, part_row, frames, &a.g.colblocks, &a.g.chunk_rows,
                    a.L.part_chunk, &nch, &grid);
  if (rc) return rc;
  a.L.nparts = 1;
  a.g.part_row[0] = 0;
  a.g.part_row[1] = (int)rows;
  a.g.rows = (int)rows;
  a.g.cols = (int)cols;
  a.g.src_pitch = in_pitch;
  a.g.pitch = out_pitch;
  a.bin = in;
  a.bout = out;
  a.in_stride = in_fs;
  a.out_stride = out_fs;
  a.sums = sums;
  a.frames = frames;
  a.chunks_per_frame = nch;
  a.work = stream_counter(dev, s);
  if (!a.work) return SK_ERR_CUDA;
  SK_CUDA(cudaMemsetAsync(sums, 0, sizeof(long long) * frames, s));
  fn<<<grid, kBlock, 0, s>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sobel_frames launch");
  return SK_OK;
}

}  // namespace sk

extern "C" int sk_sobel_frames(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                               uint8_t* d_out, int64_t out_pitch, int64_t out_frame_stride,
                               int32_t frames, int64_t rows, int64_t cols, int64_t* d_sums,
                               void* stream) {
  return sk::sobel_frames(d_in, in_pitch, in_frame_stride, d_out, out_pitch, out_frame_stride,
                          frames, rows, cols, reinterpret_cast<long long*>(d_sums),
                          static_cast<cudaStream_t>(stream));
}
