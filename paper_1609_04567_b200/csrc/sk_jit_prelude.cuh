// Device-side vocabulary for user elemental functions compiled at run time
// (NVRTC, sk_jit.cu).  A JIT program is
//
//   #include "sk_jit_prelude.cuh"        <- this file
//   <generated part>                     <- paper_1609_04567_b200/jit.py
//   #include "sk_jit_kernel.cuh"         <- the fused sweep kernel
//
// The generated part (from a Python point function, or from CUDA source the
// user wrote against this API -- the paper's elemental-function-as-kernel-
// source interface) defines the element types, the
// elemental function, the delta and the combinator.
//
// Reference semantics this restates:
//   * the window: Neighborhood.at / center / center_index, ABSENT outside the
//     grid (grid.py:201-324); IndexedNeighborhood pairs (grid.py:243-256)
//   * env.at(i, j) of an aligned read-only grid, ABSENT outside (grid.py)
//   * Python arithmetic on the values (int / float division, floor division,
//     modulo, power, round, comparisons), raising where Python raises:
//     such an element records an error code and its index, and the run
//     reports StencilError for the lowest failing index (patterns.py:29-38,
//     partition.py:357-360).
#pragma once

#include "sk_common.cuh"
#include "sk_sweep.cuh"

namespace sk {

// error codes (mapped to Python exception types in jit.py)
enum : int {
  kErrNone = 0,
  kErrAbsent = 1,      // TypeError: arithmetic / truth value of ABSENT
  kErrZeroDiv = 2,     // ZeroDivisionError
  kErrDomain = 3,      // ValueError: math domain error
  kErrOverflow = 4,    // OverflowError / ValueError: int() of inf / nan
};

struct SkErr {
  int code = 0;
  __device__ __forceinline__ void set(int c) {
    if (!code) code = c;
  }
};

// The window around one grid element, staged in shared memory.  `at` reads
// the staged value (the pad value where the slot is off-grid, replicated
// border in "edge" pad mode); `ok` says whether the slot is on the grid (the
// reference's `is not ABSENT`).  IN: the whole window is known to be on the
// grid (interior tiles), so `ok` is the constant true and every ABSENT test
// in the generated elemental folds away at compile time.
struct SkEnv;

template <class V, bool IN = false, int STRIDE = 0, class E0 = float, bool PRE = false>
struct SkNb {
  const V* c;       // centre slot in the staged tile
  int stride;       // tile row stride (elements)
  int i, j;         // global row / column of the centre
  int rows, cols;   // grid dims
  int k;            // radius
  long long eidx;   // element index of the centre in the env grids (all pitch == env.pitch[0])
  const E0* ec;     // PRE: env slot 0 at the centre, staged in shared memory
  // STRIDE: the tile row stride as a compile-time constant (0: use `stride`)
  __device__ __forceinline__ V at(int di, int dj) const {
    return c[di * (STRIDE ? STRIDE : stride) + dj];
  }
  // true when the whole window is on the grid (and, for row blocks, every
  // env row within the radius is resident): ABSENT / bounds tests fold away
  __device__ static constexpr bool inner() { return IN; }
  // env.at(*nb.center_index): slot 0 from the staged env tile when PRE
  template <class T>
  __device__ __forceinline__ T centre_env(const SkEnv& env, int slot) const;
  __device__ __forceinline__ bool ok(int di, int dj) const {
    if constexpr (IN) return true;
    return (unsigned)(i + di) < (unsigned)rows && (unsigned)(j + dj) < (unsigned)cols;
  }
  __device__ __forceinline__ V center() const { return c[0]; }
};

// Read-only environment grids (up to 4), row-major with a pitch, aligned with
// the loop grid.  get<T>(slot, i, j) reads an absolute element; ok(i, j) says
// whether (i, j) is on the grid.
struct SkEnv {
  const void* p[4];      // -> owned row 0 of each env grid (halo rows above it)
  long long pitch[4];
  int rows, cols;        // global grid dims
  int row0;              // global row of local row 0 (row blocks of a multi-rank run)
  int lo, hi;            // global rows [lo, hi) resident here (owned + halos)
  template <class T>
  __device__ __forceinline__ T get(int slot, long long i, long long j) const {
    return __ldg(static_cast<const T*>(p[slot]) + (i - row0) * pitch[slot] + j);
  }
  __device__ __forceinline__ bool ok(long long i, long long j) const {
    return i >= 0 && i < rows && j >= 0 && j < cols;
  }
  // the centre element of env grid `slot` (the common env.at(*nb.center_index))
  template <class T>
  __device__ __forceinline__ T at_centre(int slot, long long eidx) const {
    return __ldg(static_cast<const T*>(p[slot]) + eidx);
  }
  // on the grid but not resident on this rank (a row block's env rows end
  // with its halo rows)
  __device__ __forceinline__ bool resident(long long i) const { return i >= lo && i < hi; }
};

template <class V, bool IN, int STRIDE, class E0, bool PRE>
template <class T>
__device__ __forceinline__ T SkNb<V, IN, STRIDE, E0, PRE>::centre_env(const SkEnv& env,
                                                                     int slot) const {
  if constexpr (PRE) {
    if (slot == 0) return (T)*ec;
  }
  return env.at_centre<T>(slot, eidx);
}

// (i, j) within the radius of an interior window's centre: on the grid and
// resident, no checks needed (false for border windows)
template <class NB>
__device__ __forceinline__ bool sk_env_near(const NB& nb, long long i, long long j) {
  if constexpr (!NB::inner()) return false;
  const long long di = i - nb.i, dj = j - nb.j;
  return di >= -nb.k && di <= nb.k && dj >= -nb.k && dj <= nb.k;
}

// Kernel parameters of sk_jit_sweep (built on the host in sk_jit.cu).
struct JitArgs {
  Sweep2D g;
  LoopCtl L;
  SkEnv env;
};

// ---------------------------------------------------------------- Python ops
// Exact IEEE arithmetic (the program is compiled with --fmad=false).

// value of a possibly-ABSENT slot used where Python needs a number
template <class T>
__device__ __forceinline__ T py_val(T v, bool ok, SkErr& e) {
  if (!ok) e.set(kErrAbsent);
  return v;
}

// true division: int / int and float / float (Python floats raise on 0;
// numpy float32 scalars return inf / nan)
__device__ __forceinline__ double py_truediv(long long a, long long b, SkErr& e) {
  if (b == 0) {
    e.set(kErrZeroDiv);
    return 0.0;
  }
  return __ddiv_rn((double)a, (double)b);
}
__device__ __forceinline__ double py_truediv(double a, double b, SkErr& e) {
  if (b == 0.0) {
    e.set(kErrZeroDiv);
    return 0.0;
  }
  return __ddiv_rn(a, b);
}
__device__ __forceinline__ float py_truediv(float a, float b, SkErr&) { return __fdiv_rn(a, b); }

// floor division and modulo (CPython long_divmod / float_divmod; numpy
// npy_divmod for float32 scalars)
__device__ __forceinline__ long long py_floordiv(long long a, long long b, SkErr& e) {
  if (b == 0) {
    e.set(kErrZeroDiv);
    return 0;
  }
  long long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
__device__ __forceinline__ long long py_mod(long long a, long long b, SkErr& e) {
  if (b == 0) {
    e.set(kErrZeroDiv);
    return 0;
  }
  long long r = a % b;
  if (r != 0 && ((r < 0) != (b < 0))) r += b;
  return r;
}
template <class T>
__device__ __forceinline__ T py_fdivmod(T a, T b, T* modp) {
  T mod = fmod(a, b);
  T div = (a - mod) / b;
  if (mod != T(0)) {
    if ((b < T(0)) != (mod < T(0))) {
      mod += b;
      div -= T(1);
    }
  } else {
    mod = copysign(T(0), b);
  }
  T fl;
  if (div != T(0)) {
    fl = floor(div);
    if (div - fl > T(0.5)) fl += T(1);
  } else {
    fl = copysign(T(0), a / b);
  }
  *modp = mod;
  return fl;
}
__device__ __forceinline__ double py_floordiv(double a, double b, SkErr& e) {
  if (b == 0.0) {
    e.set(kErrZeroDiv);
    return 0.0;
  }
  double m;
  return py_fdivmod(a, b, &m);
}
__device__ __forceinline__ double py_mod(double a, double b, SkErr& e) {
  if (b == 0.0) {
    e.set(kErrZeroDiv);
    return 0.0;
  }
  double m;
  py_fdivmod(a, b, &m);
  return m;
}
__device__ __forceinline__ float py_floordiv(float a, float b, SkErr&) {
  if (b == 0.0f) return a / b;  // numpy: inf / nan, no exception
  float m;
  return py_fdivmod(a, b, &m);
}
__device__ __forceinline__ float py_mod(float a, float b, SkErr&) {
  if (b == 0.0f) return __int_as_float(0x7fc00000);
  float m;
  py_fdivmod(a, b, &m);
  return m;
}

// power: int ** non-negative int stays an int; otherwise float pow
__device__ __forceinline__ long long py_ipow(long long a, long long b) {
  long long r = 1;
  while (b > 0) {
    if (b & 1) r *= a;
    a *= a;
    b >>= 1;
  }
  return r;
}
__device__ __forceinline__ double py_pow(double a, double b, SkErr& e) {
  if (a == 0.0 && b < 0.0) {
    e.set(kErrZeroDiv);
    return 0.0;
  }
  if (b == 2.0) return __dmul_rn(a, a);  // CPython: exact square
  return pow(a, b);
}
__device__ __forceinline__ float py_pow(float a, float b, SkErr&) {
  if (b == 2.0f) return __fmul_rn(a, a);
  return powf(a, b);
}

// math module: results are Python floats; domain errors raise ValueError
__device__ __forceinline__ double py_sqrt(double x, SkErr& e) {
  if (x < 0.0) e.set(kErrDomain);
  return __dsqrt_rn(x);
}
__device__ __forceinline__ double py_log(double x, SkErr& e) {
  if (!(x > 0.0)) {
    if (x <= 0.0) e.set(kErrDomain);
  }
  return log(x);
}
__device__ __forceinline__ long long py_round(double x, SkErr& e) {  // round(x): half to even, int
  if (isinf(x)) e.set(kErrOverflow);
  if (isnan(x)) e.set(kErrOverflow);
  return (long long)rint(x);
}
__device__ __forceinline__ long long py_int(double x, SkErr& e) {  // int(x): truncation
  if (isinf(x) || isnan(x)) e.set(kErrOverflow);
  return (long long)trunc(x);
}
__device__ __forceinline__ long long py_floor_int(double x, SkErr& e) {  // math.floor -> int
  if (isinf(x) || isnan(x)) e.set(kErrOverflow);
  return (long long)floor(x);
}
__device__ __forceinline__ long long py_ceil_int(double x, SkErr& e) {
  if (isinf(x) || isnan(x)) e.set(kErrOverflow);
  return (long long)ceil(x);
}

// max / min of two values the way Python's builtins pick (first maximal /
// minimal argument wins; comparisons as written)
template <class T>
__device__ __forceinline__ T py_max(T a, T b) { return (b > a) ? b : a; }
template <class T>
__device__ __forceinline__ T py_min(T a, T b) { return (b < a) ? b : a; }

__device__ __forceinline__ long long py_abs(long long a) { return a < 0 ? -a : a; }
__device__ __forceinline__ double py_abs(double a) { return fabs(a); }
__device__ __forceinline__ float py_abs(float a) { return fabsf(a); }

// ---------------------------------------------------------------- combinators
// Sum and max with the engine's reduce semantics (OpCombine); custom
// combinators are generated with the same interface.
struct SkSum {
  __device__ __forceinline__ double operator()(double a, double b) const { return a + b; }
  __device__ __forceinline__ double fold(double acc, double v) const { return acc + v; }
  __device__ __forceinline__ double neutral(double) const { return 0.0; }
};
struct SkMax {
  __device__ __forceinline__ double operator()(double a, double b) const { return rmax(a, b); }
  __device__ __forceinline__ double fold(double acc, double v) const { return (v < acc) ? acc : v; }
  __device__ __forceinline__ double neutral(double) const { return -INFINITY; }
};

}  // namespace sk
