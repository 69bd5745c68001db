// reduce_all for the built-in combinators: the reference's left fold of a
// grid in row-major order from the identity (patterns.py:143-147,
// Combinator.fold patterns.py:103-108), on the device.
//
//  * integer SUM / MAX: order-free (int64 wrap-around for SUM, like numpy
//    int64) -> one grid-stride pass, block reduce, one atomic per block.
//  * floating MAX `a if b < a else b`: order matters only for NaN and for
//    equal values (+0 / -0): a NaN element makes the accumulator NaN and
//    the next element replaces it, and an element equal to the accumulator
//    replaces it.  So the result is the last element if it is NaN; else the
//    LAST element attaining the maximum of everything after the last NaN
//    (the identity counts as element -1).  Three grid-stride passes (last
//    NaN index, maximum, last index of the maximum) and a one-thread final
//    step -- bit-identical to the sequential fold.
//  * floating SUM: rounding depends on the order, so the fold is evaluated
//    sequentially in the element type (fp32 data: fp32 accumulation, numpy
//    NEP 50; fp64: fp64), op by op with round-to-nearest adds: one CTA
//    streams 2048-element tiles through shared memory (double-buffered, so
//    the loads of tile t+1 overlap the fold of tile t) and one thread folds.
//    Bit-identical to the reference; O(n) latency-bound by design.
#include <climits>
#include <cstdint>
#include <cstring>

#include "sk_internal.h"

namespace sk {
namespace fold {

constexpr int kB = 256;

template <typename T>
__device__ __forceinline__ long long widen(T v) { return (long long)v; }

template <typename T>
__global__ void int_sum(const T* d, long long n, unsigned long long* out) {
  long long s = 0;
  for (long long i = blockIdx.x * (long long)kB + threadIdx.x; i < n; i += (long long)gridDim.x * kB)
    s += widen(d[i]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ long long w[kB / 32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int k = 0; k < kB / 32; ++k) t += w[k];
    atomicAdd(out, (unsigned long long)t);  // wraps like int64
  }
}

template <typename T>
__global__ void int_max(const T* d, long long n, long long* out) {
  long long m = LLONG_MIN;
  for (long long i = blockIdx.x * (long long)kB + threadIdx.x; i < n; i += (long long)gridDim.x * kB)
    m = max(m, widen(d[i]));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ long long w[kB / 32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = LLONG_MIN;
    for (int k = 0; k < kB / 32; ++k) t = max(t, w[k]);
    atomicMax(out, t);
  }
}

// float MAX state: [0] last NaN index (-1 none), [1] max key, [2] last index of the max
struct FMax {
  long long last_nan;
  unsigned long long key;
  long long idx;
};

// totally ordered key of a non-NaN float/double with -0 == +0
__device__ __forceinline__ unsigned long long okey(double v) {
  if (v == 0.0) v = 0.0;
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

template <typename T>
__global__ void fmax_nan(const T* d, long long n, FMax* st) {
  long long j = -1;
  for (long long i = blockIdx.x * (long long)kB + threadIdx.x; i < n; i += (long long)gridDim.x * kB)
    if (d[i] != d[i]) j = i;  // grid-stride order: the thread's last hit is its largest
  for (int o = 16; o > 0; o >>= 1) j = max(j, __shfl_xor_sync(0xffffffffu, j, o));
  if ((threadIdx.x & 31) == 0 && j >= 0) atomicMax(&st->last_nan, j);
}

template <typename T>
__global__ void fmax_val(const T* d, long long n, FMax* st) {
  const long long from = st->last_nan + 1;
  unsigned long long k = 0;
  for (long long i = from + blockIdx.x * (long long)kB + threadIdx.x; i < n;
       i += (long long)gridDim.x * kB)
    k = max(k, okey((double)d[i]));
  for (int o = 16; o > 0; o >>= 1) k = max(k, __shfl_xor_sync(0xffffffffu, k, o));
  if ((threadIdx.x & 31) == 0 && k) atomicMax(&st->key, k);
}

template <typename T>
__global__ void fmax_idx(const T* d, long long n, FMax* st) {
  const long long from = st->last_nan + 1;
  const unsigned long long key = st->key;
  long long j = -1;
  for (long long i = from + blockIdx.x * (long long)kB + threadIdx.x; i < n;
       i += (long long)gridDim.x * kB)
    if (okey((double)d[i]) == key) j = i;
  for (int o = 16; o > 0; o >>= 1) j = max(j, __shfl_xor_sync(0xffffffffu, j, o));
  if ((threadIdx.x & 31) == 0 && j >= 0) atomicMax(&st->idx, j);
}

// fold the identity in front and write the result (one thread)
template <typename T>
__global__ void fmax_final(const T* d, long long n, const FMax* st, T ident, T* out) {
  const long long ln = st->last_nan;
  T r;
  if (n == 0) r = ident;
  else if (ln == n - 1) r = d[n - 1];                   // the last element is NaN
  else if (ln >= 0) r = d[st->idx];                     // everything before it is replaced
  else if (ident != ident) r = d[st->idx];              // a NaN identity is replaced
  else r = (d[st->idx] < ident) ? ident : d[st->idx];   // ties: the later element
  *out = r;
}

// sequential float SUM, one CTA: tiles of kTile elements double-buffered in smem
constexpr int kTile = 2048;  // 2 x 16 KB of fp64 in static shared memory
template <typename T>
__global__ void __launch_bounds__(kB) fsum_seq(const T* d, long long n, T ident, T* out) {
  __shared__ T buf[2][kTile];
  const long long ntiles = (n + kTile - 1) / kTile;
  auto load = [&](long long t, int b) {
    const long long base = t * kTile;
    for (int k = threadIdx.x; k < kTile; k += kB) {
      const long long i = base + k;
      if (i < n) buf[b][k] = d[i];
    }
  };
  T acc = ident;
  if (ntiles > 0) load(0, 0);
  __syncthreads();
  for (long long t = 0; t < ntiles; ++t) {
    const int b = (int)(t & 1);
    if (t + 1 < ntiles) load(t + 1, b ^ 1);  // every thread but the folder's work overlaps
    if (threadIdx.x == 0) {
      const long long m = min((long long)kTile, n - t * kTile);
      for (int k = 0; k < m; ++k) acc = xadd(acc, buf[b][k]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = acc;
}

int grid_for(long long n) {
  int dev = 0;
  cudaGetDevice(&dev);
  const long long want = (n + kB - 1) / kB;
  const long long cap = (long long)device_sms(dev) * 8;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

template <typename T>
int run_int(const void* d, long long n, int op, const void* ident, void* out, cudaStream_t s) {
  const T* p = static_cast<const T*>(d);
  SK_CUDA(cudaMemcpyAsync(out, ident, 8, cudaMemcpyHostToDevice, s));
  if (n == 0) return SK_OK;
  if (op == SK_REDUCE_SUM)
    int_sum<T><<<grid_for(n), kB, 0, s>>>(p, n, static_cast<unsigned long long*>(out));
  else
    int_max<T><<<grid_for(n), kB, 0, s>>>(p, n, static_cast<long long*>(out));
  SK_CUDA(cudaGetLastError());
  return SK_OK;
}

template <typename T>
int run_float(const void* d, long long n, int op, const void* ident, void* out, cudaStream_t s) {
  const T* p = static_cast<const T*>(d);
  T id;
  memcpy(&id, ident, sizeof(T));
  if (op == SK_REDUCE_SUM) {
    fsum_seq<T><<<1, kB, 0, s>>>(p, n, id, static_cast<T*>(out));
    SK_CUDA(cudaGetLastError());
    return SK_OK;
  }
  FMax* st = nullptr;
  SK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&st), sizeof(FMax), s));
  const FMax init{-1, 0ull, -1};
  SK_CUDA(cudaMemcpyAsync(st, &init, sizeof(FMax), cudaMemcpyHostToDevice, s));
  if (n > 0) {
    const int g = grid_for(n);
    fmax_nan<T><<<g, kB, 0, s>>>(p, n, st);
    fmax_val<T><<<g, kB, 0, s>>>(p, n, st);
    fmax_idx<T><<<g, kB, 0, s>>>(p, n, st);
  }
  fmax_final<T><<<1, 1, 0, s>>>(p, n, st, id, static_cast<T*>(out));
  SK_CUDA(cudaGetLastError());
  SK_CUDA(cudaStreamSynchronize(s));  // `init` lives on this frame
  SK_CUDA(cudaFreeAsync(st, s));
  return SK_OK;
}

}  // namespace fold
}  // namespace sk

extern "C" int sk_reduce_fold(const void* d_data, int64_t n, int32_t dtype, int32_t op,
                              const void* identity, void* d_out, void* stream) {
  using namespace sk;
  if ((!d_data && n > 0) || n < 0 || !identity || !d_out ||
      (op != SK_REDUCE_SUM && op != SK_REDUCE_MAX)) {
    set_error("sk_reduce_fold: bad arguments");
    return SK_ERR_ARG;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (dtype) {
    case SK_U8: return fold::run_int<unsigned char>(d_data, n, op, identity, d_out, s);
    case SK_I32: return fold::run_int<int>(d_data, n, op, identity, d_out, s);
    case SK_I64: return fold::run_int<long long>(d_data, n, op, identity, d_out, s);
    case SK_F32: return fold::run_float<float>(d_data, n, op, identity, d_out, s);
    case SK_F64: return fold::run_float<double>(d_data, n, op, identity, d_out, s);
    default:
      set_error("sk_reduce_fold: unsupported element type");
      return SK_ERR_UNSUPPORTED;
  }
}
