// Standalone A/B harness for the Helmholtz sweep shape (not product; tools/).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/ab tools/helm_sweep_ab.cu
// Same arithmetic as helmholtz_sweep (SQUARE delta, SUM reduce), simple
// geometry: rows x cols (cols % (VEC) == 0), Dirichlet 0 outside.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <typename T, int VEC> struct V { T v[VEC]; };

template <int MODE>
__device__ __forceinline__ float4 ld16(const void* p) {
  float4 r;
  if (MODE == 0) {
    r = __ldg(reinterpret_cast<const float4*>(p));
  } else if (MODE == 1) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  } else {
    asm volatile("ld.global.nc.L2::128B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  }
  return r;
}
template <int SMODE>
__device__ __forceinline__ void st16(void* p, float4 v) {
  if (SMODE == 0) *reinterpret_cast<float4*>(p) = v;
  else __stcs(reinterpret_cast<float4*>(p), v);
}

template <typename T, int VEC, int LMODE>
__device__ __forceinline__ V<T, VEC> ldv(const T* p) {
  V<T, VEC> r;
  constexpr int N = VEC * sizeof(T) / 16;
#pragma unroll
  for (int i = 0; i < N; ++i) *reinterpret_cast<float4*>(&r.v[i * 16 / sizeof(T)]) = ld16<LMODE>(reinterpret_cast<const char*>(p) + 16 * i);
  return r;
}
template <typename T, int VEC, int SMODE>
__device__ __forceinline__ void stv(T* p, const V<T, VEC>& r) {
  constexpr int N = VEC * sizeof(T) / 16;
#pragma unroll
  for (int i = 0; i < N; ++i) st16<SMODE>(reinterpret_cast<char*>(p) + 16 * i, *reinterpret_cast<const float4*>(&r.v[i * 16 / sizeof(T)]));
}
template <typename T, int VEC>
__device__ __forceinline__ V<T, VEC> zv() { V<T, VEC> r;
#pragma unroll
  for (int i = 0; i < VEC; ++i) r.v[i] = T(0); return r; }

__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float xmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float xadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float xsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double div_const(double x, double b, double r) {
  const double q0 = __dmul_rn(x, r); const double e = __fma_rn(-q0, b, x); return __fma_rn(e, r, q0); }
__device__ __forceinline__ float div_const(float x, float b, float r) {
  const float q0 = __fmul_rn(x, r); const float e = __fmaf_rn(-q0, b, x); return __fmaf_rn(e, r, q0); }

template <typename T>
struct Args {
  const T* src; T* dst; const T* env; long long pitch; int rows, cols, colblocks, chunk_rows, nchunks;
  T ax, ay, b, rb, keep, relax; unsigned* work; double* partials;
};

// D = prefetch depth in rows (ring of D row slots in registers)
template <typename T, int BLOCK, int VEC, int D, int MINB, int LMODE, int SMODE, int FEAT = 0>
__global__ void __launch_bounds__(BLOCK, MINB) sweep(const __grid_constant__ Args<T> a) {
  __shared__ int s_chunk;
  __shared__ double sh[BLOCK / 32];
  const int lane = threadIdx.x & 31;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_chunk = (int)atomicAdd(a.work, 1u);
    __syncthreads();
    const int c = s_chunk;
    if (c >= a.nchunks) break;
    const int rc = c / a.colblocks, cb = c - rc * a.colblocks;
    const int r0 = rc * a.chunk_rows;
    const int r1 = min(r0 + a.chunk_rows, a.rows);
    const int col = cb * (BLOCK * VEC) + (int)threadIdx.x * VEC;
    const bool active = col < a.cols;
    const bool has_l = lane == 0 && col > 0 && active;
    const bool has_r = lane == 31 && col + VEC < a.cols;
    const long long fp = a.pitch;
    const T* front = a.src + col;
    auto ldrow = [&](int r) -> V<T, VEC> {
      if (!active || r < 0 || r >= a.rows) return zv<T, VEC>();
      return ldv<T, VEC, LMODE>(front + (long long)r * fp);
    };
    V<T, VEC> up = ldrow(r0 - 1), cen = ldrow(r0);
    V<T, VEC> dn[D], fv[D];
    T ls[D], rs[D];
    auto issue = [&](int s, int rr) {
      if (rr < r1) {
        dn[s] = ldrow(rr + 1);
        fv[s] = active ? ldv<T, VEC, LMODE>(a.env + (long long)rr * fp + col) : zv<T, VEC>();
        ls[s] = has_l ? __ldg(front + (long long)rr * fp - 1) : T(0);
        rs[s] = has_r ? __ldg(front + (long long)rr * fp + VEC) : T(0);
      }
    };
#pragma unroll
    for (int s = 0; s < D; ++s) issue(s, r0 + s);
    double accs = 0.0;
    T accm = -INFINITY; bool nanseen = false;
    const T ax = a.ax, ay = a.ay, b = a.b, rb = a.rb, keep = a.keep, relax = a.relax;
    for (int r = r0; r < r1; r += D) {
#pragma unroll
      for (int u = 0; u < D; ++u) {
        const int rr = r + u;
        if (rr < r1) {
          T lv = __shfl_up_sync(~0u, cen.v[VEC - 1], 1);
          T rv = __shfl_down_sync(~0u, cen.v[0], 1);
          if (lane == 0) lv = ls[u];
          if (lane == 31) rv = rs[u];
          V<T, VEC> o;
          T dsum = T(0);
          T num[VEC], q[VEC];
          bool ok = true;
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const T l = e == 0 ? lv : cen.v[e - 1];
            const T rt = e == VEC - 1 ? rv : cen.v[e + 1];
            const T t3 = xadd(fv[u].v[e], xmul(ax, xadd(l, rt)));
            num[e] = xmul(relax, xadd(t3, xmul(ay, xadd(up.v[e], dn[u].v[e]))));
            if (FEAT & 1) { const T aa = fabs(num[e]); ok = ok && aa >= T(0x1p-60) && aa < T(0x1p60); }
          }
          if (ok) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) q[e] = div_const(num[e], b, rb);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) q[e] = num[e] / b;
          }
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const T out = xadd(xmul(keep, cen.v[e]), q[e]);
            o.v[e] = out;
            const T t = xsub(out, cen.v[e]);
            if (FEAT & 2) {
              const T d = fabs(t);
              accm = (accm != accm || d != d) ? T(NAN) : fmax(accm, d);
            } else if (FEAT & 4) {
              const T d = fabs(t);
              accm = fmax(accm, d); nanseen |= d != d;
            } else {
              dsum = xadd(dsum, xmul(t, t));
            }
          }
          accs += (double)dsum;
          if (active) stv<T, VEC, SMODE>(a.dst + (long long)rr * fp + col, o);
          up = cen;
          cen = dn[u];
          issue(u, rr + D);
        }
      }
    }
    if (FEAT & 6) accs = nanseen ? (double)NAN : (double)accm;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) accs += __shfl_xor_sync(~0u, accs, o);
    if (lane == 0) sh[threadIdx.x >> 5] = accs;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0; for (int w = 0; w < BLOCK / 32; ++w) t += sh[w];
      a.partials[c] = t;
    }
  }
}

template <typename T, int BLOCK, int VEC, int D, int MINB, int LMODE, int SMODE, int FEAT = 0>
void run(const char* name, int rows, int cols, int chunk_rows, int iters) {
  using A = Args<T>;
  long long pitch = cols;
  size_t bytes = (size_t)rows * pitch * sizeof(T);
  T *u0, *u1, *f; CK(cudaMalloc(&u0, bytes)); CK(cudaMalloc(&u1, bytes)); CK(cudaMalloc(&f, bytes));
  CK(cudaMemset(u0, 0, bytes)); CK(cudaMemset(u1, 0, bytes));
  // f = 1
  {
    T* h = (T*)malloc((size_t)pitch * sizeof(T)); for (long long i = 0; i < pitch; ++i) h[i] = T(1);
    for (int r = 0; r < rows; ++r) CK(cudaMemcpy(f + (long long)r * pitch, h, pitch * sizeof(T), cudaMemcpyHostToDevice));
    free(h);
  }
  auto fn = sweep<T, BLOCK, VEC, D, MINB, LMODE, SMODE, FEAT>;
  int per_sm = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, BLOCK, 0));
  cudaFuncAttributes fa; CK(cudaFuncGetAttributes(&fa, fn));
  int colblocks = (cols + BLOCK * VEC - 1) / (BLOCK * VEC);
  int nchunks = ((rows + chunk_rows - 1) / chunk_rows) * colblocks;
  int grid = 148 * per_sm; if (grid > nchunks) grid = nchunks;
  unsigned* work; double* part; CK(cudaMalloc(&work, 4 * iters + 64)); CK(cudaMalloc(&part, nchunks * 8));
  CK(cudaMemset(work, 0, 4 * iters + 64));
  A a{}; a.rows = rows; a.cols = cols; a.pitch = pitch; a.colblocks = colblocks; a.chunk_rows = chunk_rows; a.nchunks = nchunks;
  a.ax = 1; a.ay = 1; a.b = 5; a.rb = T(1) / T(5); a.keep = 0; a.relax = 1; a.env = f; a.partials = part;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto launch = [&](int i) {
    a.src = (i & 1) ? u1 : u0; a.dst = (i & 1) ? u0 : u1; a.work = work + i;
    fn<<<grid, BLOCK>>>(a);
  };
  for (int i = 0; i < 4; ++i) launch(i);
  CK(cudaMemset(work, 0, 4 * iters + 64));
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) launch(i);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  ms /= iters;
  double alg = 3.0 * rows * (double)cols * sizeof(T);
  printf("%-34s regs %3d occ %2d grid %5d chunk %3d: %.4f ms  %.0f GB/s  frac %.3f\n", name, fa.numRegs, per_sm, grid,
         chunk_rows, ms, alg / ms / 1e6, alg / ms / 1e6 / 6555.5);
  cudaFree(u0); cudaFree(u1); cudaFree(f); cudaFree(work); cudaFree(part);
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 23168;
  const int NF = 32768;
  const int it = 20;
  for (int ch : {32, 64, 96, 128, 225}) {
    run<double, 128, 4, 1, 8, 0, 0, 0>("f64 V4 M8 sum", N, N, ch, it);
  }
  for (int ch : {64, 128, 256}) run<float, 128, 4, 1, 5, 0, 0>("f32 V4 M5", NF, NF, ch, it);
  return 0;
}
