// Geometry shared by the row-marching sweep kernels (Helmholtz, Life).
#pragma once
#include "sk_common.cuh"

namespace sk {

struct Sweep2D {
  const void* src;       // iteration-1 front (the caller's input; never written)
  long long src_pitch;   // elements
  void* buf[2];          // ping-pong iteration buffers: out(t) -> buf[t & 1]
  long long pitch;       // elements
  const void* env;       // read-only environment grid (or null)
  long long env_pitch;   // elements
  int rows, cols;        // owned rows / columns
  int halo_top, halo_bottom;  // 1 = buffers carry a neighbour row above / below
  int colblocks;         // column blocks of BLOCK*VEC columns
  int chunk_rows;        // rows per work chunk
  int part_row[kMaxParts + 1];  // partition row boundaries (local rows)
};

// Map a chunk id to (column block, row range).  Chunks never span a
// partition, so every chunk partial belongs to exactly one partition.
__device__ __forceinline__ void chunk_geom(const LoopCtl& L, const Sweep2D& g, int c, int* cb,
                                           int* r0, int* r1) {
  int p = 0;
  while (p + 1 < L.nparts && c >= L.part_chunk[p + 1]) ++p;
  const int q = c - L.part_chunk[p];
  const int rc = q / g.colblocks;
  *cb = q - rc * g.colblocks;
  *r0 = g.part_row[p] + rc * g.chunk_rows;
  const int e = *r0 + g.chunk_rows;
  *r1 = e < g.part_row[p + 1] ? e : g.part_row[p + 1];
}

template <typename T>
union V16 {
  float4 raw;
  T v[16 / sizeof(T)];
};

template <typename T>
__device__ __forceinline__ V16<T> ldg16(const T* p) {
  V16<T> r;
  r.raw = __ldg(reinterpret_cast<const float4*>(p));
  return r;
}

template <typename T>
__device__ __forceinline__ V16<T> zero16() {
  V16<T> r;
  r.raw = make_float4(0.f, 0.f, 0.f, 0.f);
  return r;
}

// Four contiguous elements (16 B for float, 32 B for double), loaded and
// stored as 16-byte vectors.  Giving every thread 4 elements in both
// precisions keeps 4 independent arithmetic chains per thread, which the
// fp64 sweep needs to cover its longer DP latencies.
template <typename T>
union Vec4;
template <>
union Vec4<float> {
  float4 q[1];
  float v[4];
};
template <>
union Vec4<double> {
  float4 q[2];
  double v[4];
};

template <typename T>
__device__ __forceinline__ Vec4<T> ldg4(const T* p) {
  Vec4<T> r;
#pragma unroll
  for (int i = 0; i < (int)(sizeof(r.q) / 16); ++i) r.q[i] = __ldg(reinterpret_cast<const float4*>(p) + i);
  return r;
}

template <typename T>
__device__ __forceinline__ void st4(T* p, const Vec4<T>& v) {
#pragma unroll
  for (int i = 0; i < (int)(sizeof(v.q) / 16); ++i) reinterpret_cast<float4*>(p)[i] = v.q[i];
}

template <typename T>
__device__ __forceinline__ Vec4<T> zero4() {
  Vec4<T> r;
#pragma unroll
  for (int i = 0; i < (int)(sizeof(r.q) / 16); ++i) r.q[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  return r;
}

}  // namespace sk
