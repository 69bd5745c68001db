// Adaptive-median impulse detection (phase one of the two-phase denoiser).
//
// Reference: detect_kernel block route apps/denoise.py:105-135 (point route
// :88-103), amf_detect :145-157, _mask_sum :141-142.
//
// Per pixel z, for windows w = 3, 5, ..., wmax over the IN-IMAGE values only
// (off-image slots are excluded, the reference's NaN-padded sort):
//   mn, mx = extremes; med = (lo + hi) / 2 with lo/hi the ((cnt-1)/2)-th and
//   (cnt/2)-th smallest; if mn < med < mx: flag = z in {mn, mx}, stop;
//   after the last window: flag = z != med.
// Medians of even counts are half-integers; every comparison is done in
// doubled integer space (2*mn < lo+hi < 2*mx, 2*z == lo+hi), so the
// decision is exact.  Order statistics of u8 values come from an 8-step
// radix (bitwise) selection over counts -- no sorting, no fp.
//
// Integer-ALU-bound (<= 49-value windows at wmax=7).  A CTA stages a
// (TH+2K) x (TW+2K) u8 tile in shared memory; one thread per output pixel.
#include "sk_internal.h"

namespace sk {

constexpr int kTW = 32, kTH = 8;

struct AmfArgs {
  const unsigned char* in;
  unsigned char* out;
  long long in_pitch, out_pitch, in_stride, out_stride;
  int rows, cols, frames, wmax;
  int tiles_x, tiles_per_frame;
  long long* counts;  // batch mode: per-frame flagged count
  unsigned* work;     // batch mode: the stream's chunk counter (stream_counter)
  LoopCtl L;          // loop mode
  const void* src;    // loop mode: iteration-1 front
  void* buf[2];
};

template <int K>
__device__ __forceinline__ void window_stats(const unsigned char* tile, int tw, int ty, int tx,
                                             int r0, int r1, int c0, int c1, int* cnt, int* mn,
                                             int* mx, int* lo, int* hi) {
  // rows [r0, r1], cols [c0, c1] are tile coordinates of the in-image window
  int n = 0, a = 255, b = 0;
  for (int i = r0; i <= r1; ++i)
    for (int j = c0; j <= c1; ++j) {
      const int v = tile[i * tw + j];
      a = min(a, v);
      b = max(b, v);
      ++n;
    }
  const int k1 = (n - 1) >> 1;  // lo = k1-th smallest (0-based)
  int res = 0;
#pragma unroll 1
  for (int bit = 7; bit >= 0; --bit) {
    const int t = res | (1 << bit);
    int below = 0;
    for (int i = r0; i <= r1; ++i)
      for (int j = c0; j <= c1; ++j) below += tile[i * tw + j] < t;
    if (below <= k1) res = t;
  }
  int h = res;
  if (!(n & 1)) {  // hi = (k1+1)-th smallest
    int le = 0, nxt = 256;
    for (int i = r0; i <= r1; ++i)
      for (int j = c0; j <= c1; ++j) {
        const int v = tile[i * tw + j];
        le += v <= res;
        if (v > res) nxt = min(nxt, v);
      }
    h = le > k1 + 1 ? res : nxt;
  }
  *cnt = n;
  *mn = a;
  *mx = b;
  *lo = res;
  *hi = h;
}

// Full 3x3 window (the first AMF level of every interior pixel): min, max
// and median of the 9 values with a median-of-9 exchange network in
// registers (19 compare-exchanges) instead of 8 radix passes over the window.
__device__ __forceinline__ void stats3x3(const unsigned char* tile, int tw, int ly, int lx, int* mn,
                                         int* mx, int* med) {
  int p[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) p[i * 3 + j] = tile[(ly - 1 + i) * tw + lx - 1 + j];
  int a = p[0], b = p[0];
#pragma unroll
  for (int i = 1; i < 9; ++i) {
    a = min(a, p[i]);
    b = max(b, p[i]);
  }
  auto cx = [&](int i, int j) {
    const int lo = min(p[i], p[j]), hi = max(p[i], p[j]);
    p[i] = lo;
    p[j] = hi;
  };
  cx(1, 2); cx(4, 5); cx(7, 8); cx(0, 1); cx(3, 4); cx(6, 7); cx(1, 2); cx(4, 5); cx(7, 8);
  cx(0, 3); cx(5, 8); cx(4, 7); cx(3, 6); cx(1, 4); cx(2, 5); cx(4, 7); cx(4, 2); cx(6, 4);
  cx(4, 2);
  *mn = a;
  *mx = b;
  *med = p[4];
}

template <int K, bool BATCH>
__global__ void __launch_bounds__(kTW * kTH) amf_kernel(const __grid_constant__ AmfArgs a) {
  constexpr int TW = kTW + 2 * K, TH = kTH + 2 * K;
  __shared__ unsigned char tile[TH * TW];
  __shared__ double sh[kTW * kTH / 32];
  __shared__ int s_chunk;
  for (long long it = BATCH ? 1 : loop_enter(a.L); it != 0;
       it = BATCH ? 0 : loop_next<kTW * kTH>(a.L, it, sh)) {
  const unsigned char* front0;
  unsigned char* back0;
  if (BATCH) {
    front0 = a.in;
    back0 = a.out;
  } else {
    front0 = static_cast<const unsigned char*>(it == 1 ? a.src : a.buf[(it - 1) & 1]);
    back0 = static_cast<unsigned char*>(a.buf[it & 1]);
  }
  const long long fpitch = (BATCH || it == 1) ? a.in_pitch : a.out_pitch;
  const int total = BATCH ? a.frames * a.tiles_per_frame : a.L.part_chunk[a.L.nparts];
  const int tid = threadIdx.x;  // 1D block: (tx, ty) = (tid % kTW, tid / kTW)
  const int txl = tid % kTW, tyl = tid / kTW;
  const int K2 = a.wmax / 2;
  auto next = [&]() {
    return BATCH ? next_chunk_stream(a.work, total, &s_chunk) : next_chunk(a.L, &s_chunk);
  };
  for (int c = next(); c < total; c = next()) {
    const int frame = BATCH ? c / a.tiles_per_frame : 0;
    const int t = c - frame * a.tiles_per_frame;
    const int ty0 = (t / a.tiles_x) * kTH, tx0 = (t % a.tiles_x) * kTW;
    const unsigned char* front = front0 + (BATCH ? frame * a.in_stride : 0);
    unsigned char* back = back0 + (BATCH ? frame * a.out_stride : 0);
    for (int i = tid; i < TH * TW; i += kTW * kTH) {
      const int gr = ty0 - K + i / TW, gc = tx0 - K + i % TW;
      tile[i] = (gr >= 0 && gr < a.rows && gc >= 0 && gc < a.cols)
                    ? __ldg(front + (long long)gr * fpitch + gc) : 0;
    }
    __syncthreads();
    const int gr = ty0 + tyl, gc = tx0 + txl;
    int flag = 0;
    if (gr < a.rows && gc < a.cols) {
      const int ly = tyl + K, lx = txl + K;
      const int z = tile[ly * TW + lx];
      int lo = z, hi = z, decided = 0;
      int rstart = 1;
      if (K2 >= 1 && gr >= 1 && gr + 1 < a.rows && gc >= 1 && gc + 1 < a.cols) {
        int mn, mx, med;
        stats3x3(tile, TW, ly, lx, &mn, &mx, &med);
        lo = hi = med;
        if (mn < med && med < mx) {
          flag = (z == mn || z == mx);
          decided = 1;
        }
        rstart = 2;
      }
      for (int r = rstart; r <= K2 && !decided; ++r) {
        const int r0 = ly - min(r, gr), r1 = ly + min(r, a.rows - 1 - gr);
        const int c0 = lx - min(r, gc), c1 = lx + min(r, a.cols - 1 - gc);
        int cnt, mn, mx;
        window_stats<K>(tile, TW, ly, lx, r0, r1, c0, c1, &cnt, &mn, &mx, &lo, &hi);
        const int s2 = lo + hi;  // 2 * median
        if (2 * mn < s2 && s2 < 2 * mx) {
          flag = (z == mn || z == mx);
          decided = 1;
          break;
        }
      }
      if (!decided) flag = (2 * z != lo + hi);
      back[(long long)gr * (BATCH ? a.out_pitch : a.out_pitch) + gc] = (unsigned char)flag;
    }
    const double v = block_reduce<kTW * kTH>(SK_REDUCE_SUM, (double)flag, sh);
    if (tid == 0) {
      if (BATCH) atomicAdd(reinterpret_cast<unsigned long long*>(&a.counts[frame]),
                           (unsigned long long)v);
      else a.L.partials[c] = v;
    }
  }
  }  // iterations
}

// ---------------------------------------------------------------- host side

namespace {

template <bool BATCH>
using AmfFn = void (*)(const AmfArgs);

template <bool BATCH>
AmfFn<BATCH> pick(int wmax) {
  if (wmax <= 7) return amf_kernel<3, BATCH>;
  if (wmax <= 15) return amf_kernel<7, BATCH>;
  return nullptr;
}

int grid_for(int device, const void* fn, long long tiles) {
  const long long slots = (long long)device_sms(device) * occupancy(fn, kTW * kTH);
  return (int)(slots < tiles ? slots : tiles);
}

int setup(sk_run* r) {
  const int wmax = (int)r->plan.params[0];
  if (r->plan.dtype != SK_U8 || wmax < 3 || !(wmax & 1) || !pick<false>(wmax)) {
    set_error("amf: u8 grid and odd wmax in [3, 15] required");
    return SK_ERR_UNSUPPORTED;
  }
  if (r->plan.reduce_op != SK_REDUCE_SUM || r->plan.delta_op != SK_DELTA_NONE) {
    set_error("amf: only the flagged-count SUM reduce is supported");
    return SK_ERR_UNSUPPORTED;
  }
  const long long tx = (r->plan.cols + kTW - 1) / kTW, ty = (r->plan.rows + kTH - 1) / kTH;
  r->nchunks = (int)(tx * ty);
  r->nparts = 1;  // integer count: the fold order cannot change the value
  r->part_chunk[0] = 0;
  r->part_chunk[1] = r->nchunks;
  r->colblocks = (int)tx;
  r->grid = grid_for(r->device, (const void*)pick<false>(wmax), r->nchunks);
  return SK_OK;
}

int launch(sk_run* r, const LoopCtl& L, cudaStream_t s) {
  const int wmax = (int)r->plan.params[0];
  AmfArgs a{};
  a.src = r->src;
  a.buf[0] = r->buf[0];
  a.buf[1] = r->buf[1];
  a.in_pitch = r->src_pitch;
  a.out_pitch = r->pitch;
  a.rows = (int)r->plan.rows;
  a.cols = (int)r->plan.cols;
  a.frames = 1;
  a.wmax = wmax;
  a.tiles_x = r->colblocks;
  a.tiles_per_frame = r->nchunks;
  a.L = L;
  SK_CUDA(launch_kernel(pick<false>(wmax), r->grid, kTW * kTH, a, s, L.persistent != 0));
  return SK_OK;
}

void teardown(sk_run*) {}

const KernelOps kOps = {setup, launch, teardown};

}  // namespace

const KernelOps* amf_ops() { return &kOps; }

int amf_frames(const uint8_t* in, long long in_pitch, long long in_fs, uint8_t* mask,
               long long mask_pitch, long long mask_fs, int frames, long long rows,
               long long cols, int wmax, long long* counts, cudaStream_t s) {
  if (!in || !mask || !counts || frames < 1 || rows < 1 || cols < 1 || in_pitch < cols ||
      mask_pitch < cols || wmax < 3 || !(wmax & 1) || !pick<true>(wmax)) {
    set_error("sk_amf_frames: bad arguments (odd wmax in [3, 15])");
    return SK_ERR_ARG;
  }
  int dev = 0;
  SK_CUDA(cudaGetDevice(&dev));
  AmfArgs a{};
  a.in = in;
  a.out = mask;
  a.in_pitch = in_pitch;
  a.out_pitch = mask_pitch;
  a.in_stride = in_fs;
  a.out_stride = mask_fs;
  a.rows = (int)rows;
  a.cols = (int)cols;
  a.frames = frames;
  a.wmax = wmax;
  a.tiles_x = (int)((cols + kTW - 1) / kTW);
  a.tiles_per_frame = a.tiles_x * (int)((rows + kTH - 1) / kTH);
  a.counts = counts;
  a.L.nparts = 1;
  a.work = stream_counter(dev, s);
  if (!a.work) return SK_ERR_CUDA;
  SK_CUDA(cudaMemsetAsync(counts, 0, sizeof(long long) * frames, s));
  const long long tiles = (long long)a.tiles_per_frame * frames;
  pick<true>(wmax)<<<grid_for(dev, (const void*)pick<true>(wmax), tiles), kTW * kTH, 0, s>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "amf_frames launch");
  return SK_OK;
}

}  // namespace sk

extern "C" int sk_amf_frames(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                             uint8_t* d_mask, int64_t mask_pitch, int64_t mask_frame_stride,
                             int32_t frames, int64_t rows, int64_t cols, int32_t wmax,
                             int64_t* d_counts, void* stream) {
  return sk::amf_frames(d_in, in_pitch, in_frame_stride, d_mask, mask_pitch, mask_frame_stride,
                        frames, rows, cols, wmax, reinterpret_cast<long long*>(d_counts),
                        static_cast<cudaStream_t>(stream));
}
