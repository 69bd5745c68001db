// Host-side internals shared by the runtime and the per-kernel launchers.
#pragma once

#include <cuda_runtime.h>
#include <string>
#include <vector>

#include "sk_common.cuh"

struct sk_run;
struct sk_jit;

namespace sk {

void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define SK_CUDA(call)                                 \
  do {                                                \
    cudaError_t _e = (call);                          \
    if (_e != cudaSuccess) return ::sk::cuda_fail(_e, #call); \
  } while (0)

// Per-kernel hooks.  `setup` sizes the launch (grid, work chunks) and any
// extra device state; `launch` enqueues one sweep with the given loop
// control on stream `s` (plain launch or into a graph capture).
struct KernelOps {
  int (*setup)(sk_run*);
  int (*launch)(sk_run*, const LoopCtl&, cudaStream_t);
  void (*teardown)(sk_run*);
  // after a device loop whose launches compute two iterations each stopped
  // at the first of a pair: recompute that iteration's grid (may be null)
  int (*fixup)(sk_run*, long long it, cudaStream_t) = nullptr;
};

const KernelOps* helmholtz_ops();
const KernelOps* life_ops();
const KernelOps* restore_ops();
int restore_frame_status(sk_run* r, long long* iters, double* values, int* exhausted);
unsigned char* restore_chg(sk_run* r, long long it);  // null unless a restore run
const KernelOps* u8_ops();   // Sobel / Life (sk_u8stencil.cu)
const KernelOps* amf_ops();  // adaptive-median detection (sk_amf.cu)
const KernelOps* jit_ops();  // user elemental functions (sk_jit.cu)

// shared body of sk_run_begin / sk_run_begin_jit
int begin_impl(const sk_plan* plan, const sk_jit* jit, const void* d_src, int64_t src_pitch,
               const void* d_env, int64_t env_pitch, const void* const* jit_env,
               const int64_t* jit_env_pitch, int n_env, void* d_buf0, void* d_buf1, int64_t pitch,
               void* stream, sk_run** out);

int device_sms(int device);

// A device word that is 0 whenever no kernel on stream `s` is running: the
// chunk counter of one-launch batched kernels, which reset it before they
// exit (allocated once per (device, stream), never freed).
unsigned* stream_counter(int device, cudaStream_t s);

// Resident CTAs per SM for a kernel at a block size (cached per process: the
// driver query costs tens of microseconds and runs are created per frame).
int occupancy(const void* fn, int block);

// Plain launch, or a cooperative launch for persistent (whole-loop) kernels,
// which guarantees every CTA is co-resident for the in-kernel grid barrier.
template <typename A>
cudaError_t launch_kernel(void (*fn)(A), int grid, int block, const A& args, cudaStream_t s,
                          bool cooperative) {
  if (!cooperative) {
    fn<<<grid, block, 0, s>>>(args);
    return cudaGetLastError();
  }
  void* params[] = {const_cast<A*>(&args)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), grid, block, params, 0, s);
}

// Batched Sobel through the TMA row ring (sk_sobel_tma.cu); SK_ERR_UNSUPPORTED
// when the geometry does not fit it (rows wider than 2048 bytes, unaligned
// pitches), in which case sobel_frames runs the generic batched sweep.
int sobel_frames_tma(const uint8_t* in, long long in_pitch, long long in_fs, uint8_t* out,
                     long long out_pitch, long long out_fs, int frames, long long rows,
                     long long cols, long long* sums, cudaStream_t s);

// cuTensorMapEncodeTiled (PFN_cuTensorMapEncodeTiled_v12000), or null
void* tma_encoder();

// mismatches of div_const vs IEEE division over all safe fp32 numerators
// (cached per divisor; -1 if the check could not run)
long long verify_div_f32(float b, cudaStream_t s);

}  // namespace sk

struct sk_run {
  sk_plan plan{};
  int device = 0;
  cudaStream_t stream = nullptr;
  const sk::KernelOps* ops = nullptr;

  const void* src = nullptr;
  long long src_pitch = 0;
  const void* env = nullptr;
  long long env_pitch = 0;
  void* buf[2] = {nullptr, nullptr};
  long long pitch = 0;

  // launch geometry (filled by ops->setup)
  int grid = 0;
  int block = 0;
  int nparts = 1;
  int part_row[sk::kMaxParts + 1] = {};
  int part_chunk[sk::kMaxParts + 1] = {};
  int colblocks = 1;
  int chunk_rows = 1;
  int nchunks = 0;
  const int* part_chunk_dev = nullptr;  // device-computed chunk ranges (restore)
  const int* flagged_dev = nullptr;     // device-computed flagged count (restore)

  // device loop state
  sk::Status* d_status = nullptr;
  double* d_partials = nullptr;
  double* h_ring = nullptr;  // pinned, mapped
  double* d_ring = nullptr;  // device alias of h_ring
  long long launched = 0;
  long long total_launches = 0;
  bool combined = false;  // cross-rank combine in use
  bool persistent_done = false;  // the loop ran as one persistent launch
  cudaEvent_t ev_done[sk::kRing] = {};

  // optional per-sweep timing
  bool timing = false;
  std::vector<cudaEvent_t> t_start, t_stop;
  std::vector<long long> t_iter;

  // device-loop graph
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap_stream = nullptr;

  // user elemental kernel (SK_KERNEL_JIT)
  const sk_jit* jit = nullptr;
  const void* jit_env[4] = {};
  long long jit_env_pitch[4] = {};
  int jit_nenv = 0;
  bool no_graph = false;  // the kernel cannot drive a graph WHILE node
  bool has_peers = false;  // peer transport attached (sk_run_set_peers)
  sk_peers peers{};
  int steps_per_launch = 1;  // 2: launches compute iterations 2L+1, 2L+2 (results in buf[L & 1])

  // kernel-specific device state (restore: flagged list, change flags)
  void* aux[8] = {};  // kernel-specific device allocations
  long long aux_n[8] = {};
};
