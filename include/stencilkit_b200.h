/*
 * stencilkit_b200 -- C ABI of the B200-native loop-of-stencil-reduce engine.
 *
 * This is the drop-in boundary for the reference package `stencilkit`
 * (/root/reference/pkg/src/stencilkit).  The reference's plugin point is the
 * Executor protocol (loop.py:124-137: begin(plan, grid) -> run; step(run) ->
 * reduce value; finish(run) -> (Grid, CopyLedger); abort(run)) driven by
 * _drive (loop.py:198-224).  The Python `DeviceExecutor` in
 * paper_1609_04567_b200/partition.py implements that protocol on top of the
 * functions below, loaded with ctypes.
 *
 * Conventions: plain C types only; every function returns SK_OK (0) or an
 * SK_ERR_* code and never throws; sk_last_error() gives the message of the
 * calling thread's last failure.  Pointers named d_* are CUDA device
 * pointers (any allocator); `stream` is a cudaStream_t (NULL = legacy
 * default stream).  One sk_run is single-owner; distinct runs are
 * independent and may be driven from different host threads.
 */
#ifndef STENCILKIT_B200_H
#define STENCILKIT_B200_H

#ifndef __CUDACC_RTC__
#include <stdint.h>
#else /* NVRTC (user elemental kernels, sk_jit_*) */
typedef signed char int8_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned char uint8_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SK_ABI_VERSION 1

/* status codes */
#define SK_OK 0
#define SK_ERR_ARG 1
#define SK_ERR_CUDA 2
#define SK_ERR_STATE 3
#define SK_ERR_UNSUPPORTED 4

/* element types */
#define SK_U8 1
#define SK_I32 2 /* reduce_all only */
#define SK_F32 3
#define SK_F64 4
#define SK_I64 5 /* reduce_all only */

/* device kernels: the reference's block kernels, one per app
 * (apps/helmholtz.py:85-92, apps/sobel.py:47-66, apps/denoise.py:105-135,
 *  apps/denoise.py:209-246, apps/life.py:35-43) */
#define SK_KERNEL_HELMHOLTZ 1 /* params: ax, ay, b, keep, relax           */
#define SK_KERNEL_SOBEL 2     /* u8 in/out, off-image reads = centre      */
#define SK_KERNEL_AMF 3       /* params: wmax; u8 in, u8 0/1 out          */
#define SK_KERNEL_RESTORE 4   /* params: beta, phi_eps[, pa, pb]; f64 work, u8 mask.
                                 pb > 0: the run computes partitions [pa, pb) only
                                 (a frame split across runs / GPUs) */
#define SK_KERNEL_LIFE 5      /* u8 0/1 board                             */
#define SK_KERNEL_JIT 6       /* user elemental function (sk_jit_compile)  */

/* Combinator kinds (patterns.py:195-211) and Delta kinds
 * (apps/helmholtz.py:98-100, apps/denoise.py:252-254) */
#define SK_REDUCE_SUM 1
#define SK_REDUCE_MAX 2
#define SK_REDUCE_CUSTOM 3 /* JIT kernels: the combinator compiled into the program */
#define SK_DELTA_NONE 0
#define SK_DELTA_ABS 1
#define SK_DELTA_SQUARE 2

/* device-evaluable loop conditions (Condition, loop.py:43-57):
 *   HOST     : never stops on the device; the host evaluates its predicate
 *   LT       : value < a                      (e.g. max|delta| < 1e-4)
 *   RMS_LT   : sqrt(value / n) < a            (apps/helmholtz.py:128-131)
 *   MEAN_LT  : value / n < a                  (apps/denoise.py:282-283)
 *   ITER_GE  : iteration >= n                 (stop_after, loop.py:70-74)
 *   MEAN_FLAGGED_LT : value / max(F, 1) < a   with F the run's flagged-pixel
 *              count (restore runs; restore_regularize, apps/denoise.py:279-283)
 * all evaluated in fp64 exactly as the Python predicate. */
#define SK_COND_HOST 0
#define SK_COND_LT 1
#define SK_COND_RMS_LT 2
#define SK_COND_MEAN_LT 3
#define SK_COND_ITER_GE 4
#define SK_COND_MEAN_FLAGGED_LT 5

/* One loop plan = the reference's LoopPlan (loop.py:101-110) reduced to
 * device terms.  Grids are row-major with a row pitch in elements. */
typedef struct sk_plan {
  int32_t kernel;      /* SK_KERNEL_* */
  int32_t dtype;       /* element type of the iterated grid */
  int64_t rows, cols;  /* owned rows x columns */
  int32_t partitions;  /* row partitions for the reduce fold (partition.py:187-195) */
  int32_t reduce_op;   /* SK_REDUCE_* */
  int32_t delta_op;    /* SK_DELTA_* */
  int32_t halo_top;    /* neighbour-owned rows the buffers carry above row 0
                          (Helmholtz: 0 or 1; user elementals: 0 or the radius k) */
  int32_t halo_bottom; /* likewise below row rows-1 */
  int32_t flags;       /* SK_FLAG_* */
  double identity;     /* combinator identity */
  double params[8];    /* kernel parameters, see SK_KERNEL_* */
} sk_plan;

#define SK_FLAG_TIMING 1 /* record CUDA events around every sweep launch */
#define SK_FLAG_FRAMES 2 /* restore: the `partitions` row blocks are independent
                            frames, each with its own loop (video farm batch) */

typedef struct sk_cond {
  int32_t kind; /* SK_COND_* */
  int32_t pad;
  double a;
  double n;
  int64_t max_iterations;
} sk_cond;

typedef struct sk_run sk_run;

#ifndef __CUDACC_RTC__ /* device programs (NVRTC) need only the constants and types above */
const char* sk_last_error(void);
int sk_abi_version(void);

/* Executor.begin (loop.py:124-137; ParallelExecutor.begin partition.py:607-625).
 * d_src   : the input grid (read, never written: loop.py:157-161), layout
 *           (halo_top + rows + halo_bottom) x src_pitch.  Iteration 1 reads it.
 * d_env   : read-only environment grid (same row layout; env_pitch), or NULL.
 *           Helmholtz: f (same dtype).  Restore: the 0/1 noise map (u8).
 * d_buf0/1: the executor's two iteration buffers (PartitionSet.buffer_allocations,
 *           partition.py:160), layout (halo_top + rows + halo_bottom) x pitch.
 * pitch / src_pitch / env_pitch must be multiples of 16 bytes / sizeof(elem)
 * (Helmholtz: also of 4 elements) and the pointers 16-byte aligned (the
 * Python layer stages otherwise). */
int sk_run_begin(const sk_plan* plan, const void* d_src, int64_t src_pitch,
                 const void* d_env, int64_t env_pitch, void* d_buf0, void* d_buf1,
                 int64_t pitch, void* stream, sk_run** out);

/* Executor.step (loop.py:209-213): enqueue `n` iterations (async).  Iterations
 * past a device-decided stop are no-ops. */
int sk_run_launch(sk_run* run, int32_t n);

/* Wait for iteration `it` (1-based, already launched) and return its
 * combined reduce value. */
int sk_run_value(sk_run* run, int64_t it, double* value);

/* Whole _drive loop on the device (loop.py:198-224) for a device-evaluable
 * condition: one CUDA-graph launch with a conditional WHILE node (or batched
 * launches when timing).  Outputs: completed iterations, the final reduce
 * value, and whether the cap was hit without the condition holding. */
int sk_run_loop(sk_run* run, const sk_cond* cond, int64_t* iterations, double* final_value,
                int32_t* exhausted);

/* Executor.finish (partition.py:658-661): which iteration buffer holds the
 * result of iteration `it`: 0 or 1 (-1 means the input itself, it == 0). */
int sk_run_result(sk_run* run, int64_t it, int32_t* which);

/* Device address of the run's status value (double) for the most recent
 * iteration -- the per-rank partial a multi-GPU driver all-gathers. */
int sk_run_value_ptr(sk_run* run, void** d_value);

/* Multi-GPU (one run per rank, row blocks): after iteration t's sweep and
 * the all-gather of every rank's sk_run_value_ptr value into d_partials[n]
 * (rank order), fold them in ascending rank order from the identity (the
 * reference's host combine, partition.py:642-646), evaluate `cond` for
 * iteration t on the device and stop the run if it holds.  Enqueued on the
 * run's stream; later sweeps of a stopped run are no-ops, so a driver may
 * enqueue several iterations ahead without reading anything back. */
int sk_run_combine(sk_run* run, const double* d_partials, int32_t n, const sk_cond* cond);

/* ---- peer transport (multi-GPU without a collective library) ----------
 * Replaces the NCCL halo send/recv + all-gather of the reference's
 * halo_exchange / partial fold (partition.py:247-262, 642-646) for ranks on
 * one node.  The Helmholtz sweep stores its first / last owned row straight
 * into the neighbours' halo rows (peer memory: NVLink, or the same device),
 * and the launch's finalizing CTA writes this rank's value into every
 * rank's mailbox and then the launch sequence number into every rank's
 * flag word (system-scope fences in between).  The host then enqueues
 * sk_run_peer_wait (a stream wait on the local flags -- no SM spins) and
 * sk_run_combine over the local mailbox. */
#define SK_MAX_PEERS 8

typedef struct sk_peers {
  int32_t rank, world; /* world in [2, SK_MAX_PEERS] */
  void* up_rows[2];    /* rank-1's bottom halo row in its buf0 / buf1 (NULL on rank 0) */
  void* down_rows[2];  /* rank+1's top halo row in its buf0 / buf1 (NULL on the last rank) */
  double* mail[SK_MAX_PEERS];  /* rank p's mailbox, double[2][world] (mapped here) */
  uint32_t* flags[SK_MAX_PEERS]; /* rank p's flag words, uint32[world], zero at start */
} sk_peers;

/* Attach the peer transport to a Helmholtz run (before its first launch);
 * every later launch publishes its value and sequence number (1, 2, ...). */
int sk_run_set_peers(sk_run* run, const sk_peers* peers);

/* Enqueue on the run's stream: wait until every other rank has published
 * launch `seq` (its flag word here >= seq).  The mailbox row to combine is
 * mail[rank] + (seq & 1) * world. */
int sk_run_peer_wait(sk_run* run, int64_t seq);

/* Halo exchange between two runs of the same geometry that split one grid
 * (partition.py:247-262; e.g. a frame restored 1:n across GPUs, each run
 * computing its own partitions over a full-size replica): copy rows
 * [row_lo, row_hi) of iteration `it`'s result buffer -- and, for restore
 * runs, of its change-flag plane -- from `src` to `dst` (any devices:
 * peer copies over NVLink).  Enqueued on src's stream after iteration `it`;
 * dst's stream waits for the copy before its next launch.  No host sync. */
int sk_run_exchange_rows(sk_run* dst, sk_run* src, int64_t row_lo, int64_t row_hi, int64_t it);

/* Device memory that other processes can map (cudaMalloc + CUDA IPC):
 * allocate (zeroed), export a 64-byte handle, map a peer's handle, unmap,
 * free. */
int sk_ipc_alloc(int64_t bytes, void** d_ptr);
int sk_ipc_handle(void* d_ptr, uint8_t handle[64]);
int sk_ipc_open(const uint8_t handle[64], void** d_ptr);
int sk_ipc_close(void* d_ptr);
int sk_ipc_free(void* d_ptr);

/* Synchronise the run's stream and read its loop status: completed
 * iterations, the last combined value (cross-rank if sk_run_combine is used),
 * whether the loop stopped and whether the cap was hit. */
int sk_run_status(sk_run* run, int64_t* iterations, double* value, int32_t* stopped,
                  int32_t* exhausted);

/* Frame-batch restore runs (SK_FLAG_FRAMES): per-frame loop outcome after
 * sk_run_loop -- completed iterations (the frame's result is in buffer
 * iters[f] & 1), last reduce value, cap hit.  Arrays of `partitions`. */
int sk_run_frame_status(sk_run* run, int64_t* iterations, double* values, int32_t* exhausted);

/* Sum of CUDA-event durations of all timed sweep launches (SK_FLAG_TIMING). */
int sk_run_kernel_time(sk_run* run, double* total_ms, int64_t* launches);

/* Number of sweep kernels this run has launched (including no-op launches
 * past a device-decided stop). */
int sk_run_launches(sk_run* run, int64_t* launches);

/* Executor.abort / end of finish: release device state. */
int sk_run_destroy(sk_run* run);

/* Self-check of the engine's exact division by a run constant (see
 * sk_common.cuh div_const): number of fp32 numerators in the fast range whose
 * result differs from IEEE division x / b (0 expected; -1 = check failed). */
long long sk_verify_div_f32(float b, void* stream);

/* reduce_all for SUM / MAX (patterns.py:143-147): the left fold
 * acc = identity; for v in data: acc = fn(acc, v), row-major, on the device.
 * dtype SK_U8 / SK_I32 / SK_I64 (identity and result: int64; SUM wraps like
 * int64), SK_F32 / SK_F64 (identity and result in the element type; SUM is
 * folded sequentially in that type, MAX keeps `a if b < a else b`'s NaN and
 * tie behaviour): bit-identical to the sequential fold.  `identity` is a host
 * pointer (8 bytes; 4 for SK_F32), `d_out` device memory (8 bytes). */
int sk_reduce_fold(const void* d_data, int64_t n, int32_t dtype, int32_t op, const void* identity,
                   void* d_out, void* stream);

/* ---- batched map-only stencils for frame streams (config C2) -----------
 * Sobel edge magnitude (apps/sobel.py:47-66) over `frames` frames of
 * rows x cols u8 pixels, frame f at d_in + f*frame_stride (pitch bytes per
 * row), output likewise; d_sums[f] receives the frame's pixel sum (the
 * reference's _pixel_sum reduce, apps/sobel.py:73-74). */
int sk_sobel_frames(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride, uint8_t* d_out,
                    int64_t out_pitch, int64_t out_frame_stride, int32_t frames, int64_t rows,
                    int64_t cols, int64_t* d_sums, void* stream);

/* Adaptive-median noise detection (apps/denoise.py:105-135) over frames;
 * d_counts[f] receives the number of flagged pixels. */
int sk_amf_frames(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride, uint8_t* d_mask,
                  int64_t mask_pitch, int64_t mask_frame_stride, int32_t frames, int64_t rows,
                  int64_t cols, int32_t wmax, int64_t* d_counts, void* stream);

/* ---- user elemental functions (run-time compiled) -----------------------
 * The paper's API passes the elemental function, combinator and delta as
 * kernel source; the reference package passes Python
 * callables (ElementalFn.point, patterns.py:41-68; Combinator/Delta
 * patterns.py:85-122).  paper_1609_04567_b200/jit.py renders either as one
 * CUDA program against csrc/sk_jit_prelude.cuh; sk_jit_compile builds it
 * with NVRTC for sm_100a (no GPU needed) and keeps the cubin; the kernel is
 * loaded per device when a run starts. */
typedef struct sk_jit sk_jit;

int sk_jit_compile(const char* source, const char* name, sk_jit** out);
/* NVRTC log of the compile (owned by the program; may be empty) */
const char* sk_jit_log(const sk_jit* program);
int64_t sk_jit_cubin_size(const sk_jit* program);
/* copy the sm_100a cubin (sk_jit_cubin_size bytes) -- for cuobjdump / caching */
int sk_jit_cubin(const sk_jit* program, void* dst);
int sk_jit_destroy(sk_jit* program);

/* Executor.begin for a compiled elemental (plan->kernel = SK_KERNEL_JIT,
 * reduce_op SUM / MAX / CUSTOM).  plan->params: [0] rows per staged tile
 * (the program's SK_TH), [1] global row of owned row 0 and [2] global row
 * count when this run is one rank's row block of a larger grid (0, 0 for a
 * whole grid).  Each d_env[i] points at the env row of owned row 0; a row
 * block's env carries the same halo rows as its grid, before and after;
 * all env grids share one pitch (in elements).   d_src is the input grid (element type of
 * the program's sk_in_t), d_buf0/1 the iteration buffers (sk_val_t); d_env
 * holds n_env (0..4) read-only grids aligned with the loop grid, each with
 * its own pitch in elements.  Other calls as for sk_run_begin. */
int sk_run_begin_jit(const sk_plan* plan, const sk_jit* program, const void* d_src,
                     int64_t src_pitch, const void* const* d_env, const int64_t* env_pitch,
                     int32_t n_env, void* d_buf0, void* d_buf1, int64_t pitch, void* stream,
                     sk_run** out);

/* First elemental failure of a JIT run (the reference raises StencilError,
 * patterns.py:29-38): code 0 = none, 1 = ABSENT used as a number
 * (TypeError), 2 = division by zero, 3 = math domain error, 4 = int() of
 * inf/nan, 5 = returned None, 6 = env index off the grid (GridError),
 * 7 = window offset beyond the radius (IndexError), 8 = int ** negative int;
 * index = row-major element index (lowest failing); iteration = the failing
 * iteration.  A failed iteration's ring value (sk_run_value) is NaN and the
 * loop stops there. */
int sk_run_error(sk_run* run, int32_t* code, int64_t* index, int64_t* iteration);
#endif /* __CUDACC_RTC__ */

#ifdef __cplusplus
}
#endif

#endif /* STENCILKIT_B200_H */
