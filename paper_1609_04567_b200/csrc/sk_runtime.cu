// C-ABI runtime: run lifecycle, device-resident loop (CUDA graph WHILE),
// host-driven steps with asynchronous value readback, per-sweep timing.
//
// Maps the reference's Executor protocol (loop.py:124-137) and _drive
// (loop.py:198-224) onto device state.  See include/stencilkit_b200.h.
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>

#include <cuda.h>
#include <cstring>

#include "sk_internal.h"

namespace sk {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return SK_ERR_CUDA;
}

int device_sms(int device) {
  static std::mutex mu;
  static int cache[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0)
      n = 148;
    cache[device] = n;
  }
  return cache[device];
}

// The runs' small and per-run buffers come from the device's default
// stream-ordered pool (cudaMallocAsync).  Its release threshold defaults to
// 0: every synchronisation hands unused pool memory back to the driver, so
// a stream of runs (a farm restoring batch after batch) re-maps hundreds of
// MB per batch.  Keep it: the threshold goes to the maximum once per device.
void keep_pool(int device) {
  static std::mutex mu;
  static bool done[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64 || done[device]) return;
  done[device] = true;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

unsigned* stream_counter(int device, cudaStream_t s) {
  constexpr int kSlab = 4096;
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, unsigned*> slots;
  static unsigned* slab[64] = {};
  static int used[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64) return nullptr;
  auto key = std::make_pair(device, s);
  auto it = slots.find(key);
  if (it != slots.end()) return it->second;
  unsigned* p = nullptr;
  if (!slab[device]) {
    if (cudaMalloc(reinterpret_cast<void**>(&slab[device]), kSlab * sizeof(unsigned)) != cudaSuccess ||
        cudaMemset(slab[device], 0, kSlab * sizeof(unsigned)) != cudaSuccess) {
      set_error("stream_counter: cannot allocate the counter slab");
      slab[device] = nullptr;
      return nullptr;
    }
  }
  if (used[device] < kSlab) {
    p = slab[device] + used[device]++;
  } else if (cudaMalloc(reinterpret_cast<void**>(&p), sizeof(unsigned)) != cudaSuccess ||
             cudaMemset(p, 0, sizeof(unsigned)) != cudaSuccess) {
    set_error("stream_counter: cannot allocate a counter");
    return nullptr;
  }
  slots[key] = p;
  return p;
}

int occupancy(const void* fn, int block) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(fn, block);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, 0) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 1;
  }
  cache[key] = n;
  return n;
}

// Pinned, device-mapped arena for the per-run value rings (cudaHostAlloc is
// far too slow to call per run in a frame stream).
namespace {
struct RingArena {
  std::mutex mu;
  double* host = nullptr;
  double* dev = nullptr;
  std::vector<int> free_slots;
  static constexpr int kSlots = 1024;
  int init() {
    if (host) return SK_OK;
    SK_CUDA(cudaHostAlloc(&host, sizeof(double) * kRing * kSlots, cudaHostAllocMapped | cudaHostAllocPortable));
    SK_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), host, 0));
    for (int i = kSlots - 1; i >= 0; --i) free_slots.push_back(i);
    return SK_OK;
  }
  int take(double** h, double** d) {
    std::lock_guard<std::mutex> lk(mu);
    int rc = init();
    if (rc) return rc;
    if (free_slots.empty()) {
      set_error("too many concurrent runs (value-ring arena exhausted)");
      return SK_ERR_STATE;
    }
    int s = free_slots.back();
    free_slots.pop_back();
    *h = host + (size_t)s * kRing;
    *d = dev + (size_t)s * kRing;
    return SK_OK;
  }
  void give(double* h) {
    if (!h) return;
    std::lock_guard<std::mutex> lk(mu);
    free_slots.push_back((int)((h - host) / kRing));
  }
};
RingArena g_ring;
}  // namespace

// `c` set: a device loop (sk_run_loop), whose values the host never reads
// per iteration -- no writes to the host-mapped value ring.
static LoopCtl make_ctl(sk_run* r, const sk_cond* c, bool graph, cudaGraphConditionalHandle gh) {
  LoopCtl L;
  L.st = r->d_status;
  L.partials = r->d_partials;
  L.nparts = r->nparts;
  for (int i = 0; i <= r->nparts; ++i) L.part_chunk[i] = r->part_chunk[i];
  L.part_chunk_dev = r->part_chunk_dev;
  L.flagged_dev = r->flagged_dev;
  L.reduce = r->plan.reduce_op;
  L.identity = r->plan.identity;
  L.ring = c ? nullptr : r->d_ring;
  if (c) {
    L.cond.kind = c->kind;
    L.cond.a = c->a;
    L.cond.n = c->n;
    L.cond.max_it = c->max_iterations;
  } else {
    L.cond.kind = SK_COND_HOST;
    L.cond.a = 0;
    L.cond.n = 0;
    L.cond.max_it = (long long)1 << 62;
  }
  L.gh = gh;
  L.use_graph = graph ? 1 : 0;
  L.persistent = 0;
  L.peer.rank = L.peer.world = 0;
  L.peer.seq = 0;
  for (int p = 0; p < kMaxPeers; ++p) {
    L.peer.mail[p] = nullptr;
    L.peer.flag[p] = nullptr;
  }
  if (r->has_peers) {
    L.peer.rank = r->peers.rank;
    L.peer.world = r->peers.world;
    for (int p = 0; p < r->peers.world; ++p) {
      L.peer.mail[p] = r->peers.mail[p];
      L.peer.flag[p] = r->peers.flags[p];
    }
  }
  return L;
}

// Status read-back through a pinned, per-thread staging block: a copy into
// pageable stack memory is a staged, synchronous driver copy on top of the
// stream synchronise (~10 us per loop on the C1 path).
static int read_status(sk_run* r, Status* out) {
  thread_local Status* pinned = nullptr;
  if (!pinned && cudaMallocHost(reinterpret_cast<void**>(&pinned), sizeof(Status)) != cudaSuccess) {
    pinned = nullptr;
    cudaGetLastError();
  }
  if (pinned) {
    SK_CUDA(cudaMemcpyAsync(pinned, r->d_status, sizeof(Status), cudaMemcpyDeviceToHost, r->stream));
    SK_CUDA(cudaStreamSynchronize(r->stream));
    *out = *pinned;
  } else {
    SK_CUDA(cudaMemcpyAsync(out, r->d_status, sizeof(Status), cudaMemcpyDeviceToHost, r->stream));
    SK_CUDA(cudaStreamSynchronize(r->stream));
  }
  return SK_OK;
}

static int launch_timed(sk_run* r, const LoopCtl& L0) {
  LoopCtl L = L0;
  L.peer.seq = (unsigned)(r->launched + 1);  // this launch's sequence number
  cudaEvent_t a = nullptr, b = nullptr;
  if (r->timing) {
    SK_CUDA(cudaEventCreate(&a));
    SK_CUDA(cudaEventCreate(&b));
    SK_CUDA(cudaEventRecord(a, r->stream));
  }
  int rc = r->ops->launch(r, L, r->stream);
  if (rc) return rc;
  r->launched += 1;
  r->total_launches += 1;
  if (r->timing) {
    SK_CUDA(cudaEventRecord(b, r->stream));
    r->t_start.push_back(a);
    r->t_stop.push_back(b);
    // first iteration this launch computes (two per launch: 2L+1)
    r->t_iter.push_back(r->steps_per_launch == 2 ? 2 * r->launched - 1 : r->launched);
  }
  cudaEvent_t& ev = r->ev_done[r->launched % kRing];
  if (!ev) SK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  SK_CUDA(cudaEventRecord(ev, r->stream));
  return SK_OK;
}

// Cross-rank combine: one thread folds the gathered per-rank partials in
// rank order from the identity and decides the iteration.
__global__ void combine_kernel(Status* st, const double* parts, int n, int reduce,
                               double identity, CondDev cond, volatile double* ring) {
  const long long it = st->iter;
  if (st->stop || it == 0 || st->gdecided >= it) return;  // no new iteration to decide
  double acc = identity;
  for (int i = 0; i < n; ++i) {
    const double v = parts[i];
    if (reduce == SK_REDUCE_SUM) acc = acc + v;
    else acc = (v < acc) ? acc : v;
  }
  const int c = eval_cond(cond, acc, it);
  const int capped = it >= cond.max_it;
  st->gvalue = acc;
  st->gdecided = it;
  st->cond_true = c;
  st->exhausted = !c && capped;
  st->stop = c || capped;
  if (ring) ring[it % kRing] = acc;
}

}  // namespace sk

using namespace sk;

extern "C" {

const char* sk_last_error(void) { return g_err.c_str(); }

int sk_abi_version(void) { return SK_ABI_VERSION; }

int sk_run_begin(const sk_plan* plan, const void* d_src, int64_t src_pitch, const void* d_env,
                 int64_t env_pitch, void* d_buf0, void* d_buf1, int64_t pitch, void* stream,
                 sk_run** out) {
  return sk::begin_impl(plan, nullptr, d_src, src_pitch, d_env, env_pitch, nullptr, nullptr, 0, d_buf0,
                        d_buf1, pitch, stream, out);
}

}  // extern "C"

namespace sk {

int begin_impl(const sk_plan* plan, const sk_jit* jit, const void* d_src, int64_t src_pitch,
               const void* d_env, int64_t env_pitch, const void* const* jit_env,
               const int64_t* jit_env_pitch, int n_env, void* d_buf0, void* d_buf1, int64_t pitch,
               void* stream, sk_run** out) {
  if (!plan || !out || !d_buf0 || !d_buf1 || !d_src) {
    set_error("sk_run_begin: null argument");
    return SK_ERR_ARG;
  }
  *out = nullptr;
  if (plan->rows < 1 || plan->cols < 1 || plan->rows > (1ll << 31) - 2 || plan->cols > (1ll << 31) - 64) {
    set_error("sk_run_begin: bad grid dims");
    return SK_ERR_ARG;
  }
  if (plan->partitions < 1 || plan->partitions > kMaxParts || plan->partitions > plan->rows) {
    set_error("sk_run_begin: partitions must be in [1, min(rows, 64)]");
    return SK_ERR_ARG;
  }
  if (plan->reduce_op != SK_REDUCE_SUM && plan->reduce_op != SK_REDUCE_MAX &&
      !(jit && plan->reduce_op == SK_REDUCE_CUSTOM)) {
    set_error("sk_run_begin: unknown reduce op");
    return SK_ERR_ARG;
  }
  if ((plan->kernel == SK_KERNEL_JIT) != (jit != nullptr)) {
    set_error("sk_run_begin: user elemental kernels start with sk_run_begin_jit");
    return SK_ERR_ARG;
  }
  if (n_env < 0 || n_env > 4 || (n_env > 0 && (!jit_env || !jit_env_pitch))) {
    set_error("sk_run_begin_jit: 0..4 env grids");
    return SK_ERR_ARG;
  }
  const KernelOps* ops = nullptr;
  switch (plan->kernel) {
    case SK_KERNEL_JIT: ops = jit_ops(); break;
    case SK_KERNEL_HELMHOLTZ: ops = helmholtz_ops(); break;
    case SK_KERNEL_LIFE: ops = life_ops(); break;
    case SK_KERNEL_RESTORE: ops = restore_ops(); break;
    case SK_KERNEL_SOBEL: ops = u8_ops(); break;
    case SK_KERNEL_AMF: ops = amf_ops(); break;
    default:
      set_error("sk_run_begin: unknown kernel id");
      return SK_ERR_ARG;
  }
  // Keep stream-ordered allocations resident between runs: with the default
  // release threshold (0) the pool unmaps freed memory at every synchronise
  // and the next run's setup pays for re-mapping it.
  {
    static std::once_flag once[64];
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64)
      std::call_once(once[dev], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          unsigned long long thr = ~0ull;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
      });
  }
  sk_run* r = new sk_run();
  r->plan = *plan;
  r->ops = ops;
  r->stream = static_cast<cudaStream_t>(stream);
  r->src = d_src;
  r->src_pitch = src_pitch;
  r->env = d_env;
  r->env_pitch = env_pitch;
  r->buf[0] = d_buf0;
  r->buf[1] = d_buf1;
  r->pitch = pitch;
  r->timing = (plan->flags & SK_FLAG_TIMING) != 0;
  r->jit = jit;
  r->jit_nenv = n_env;
  for (int i = 0; i < n_env; ++i) {
    r->jit_env[i] = jit_env[i];
    r->jit_env_pitch[i] = jit_env_pitch[i];
  }
  r->no_graph = jit != nullptr;  // JIT kernels never set a graph condition
  int rc = SK_OK;
  cudaError_t ce = cudaGetDevice(&r->device);
  if (ce != cudaSuccess) {
    delete r;
    return cuda_fail(ce, "cudaGetDevice");
  }
  // partition row boundaries: remainder to the lowest partitions
  // (_split_ranges, partition.py:187-195)
  r->nparts = plan->partitions;
  {
    const long long base = plan->rows / r->nparts, rem = plan->rows % r->nparts;
    long long b = 0;
    r->part_row[0] = 0;
    for (int i = 0; i < r->nparts; ++i) {
      b += base + (i < rem ? 1 : 0);
      r->part_row[i + 1] = (int)b;
    }
  }
  keep_pool(r->device);
  rc = r->ops->setup(r);
  if (rc) {
    delete r;
    return rc;
  }
  auto fail = [&](cudaError_t e, const char* what) {
    int code = cuda_fail(e, what);
    sk_run_destroy(r);
    return code;
  };
  if ((ce = cudaMallocAsync(reinterpret_cast<void**>(&r->d_status), sizeof(Status), r->stream)))
    return fail(ce, "cudaMallocAsync(status)");
  if ((ce = cudaMemsetAsync(r->d_status, 0, sizeof(Status), r->stream)))
    return fail(ce, "cudaMemsetAsync(status)");
  // two partials slots per chunk: two-iteration launches reduce both
  const size_t np = 2 * ((size_t)(r->nchunks > r->grid ? r->nchunks : r->grid) + 1);
  if ((ce = cudaMallocAsync(reinterpret_cast<void**>(&r->d_partials), np * sizeof(double), r->stream)))
    return fail(ce, "cudaMallocAsync(partials)");
  if ((rc = g_ring.take(&r->h_ring, &r->d_ring))) {
    sk_run_destroy(r);
    return rc;
  }
  *out = r;
  return SK_OK;
}

}  // namespace sk

extern "C" {

int sk_run_launch(sk_run* r, int32_t n) {
  if (!r || n < 0) {
    set_error("sk_run_launch: bad argument");
    return SK_ERR_ARG;
  }
  LoopCtl L = make_ctl(r, nullptr, false, 0);
  for (int i = 0; i < n; ++i) {
    int rc = launch_timed(r, L);
    if (rc) return rc;
  }
  return SK_OK;
}

int sk_run_value(sk_run* r, int64_t it, double* value) {
  if (!r || !value || it < 1 || it > r->launched || it <= r->launched - kRing) {
    set_error("sk_run_value: iteration not in the launched window");
    return SK_ERR_ARG;
  }
  SK_CUDA(cudaEventSynchronize(r->ev_done[it % kRing]));
  *value = static_cast<volatile double*>(r->h_ring)[it % kRing];
  return SK_OK;
}

int sk_run_loop(sk_run* r, const sk_cond* c, int64_t* iterations, double* final_value,
                int32_t* exhausted) {
  if (!r || !c || c->max_iterations < 1) {
    set_error("sk_run_loop: bad argument");
    return SK_ERR_ARG;
  }
  if (r->launched != 0) {
    set_error("sk_run_loop: the run already has host-driven iterations");
    return SK_ERR_STATE;
  }
  int rc = SK_OK;
  // SK_NO_GRAPH=1 forces plain launches (profilers cannot see kernels inside
  // conditional graph nodes)
  const char* ng = getenv("SK_NO_GRAPH");
  const char* np = getenv("SK_NO_PERSIST");
  bool use_graph = !r->timing && !r->no_graph && !(ng && ng[0] == '1');
  bool persistent = !r->timing && !(np && np[0] == '1');
  if (persistent) {
    // One cooperative launch runs every iteration (in-kernel grid barrier
    // carrying the convergence decision); no per-iteration launches at all.
    LoopCtl L = make_ctl(r, c, false, 0);
    L.persistent = 1;
    rc = r->ops->launch(r, L, r->stream);
    if (rc == SK_OK) {
      use_graph = false;
      r->total_launches += 1;
      r->persistent_done = true;
    } else {
      cudaGetLastError();  // e.g. cooperative launch unavailable: fall back
      rc = SK_OK;
    }
  }
  if (use_graph && !r->persistent_done) {
    // One graph: conditional WHILE node whose body is one sweep; the sweep's
    // finalizing CTA clears the condition when the loop is over.
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ex = nullptr;
    cudaGraphConditionalHandle h;
    cudaError_t ce = cudaGraphCreate(&g, 0);
    if (ce == cudaSuccess) ce = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {};
    cudaGraphNode_t node;
    if (ce == cudaSuccess) {
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      ce = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
    }
    if (ce == cudaSuccess && !r->cap_stream) ce = cudaStreamCreateWithFlags(&r->cap_stream, cudaStreamNonBlocking);
    if (ce == cudaSuccess) {
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      ce = cudaStreamBeginCaptureToGraph(r->cap_stream, body, nullptr, nullptr, 0,
                                         cudaStreamCaptureModeRelaxed);
      if (ce == cudaSuccess) {
        LoopCtl L = make_ctl(r, c, true, h);
        rc = r->ops->launch(r, L, r->cap_stream);
        cudaGraph_t body2 = body;
        cudaError_t ce2 = cudaStreamEndCapture(r->cap_stream, &body2);
        if (rc) {
          cudaGraphDestroy(g);
          return rc;
        }
        ce = ce2;
      }
    }
    if (ce == cudaSuccess) ce = cudaGraphInstantiate(&ex, g, 0);
    if (g) cudaGraphDestroy(g);
    if (ce == cudaSuccess) {
      ce = cudaGraphLaunch(ex, r->stream);
      if (ce == cudaSuccess) r->gexec = ex;
      else cudaGraphExecDestroy(ex);
    }
    if (ce != cudaSuccess) {
      cudaGetLastError();  // clear; fall back to batched launches
      use_graph = false;
    }
  }
  if (!use_graph && !r->persistent_done) {
    // Batched launches: iterations after the device-decided stop are no-ops.
    LoopCtl L = make_ctl(r, c, false, 0);
    const int batch = 8;
    for (;;) {
      for (int i = 0; i < batch; ++i)
        if ((rc = launch_timed(r, L))) return rc;
      Status st;
      if (int rs = read_status(r, &st)) return rs;
      if (st.stop) break;
    }
  }
  Status st;
  if (int rs = read_status(r, &st)) return rs;
  if (!st.stop) {
    set_error("sk_run_loop: device loop ended without a decision");
    return SK_ERR_STATE;
  }
  if (use_graph)  // one sweep kernel per WHILE-body execution
    r->total_launches += r->steps_per_launch == 2 ? (st.iter + 1) / 2 : st.iter;
  if (st.fix) {  // stopped at the first iteration of a two-iteration launch
    if (!r->ops->fixup) {
      set_error("sk_run_loop: kernel cannot recompute a skipped iteration");
      return SK_ERR_STATE;
    }
    if ((rc = r->ops->fixup(r, st.iter, r->stream))) return rc;
    r->total_launches += 1;
    SK_CUDA(cudaStreamSynchronize(r->stream));
  }
  r->launched = st.iter;  // committed iterations
  if (iterations) *iterations = st.iter;
  if (final_value) *final_value = st.value;
  if (exhausted) *exhausted = st.exhausted;
  return SK_OK;
}

int sk_run_result(sk_run* r, int64_t it, int32_t* which) {
  if (!r || !which || it < 0 || it > r->launched) {
    set_error("sk_run_result: iteration out of range");
    return SK_ERR_ARG;
  }
  if (it == 0) *which = -1;
  else if (r->steps_per_launch == 2) *which = (int32_t)(((it - 1) >> 1) & 1);
  else *which = (int32_t)(it & 1);
  return SK_OK;
}

static size_t dtype_size(int dt) {
  switch (dt) {
    case SK_U8: return 1;
    case SK_F32: return 4;
    case SK_F64: return 8;
    default: return 8;
  }
}

int sk_run_exchange_rows(sk_run* dst, sk_run* src, int64_t row_lo, int64_t row_hi, int64_t it) {
  if (!dst || !src || dst == src || row_lo < 0 || row_hi > src->plan.rows || row_lo >= row_hi ||
      it < 1 || it > src->launched || dst->plan.rows != src->plan.rows ||
      dst->plan.cols != src->plan.cols || dst->plan.dtype != src->plan.dtype ||
      dst->plan.kernel != src->plan.kernel || dst->plan.halo_top != src->plan.halo_top ||
      src->steps_per_launch != 1 || dst->steps_per_launch != 1) {
    set_error("sk_run_exchange_rows: runs of one geometry, rows inside the grid, a launched iteration");
    return SK_ERR_ARG;
  }
  const size_t esz = dtype_size(src->plan.dtype);
  const int b = (int)(it & 1);
  const long long off_rows = src->plan.halo_top + row_lo;
  const size_t width = (size_t)src->plan.cols * esz;
  const char* sp = static_cast<const char*>(src->buf[b]) + off_rows * src->pitch * esz;
  char* dp = static_cast<char*>(dst->buf[b]) + off_rows * dst->pitch * esz;
  SK_CUDA(cudaMemcpy2DAsync(dp, dst->pitch * esz, sp, src->pitch * esz, width,
                            (size_t)(row_hi - row_lo), cudaMemcpyDefault, src->stream));
  unsigned char* sc = restore_chg(src, it);
  unsigned char* dc = restore_chg(dst, it);
  if (sc && dc) {
    const size_t n = (size_t)(row_hi - row_lo) * src->plan.cols;
    SK_CUDA(cudaMemcpyAsync(dc + row_lo * src->plan.cols, sc + row_lo * src->plan.cols, n,
                            cudaMemcpyDefault, src->stream));
  }
  cudaEvent_t ev = nullptr;
  SK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  cudaError_t e1 = cudaEventRecord(ev, src->stream);
  cudaError_t e2 = e1 == cudaSuccess ? cudaStreamWaitEvent(dst->stream, ev, 0) : e1;
  cudaEventDestroy(ev);  // released once the wait has been satisfied
  if (e2 != cudaSuccess) return cuda_fail(e2, "sk_run_exchange_rows");
  return SK_OK;
}

int sk_run_value_ptr(sk_run* r, void** d_value) {
  if (!r || !d_value) {
    set_error("sk_run_value_ptr: null argument");
    return SK_ERR_ARG;
  }
  *d_value = reinterpret_cast<char*>(r->d_status) + offsetof(Status, value);
  return SK_OK;
}

int sk_run_kernel_time(sk_run* r, double* total_ms, int64_t* launches) {
  if (!r || !total_ms || !launches) {
    set_error("sk_run_kernel_time: null argument");
    return SK_ERR_ARG;
  }
  // Only sweeps that computed an iteration count (over-launched no-ops after
  // the device-decided stop are excluded).
  Status st;
  if (int rs = read_status(r, &st)) return rs;
  double tot = 0;
  long long n = 0;
  for (size_t i = 0; i < r->t_start.size(); ++i) {
    if (r->t_iter[i] > st.iter) continue;
    float ms = 0;
    SK_CUDA(cudaEventElapsedTime(&ms, r->t_start[i], r->t_stop[i]));
    tot += ms;
    ++n;
  }
  *total_ms = tot;
  *launches = n;
  return SK_OK;
}

int sk_run_combine(sk_run* r, const double* d_partials, int32_t n, const sk_cond* c) {
  if (!r || !d_partials || n < 1 || !c) {
    set_error("sk_run_combine: bad argument");
    return SK_ERR_ARG;
  }
  CondDev cd;
  cd.kind = c->kind;
  cd.a = c->a;
  cd.n = c->n;
  cd.max_it = c->max_iterations;
  combine_kernel<<<1, 1, 0, r->stream>>>(r->d_status, d_partials, n, r->plan.reduce_op,
                                         r->plan.identity, cd, r->d_ring);
  SK_CUDA(cudaGetLastError());
  r->combined = true;
  return SK_OK;
}

int sk_run_set_peers(sk_run* r, const sk_peers* p) {
  if (!r || !p || p->world < 2 || p->world > SK_MAX_PEERS || p->rank < 0 || p->rank >= p->world) {
    set_error("sk_run_set_peers: bad argument");
    return SK_ERR_ARG;
  }
  if (r->plan.kernel != SK_KERNEL_HELMHOLTZ) {
    set_error("sk_run_set_peers: the peer transport is implemented for the Helmholtz sweep");
    return SK_ERR_UNSUPPORTED;
  }
  if (r->launched != 0) {
    set_error("sk_run_set_peers: attach before the first launch");
    return SK_ERR_STATE;
  }
  for (int q = 0; q < p->world; ++q)
    if (!p->mail[q] || !p->flags[q]) {
      set_error("sk_run_set_peers: every rank needs a mailbox and flag words");
      return SK_ERR_ARG;
    }
  if ((p->rank > 0) != (p->up_rows[0] && p->up_rows[1]) ||
      (p->rank < p->world - 1) != (p->down_rows[0] && p->down_rows[1]) ||
      (p->rank > 0) != (r->plan.halo_top == 1) || (p->rank < p->world - 1) != (r->plan.halo_bottom == 1)) {
    set_error("sk_run_set_peers: neighbour halo rows do not match the run's halo layout");
    return SK_ERR_ARG;
  }
  r->peers = *p;
  r->has_peers = true;
  return SK_OK;
}

int sk_run_peer_wait(sk_run* r, int64_t seq) {
  if (!r || !r->has_peers || seq < 1) {
    set_error("sk_run_peer_wait: run has no peer transport, or bad sequence number");
    return SK_ERR_ARG;
  }
  static decltype(&cuStreamWaitValue32) wait32 = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &f, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      wait32 = reinterpret_cast<decltype(&cuStreamWaitValue32)>(f);
  });
  if (!wait32) {
    set_error("sk_run_peer_wait: cuStreamWaitValue32 unavailable");
    return SK_ERR_UNSUPPORTED;
  }
  const sk_peers& p = r->peers;
  uint32_t* mine = p.flags[p.rank];
  for (int q = 0; q < p.world; ++q) {
    if (q == p.rank) continue;
    CUresult e = wait32(reinterpret_cast<CUstream>(r->stream), reinterpret_cast<CUdeviceptr>(mine + q),
                        (cuuint32_t)seq, CU_STREAM_WAIT_VALUE_GEQ);
    if (e != CUDA_SUCCESS) {
      set_error("sk_run_peer_wait: cuStreamWaitValue32 failed (" + std::to_string((int)e) + ")");
      return SK_ERR_CUDA;
    }
  }
  return SK_OK;
}

int sk_ipc_alloc(int64_t bytes, void** d_ptr) {
  if (bytes < 1 || !d_ptr) {
    set_error("sk_ipc_alloc: bad argument");
    return SK_ERR_ARG;
  }
  SK_CUDA(cudaMalloc(d_ptr, (size_t)bytes));
  SK_CUDA(cudaMemset(*d_ptr, 0, (size_t)bytes));
  return SK_OK;
}

int sk_ipc_handle(void* d_ptr, uint8_t handle[64]) {
  if (!d_ptr || !handle) {
    set_error("sk_ipc_handle: null argument");
    return SK_ERR_ARG;
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  SK_CUDA(cudaIpcGetMemHandle(&h, d_ptr));
  memcpy(handle, &h, 64);
  return SK_OK;
}

int sk_ipc_open(const uint8_t handle[64], void** d_ptr) {
  if (!handle || !d_ptr) {
    set_error("sk_ipc_open: null argument");
    return SK_ERR_ARG;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  SK_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SK_OK;
}

int sk_ipc_close(void* d_ptr) {
  if (!d_ptr) return SK_OK;
  SK_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return SK_OK;
}

int sk_ipc_free(void* d_ptr) {
  if (!d_ptr) return SK_OK;
  SK_CUDA(cudaFree(d_ptr));
  return SK_OK;
}

int sk_run_status(sk_run* r, int64_t* iterations, double* value, int32_t* stopped,
                  int32_t* exhausted) {
  if (!r) {
    set_error("sk_run_status: null run");
    return SK_ERR_ARG;
  }
  Status st;
  if (int rs = read_status(r, &st)) return rs;
  if (iterations) *iterations = st.iter;
  if (value) *value = r->combined ? st.gvalue : st.value;
  if (stopped) *stopped = st.stop;
  if (exhausted) *exhausted = st.exhausted;
  return SK_OK;
}

int sk_run_frame_status(sk_run* r, int64_t* iterations, double* values, int32_t* exhausted) {
  if (!r || !iterations || !values || !exhausted) {
    set_error("sk_run_frame_status: null argument");
    return SK_ERR_ARG;
  }
  static_assert(sizeof(long long) == sizeof(int64_t), "");
  return restore_frame_status(r, reinterpret_cast<long long*>(iterations), values,
                              reinterpret_cast<int*>(exhausted));
}

int sk_run_launches(sk_run* r, int64_t* launches) {
  if (!r || !launches) {
    set_error("sk_run_launches: null argument");
    return SK_ERR_ARG;
  }
  *launches = r->total_launches;
  return SK_OK;
}

int sk_run_destroy(sk_run* r) {
  if (!r) return SK_OK;
  int rc = SK_OK;
  // the run's stream may still be executing: wait before freeing
  if (r->stream || true) {
    cudaError_t e = cudaStreamSynchronize(r->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaStreamSynchronize(destroy)");
  }
  if (r->ops && r->ops->teardown) r->ops->teardown(r);
  if (r->gexec) cudaGraphExecDestroy(r->gexec);
  if (r->cap_stream) cudaStreamDestroy(r->cap_stream);
  for (auto& e : r->ev_done)
    if (e) cudaEventDestroy(e);
  for (auto e : r->t_start) cudaEventDestroy(e);
  for (auto e : r->t_stop) cudaEventDestroy(e);
  if (r->d_status) cudaFreeAsync(r->d_status, r->stream);
  if (r->d_partials) cudaFreeAsync(r->d_partials, r->stream);
  g_ring.give(r->h_ring);
  delete r;
  return rc;
}

}  // extern "C"
