// Run-time compiled user elemental functions (SURVEY next-1 / next-2).
//
// The paper's API takes the elemental function, the combinator and the
// delta as kernel source (Fig. 1); the
// reference package takes Python callables (ElementalFn.point,
// patterns.py:41-68).  paper_1609_04567_b200/jit.py turns either into a CUDA
// program (sk_jit_prelude.cuh + generated part + sk_jit_kernel.cuh); this
// file compiles it with NVRTC for sm_100a, loads it per device through the
// driver API (entry points fetched from the runtime, so the library does not
// link libcuda), and plugs the kernel into the run machinery as one more
// KernelOps (SK_KERNEL_JIT): the same device-resident loop, reduce fold and
// loop test as the built-in kernels.
#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "sk_internal.h"
#include "sk_jit_prelude.cuh"
#include "sk_sweep.cuh"

// the headers NVRTC sees (generated at build time from the files above)
#include "sk_jit_headers.inc"

struct sk_jit {
  std::string log;
  std::vector<char> cubin;
  std::mutex mu;
  CUmodule mod[64] = {};
  CUfunction fn[64] = {};
  int occ[64] = {};
  int smem[64] = {};  // dynamic shared memory bytes per launch
  int block = 256;
};

namespace sk {
namespace {

// ---------------------------------------------------------------- NVRTC
struct Nvrtc {
  bool ok = false;
  std::string why;
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcGetErrorString) err = nullptr;
};

const Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
    void* h = nullptr;
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      n.why = "libnvrtc.so.12 not found";
      return;
    }
#define SK_SYM(f, s) n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, s))
    SK_SYM(create, "nvrtcCreateProgram");
    SK_SYM(compile, "nvrtcCompileProgram");
    SK_SYM(log_size, "nvrtcGetProgramLogSize");
    SK_SYM(log, "nvrtcGetProgramLog");
    SK_SYM(cubin_size, "nvrtcGetCUBINSize");
    SK_SYM(cubin, "nvrtcGetCUBIN");
    SK_SYM(destroy, "nvrtcDestroyProgram");
    SK_SYM(err, "nvrtcGetErrorString");
#undef SK_SYM
    n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy && n.err;
    if (!n.ok) n.why = "libnvrtc is missing symbols";
  });
  return n;
}

// ---------------------------------------------------------------- driver API
struct Driver {
  bool ok = false;
  decltype(&cuModuleLoadData) load = nullptr;
  decltype(&cuModuleGetFunction) get = nullptr;
  decltype(&cuModuleUnload) unload = nullptr;
  decltype(&cuLaunchKernel) launch = nullptr;
  decltype(&cuLaunchCooperativeKernel) launch_coop = nullptr;
  decltype(&cuOccupancyMaxActiveBlocksPerMultiprocessor) occupancy = nullptr;
  decltype(&cuGetErrorName) err = nullptr;
  decltype(&cuModuleGetGlobal) global = nullptr;
  decltype(&cuMemcpyDtoH) dtoh = nullptr;
  decltype(&cuFuncSetAttribute) setattr = nullptr;
};

const Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* s, void** f) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPointByVersion(s, f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *f;
    };
    bool ok = true;
    ok &= get("cuModuleLoadData", reinterpret_cast<void**>(&d.load));
    ok &= get("cuModuleGetFunction", reinterpret_cast<void**>(&d.get));
    ok &= get("cuModuleUnload", reinterpret_cast<void**>(&d.unload));
    ok &= get("cuLaunchKernel", reinterpret_cast<void**>(&d.launch));
    ok &= get("cuLaunchCooperativeKernel", reinterpret_cast<void**>(&d.launch_coop));
    ok &= get("cuOccupancyMaxActiveBlocksPerMultiprocessor", reinterpret_cast<void**>(&d.occupancy));
    ok &= get("cuGetErrorName", reinterpret_cast<void**>(&d.err));
    ok &= get("cuModuleGetGlobal", reinterpret_cast<void**>(&d.global));
    ok &= get("cuMemcpyDtoH", reinterpret_cast<void**>(&d.dtoh));
    ok &= get("cuFuncSetAttribute", reinterpret_cast<void**>(&d.setattr));
    d.ok = ok;
    cudaGetLastError();
  });
  return d;
}

int cu_fail(CUresult r, const char* what) {
  const char* nm = nullptr;
  if (driver().err) driver().err(r, &nm);
  set_error(std::string(what) + ": " + (nm ? nm : "CUDA driver error"));
  return SK_ERR_CUDA;
}

// The program's kernel on the current device (module loaded on first use).
int jit_function(sk_jit* j, int dev, CUfunction* fn) {
  if (dev < 0 || dev >= 64) {
    set_error("sk_jit: device index out of range");
    return SK_ERR_ARG;
  }
  std::lock_guard<std::mutex> lk(j->mu);
  if (!j->fn[dev]) {
    const Driver& d = driver();
    if (!d.ok) {
      set_error("sk_jit: CUDA driver entry points unavailable");
      return SK_ERR_CUDA;
    }
    SK_CUDA(cudaFree(nullptr));  // the device's primary context is current
    CUmodule m;
    CUresult r = d.load(&m, j->cubin.data());
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuModuleLoadData(user elemental)");
    CUfunction f;
    r = d.get(&f, m, "sk_jit_sweep");
    if (r != CUDA_SUCCESS) {
      d.unload(m);
      return cu_fail(r, "cuModuleGetFunction(sk_jit_sweep)");
    }
    // the tile buffers are dynamic shared memory; the program says how much
    // (sk_jit_smem_bytes), which may pass the 48 KB default
    int smem = 0;
    CUdeviceptr gp = 0;
    size_t gsz = 0;
    if (d.global(&gp, &gsz, m, "sk_jit_smem_bytes") != CUDA_SUCCESS || gsz != sizeof(int) ||
        d.dtoh(&smem, gp, sizeof(int)) != CUDA_SUCCESS) {
      d.unload(m);
      set_error("sk_jit: program lacks sk_jit_smem_bytes");
      return SK_ERR_STATE;
    }
    r = d.setattr(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem);
    if (r != CUDA_SUCCESS) {
      d.unload(m);
      return cu_fail(r, "cuFuncSetAttribute(user elemental shared memory)");
    }
    int occ = 0;
    if (d.occupancy(&occ, f, j->block, (size_t)smem) != CUDA_SUCCESS || occ < 1) occ = 1;
    j->mod[dev] = m;
    j->fn[dev] = f;
    j->occ[dev] = occ;
    j->smem[dev] = smem;
  }
  *fn = j->fn[dev];
  return SK_OK;
}

constexpr int kTW = 128;  // sk_jit_kernel.cuh tile width; rows per tile = plan.params[0]

int jit_setup(sk_run* r) {
  sk_jit* j = const_cast<sk_jit*>(r->jit);
  if (r->plan.halo_top < 0 || r->plan.halo_bottom < 0) {
    set_error("negative halo rows");
    return SK_ERR_ARG;
  }
  for (int i = 1; i < r->jit_nenv; ++i)
    if (r->jit_env_pitch[i] != r->jit_env_pitch[0]) {
      set_error("sk_run_begin_jit: env grids must share one pitch (elements)");
      return SK_ERR_ARG;
    }
  CUfunction f;
  int rc = jit_function(j, r->device, &f);
  if (rc) return rc;
  r->block = j->block;
  // params[3] == 1: a rank-1 grid (one column, pitch 1) run with contiguous
  // element tiles of SK_TH * SK_TW (program compiled with SK_NDIM 1)
  const bool rank1 = r->plan.params[3] == 1.0;
  if (rank1 && r->plan.cols != 1) {
    set_error("sk_run_begin_jit: a rank-1 program runs on a one-column grid");
    return SK_ERR_ARG;
  }
  r->colblocks = rank1 ? 1 : (int)((r->plan.cols + kTW - 1) / kTW);
  const int kTH = r->plan.params[0] >= 1 ? (int)r->plan.params[0] : 16;  // the program's SK_TH
  const int tile_rows = rank1 ? kTH * kTW : kTH;  // rows (= elements, rank 1) per tile
  // chunk = a run of tiles: as tall as possible (<= 8 tiles) while leaving
  // ~4 chunks per resident CTA for balance
  {
    const long long slots = (long long)device_sms(r->device) * j->occ[r->device];
    const long long tiles = ((r->plan.rows + tile_rows - 1) / tile_rows) * r->colblocks;
    long long m = tiles / (4 * slots);
    m = m < 1 ? 1 : (m > 8 ? 8 : m);
    r->chunk_rows = (int)(tile_rows * m);
  }
  int n = 0;
  r->part_chunk[0] = 0;
  for (int i = 0; i < r->nparts; ++i) {
    const int pr = r->part_row[i + 1] - r->part_row[i];
    n += ((pr + r->chunk_rows - 1) / r->chunk_rows) * r->colblocks;
    r->part_chunk[i + 1] = n;
  }
  r->nchunks = n;
  const long long slots = (long long)device_sms(r->device) * j->occ[r->device];
  r->grid = (int)(slots < n ? slots : n);
  if (r->grid < 1) r->grid = 1;
  return SK_OK;
}

int jit_launch(sk_run* r, const LoopCtl& L, cudaStream_t s) {
  sk_jit* j = const_cast<sk_jit*>(r->jit);
  CUfunction f;
  int rc = jit_function(j, r->device, &f);
  if (rc) return rc;
  JitArgs a;
  memset(&a, 0, sizeof(a));
  Sweep2D& g = a.g;
  g.src = r->src;
  g.src_pitch = r->src_pitch;
  g.buf[0] = r->buf[0];
  g.buf[1] = r->buf[1];
  g.pitch = r->pitch;
  g.rows = (int)r->plan.rows;
  g.cols = (int)r->plan.cols;
  g.halo_top = r->plan.halo_top;
  g.halo_bottom = r->plan.halo_bottom;
  g.colblocks = r->colblocks;
  g.chunk_rows = r->chunk_rows;
  for (int i = 0; i <= r->nparts; ++i) g.part_row[i] = r->part_row[i];
  a.L = L;
  // a row block of a larger grid: global row of owned row 0, global rows
  const int row0 = (int)r->plan.params[1];
  const int grows = r->plan.params[2] >= 1 ? (int)r->plan.params[2] : g.rows;
  for (int i = 0; i < r->jit_nenv; ++i) {
    a.env.p[i] = r->jit_env[i];  // -> owned row 0 (halo rows, if any, precede it)
    a.env.pitch[i] = r->jit_env_pitch[i];
  }
  a.env.rows = grows;
  a.env.cols = g.cols;
  a.env.row0 = row0;
  a.env.lo = row0 - g.halo_top;
  a.env.hi = row0 + g.rows + g.halo_bottom;
  void* params[] = {&a};
  const Driver& d = driver();
  CUresult cr;
  if (L.persistent) {
    const int slots = device_sms(r->device) * j->occ[r->device];
    const int grid = r->grid < slots ? r->grid : slots;
    cr = d.launch_coop(f, grid, 1, 1, r->block, 1, 1, (unsigned)j->smem[r->device],
                       reinterpret_cast<CUstream>(s), params);
  } else {
    cr = d.launch(f, r->grid, 1, 1, r->block, 1, 1, (unsigned)j->smem[r->device],
                  reinterpret_cast<CUstream>(s), params, nullptr);
  }
  if (cr != CUDA_SUCCESS) return cu_fail(cr, "cuLaunchKernel(user elemental)");
  return SK_OK;
}

void jit_teardown(sk_run*) {}

const KernelOps kJitOps = {jit_setup, jit_launch, jit_teardown};

// JitArgs is built on the host and read by NVRTC-compiled code: both sides
// compile the same headers, the size check below catches drift.
static_assert(sizeof(SkEnv) == 4 * 8 + 4 * 8 + 5 * 4 + 4, "SkEnv layout");

}  // namespace

const KernelOps* jit_ops() { return &kJitOps; }

}  // namespace sk

using namespace sk;

extern "C" {

int sk_jit_compile(const char* source, const char* name, sk_jit** out) {
  if (!source || !out) {
    set_error("sk_jit_compile: null argument");
    return SK_ERR_ARG;
  }
  *out = nullptr;
  const Nvrtc& n = nvrtc();
  if (!n.ok) {
    set_error("sk_jit_compile: " + n.why);
    return SK_ERR_UNSUPPORTED;
  }
  nvrtcProgram prog;
  nvrtcResult res = n.create(&prog, source, name ? name : "sk_user_elemental.cu", kJitHeaderCount,
                             kJitHeaderSrcs, kJitHeaderNames);
  if (res != NVRTC_SUCCESS) {
    set_error(std::string("nvrtcCreateProgram: ") + n.err(res));
    return SK_ERR_ARG;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo",
                        "-DSK_JIT=1"};
  res = n.compile(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  sk_jit* j = new sk_jit();
  size_t ls = 0;
  if (n.log_size(prog, &ls) == NVRTC_SUCCESS && ls > 1) {
    j->log.resize(ls);
    n.log(prog, &j->log[0]);
    j->log.resize(strlen(j->log.c_str()));
  }
  if (res != NVRTC_SUCCESS) {
    set_error("sk_jit_compile: " + std::string(n.err(res)) + "\n" + j->log);
    n.destroy(&prog);
    delete j;
    return SK_ERR_ARG;
  }
  size_t cs = 0;
  if (n.cubin_size(prog, &cs) != NVRTC_SUCCESS || cs == 0) {
    set_error("sk_jit_compile: no cubin produced");
    n.destroy(&prog);
    delete j;
    return SK_ERR_STATE;
  }
  j->cubin.resize(cs);
  n.cubin(prog, j->cubin.data());
  n.destroy(&prog);
  *out = j;
  return SK_OK;
}

const char* sk_jit_log(const sk_jit* j) { return j ? j->log.c_str() : ""; }

int64_t sk_jit_cubin_size(const sk_jit* j) { return j ? (int64_t)j->cubin.size() : 0; }

int sk_jit_cubin(const sk_jit* j, void* dst) {
  if (!j || !dst) {
    set_error("sk_jit_cubin: null argument");
    return SK_ERR_ARG;
  }
  memcpy(dst, j->cubin.data(), j->cubin.size());
  return SK_OK;
}

int sk_jit_destroy(sk_jit* j) {
  if (!j) return SK_OK;
  const Driver& d = driver();
  for (int i = 0; i < 64; ++i)
    if (j->mod[i] && d.unload) {
      int prev = 0;
      cudaGetDevice(&prev);
      if (cudaSetDevice(i) == cudaSuccess) d.unload(j->mod[i]);
      cudaSetDevice(prev);
    }
  delete j;
  return SK_OK;
}

int sk_run_begin_jit(const sk_plan* plan, const sk_jit* jit, const void* d_src, int64_t src_pitch,
                     const void* const* d_env, const int64_t* env_pitch, int32_t n_env, void* d_buf0,
                     void* d_buf1, int64_t pitch, void* stream, sk_run** out) {
  if (!jit) {
    set_error("sk_run_begin_jit: null program");
    return SK_ERR_ARG;
  }
  return begin_impl(plan, jit, d_src, src_pitch, nullptr, 0, d_env, env_pitch, n_env, d_buf0, d_buf1,
                    pitch, stream, out);
}

int sk_run_error(sk_run* r, int32_t* code, int64_t* index, int64_t* iteration) {
  if (!r || !code || !index || !iteration) {
    set_error("sk_run_error: null argument");
    return SK_ERR_ARG;
  }
  Status st;
  SK_CUDA(cudaMemcpyAsync(&st, r->d_status, sizeof(Status), cudaMemcpyDeviceToHost, r->stream));
  SK_CUDA(cudaStreamSynchronize(r->stream));
  *iteration = st.err_iter;
  if (st.err == 0) {
    *code = 0;
    *index = -1;
  } else {
    const unsigned long long k = ~st.err;
    *code = (int32_t)(k & 0xff);
    *index = (int64_t)(k >> 8);
  }
  return SK_OK;
}

}  // extern "C"
