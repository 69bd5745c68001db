// Latency of the resident loop's grid step on B200, standalone (tools/, not
// product): N iterations of {arrive, wait} over 128 co-resident CTAs,
// flat (every CTA on one global counter) vs hierarchical (cluster barrier,
// one CTA per cluster on the global counter, cluster barrier) and the
// cluster barrier alone.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gs tools/grid_step_ab.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1;} } while (0)

__device__ __forceinline__ void flat_step(unsigned* cnt, unsigned want) {
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    unsigned seen;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
    } while ((int)(seen - want) < 0);
  }
  __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) steps(unsigned* cnt, int iters, long long* out) {
  long long t0 = clock64();
  const int nb = gridDim.x;
  cg::cluster_group cl = cg::this_cluster();
  const int ncl = nb / (int)cl.num_blocks();
  for (int it = 1; it <= iters; ++it) {
    if (MODE == 0) {
      flat_step(cnt, (unsigned)(nb * it));
    } else if (MODE == 1) {
      cl.sync();
      if (cl.block_rank() == 0) flat_step(cnt, (unsigned)(ncl * it));
      cl.sync();
    } else if (MODE == 2) {
      cl.sync();
    } else {
      // hierarchical with split arrive/wait on the cluster barrier
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      if (cl.block_rank() == 0) flat_step(cnt, (unsigned)(ncl * it));
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = clock64() - t0;
}

// LL halo exchange: every CTA stores its two edge rows as (value, tag)
// 8-byte pairs and polls its neighbours' rows until every tag equals the
// iteration (no barrier, no fence, one L2 round trip); the global counter
// is arrived on but waited for only two iterations later (lagged decision).
__global__ void __launch_bounds__(512, 1) ll_steps(unsigned* cnt, unsigned long long* xb, int iters, int cols,
                                                   long long* out, int lag) {
  const int nb = gridDim.x, b = blockIdx.x;
  float acc = 0.f;
  for (int it = 1; it <= iters; ++it) {
    unsigned long long* mine = xb + ((size_t)((it & 1) * nb + b) * 2) * cols;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
      const unsigned long long v = ((unsigned long long)(unsigned)it << 32) | __float_as_uint(acc + c);
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(mine + c), "l"(v) : "memory");
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(mine + cols + c), "l"(v) : "memory");
    }
    if (lag >= 0 && threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      if (it > lag) {
        const unsigned want = (unsigned)(nb * (it - lag));
        unsigned seen;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
        } while ((int)(seen - want) < 0);
      }
    }
    // neighbours' rows of `it`
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
      if (b > 0) {
        const unsigned long long* p = xb + ((size_t)((it & 1) * nb + b - 1) * 2 + 1) * cols + c;
        unsigned long long v;
        do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); } while ((unsigned)(v >> 32) != (unsigned)it);
        acc += __uint_as_float((unsigned)v) * 1e-9f;
      }
      if (b + 1 < nb) {
        const unsigned long long* p = xb + ((size_t)((it & 1) * nb + b + 1) * 2) * cols + c;
        unsigned long long v;
        do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); } while ((unsigned)(v >> 32) != (unsigned)it);
        acc += __uint_as_float((unsigned)v) * 1e-9f;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && b == 0) *out = (long long)acc;
}

int run_ll(int nb, int iters, int lag) {
  unsigned* cnt; long long* out; unsigned long long* xb;
  const int cols = 1024;
  CK(cudaMalloc(&cnt, 4)); CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&xb, (size_t)2 * nb * 2 * cols * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaMemset(cnt, 0, 4)); CK(cudaMemset(xb, 0, (size_t)2 * nb * 2 * cols * 8));
    void* args[] = {&cnt, &xb, &iters, (void*)&cols, &out, &lag};
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)ll_steps, nb, 512, args, 0, 0));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("LL neighbour exchange (lag %2d)       nb %3d: %.3f us per step\n", lag, nb, best * 1e3 / iters);
  cudaFree(cnt); cudaFree(out); cudaFree(xb);
  return 0;
}

template <int MODE>
int run(const char* name, int nb, int cluster, int iters) {
  unsigned* cnt; long long* out;
  CK(cudaMalloc(&cnt, 4)); CK(cudaMalloc(&out, 8));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb); cfg.blockDim = dim3(256);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  if (cluster > 8) { CK(cudaFuncSetAttribute(steps<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)); }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaMemset(cnt, 0, 4));
    cudaEventRecord(e0);
    CK(cudaLaunchKernelEx(&cfg, steps<MODE>, cnt, iters, out));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("%-36s nb %3d cluster %2d: %.3f us per step (%d steps, launch incl.)\n", name, nb, cluster,
         best * 1e3 / iters, iters);
  cudaFree(cnt); cudaFree(out);
  return 0;
}

int main() {
  const int it = 2000;
  run<0>("flat global counter", 128, 1, it);
  run<0>("flat global counter", 148, 1, it);
  run<0>("flat global counter (cluster 8 launch)", 128, 8, it);
  run<1>("cluster.sync + global + cluster.sync", 128, 8, it);
  run<1>("cluster.sync + global + cluster.sync", 128, 16, it);
  run<3>("split cluster + global + cluster", 128, 16, it);
  run<2>("cluster.sync only", 128, 8, it);
  run<2>("cluster.sync only", 128, 16, it);
  run_ll(147, it, -1);
  run_ll(147, it, 1);
  run_ll(147, it, 2);
  run_ll(147, it, 0);
  return 0;
}
