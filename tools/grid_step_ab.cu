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
  return 0;
}
