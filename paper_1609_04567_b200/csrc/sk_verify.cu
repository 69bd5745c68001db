// Exhaustive on-device check of the 3-op division by a run constant
// (div_const, sk_common.cuh) against IEEE division, for every fp32 numerator
// in the fast path's range.  2^32 candidates take a few milliseconds on a
// B200, so the engine verifies each new divisor once per process before it
// trusts the fast path (falling back to IEEE division on any mismatch).
#include <map>
#include <mutex>

#include "sk_internal.h"

namespace sk {

__global__ void verify_div_kernel(float b, unsigned long long* bad) {
  const float r = __frcp_rn(b);
  unsigned long long mine = 0;
  const unsigned long long n = 1ull << 32;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const float x = __uint_as_float((unsigned)i);
    if (!div_safe(x)) continue;
    const float q = div_const(x, b, r);
    const float w = __fdiv_rn(x, b);
    mine += (__float_as_uint(q) != __float_as_uint(w));
  }
  if (mine) atomicAdd(bad, mine);
}

long long verify_div_f32(float b, cudaStream_t s) {
  static std::mutex mu;
  static std::map<unsigned, long long> cache;
  unsigned key = 0;
  memcpy(&key, &b, 4);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  unsigned long long* d = nullptr;
  unsigned long long h = 0;
  long long res = -1;
  if (cudaMallocAsync(&d, sizeof(*d), s) == cudaSuccess &&
      cudaMemsetAsync(d, 0, sizeof(*d), s) == cudaSuccess) {
    int dev = 0;
    cudaGetDevice(&dev);
    verify_div_kernel<<<device_sms(dev) * 8, 256, 0, s>>>(b, d);
    if (cudaGetLastError() == cudaSuccess &&
        cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s) == cudaSuccess &&
        cudaStreamSynchronize(s) == cudaSuccess)
      res = (long long)h;
  }
  if (d) cudaFreeAsync(d, s);
  cudaGetLastError();
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = res;
  return res;
}

}  // namespace sk

extern "C" long long sk_verify_div_f32(float b, void* stream) {
  return sk::verify_div_f32(b, static_cast<cudaStream_t>(stream));
}
