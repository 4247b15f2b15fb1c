// probe.cu -- live bandwidth probes for the roofline denominators.
//
// BASELINE.json defines the gather roofline as  t_roof = U / BW_HBM + G / BW_L2.
// MEASURED_PEAKS.json carries BW_HBM (a driver-measured copy); BW_L2 is not
// in it, so bench.py measures it here on the same GPU in the same run:
// 128-bit read-only loads that re-read an L2-resident buffer from every SM.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "lffn_gpu.h"
#include "lffn_internal.h"

namespace {

__global__ void l2_read_kernel(const float4* __restrict__ p, size_t n4_mask, int passes,
                               float* out) {
  float acc = 0.f;
  const size_t start = (size_t)blockIdx.x * 4096u;
  for (int ps = 0; ps < passes; ++ps) {
    for (size_t i = threadIdx.x; i <= n4_mask; i += (size_t)blockDim.x * 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcg(p + ((i + u * blockDim.x + start) & n4_mask));
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  }
  if (acc == 1234.5f) *out = acc;
}

__global__ void hbm_read_kernel(const float4* __restrict__ p, size_t n4, float* out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride * 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t j = i + u * stride;
      v[u] = j < n4 ? __ldcs(p + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) *out = acc;
}

// Random 512-byte segments (one per warp load, 32 x 16 B) of an L2-resident
// buffer: the gather's access granularity without its arithmetic.  Every
// lane keeps 8 independent segments in flight.
__global__ void l2_random_kernel(const float4* __restrict__ p, uint32_t nseg_mask, int iters,
                                 float* out) {
  const int lane = threadIdx.x & 31;
  uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  h = h * 2654435761u + 12345u;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h ^= h << 13; h ^= h >> 17; h ^= h << 5;  // xorshift, warp-uniform
      v[u] = __ldg(p + (size_t)(h & nseg_mask) * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) *out = acc;
}

}  // namespace

extern "C" {

// which = 0: L2 read bandwidth (32 MiB working set, sequential 128-bit
// re-reads), 1: HBM read bandwidth (4 GiB stream), 2: L2 read bandwidth
// for random 512-byte segments of a 32 MiB buffer (the gather's pattern).  Best of `reps` timed launches, GB/s of bytes loaded.
int lffn_probe_bandwidth(int device, int which, int reps, double* gbs) {
  using lffn_gpu::fail;
  if (!gbs) return fail(LFFN_ERR_USAGE, "probe: null output");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess)
    return fail(LFFN_ERR_RUNTIME, "probe: no device");
  const int sms = prop.multiProcessorCount;
  const size_t bytes = which == 1 ? (size_t(4) << 30) : (size_t(32) << 20);
  void* buf = nullptr;
  float* out = nullptr;
  cudaEvent_t a, b;
  if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&out, 16) != cudaSuccess)
    return fail(LFFN_ERR_RUNTIME, "probe: allocation failed");
  cudaMemset(buf, 0, bytes);
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 0.0;
  const int passes = 16;
  for (int r = 0; r < reps + 1; ++r) {
    cudaEventRecord(a);
    const int rit = 64;
    if (which == 2)
      l2_random_kernel<<<sms * 2, 1024>>>(static_cast<const float4*>(buf), uint32_t(bytes / 512 - 1),
                                          rit, out);
    else if (which == 0)
      l2_read_kernel<<<sms * 2, 1024>>>(static_cast<const float4*>(buf), bytes / 16 - 1, passes,
                                        out);
    else
      hbm_read_kernel<<<sms * 8, 512>>>(static_cast<const float4*>(buf), bytes / 16, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double moved = which == 0 ? double(bytes) * passes * sms * 2
                         : which == 2 ? double(sms) * 2 * 32 * rit * 8 * 512.0
                                      : double(bytes);
    if (r > 0 && ms > 0.f) best = std::max(best, moved / (ms * 1e6));
  }
  const cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  cudaFree(out);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(LFFN_ERR_RUNTIME, std::string("probe: ") + cudaGetErrorString(e));
  *gbs = best;
  return LFFN_OK;
}

}  // extern "C"
