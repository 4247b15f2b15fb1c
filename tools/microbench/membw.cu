// Memory-hierarchy probes for the LookupFFN gather roofline on B200 (sm_100a).
//
// The gather roofline in BASELINE.json is  t_roof = U / BW_HBM + G / BW_L2,
// and MEASURED_PEAKS.json only carries BW_HBM.  This probe measures, with
// CUDA events after warm-up:
//   hbm   : streaming 128-bit reads over a 4 GiB buffer (read-only bytes)
//   l2    : 128-bit re-reads of an L2-resident buffer (16..96 MiB)
//   smem  : LDS.128 throughput per SM x 148
//   gather: random 3 KiB row gathers out of a 201 MB table (the c2 access
//           pattern without the arithmetic)
//   fp64  : dependent-free DADD throughput
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membw membw.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void read_stream(const float4* __restrict__ p, size_t n4, float* out) {
  float acc = 0.f;
  size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += stride * 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      size_t j = i + u * stride;
      v[u] = j < n4 ? __ldcs(p + j) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) *out = acc;
}

// Each CTA walks the whole (L2-resident) buffer `passes` times from a
// CTA-dependent start so the chip keeps reading distinct lines.
__global__ void read_l2(const float4* __restrict__ p, size_t n4, int passes, float* out) {
  float acc = 0.f;
  size_t chunk = n4 / gridDim.x;
  size_t start = chunk * blockIdx.x;
  for (int ps = 0; ps < passes; ++ps) {
    for (size_t i = threadIdx.x; i < n4; i += blockDim.x * 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        size_t j = (i + u * blockDim.x + start) & (n4 - 1);
        v[u] = __ldcg(p + j);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  }
  if (acc == 1234.5f) *out = acc;
}

__global__ void smem_bw(int iters, float* out) {
  extern __shared__ float4 sm[];
  const int n = 2048;  // 32 KiB of float4
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_float4(i, 1, 2, 3);
  __syncthreads();
  float acc = 0.f;
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float4 v = sm[(idx + u * 256) & (n - 1)];
      acc += v.x;
    }
    idx = (idx + 32) & (n - 1);
  }
  if (acc == 1234.5f) *out = acc;
}

// Random row gathers: warp w handles tokens; per token, per table, one
// 3 KiB row (768 floats) chosen by a hash of (token, table).
template <bool kCG>
__global__ void gather_rows(const float4* __restrict__ tab, int rows_per_table, int tables,
                            int row4, int tokens, float* out) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < tokens; t += nwarps) {
    float4 acc[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) acc[c] = make_float4(0, 0, 0, 0);
    for (int k = 0; k < tables; ++k) {
      uint32_t hsh = (uint32_t)t * 2654435761u ^ (uint32_t)k * 40503u;
      hsh ^= hsh >> 13; hsh *= 0x5bd1e995u; hsh ^= hsh >> 15;
      int code = hsh % rows_per_table;
      const float4* r = tab + ((size_t)k * rows_per_table + code) * row4;
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        float4 v = kCG ? __ldcg(r + lane + 32 * c) : __ldg(r + lane + 32 * c);
        acc[c].x += v.x; acc[c].y += v.y; acc[c].z += v.z; acc[c].w += v.w;
      }
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < 6; ++c) s += acc[c].x + acc[c].y + acc[c].z + acc[c].w;
    if (s == 1234.5f) *out = s;
  }
}

__global__ void dadd_rate(int iters, double* out) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  double b = 1e-9;
  for (int i = 0; i < iters; ++i) {
    a0 += b; a1 -= b; a2 += b; a3 -= b; a4 += b; a5 -= b; a6 += b; a7 -= b;
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 1234.5) *out = s;
}

template <typename F>
float time_ms(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) f();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs %d L2 %d MB smem/SM %zu\n", prop.name, prop.multiProcessorCount,
         prop.l2CacheSize >> 20, prop.sharedMemPerMultiprocessor);
  int sms = prop.multiProcessorCount;
  float* out; CK(cudaMalloc(&out, 64));
  size_t big = size_t(4) << 30;
  float4* buf; CK(cudaMalloc(&buf, big));
  CK(cudaMemset(buf, 0, big));
  {
    size_t n4 = big / 16;
    float ms = time_ms([&] { read_stream<<<sms * 8, 512>>>(buf, n4, out); }, 10);
    printf("hbm_read_gbs %.1f\n", big / ms / 1e6);
  }
  for (size_t mb : {16, 32, 48, 64, 96}) {
    size_t bytes = mb << 20, n4 = bytes / 16;
    int passes = 16;
    for (int tpb : {512, 1024}) {
      float ms = time_ms([&] { read_l2<<<sms * (tpb == 512 ? 4 : 2), tpb>>>(buf, n4, passes, out); }, 5);
      double tot = double(bytes) * passes * sms * (tpb == 512 ? 4 : 2);
      printf("l2_read_gbs buf=%zuMB tpb=%d %.1f\n", mb, tpb, tot / ms / 1e6);
    }
  }
  {
    CK(cudaFuncSetAttribute(smem_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024));
    int iters = 20000;
    float ms = time_ms([&] { smem_bw<<<sms * 4, 256, 48 * 1024>>>(iters, out); }, 5);
    double bytes = double(sms) * 4 * 256 * iters * 8 * 16;
    printf("smem_lds128_gbs %.1f\n", bytes / ms / 1e6);
  }
  {
    int tables = 256, rows = 256, row4 = 192, tokens = 16384;
    float ms = time_ms([&] { gather_rows<false><<<sms * 8, 256>>>(buf, rows, tables, row4, tokens, out); }, 5);
    double g = double(tokens) * tables * row4 * 16;
    printf("gather_c2_fp32_gbs %.1f ms %.3f\n", g / ms / 1e6, ms);
    for (int bpm : {4, 16}) {
      float ms2 = time_ms([&] { gather_rows<true><<<sms * bpm, 256>>>(buf, rows, tables, row4, tokens, out); }, 5);
      printf("gather_c2_fp32_cg_gbs(bps=%d) %.1f ms %.3f\n", bpm, g / ms2 / 1e6, ms2);
    }
  }
  {
    int iters = 100000;
    double* o; CK(cudaMalloc(&o, 64));
    float ms = time_ms([&] { dadd_rate<<<sms * 8, 256>>>(iters, o); }, 3);
    double flops = double(sms) * 8 * 256 * iters * 8;
    printf("dadd_gflops %.1f\n", flops / ms / 1e6);
  }
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("clock_khz %d\n", clk);
  return 0;
}
