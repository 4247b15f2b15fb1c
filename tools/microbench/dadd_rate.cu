// fp64 add issue rate per SM as a function of resident warps per scheduler:
// does one warp's stream of independent butterflies (the K1f inner loop: 64
// float64 registers, six in-register stages) saturate the fp64 pipe, or does
// it take several warps?  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o dadd_rate dadd_rate.cu ; run: ./dadd_rate
#include <cstdio>
#include <cuda_runtime.h>

template <int NV>
__global__ void __launch_bounds__(NV == 64 ? 384 : 512, 1) dadd_kernel(double* out, int iters, double seed) {
  double v[NV];
#pragma unroll
  for (int r = 0; r < NV; ++r) v[r] = seed * (r + 1) + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 1; k < NV; k <<= 1) {
#pragma unroll
      for (int r = 0; r < NV; ++r) {
        if (r & k) continue;
        const double a = v[r], b = v[r | k];
        v[r] = __dadd_rn(a, b);
        v[r | k] = __dsub_rn(a, b);
      }
    }
#pragma unroll
    for (int r = 0; r < NV; ++r) v[r] *= 1e-2;  // keep finite (counts as fp64 work too)
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < NV; ++r) s += v[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NV>
void run(int threads) {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 512);
  const int iters = 400;
  int logn = 0;
  while ((1 << logn) < NV) ++logn;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dadd_kernel<NV><<<sms, threads>>>(out, 10, 1.0);
  cudaDeviceSynchronize();
  float best = 1e9f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dadd_kernel<NV><<<sms, threads>>>(out, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double ops = double(iters) * (NV * logn + NV) * threads * sms;  // lane ops
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("NV=%2d threads/SM=%4d (warps/scheduler %.2f): %.3f ms  %.1f fp64 lane-ops/clk/SM at %d MHz nominal\n", NV,
         threads, threads / 128.0, best, ops / (best * 1e-3) / (double(clk) * 1e3) / sms, clk / 1000);
  cudaFree(out);
}

int main() {
  for (int t : {128, 256, 384}) run<64>(t);
  for (int t : {128, 256, 384, 512}) run<32>(t);
  for (int t : {128, 256, 512}) run<16>(t);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("CUDA error: %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
