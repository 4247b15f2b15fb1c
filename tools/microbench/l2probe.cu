// l2probe.cu -- which L2 read rate is the gather's ceiling on B200?
//
// The gather roofline needs one L2 bandwidth figure (BW_L2).  Round 1 had two
// probes that disagreed (28.2 TB/s for the sliding sequential re-read in
// csrc/probe.cu, ~20 TB/s for membw.cu's per-CTA chunks).  This tool runs the
// access patterns side by side, all L2-resident, 128-bit loads, CUDA events,
// best of 5 after a warm-up:
//   seq_slide   csrc/probe.cu which=0 (CTA b starts 64 KiB * b into the buffer)
//   seq_chunk   membw.cu read_l2 (CTA b starts at b * size / grid)
//   rand_S      one warp reads a random S-byte segment (S = 512 .. 4096) per
//               load group, 8 groups in flight per lane, warp-uniform hash
//   rows_c2     random 3 KiB rows of a [256 x 256 x 768] fp32 table stack
//               (the c2 gather without arithmetic), buffer size varied
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o l2probe l2probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e = (x);                                                                 \
    if (e != cudaSuccess) {                                                              \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
      exit(1);                                                                           \
    }                                                                                    \
  } while (0)

__global__ void seq_slide(const float4* __restrict__ p, size_t mask, int passes, float* out) {
  float acc = 0.f;
  const size_t start = (size_t)blockIdx.x * 4096u;
  for (int ps = 0; ps < passes; ++ps)
    for (size_t i = threadIdx.x; i <= mask; i += (size_t)blockDim.x * 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcg(p + ((i + u * blockDim.x + start) & mask));
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  if (acc == 1234.5f) *out = acc;
}

__global__ void seq_chunk(const float4* __restrict__ p, size_t n4, int passes, float* out) {
  float acc = 0.f;
  const size_t start = (n4 / gridDim.x) * blockIdx.x & ~size_t(31);
  for (int ps = 0; ps < passes; ++ps)
    for (size_t i = threadIdx.x; i < n4; i += blockDim.x * 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcg(p + ((i + u * blockDim.x + start) & (n4 - 1)));
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  if (acc == 1234.5f) *out = acc;
}

// SEG16 = segment length in 16-byte units (multiple of 32: whole warp loads)
template <int SEG16, bool CG>
__global__ void rand_seg(const float4* __restrict__ p, uint32_t nseg_mask, int iters, float* out) {
  constexpr int L = SEG16 / 32;  // loads per lane per segment
  constexpr int INFL = L >= 8 ? 1 : 8 / L;
  const int lane = threadIdx.x & 31;
  uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  h = h * 2654435761u + 12345u;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float4 v[INFL][L];
#pragma unroll
    for (int u = 0; u < INFL; ++u) {
      h ^= h << 13; h ^= h >> 17; h ^= h << 5;
      const float4* s = p + (size_t)(h & nseg_mask) * SEG16 + lane;
#pragma unroll
      for (int l = 0; l < L; ++l) v[u][l] = CG ? __ldcg(s + 32 * l) : __ldg(s + 32 * l);
    }
#pragma unroll
    for (int u = 0; u < INFL; ++u)
#pragma unroll
      for (int l = 0; l < L; ++l) acc += v[u][l].x + v[u][l].y + v[u][l].z + v[u][l].w;
  }
  if (acc == 1234.5f) *out = acc;
}

template <typename F>
float best_ms(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

template <int SEG16>
void run_rand(const float4* buf, size_t bytes, int sms, float* out, int tpb, int ctas_per_sm) {
  const uint32_t nseg = uint32_t(bytes / (SEG16 * 16));
  uint32_t m = 1;
  while (m * 2 <= nseg) m *= 2;
  const int iters = 64 * 512 / (SEG16 * 16 / 64);  // ~constant bytes per launch
  constexpr int L = SEG16 / 32;
  constexpr int INFL = L >= 8 ? 1 : 8 / L;
  const double moved = double(sms) * ctas_per_sm * (tpb / 32) * double(iters) * INFL * SEG16 * 16;
  const float ms = best_ms([&] { rand_seg<SEG16, false><<<sms * ctas_per_sm, tpb>>>(buf, m - 1, iters, out); }, 5);
  const float ms2 = best_ms([&] { rand_seg<SEG16, true><<<sms * ctas_per_sm, tpb>>>(buf, m - 1, iters, out); }, 5);
  printf("rand_seg bytes=%d buf=%zuMB tpb=%d ctas/sm=%d  ldg %.1f GB/s  ldcg %.1f GB/s\n", SEG16 * 16,
         bytes >> 20, tpb, ctas_per_sm, moved / ms / 1e6, moved / ms2 / 1e6);
}

int main(int argc, char** argv) {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  printf("device %s SMs %d L2 %d MB\n", prop.name, sms, prop.l2CacheSize >> 20);
  float* out;
  CK(cudaMalloc(&out, 64));
  const size_t big = size_t(256) << 20;
  float4* buf;
  CK(cudaMalloc(&buf, big));
  CK(cudaMemset(buf, 0, big));
  const bool quick = argc > 1;  // ncu mode: one launch of each main pattern
  for (size_t mb : {size_t(32)}) {
    const size_t bytes = mb << 20;
    const int passes = 16;
    float ms = best_ms([&] { seq_slide<<<sms * 2, 1024>>>(buf, bytes / 16 - 1, passes, out); }, quick ? 1 : 5);
    printf("seq_slide buf=%zuMB %.1f GB/s\n", mb, double(bytes) * passes * sms * 2 / ms / 1e6);
    ms = best_ms([&] { seq_chunk<<<sms * 2, 1024>>>(buf, bytes / 16, passes, out); }, quick ? 1 : 5);
    printf("seq_chunk buf=%zuMB %.1f GB/s\n", mb, double(bytes) * passes * sms * 2 / ms / 1e6);
  }
  if (quick) {
    run_rand<32>(buf, size_t(32) << 20, sms, out, 1024, 2);
    run_rand<192>(buf, size_t(32) << 20, sms, out, 1024, 2);
    return 0;
  }
  for (size_t mb : {size_t(8), size_t(32), size_t(96)}) {
    run_rand<32>(buf, mb << 20, sms, out, 1024, 2);
    run_rand<64>(buf, mb << 20, sms, out, 1024, 2);
    run_rand<128>(buf, mb << 20, sms, out, 1024, 2);
    run_rand<192>(buf, mb << 20, sms, out, 1024, 2);
    run_rand<256>(buf, mb << 20, sms, out, 1024, 2);
  }
  run_rand<32>(buf, size_t(32) << 20, sms, out, 256, 8);
  run_rand<192>(buf, size_t(32) << 20, sms, out, 256, 8);
  run_rand<192>(buf, size_t(32) << 20, sms, out, 512, 2);
  run_rand<192>(buf, size_t(32) << 20, sms, out, 1024, 1);
  return 0;
}
