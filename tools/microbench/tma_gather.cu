// Random-row gather throughput: TMA bulk copies (cp.async.bulk global ->
// shared, mbarrier completion) vs 128-bit register loads, on an L2-resident
// or HBM-sized row table.  Question: can whole-row bulk copies beat the
// ~19-20 TB/s that random 512-byte LDG segments reach?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_gather tma_gather.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
               "@!p bra W_%=;\n\t}\n" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

__device__ __forceinline__ uint32_t rnd(uint32_t& h) { h ^= h << 13; h ^= h >> 17; h ^= h << 5; return h; }

// One producer thread per CTA keeps NS slots of ROW bytes in flight; each
// slot is consumed by consumer warp (slot % CW) which reads it with LDS.128
// and accumulates.  Rows per CTA: iters.
template <int ROW, int NS, int CW, int PL>
__global__ void __launch_bounds__(32 * (CW + 1), 1) tma_gather(const char* __restrict__ T, uint32_t nrows,
                                                                int iters, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + NS;
  unsigned char* ring = sm + 2048;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { bar_init(full + s, 1); bar_init(empty + s, 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == CW) {
    if (lane < PL) {
      uint32_t h = blockIdx.x * 7919u + 13u + lane * 104729u;
      for (int i = lane; i < iters; i += PL) {
        const int s = i % NS;
        const uint32_t use = i / NS;
        if (use > 0) bar_wait(empty + s, (use - 1) & 1);
        const uint32_t r = rnd(h) % nrows;
        bar_expect(full + s, ROW);
        bulk_g2s(ring + (size_t)s * ROW, T + (size_t)r * ROW, ROW, full + s);
      }
    }
  } else {
    float acc = 0.f;
    for (int i = warp; i < iters; i += CW) {
      const int s = i % NS;
      bar_wait(full + s, (i / NS) & 1);
      const float4* q = reinterpret_cast<const float4*>(ring + (size_t)s * ROW);
#pragma unroll
      for (int j = lane; j < ROW / 16; j += 32) { const float4 v = q[j]; acc += v.x + v.y + v.z + v.w; }
      __syncwarp();
      if (lane == 0) bar_arrive(empty + s);
    }
    if (acc == 1234.5f) *out = acc;
  }
}

// LDG baseline: one warp per row, rows in flight per lane = IF.
template <int ROW, int IF>
__global__ void __launch_bounds__(256, 2) ldg_gather(const char* __restrict__ T, uint32_t nrows, int iters, float* out) {
  const int lane = threadIdx.x & 31;
  uint32_t h = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 7919u + 13u;
  float acc = 0.f;
  constexpr int PER = ROW / 512;  // 512 B per warp load
  for (int i = 0; i < iters; i += IF) {
    float4 v[IF][PER];
#pragma unroll
    for (int f = 0; f < IF; ++f) {
      const uint32_t r = rnd(h) % nrows;
      const float4* q = reinterpret_cast<const float4*>(T + (size_t)r * ROW);
#pragma unroll
      for (int c = 0; c < PER; ++c) v[f][c] = __ldg(q + c * 32 + lane);
    }
#pragma unroll
    for (int f = 0; f < IF; ++f)
#pragma unroll
      for (int c = 0; c < PER; ++c) acc += v[f][c].x + v[f][c].y + v[f][c].z + v[f][c].w;
  }
  if (acc == 1234.5f) *out = acc;
}

template <int ROW, int NS, int CW, int PL = 1>
void run_tma(const char* T, uint32_t nrows, int sms, int ctas_per_sm, float* out, const char* tag) {
  const size_t smem = 2048 + size_t(NS) * ROW;
  auto k = tma_gather<ROW, NS, CW, PL>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(a);
    k<<<sms * ctas_per_sm, 32 * (CW + 1), smem>>>(T, nrows, iters, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  const double bytes = double(sms) * ctas_per_sm * iters * ROW;
  printf("tma  %-10s row=%5d slots=%2d cw=%d producers=%2d ctas/sm=%d smem=%6zu: %8.1f GB/s\n", tag, ROW, NS, CW, PL, ctas_per_sm,
         smem, bytes / (best * 1e6));
}

template <int ROW, int IF>
void run_ldg(const char* T, uint32_t nrows, int sms, float* out, const char* tag) {
  const int iters = 512;
  const int grid = sms * 2;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(a);
    ldg_gather<ROW, IF><<<grid, 256>>>(T, nrows, iters, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  const double bytes = double(grid) * 8 * iters * ROW;
  printf("ldg  %-10s row=%5d inflight=%d: %8.1f GB/s\n", tag, ROW, IF, bytes / (best * 1e6));
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* out;
  CK(cudaMalloc(&out, 16));
  for (size_t mb : {32, 201}) {
    char* T;
    const size_t bytes = mb << 20;
    CK(cudaMalloc(&T, bytes));
    CK(cudaMemset(T, 0, bytes));
    char tag[32];
    snprintf(tag, sizeof tag, "%zuMB", mb);
    run_ldg<3072, 4>(T, bytes / 3072, sms, out, tag);
    run_ldg<2048, 4>(T, bytes / 2048, sms, out, tag);
    run_tma<3072, 32, 4, 1>(T, bytes / 3072, sms, 1, out, tag);
    run_tma<3072, 32, 4, 8>(T, bytes / 3072, sms, 1, out, tag);
    run_tma<3072, 32, 4, 32>(T, bytes / 3072, sms, 1, out, tag);
    run_tma<3072, 64, 8, 32>(T, bytes / 3072, sms, 1, out, tag);
    run_tma<3072, 32, 4, 32>(T, bytes / 3072, sms, 2, out, tag);
    run_tma<2048, 96, 8, 32>(T, bytes / 2048, sms, 1, out, tag);
    run_tma<8192, 24, 8, 24>(T, bytes / 8192, sms, 1, out, tag);
    run_tma<512, 128, 8, 32>(T, bytes / 512, sms, 1, out, tag);
    CK(cudaFree(T));
  }
  return 0;
}
