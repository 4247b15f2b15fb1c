// mma_rate.cu -- issue-rate microbenchmark for tcgen05.mma (no loads in the
// loop): one CTA per SM, one thread issues `iters` MMAs from a resident smem
// tile into TMEM, commits, waits; cycles per MMA from clock64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, int sw128) {
  uint64_t d = uint64_t((addr >> 4) & 0x3FFF);
  if (sw128) {
    d |= uint64_t(1) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(2) << 61;
  } else {
    d |= uint64_t(128 >> 4) << 16;
    d |= uint64_t(1024 >> 4) << 32;
  }
  d |= uint64_t(1) << 46;
  return d;
}

template <int KIND>  // 0 tf32, 1 bf16 (kind::f16)
__global__ void __launch_bounds__(128, 1) mma_rate(int m, int n, int iters, int sw, int fill, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* tile = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + 12345u;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    // random values in [-2, 2) (tf32 / bf16 read the high bits)
    const float f = (float)(h & 0xFFFFFF) / 4194304.0f - 2.0f;
    reinterpret_cast<float*>(tile)[i] = fill ? f : 0.f;
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  uint32_t idesc = 1u << 4;
  if (KIND == 0) idesc |= (2u << 7) | (2u << 10);
  else idesc |= (1u << 7) | (1u << 10);
  idesc |= uint32_t(n >> 3) << 17;
  idesc |= uint32_t(m >> 4) << 24;
  if (threadIdx.x == 0) {
    const uint32_t a = su32(tile), b = a + 32768;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t adv = uint32_t(i & 3) * 32;
      const uint64_t da = desc(a + adv, sw), db = desc(b + adv, sw);
      const uint32_t acc = i > 0;
      if (KIND == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred d;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], 0;\n\t@!d bra W;\n\t}\n" ::"r"(su32(&bar)) : "memory");
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  long long h[148];
  const int iters = 4096;
  struct C { int kind, m, n, sw; const char* name; } cs[] = {
      {0, 128, 128, 1, "tf32 128x128x8  sw128"}, {0, 128, 256, 1, "tf32 128x256x8  sw128"},
      {0, 128, 64, 1, "tf32 128x64x8   sw128"},  {0, 128, 128, 0, "tf32 128x128x8  none"},
      {1, 128, 128, 1, "bf16 128x128x16 sw128"}, {1, 128, 256, 1, "bf16 128x256x16 sw128"}};
  for (int fill = 0; fill < 2; ++fill)
  for (auto& c : cs) {
    auto k = c.kind == 0 ? mma_rate<0> : mma_rate<1>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    for (int rep = 0; rep < 2; ++rep) k<<<148, 128, 65536 + 1024>>>(c.m, c.n, iters, c.sw, fill, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148.0;
    const int kk = c.kind == 0 ? 8 : 16;
    const double fma = double(c.m) * c.n * kk;
    printf("fill=%d %s: %s  %.1f cyc/mma  %.0f FMA/cyc/SM\n", fill, c.name, cudaGetErrorString(e), avg / iters,
           fma / (avg / iters));
  }
  return 0;
}
