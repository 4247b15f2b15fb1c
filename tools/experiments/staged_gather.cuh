// staged_gather.cuh -- EXPERIMENT (not built into liblffn_gpu.so): K3s, the
// gather-accumulate with table tiles staged in shared memory (fp32 tables,
// up to 256 rows per table).  Measured at c2 (16384 tokens): 1.06-1.18 ms
// with cp.async + a CTA barrier per table, 0.759 ms with TMA tiles and
// producer / consumer mbarriers (bit-identical y), against 0.641 ms for the
// row-per-warp kernel; ncu (TMA version): shared-memory load wavefronts at
// 49 % of peak with the LSU data pipe at 85 % (record loads, spills), stalls
// short / long scoreboard.  Its ceiling -- every gathered byte read once
// from shared memory plus the tile writes -- is ~0.43-0.5 ms at c2.  (A
// `#pragma unroll 1` over the four tables of a record group raced: the
// eight LDS of a table moved past the stage release; keep it unrolled.)
//
// Why: the row-per-warp gather (K3, gather_kernels.cuh) reads every gathered
// byte from L2 and runs at the L2 tag-rate ceiling (~20 TB/s of distinct
// sectors, profiles/r2_l2_probe.md).  Here a CTA owns a block of TB = 1024
// tokens and a 32-column slice of the output: per table it copies the
// table's (rows x 32-column) tile once into shared memory (cp.async, a
// three-stage ring) and every token of the block reads its row segment from
// there -- L2 lookups per gathered byte drop by TB / rows (4x at c2), and
// the bound becomes the shared-memory data path (each gathered byte read
// once from shared memory, each tile byte written once).
//
// Layout: one thread per token; its 32 fp32 accumulators are the token's
// column slice.  Tile rows are stored unswizzled (128 B = all 32 banks), and
// at step j lane l reads 16-byte chunk (j + l) mod 8 of its row into
// accumulator slot j, so the eight lanes of a quarter-warp always hit eight
// different bank groups whatever their rows (conflict-free LDS.128); the
// slot -> column rotation is undone at the store.
//
// Reference: lookup_gather_f32 (bench.cpp:182-194), the gather loop of
// forward_impl (lookup.cpp:223-268): y_i = sum_k coeff[i,k] T_k[code[i,k]],
// tables ascending, fp32 accumulation per column -- the same order and
// rounding as the row-per-warp kernel, so y is bit-identical to it.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "dense_tcgen05.cuh"
#include "gather_kernels.cuh"

namespace lffn_gpu {

constexpr int kStagedTB = 1024;      // tokens per block (= threads per CTA)
constexpr int kStagedCW = 32;        // columns per slice (fp32: one 128-byte row segment)
constexpr int kStagedStages = 6;     // tile ring depth (5 tables of lookahead: ~2.5 us)
constexpr int kStagedMaxRows = 256;  // rows per table (tile <= 32 KB)

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
               "l"(gmem_src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// items = (token block, column slice), slice-fastest so the CTAs running at
// the same time walk the same tables (they stay L2-resident between them)
__global__ void __launch_bounds__(kStagedTB, 1) gather_staged_kernel(GatherParams p, int nitems) {
  extern __shared__ __align__(16) float tiles[];  // [stages][rows][32]
  const int tid = threadIdx.x, lane = tid & 31;
  const int rows = p.rows;
  const int tile_floats = rows * kStagedCW;
  const int nslices = p.d_out / kStagedCW;
  const float* T = static_cast<const float*>(p.T);
  const int64_t tstride = (int64_t)rows * p.d_out;
  int bad = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int slice = item % nslices;
    const int64_t token = (int64_t)(item / nslices) * kStagedTB + tid;
    const bool live = token < p.n;
    const int c0 = slice * kStagedCW;
    // the tile of table k: rows x 128 B at column c0, 16-byte chunks
    auto issue = [&](int k) {
      if (k < p.nk) {
        float* dst = tiles + (k % kStagedStages) * tile_floats;
        const float* src = T + (int64_t)k * tstride + c0;
        for (int q = tid; q < rows * 8; q += kStagedTB) {
          const int r = q >> 3, ch = q & 7;
          cp_async16(dst + r * kStagedCW + ch * 4, src + (int64_t)r * p.d_out + ch * 4);
        }
      }
      cp_async_commit();
    };
    float acc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    const uint32_t* cr = p.codes + (live ? token : 0) * p.ld;
    const float* wr = p.coeff + (live ? token : 0) * p.ld;
    __syncthreads();  // the previous item's last tiles are consumed
#pragma unroll
    for (int s = 0; s < kStagedStages - 1; ++s) issue(s);
    for (int kg = 0; kg < p.nk; kg += 4) {
      // this token's records of the next four tables (32 warps per SM hide
      // the load; no prefetch registers at the 64-register budget)
      const uint4 cc = live ? __ldg(reinterpret_cast<const uint4*>(cr + kg)) : make_uint4(0u, 0u, 0u, 0u);
      const float4 ww = live ? __ldg(reinterpret_cast<const float4*>(wr + kg)) : make_float4(0.f, 0.f, 0.f, 0.f);
      const uint32_t code4[4] = {cc.x, cc.y, cc.z, cc.w};
      const float w4[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = kg + q;
        cp_async_wait<kStagedStages - 2>();
        __syncthreads();                       // tile k landed; tile k-1 consumed by all
        issue(k + kStagedStages - 1);          // into the stage tile k-1 used
        const float* row = tiles + (k % kStagedStages) * tile_floats + (int)code4[q] * kStagedCW;
        const float w = w4[q];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v = *reinterpret_cast<const float4*>(row + 4 * ((j + lane) & 7));
          acc[j][0] = fmaf(w, v.x, acc[j][0]);
          acc[j][1] = fmaf(w, v.y, acc[j][1]);
          acc[j][2] = fmaf(w, v.z, acc[j][2]);
          acc[j][3] = fmaf(w, v.w, acc[j][3]);
        }
      }
    }
    cp_async_wait<0>();
    if (live) {
      float* yr = p.y + token * p.d_out + c0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float* dst = yr + 4 * ((j + lane) & 7);
        float4 o = make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]);
        if (p.accumulate) {
          const float4 a = *reinterpret_cast<const float4*>(dst);
          o.x += a.x; o.y += a.y; o.z += a.z; o.w += a.w;
        }
        if (!isfinite(o.x) || !isfinite(o.y) || !isfinite(o.z) || !isfinite(o.w)) bad = 4;
        *reinterpret_cast<float4*>(dst) = o;
      }
    }
  }
  if (bad) atomicOr(p.flag, bad);
}

// K3s with TMA: the tile of table k arrives by one 2-D bulk tensor copy
// (rows x 32 floats, no swizzle) issued by a producer warp into a ring of
// kStagedTmaStages stages; 31 consumer warps (992 tokens) wait on the stage's
// "full" mbarrier, accumulate, and release it through its "empty" mbarrier --
// no CTA-wide barrier per table, so warps drift freely within the ring.
constexpr int kStagedTmaStages = 6;
constexpr int kStagedTmaTB = 992;  // 31 consumer warps, one token per thread

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(1024, 1)
    gather_staged_tma_kernel(const __grid_constant__ CUtensorMap map, GatherParams p, int nitems) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  const int rows = p.rows;
  const int tile_floats = rows * kStagedCW;
  const uint32_t tile_bytes = uint32_t(tile_floats) * 4u;
  float* tiles = reinterpret_cast<float*>(sm_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm_raw + size_t(kStagedTmaStages) * tile_bytes);
  uint64_t* empty = full + kStagedTmaStages;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nslices = p.d_out / kStagedCW;
  if (tid == 0) {
    for (int s = 0; s < kStagedTmaStages; ++s) {
      umma::mbar_init(&full[s], 1);
      umma::mbar_init(&empty[s], 31);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  int bad = 0;
  if (warp == 31) {
    // producer: one elected lane walks every (item, table) in consumption order
    if (lane == 0) {
      int64_t idx = 0;
      for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
        const int c0 = (item % nslices) * kStagedCW;
        for (int k = 0; k < p.nk; ++k, ++idx) {
          const int s = int(idx % kStagedTmaStages);
          const int64_t u = idx / kStagedTmaStages;
          if (u > 0) umma::mbar_wait(&empty[s], uint32_t((u - 1) & 1));
          mbar_expect_tx(&full[s], tile_bytes);
          tma_load_2d(umma::smem_u32(tiles + s * tile_floats), &map, c0, k * rows, &full[s]);
        }
      }
    }
    return;
  }
  int64_t idx = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int slice = item % nslices;
    const int64_t token = (int64_t)(item / nslices) * kStagedTmaTB + tid;
    const bool live = token < p.n;
    const int c0 = slice * kStagedCW;
    float acc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    const uint32_t* cr = p.codes + (live ? token : 0) * p.ld;
    const float* wr = p.coeff + (live ? token : 0) * p.ld;
    for (int kg = 0; kg < p.nk; kg += 4) {
      const uint4 cc = live ? __ldg(reinterpret_cast<const uint4*>(cr + kg)) : make_uint4(0u, 0u, 0u, 0u);
      const float4 ww = live ? __ldg(reinterpret_cast<const float4*>(wr + kg)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int q = 0; q < 4; ++q, ++idx) {
        // one table's eight loads in flight at a time (64-register budget)
        const uint32_t code = q == 0 ? cc.x : q == 1 ? cc.y : q == 2 ? cc.z : cc.w;
        const float w = q == 0 ? ww.x : q == 1 ? ww.y : q == 2 ? ww.z : ww.w;
        const int s = int(idx % kStagedTmaStages);
        umma::mbar_wait(&full[s], uint32_t((idx / kStagedTmaStages) & 1));
        const float* row = tiles + s * tile_floats + (int)code * kStagedCW;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v = *reinterpret_cast<const float4*>(row + 4 * ((j + lane) & 7));
          acc[j][0] = fmaf(w, v.x, acc[j][0]);
          acc[j][1] = fmaf(w, v.y, acc[j][1]);
          acc[j][2] = fmaf(w, v.z, acc[j][2]);
          acc[j][3] = fmaf(w, v.w, acc[j][3]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
    if (live) {
      float* yr = p.y + token * p.d_out + c0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float* dst = yr + 4 * ((j + lane) & 7);
        float4 o = make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]);
        if (p.accumulate) {
          const float4 a = *reinterpret_cast<const float4*>(dst);
          o.x += a.x; o.y += a.y; o.z += a.z; o.w += a.w;
        }
        if (!isfinite(o.x) || !isfinite(o.y) || !isfinite(o.z) || !isfinite(o.w)) bad = 4;
        *reinterpret_cast<float4*>(dst) = o;
      }
    }
  }
  if (bad) atomicOr(p.flag, bad);
}

}  // namespace lffn_gpu
