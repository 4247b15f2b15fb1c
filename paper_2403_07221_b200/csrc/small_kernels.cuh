// small_kernels.cuh -- K5: the whole forward for small batches (serving:
// BASELINE c5's 1 / 8 / 64 tokens) in one launch, signflip at D = 2048.
//
// With a handful of tokens the two-kernel path is latency-bound: one token's
// hash is a serial chain on one warp (~14 us) and its gather a serial walk of
// 256 tables (~12 us).  Here a CTA (token i, table group g) of 256 threads
// runs token i's three transforms with 8 coordinates per thread (register,
// shuffle and one shared-memory exchange per transform), computes the codes
// and top-1 coefficients of group g's tables, and gathers those tables for
// all columns; the token's G CTAs form a thread-block cluster and its G
// partial rows meet in distributed shared memory, summed in group order --
// deterministic, no atomics, no global round trip.  Every CTA of a token recomputes its hash (the
// hash is not table-separable), which costs nothing at these sizes and
// removes the hash -> gather launch dependency.
//
// Reference path (/root/reference/proj): Projection::forward signflip
// (projection.cpp:200-263, fwht_kernel fwht.hpp:28-41), compute_codes /
// top1_weight (lookup.cpp:74-100, 185-189), the gather of forward_impl
// (lookup.cpp:223-268).  Numerics: float64 transform with the stages in a
// different order than fwht_kernel (they commute; ~1e-16 relative), codes
// bit-exact wherever |z| > 1e-5, the weight in the reference's order over
// the table's coordinates, fp32 gather (tables ascending within a group,
// groups ascending).
#pragma once

#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "checked.cuh"
#include "gather_kernels.cuh"
#include "hash_kernels.cuh"

namespace lffn_gpu {

struct SmallParams {
  const float* x;            // [n x d_in]
  int64_t n;
  int d_in;
  int code_width;            // h * tau
  int tau;
  int kb, ke;                // tables owned: [kb, ke)
  int scaled;
  int groups;                // G: table groups per token (grid.y)
  int tpg;                   // tables per group
  const uint32_t* signmask;  // 3 x (D / 32) words, bit set = -1
  const void* T;             // [hl][2^tau][d_out], f32 or bf16
  int rows;
  int d_out;
  float* y;                  // [n x d_out]
  int accumulate;
  int* flag;
};

constexpr int kSmallThreads = 256;
constexpr int kSmallMaxTpg = 256;
constexpr int kSmallMaxGroups = 16;  // cluster size (16: non-portable, allowed on B200)

// D = 2048 layouts: P -- thread t holds indices 8 t + r (bits 0-2 in
// registers, 3-7 across the lanes, 8-10 across the warps); Q -- thread t
// holds t + 256 r (bits 0-7 across the threads, 8-10 in registers).
__device__ __forceinline__ int small_pos(int i) { return i + 2 * (i >> 4); }
constexpr int kSmallPad = 2048 + 2 * (2048 >> 4);

template <int B0, int B1>
__device__ __forceinline__ void small_reg_stages(double (&v)[8]) {
#pragma unroll
  for (int k = B0; k < B1; ++k)
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r & (1 << k)) continue;
      const double a = v[r], b = v[r | (1 << k)];
      v[r] = __dadd_rn(a, b);
      v[r | (1 << k)] = __dsub_rn(a, b);
    }
}

// index bits 3-7 = lane bits 0-4: butterflies across lanes
__device__ __forceinline__ void small_lane_stages(double (&v)[8], int lane) {
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const bool upper = (lane >> j) & 1;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const double o = __shfl_xor_sync(0xffffffffu, v[r], 1 << j);
      v[r] = upper ? __dsub_rn(o, v[r]) : __dadd_rn(v[r], o);
    }
  }
}

__device__ __forceinline__ void small_flip(double& v, uint32_t bit) {
  v = __hiloint2double(__double2hiint(v) ^ (int)(bit << 31), __double2loint(v));
}

template <typename TT, int MAXCH>
__global__ void __launch_bounds__(kSmallThreads) forward_small_kernel(SmallParams p) {
  __shared__ __align__(16) double buf[2][kSmallPad];
  __shared__ uint32_t s_code[kSmallMaxTpg];
  __shared__ float s_coeff[kSmallMaxTpg];
  const int tid = threadIdx.x, lane = tid & 31;
  const int g = blockIdx.x;         // table group = rank in the token's cluster
  const int64_t token = blockIdx.y;
  int bad = 0;
  constexpr int W = 2048 / 32;  // sign words per transform
  // ---- x -> layout P (two float4 loads per thread)
  double v[8];
  {
    const float* xr = p.x + token * (int64_t)p.d_in;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int a = 8 * tid + r;
      const float f = a < p.d_in ? __ldg(xr + a) : 0.f;
      if (!isfinite(f)) bad |= 1;
      v[r] = (double)f;
    }
  }
  // every sign word this thread needs, loaded up front with x (the three
  // transforms would otherwise wait on three dependent L2 round trips)
  const uint32_t m0 = __ldg(p.signmask + 0 * W + (tid >> 2)) >> (8 * (tid & 3));
  const uint32_t m2 = __ldg(p.signmask + 2 * W + (tid >> 2)) >> (8 * (tid & 3));
  uint32_t m1 = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = tid + 256 * r;
    m1 |= ((__ldg(p.signmask + 1 * W + (i >> 5)) >> (i & 31)) & 1u) << r;
  }
  auto flip = [&](uint32_t m) {
#pragma unroll
    for (int r = 0; r < 8; ++r) small_flip(v[r], (m >> r) & 1u);
  };
  auto store_P = [&](double* b) {
#pragma unroll
    for (int r = 0; r < 8; r += 2)
      *reinterpret_cast<double2*>(b + small_pos(8 * tid + r)) = make_double2(v[r], v[r + 1]);
  };
  auto load_P = [&](const double* b) {
#pragma unroll
    for (int r = 0; r < 8; r += 2) {
      const double2 w = *reinterpret_cast<const double2*>(b + small_pos(8 * tid + r));
      v[r] = w.x;
      v[r + 1] = w.y;
    }
  };
  auto store_Q = [&](double* b) {
#pragma unroll
    for (int r = 0; r < 8; ++r) b[small_pos(tid + 256 * r)] = v[r];
  };
  auto load_Q = [&](const double* b) {
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = b[small_pos(tid + 256 * r)];
  };
  // transform 0: P (bits 0-7) -> Q (bits 8-10)
  flip(m0);
  small_reg_stages<0, 3>(v);
  small_lane_stages(v, lane);
  store_P(buf[0]);
  __syncthreads();
  load_Q(buf[0]);
  small_reg_stages<0, 3>(v);
  // transform 1: Q (bits 8-10) -> P (bits 0-7)
  flip(m1);
  small_reg_stages<0, 3>(v);
  store_Q(buf[1]);
  __syncthreads();
  load_P(buf[1]);
  small_reg_stages<0, 3>(v);
  small_lane_stages(v, lane);
  // transform 2: P -> Q
  flip(m2);
  small_reg_stages<0, 3>(v);
  small_lane_stages(v, lane);
  store_P(buf[0]);
  __syncthreads();
  load_Q(buf[0]);
  small_reg_stages<0, 3>(v);
  // z in natural order for the epilogue
  store_Q(buf[1]);
  __syncthreads();
  // ---- codes / coefficients of this group's tables (lookup.cpp:74-100, 185-189)
  const int k0 = p.kb + g * p.tpg;
  const int nk = min(p.tpg, p.ke - k0);
  const double* z = buf[1];
  for (int j = tid; j < nk; j += kSmallThreads) {
    const int base = (k0 + j) * p.tau;
    LFFN_DCHECK(j < kSmallMaxTpg && small_pos(base + p.tau - 1) < kSmallPad);
    uint32_t code = 0;
    double w = 1.0, sum_abs = 0.0;
    for (int q = 0; q < p.tau; ++q) {
      const double zq = z[small_pos(base + q)];
      if (!isfinite(zq)) bad |= 2;
      code |= (zq >= 0.0 ? 1u : 0u) << q;
      const double az = fabs(zq);
      sum_abs = __dadd_rn(sum_abs, az);
      if (az < 18.5) w = __ddiv_rn(w, __dadd_rn(1.0, exp(-2.0 * az)));
    }
    s_code[j] = code;
    s_coeff[j] = (float)(p.scaled ? __dmul_rn(w, sum_abs) : w);
  }
  __syncthreads();
  // ---- gather of the group's tables, all columns (MAXCH 16-byte chunks per thread)
  constexpr int VEC = Raw<TT>::VEC;
  const TT* T = reinterpret_cast<const TT*>(p.T);
  const int64_t tstride = (int64_t)p.rows * p.d_out;
  const int nchunks = p.d_out / VEC;
  float acc[MAXCH][VEC];
#pragma unroll
  for (int c = 0; c < MAXCH; ++c)
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[c][e] = 0.f;
  const int kl0 = k0 - p.kb;  // first local table of the group
  // RB rows in flight per thread: with one group of <= 16 tables (n = 1)
  // every row of the group is requested before the first arrives
  constexpr int RB = 16 / MAXCH;
  int j = 0;
  for (; j + RB <= nk; j += RB) {
    uint4 raw[RB][MAXCH];
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      LFFN_DCHECK(s_code[j + q] < (uint32_t)p.rows);
      const TT* rp = T + (int64_t)(kl0 + j + q) * tstride + (int64_t)s_code[j + q] * p.d_out;
#pragma unroll
      for (int c = 0; c < MAXCH; ++c) {
        const int ch = tid + c * kSmallThreads;
        raw[q][c] = ch < nchunks ? Raw<TT>::load(rp + ch * VEC) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int q = 0; q < RB; ++q)
#pragma unroll
      for (int c = 0; c < MAXCH; ++c) Raw<TT>::fma(acc[c], s_coeff[j + q], raw[q][c]);
  }
  for (; j + 4 <= nk; j += 4) {
    uint4 raw[4][MAXCH];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const TT* rp = T + (int64_t)(kl0 + j + q) * tstride + (int64_t)s_code[j + q] * p.d_out;
#pragma unroll
      for (int c = 0; c < MAXCH; ++c) {
        const int ch = tid + c * kSmallThreads;
        raw[q][c] = ch < nchunks ? Raw<TT>::load(rp + ch * VEC) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < MAXCH; ++c) Raw<TT>::fma(acc[c], s_coeff[j + q], raw[q][c]);
  }
  for (; j < nk; ++j) {
    const TT* rp = T + (int64_t)(kl0 + j) * tstride + (int64_t)s_code[j] * p.d_out;
#pragma unroll
    for (int c = 0; c < MAXCH; ++c) {
      const int ch = tid + c * kSmallThreads;
      if (ch < nchunks) Raw<TT>::fma(acc[c], s_coeff[j], Raw<TT>::load(rp + ch * VEC));
    }
  }
  // ---- the G partial rows of a token meet in distributed shared memory:
  // the token's G CTAs form one thread-block cluster; each parks its partial
  // in its own shared memory, and CTA g sums columns slice g over the
  // cluster's CTAs in group order (deterministic, no atomics, no global
  // round trip)
  float* yr = p.y + token * p.d_out;
  auto finish4 = [&](int c4, float4 q) {
    if (p.accumulate) {
      const float4 a = *reinterpret_cast<const float4*>(yr + 4 * c4);
      q.x += a.x; q.y += a.y; q.z += a.z; q.w += a.w;
    }
    if (!isfinite(q.x) || !isfinite(q.y) || !isfinite(q.z) || !isfinite(q.w)) bad |= 4;
    *reinterpret_cast<float4*>(yr + 4 * c4) = q;
  };
  if (p.groups == 1) {
#pragma unroll
    for (int c = 0; c < MAXCH; ++c) {
      const int ch = tid + c * kSmallThreads;
      if (ch < nchunks)
#pragma unroll
        for (int e = 0; e < VEC; e += 4)
          finish4(ch * (VEC / 4) + e / 4, make_float4(acc[c][e], acc[c][e + 1], acc[c][e + 2], acc[c][e + 3]));
    }
  } else {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    float* part = reinterpret_cast<float*>(buf[0]);  // free since transform 2
#pragma unroll
    for (int c = 0; c < MAXCH; ++c) {
      const int ch = tid + c * kSmallThreads;
      if (ch < nchunks)
#pragma unroll
        for (int e = 0; e < VEC; e += 4)
          *reinterpret_cast<float4*>(part + ch * VEC + e) =
              make_float4(acc[c][e], acc[c][e + 1], acc[c][e + 2], acc[c][e + 3]);
    }
    cluster.sync();
    const int n4 = p.d_out / 4;
    const int per = (n4 + p.groups - 1) / p.groups;
    const int c_end = min(n4, (g + 1) * per);
    for (int c4 = g * per + tid; c4 < c_end; c4 += kSmallThreads) {
      float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int rk = 0; rk < p.groups; ++rk) {
        const float4 a = *reinterpret_cast<const float4*>(cluster.map_shared_rank(part, rk) + 4 * c4);
        sum.x += a.x; sum.y += a.y; sum.z += a.z; sum.w += a.w;
      }
      finish4(c4, sum);
    }
    cluster.sync();  // the partials stay readable until every CTA is done
  }
  if (bad) atomicOr(p.flag, bad);
}

// The non-finite flag to mapped host memory, and its reset, in stream order
// (the host path of small batches polls it: lffn_gpu.cu forward_host_direct).
__global__ void flag_to_host_kernel(int* d_flag, volatile int* h_flag) {
  const int f = *d_flag;
  *d_flag = 0;
  *h_flag = f;
  __threadfence_system();
}

}  // namespace lffn_gpu
