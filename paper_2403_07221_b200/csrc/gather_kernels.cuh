// gather_kernels.cuh -- K3: the gather-accumulate stage
//   y_i (+)= sum_{k=kb}^{ke-1} coeff[i,k] * T[k][code[i,k]][:]
// replacing lookup_gather_f32 (bench.cpp:182-194) and the gather loop of
// forward_impl (lookup.cpp:223-268).  Tables are walked in ascending order
// with fp32 accumulators in registers, as the reference's f32 path does.
//
// Kernels: gather_row_persistent_kernel (the default: one warp per token or
// part of its row, persistent grid, several tables' 128-bit row segments in
// flight per lane), gather_row_kernel (same without the 4-record layout) and
// gather_direct_kernel (any width; NTOK tokens x one column chunk per warp).
// Records are (table, neighbour) pairs, table-major: with neighbor_count nc
// record r reads table r / nc.  The row kernels serve nc = 1 (the top-1
// default); nc > 1 takes gather_direct_kernel.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "checked.cuh"

namespace lffn_gpu {

struct GatherParams {
  const void* T;            // first table of this launch: [nk][R][d_out], f32 or bf16
  const uint32_t* codes;    // [n x ld], column 0 = first table of this launch
  const float* coeff;       // [n x ld]
  float* y;                 // [n x d_out]
  int64_t n;
  int ld;                   // row stride of codes / coeff (tables owned by the ctx)
  int nk;                   // tables accumulated by this launch
  int rows;                 // R = 2^tau
  int d_out;
  int accumulate;
  int* flag;
  int reverse_odd_rounds;   // persistent kernel: odd rounds walk the tables backwards
  int nc;                   // records per table (neighbor_count): record r reads table r / nc
  int bf16w;                // bf16 tables: FHFMA path for groups of bf16-exact coefficients
};

// table of record r (records are (table, neighbour) pairs, table-major)
__device__ __forceinline__ int64_t rec_table(const GatherParams& p, int r) {
  return p.nc == 1 ? r : r / p.nc;
}

template <typename TT, int VEC>
struct RowLoad;

template <>
struct RowLoad<float, 4> {
  static __device__ __forceinline__ void load(const float* p, float (&v)[4]) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
};

template <>
struct RowLoad<float, 1> {
  static __device__ __forceinline__ void load(const float* p, float (&v)[1]) { v[0] = __ldg(p); }
};

__device__ __forceinline__ float bf16lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

template <>
struct RowLoad<__nv_bfloat16, 8> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float (&v)[8]) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(p));
    v[0] = bf16lo(q.x); v[1] = bf16hi(q.x); v[2] = bf16lo(q.y); v[3] = bf16hi(q.y);
    v[4] = bf16lo(q.z); v[5] = bf16hi(q.z); v[6] = bf16lo(q.w); v[7] = bf16hi(q.w);
  }
};

template <>
struct RowLoad<__nv_bfloat16, 1> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float (&v)[1]) {
    const unsigned short s = __ldg(reinterpret_cast<const unsigned short*>(p));
    v[0] = __uint_as_float(uint32_t(s) << 16);
  }
};

template <typename TT, int VEC, int NTOK>
__global__ void __launch_bounds__(256) gather_direct_kernel(GatherParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int chunk_cols = 32 * VEC;
  const int nchunks = (p.d_out + chunk_cols - 1) / chunk_cols;
  const int64_t tgroup = gwarp / nchunks;
  const int chunk = (int)(gwarp - tgroup * nchunks);
  const int64_t i0 = tgroup * NTOK;
  if (i0 >= p.n) return;
  const int col = chunk * chunk_cols + lane * VEC;
  const bool colok = col < p.d_out;
  const TT* T = reinterpret_cast<const TT*>(p.T);
  const int64_t table_stride = (int64_t)p.rows * p.d_out;

  float acc[NTOK][VEC];
#pragma unroll
  for (int t = 0; t < NTOK; ++t)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[t][v] = 0.f;

  const uint32_t* cbase = p.codes + i0 * p.ld;
  const float* wbase = p.coeff + i0 * p.ld;
  const int ntok = (p.n - i0) < NTOK ? (int)(p.n - i0) : NTOK;

  for (int k = 0; k < p.nk; ++k) {
    float vals[NTOK][VEC];
    float w[NTOK];
#pragma unroll
    for (int t = 0; t < NTOK; ++t) {
      w[t] = 0.f;
#pragma unroll
      for (int v = 0; v < VEC; ++v) vals[t][v] = 0.f;
      if (t < ntok) {
        const uint32_t code = __ldg(cbase + (int64_t)t * p.ld + k);
        LFFN_DCHECK(code < (uint32_t)p.rows);
        w[t] = __ldg(wbase + (int64_t)t * p.ld + k);
        if (colok) RowLoad<TT, VEC>::load(T + rec_table(p, k) * table_stride + (int64_t)code * p.d_out + col, vals[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < NTOK; ++t)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[t][v] = fmaf(w[t], vals[t][v], acc[t][v]);
  }

  if (!colok) return;
  int bad = 0;
#pragma unroll
  for (int t = 0; t < NTOK; ++t) {
    if (t >= ntok) break;
    float* yr = p.y + (i0 + t) * p.d_out + col;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      float o = acc[t][v];
      if (p.accumulate) o += yr[v];
      if (!isfinite(o)) bad = 4;
      yr[v] = o;
    }
  }
  if (bad) atomicOr(p.flag, bad);
}

// Row-per-warp gather: one warp owns one token and up to MAXC chunks of
// 32*VEC columns of its output row (several warps per token for wide rows).
// Per table every lane issues its MAXC 128-bit row loads back to back; two
// tables are in flight at once, and the (code, coeff) records of the next
// four tables are prefetched while the current four are consumed, so no
// row load waits on a dependent record load.  Small per-warp register
// footprint -> high occupancy -> many L2 requests in flight per SM.
template <typename TT, int VEC, int MAXC, bool REC4>
__global__ void __launch_bounds__(256) gather_row_kernel(GatherParams p, int warps_per_token) {
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t token = gwarp / warps_per_token;
  if (token >= p.n) return;
  const int part = (int)(gwarp - token * warps_per_token);
  constexpr int CHUNK = 32 * VEC;
  const int nchunks = (p.d_out + CHUNK - 1) / CHUNK;
  const int c0 = part * MAXC;
  const int nck = min(MAXC, nchunks - c0);
  const int colbase = c0 * CHUNK + lane * VEC;
  const TT* T = reinterpret_cast<const TT*>(p.T);
  const int64_t tstride = (int64_t)p.rows * p.d_out;
  const uint32_t* cr = p.codes + token * p.ld;
  const float* wr = p.coeff + token * p.ld;

  float acc[MAXC][VEC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[c][v] = 0.f;

  auto row_loads = [&](int k, uint32_t code, float (&vals)[MAXC][VEC]) {
    LFFN_DCHECK(code < (uint32_t)p.rows && k < p.nk);
    const TT* rp = T + k * tstride + (int64_t)code * p.d_out + colbase;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      if (c < nck && colbase + c * CHUNK < p.d_out) RowLoad<TT, VEC>::load(rp + c * CHUNK, vals[c]);
      else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) vals[c][v] = 0.f;
      }
    }
  };
  auto fma_row = [&](float w, const float (&vals)[MAXC][VEC]) {
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[c][v] = fmaf(w, vals[c][v], acc[c][v]);
  };

  if constexpr (REC4) {
    // records of 4 tables per 128-bit broadcast load
    uint4 cc = __ldg(reinterpret_cast<const uint4*>(cr));
    float4 ww = __ldg(reinterpret_cast<const float4*>(wr));
    for (int kg = 0; kg < p.nk; kg += 4) {
      uint4 cn = cc;
      float4 wn = ww;
      if (kg + 4 < p.nk) {
        cn = __ldg(reinterpret_cast<const uint4*>(cr + kg + 4));
        wn = __ldg(reinterpret_cast<const float4*>(wr + kg + 4));
      }
      float va[MAXC][VEC], vb[MAXC][VEC];
      row_loads(kg + 0, cc.x, va);
      row_loads(kg + 1, cc.y, vb);
      fma_row(ww.x, va);
      fma_row(ww.y, vb);
      row_loads(kg + 2, cc.z, va);
      row_loads(kg + 3, cc.w, vb);
      fma_row(ww.z, va);
      fma_row(ww.w, vb);
      cc = cn;
      ww = wn;
    }
  } else {
    uint32_t cc = __ldg(cr);
    float ww = __ldg(wr);
    for (int k = 0; k < p.nk; ++k) {
      uint32_t cn = cc;
      float wn = ww;
      if (k + 1 < p.nk) {
        cn = __ldg(cr + k + 1);
        wn = __ldg(wr + k + 1);
      }
      float va[MAXC][VEC];
      row_loads(k, cc, va);
      fma_row(ww, va);
      cc = cn;
      ww = wn;
    }
  }

  int bad = 0;
  float* yr = p.y + token * p.d_out;
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    const int col = colbase + c * CHUNK;
    if (c < nck && col < p.d_out) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        float o = acc[c][v];
        if (p.accumulate) o += yr[col + v];
        if (!isfinite(o)) bad = 4;
        acc[c][v] = o;
      }
      if constexpr (VEC == 4) {
        *reinterpret_cast<float4*>(yr + col) = make_float4(acc[c][0], acc[c][1], acc[c][2], acc[c][3]);
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) yr[col + v] = acc[c][v];
      }
    }
  }
  if (bad) atomicOr(p.flag, bad);
}

// 128-bit raw row segment: kept packed while in flight (4 registers for 4
// fp32 or 8 bf16 values) and widened to fp32 only at the FMA.
template <typename TT>
struct Raw {
  static constexpr int VEC = sizeof(uint4) / sizeof(TT);
  static __device__ __forceinline__ uint4 load(const TT* p) {
    return __ldg(reinterpret_cast<const uint4*>(p));
  }
  static __device__ __forceinline__ void fma(float (&acc)[VEC], float w, const uint4& r) {
    if constexpr (VEC == 4) {
      acc[0] = fmaf(w, __uint_as_float(r.x), acc[0]);
      acc[1] = fmaf(w, __uint_as_float(r.y), acc[1]);
      acc[2] = fmaf(w, __uint_as_float(r.z), acc[2]);
      acc[3] = fmaf(w, __uint_as_float(r.w), acc[3]);
    } else {
      acc[0] = fmaf(w, bf16lo(r.x), acc[0]);
      acc[1] = fmaf(w, bf16hi(r.x), acc[1]);
      acc[2] = fmaf(w, bf16lo(r.y), acc[2]);
      acc[3] = fmaf(w, bf16hi(r.y), acc[3]);
      acc[4] = fmaf(w, bf16lo(r.z), acc[4]);
      acc[5] = fmaf(w, bf16hi(r.z), acc[5]);
      acc[6] = fmaf(w, bf16lo(r.w), acc[6]);
      acc[7] = fmaf(w, bf16hi(r.w), acc[7]);
    }
  }
  // Exact bf16 coefficient path (bf16 tables only): when w is a bf16 value
  // (low 16 bits zero -- every top-1 weight of 1.0, the common case for the
  // unnormalised signflip transform), w * t is exact in fp32 for bf16 t, so
  // the mixed-precision FHFMA (fma.rn.f32.bf16: bf16 x bf16 + f32, one
  // rounding) equals fmaf(w, float(t), acc) bit for bit while reading the
  // packed halves directly -- 8 instead of 16 instructions per 16 bytes.
  static __device__ __forceinline__ void fma_bf16w(float (&acc)[VEC], uint16_t w16, const uint4& r) {
    if constexpr (VEC == 8) {
      const uint32_t q[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint16_t lo, hi;
        asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(q[i]));
        asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(acc[2 * i]) : "h"(lo), "h"(w16));
        asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(acc[2 * i + 1]) : "h"(hi), "h"(w16));
      }
    }
  }
};

// true when every coefficient of the group is a bf16 value (warp-uniform:
// the records are the same in every lane)
template <int G>
__device__ __forceinline__ bool coeffs_bf16_exact(const float (&w)[G]) {
  uint32_t lowbits = 0;
#pragma unroll
  for (int q = 0; q < G; ++q) lowbits |= __float_as_uint(w[q]);
  return (lowbits & 0xffffu) == 0u;
}

// Persistent row kernel (the default): one warp per (token, part of its
// row), the grid covers the SMs MINB CTAs deep and walks tokens with a grid
// stride, and every lane keeps TIF tables' 128-bit row segments in flight
// (packed) while the (code, coeff) records of the next four tables are
// prefetched.  Requires the 4-table record layout (nk % 4 == 0, ld % 4 == 0,
// 16-byte aligned record pointers); 16-byte aligned rows (d_out % VEC == 0).
template <typename TT, int MAXC, int TIF, int MINB, bool PM = false>
__global__ void __launch_bounds__(256, MINB) gather_row_persistent_kernel(GatherParams p,
                                                                          int warps_per_token) {
  constexpr int VEC = Raw<TT>::VEC;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int CHUNK = 32 * VEC;
  const int nchunks = (p.d_out + CHUNK - 1) / CHUNK;
  const TT* T = reinterpret_cast<const TT*>(p.T);
  const int64_t tstride = (int64_t)p.rows * p.d_out;
  int bad = 0;
  for (int64_t item = gwarp; item < p.n * warps_per_token; item += nwarps) {
    // part-major order: the resident warps work on one column part of many
    // tokens, so a round of resident warps touches only that part of each
    // table row -- HBM re-reads of an over-L2 table stack drop by the number
    // of parts (c4: 4x), the gathered bytes are unchanged
    int part;
    int64_t token;
    if constexpr (PM) {
      part = (int)(item / p.n);
      token = item - (int64_t)part * p.n;
    } else {
      token = item / warps_per_token;
      part = (int)(item - token * warps_per_token);
    }
    const int c0 = part * MAXC;
    const int colbase = c0 * CHUNK + lane * VEC;
    bool ok[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) ok[c] = (c0 + c < nchunks) && (colbase + c * CHUNK < p.d_out);
    const uint32_t* cr = p.codes + token * p.ld;
    const float* wr = p.coeff + token * p.ld;
    float acc[MAXC][VEC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[c][v] = 0.f;
    // Optionally every other round of tokens walks the tables backwards, so
    // the tables a round finishes with (still in L2) are the first the next
    // round reads.
    const int rmask = (p.reverse_odd_rounds && ((item / nwarps) & 1)) ? -1 : 0;
    // records in groups of G (= TIF, at least 4): G/4 128-bit loads each
    constexpr int G = TIF > 4 ? TIF : 4;
    auto group_of = [&](int it) { return rmask ? p.nk - G - it : it; };
    uint4 cc[G / 4];
    float4 ww[G / 4];
#pragma unroll
    for (int g = 0; g < G / 4; ++g) {
      cc[g] = __ldg(reinterpret_cast<const uint4*>(cr + group_of(0)) + g);
      ww[g] = __ldg(reinterpret_cast<const float4*>(wr + group_of(0)) + g);
    }
    for (int it = 0; it < p.nk; it += G) {
      const int kg = group_of(it);
      uint4 cn[G / 4];
      float4 wn[G / 4];
#pragma unroll
      for (int g = 0; g < G / 4; ++g) {
        cn[g] = cc[g];
        wn[g] = ww[g];
      }
      if (it + G < p.nk) {
#pragma unroll
        for (int g = 0; g < G / 4; ++g) {
          cn[g] = __ldg(reinterpret_cast<const uint4*>(cr + group_of(it + G)) + g);
          wn[g] = __ldg(reinterpret_cast<const float4*>(wr + group_of(it + G)) + g);
        }
      }
      uint32_t codesG[G];
      float wG[G];
#pragma unroll
      for (int g = 0; g < G / 4; ++g) {
        codesG[4 * g] = cc[g].x; codesG[4 * g + 1] = cc[g].y;
        codesG[4 * g + 2] = cc[g].z; codesG[4 * g + 3] = cc[g].w;
        wG[4 * g] = ww[g].x; wG[4 * g + 1] = ww[g].y;
        wG[4 * g + 2] = ww[g].z; wG[4 * g + 3] = ww[g].w;
      }
      const bool fastw = p.bf16w && coeffs_bf16_exact<G>(wG);
#pragma unroll
      for (int q0 = 0; q0 < G; q0 += TIF) {
        uint4 raw[TIF][MAXC];
#pragma unroll
        for (int q = 0; q < TIF; ++q) {
          LFFN_DCHECK(codesG[q0 + q] < (uint32_t)p.rows && kg + q0 + q < p.nk && kg + q0 + q >= 0);
          const TT* rp = T + (kg + q0 + q) * tstride + (int64_t)codesG[q0 + q] * p.d_out + colbase;
#pragma unroll
          for (int c = 0; c < MAXC; ++c)
            raw[q][c] = ok[c] ? Raw<TT>::load(rp + c * CHUNK) : make_uint4(0u, 0u, 0u, 0u);
        }
        if (sizeof(TT) == 2 && fastw) {
#pragma unroll
          for (int q = 0; q < TIF; ++q)
#pragma unroll
            for (int c = 0; c < MAXC; ++c)
              Raw<TT>::fma_bf16w(acc[c], (uint16_t)(__float_as_uint(wG[q0 + q]) >> 16), raw[q][c]);
        } else {
#pragma unroll
          for (int q = 0; q < TIF; ++q)
#pragma unroll
            for (int c = 0; c < MAXC; ++c) Raw<TT>::fma(acc[c], wG[q0 + q], raw[q][c]);
        }
      }
#pragma unroll
      for (int g = 0; g < G / 4; ++g) {
        cc[g] = cn[g];
        ww[g] = wn[g];
      }
    }
    float* yr = p.y + token * p.d_out;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      if (!ok[c]) continue;
      const int col = colbase + c * CHUNK;
      if (p.accumulate) {
#pragma unroll
        for (int v = 0; v < VEC; v += 4) {
          const float4 a = *reinterpret_cast<const float4*>(yr + col + v);
          acc[c][v] += a.x; acc[c][v + 1] += a.y; acc[c][v + 2] += a.z; acc[c][v + 3] += a.w;
        }
      }
#pragma unroll
      for (int v = 0; v < VEC; ++v)
        if (!isfinite(acc[c][v])) bad = 4;
#pragma unroll
      for (int v = 0; v < VEC; v += 4)
        *reinterpret_cast<float4*>(yr + col + v) =
            make_float4(acc[c][v], acc[c][v + 1], acc[c][v + 2], acc[c][v + 3]);
    }
  }
  if (bad) atomicOr(p.flag, bad);
}

}  // namespace lffn_gpu

namespace lffn_gpu {

// Split-table gather for batches smaller than the resident warp slots (small
// serving batches, the host path's pipeline chunks): S warps of a CTA share
// one (token, column part) and each walks a contiguous 1/S of the tables
// (ascending, TIF tables' 128-bit row segments in flight per lane), so the
// per-token chain of dependent table rounds is S times shorter.  The S fp32
// partials meet in shared memory and are summed in split order (tables
// ascending within each split) -- deterministic, no atomics.  A CTA of 256
// threads holds 8 / S items.  Requires the 4-record layout with
// (nk / S) % 4 == 0 and 16-byte aligned rows.
template <typename TT, int MAXC, int TIF, int S>
__global__ void __launch_bounds__(256, 2) gather_split_kernel(GatherParams p, int parts) {
  constexpr int VEC = Raw<TT>::VEC;
  constexpr int CHUNK = 32 * VEC;
  constexpr int IPC = 8 / S;  // items per CTA
  __shared__ float4 part_sm[8][MAXC][VEC / 4][32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int split = wib % S;
  const int64_t item = (int64_t)blockIdx.x * IPC + wib / S;
  const int nchunks = (p.d_out + CHUNK - 1) / CHUNK;
  const bool live = item < p.n * parts;
  const int64_t token = live ? item / parts : 0;
  const int part = live ? (int)(item - token * parts) : 0;
  const int c0 = part * MAXC;
  const int colbase = c0 * CHUNK + lane * VEC;
  bool ok[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) ok[c] = live && (c0 + c < nchunks) && (colbase + c * CHUNK < p.d_out);
  const TT* T = reinterpret_cast<const TT*>(p.T);
  const int64_t tstride = (int64_t)p.rows * p.d_out;
  const int per = p.nk / S;
  const int kb = split * per;
  const uint32_t* cr = p.codes + token * p.ld + kb;
  const float* wr = p.coeff + token * p.ld + kb;
  float acc[MAXC][VEC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[c][v] = 0.f;
  if (live) {
    uint4 cc = __ldg(reinterpret_cast<const uint4*>(cr));
    float4 ww = __ldg(reinterpret_cast<const float4*>(wr));
    for (int it = 0; it < per; it += 4) {
      uint4 cn = cc;
      float4 wn = ww;
      if (it + 4 < per) {
        cn = __ldg(reinterpret_cast<const uint4*>(cr + it + 4));
        wn = __ldg(reinterpret_cast<const float4*>(wr + it + 4));
      }
      const uint32_t code4[4] = {cc.x, cc.y, cc.z, cc.w};
      const float w4[4] = {ww.x, ww.y, ww.z, ww.w};
      const bool fastw = p.bf16w && coeffs_bf16_exact<4>(w4);
#pragma unroll
      for (int q0 = 0; q0 < 4; q0 += TIF) {
        uint4 raw[TIF][MAXC];
#pragma unroll
        for (int q = 0; q < TIF; ++q) {
          LFFN_DCHECK(code4[q0 + q] < (uint32_t)p.rows && kb + it + q0 + q < p.nk);
          const TT* rp = T + (int64_t)(kb + it + q0 + q) * tstride + (int64_t)code4[q0 + q] * p.d_out + colbase;
#pragma unroll
          for (int c = 0; c < MAXC; ++c)
            raw[q][c] = ok[c] ? Raw<TT>::load(rp + c * CHUNK) : make_uint4(0u, 0u, 0u, 0u);
        }
        if (sizeof(TT) == 2 && fastw) {
#pragma unroll
          for (int q = 0; q < TIF; ++q)
#pragma unroll
            for (int c = 0; c < MAXC; ++c)
              Raw<TT>::fma_bf16w(acc[c], (uint16_t)(__float_as_uint(w4[q0 + q]) >> 16), raw[q][c]);
        } else {
#pragma unroll
          for (int q = 0; q < TIF; ++q)
#pragma unroll
            for (int c = 0; c < MAXC; ++c) Raw<TT>::fma(acc[c], w4[q0 + q], raw[q][c]);
        }
      }
      cc = cn;
      ww = wn;
    }
  }
  if (split != 0) {
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
#pragma unroll
      for (int v = 0; v < VEC; v += 4)
        part_sm[wib][c][v / 4][lane] = make_float4(acc[c][v], acc[c][v + 1], acc[c][v + 2], acc[c][v + 3]);
  }
  __syncthreads();
  if (split != 0 || !live) return;
#pragma unroll
  for (int s = 1; s < S; ++s)
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
#pragma unroll
      for (int v = 0; v < VEC; v += 4) {
        const float4 q = part_sm[wib + s][c][v / 4][lane];
        acc[c][v] += q.x; acc[c][v + 1] += q.y; acc[c][v + 2] += q.z; acc[c][v + 3] += q.w;
      }
  int bad = 0;
  float* yr = p.y + token * p.d_out;
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    if (!ok[c]) continue;
    const int col = colbase + c * CHUNK;
#pragma unroll
    for (int v = 0; v < VEC; v += 4) {
      float4 o = make_float4(acc[c][v], acc[c][v + 1], acc[c][v + 2], acc[c][v + 3]);
      if (p.accumulate) {
        const float4 a = *reinterpret_cast<const float4*>(yr + col + v);
        o.x += a.x; o.y += a.y; o.z += a.z; o.w += a.w;
      }
      if (!isfinite(o.x) || !isfinite(o.y) || !isfinite(o.z) || !isfinite(o.w)) bad = 4;
      *reinterpret_cast<float4*>(yr + col + v) = o;
    }
  }
  if (bad) atomicOr(p.flag, bad);
}

}  // namespace lffn_gpu
