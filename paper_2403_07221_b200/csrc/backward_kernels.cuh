// backward_kernels.cuh -- the LookupFFN backward on the device (SURVEY.md
// 8f-4): lookup_backward (lookup.cpp:292-347) and Projection::backward
// (projection.cpp:279-386) for the signflip and dense kinds.
//
//   KB1 bwd_gradz_kernel   per (token, table, neighbour) record: gdott =
//                          <grad_y_i, T_k[code]> (fp32 products, float64
//                          warp reduction), then the straight-through
//                          gradient of every coordinate,
//                          gz_j += gdott * w (s_j - tanh z_j)            (softmax)
//                          gz_j += gdott * w (s_j (1 + dot) - dot tanh z_j)  (scaled)
//                          with w, dot recomputed from z exactly as the
//                          forward does (top-1 weight / exp(dot - logden)).
//   KB2 grad_T             records bucketed per (table, code) row with
//                          deterministic stable ranks (token blocks ranked
//                          in order, block offsets, row starts by scan), then
//                          one warp per row sums coeff * grad_y over its
//                          records in the reference's order (tokens, then
//                          neighbours ascending; float32) and writes the row
//                          once -- no atomics on the gradient, run-to-run
//                          identical.
//   KB3 projection         signflip: the transposed network per token, in
//                          float64 with the reference's stage order --
//                          FWHT, x s_2, FWHT, x s_1, FWHT, x s_0 -- run as K1's
//                          pre-flip phases with masks (0, s_2, s_1) and a final
//                          flip by s_0: grad_x bit-identical to the reference
//                          for the same grad_z.  dense: two exact float64
//                          GEMMs, grad_x = g W^T (j ascending) and grad_W =
//                          x^T g (tokens ascending), bit-identical as well.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "hash_kernels.cuh"
#include "lffn_internal.h"

namespace lffn_gpu {

struct BwdParams {
  const double* z;       // [n x code_width] forward projection output (float64)
  const uint32_t* codes; // [n x hl x nc] records of the forward
  const float* coeff;    // [n x hl x nc] forward coefficients
  const float* gy;       // [n x d_out]
  const void* T;         // this context's tables [hl][rows][d_out], f32 or bf16
  int64_t n;
  int d_out, code_width, tau, kb, hl, nc, rows, scaled;
  double* gz;            // [n x code_width]: owned columns written, others untouched
  uint32_t* offs;        // [hl * rows + 1] counts, then row starts
  uint32_t* list;        // [n * hl * nc] record ids grouped by row
  float* gT;             // [hl][rows][d_out]
  int* flag;
};

// tanh(z) with the saturated range short-cut: for |z| >= 19.5 the true value
// is within 2 e^{-39} < 2^-54 of +-1, so the correctly rounded (and the
// reference's std::tanh) result is exactly +-1.0 -- no transcendental for the
// large |z| that the unnormalised transforms produce.
__device__ __forceinline__ double tanh_exact(double z) {
  return fabs(z) >= 19.5 ? copysign(1.0, z) : tanh(z);
}

template <typename TT>
__device__ __forceinline__ float tload(const TT* p);
template <>
__device__ __forceinline__ float tload<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float tload<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

// KB1: one warp per token.  Lane j < tau owns coordinate j of the current
// table; the sequential float64 reductions of the reference (sum |z|, the
// top-1 divisions, log_denominator, code_dot) run on lane 0 over shuffled
// coordinates, in the reference's order.
template <typename TT, int VEC>
__global__ void __launch_bounds__(256) bwd_gradz_kernel(BwdParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t token = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (token >= p.n) return;
  const int tau = p.tau;
  const float* gyr = p.gy + token * p.d_out;
  const TT* T = static_cast<const TT*>(p.T);
  int bad = 0;
  for (int j = lane; j < p.d_out; j += 32)
    if (!isfinite(gyr[j])) bad |= kFlagBwdInput;
  for (int k = 0; k < p.hl; ++k) {
    const double* zk = p.z + token * p.code_width + (int64_t)(p.kb + k) * tau;
    const double zj = lane < tau ? zk[lane] : 0.0;
    const double aj = fabs(zj);
    // per-coordinate terms, then lane 0 folds them in order
    const double fj = aj < 18.5 ? 1.0 + exp(-2.0 * aj) : 1.0;      // top-1 factor
    const double lj = p.nc > 1 ? aj + log1p(exp(-2.0 * aj)) : 0.0;  // log_denominator term
    double sum_abs = 0.0, w1 = 1.0, logden = 0.0;
    for (int j = 0; j < tau; ++j) {
      const double a = __shfl_sync(0xffffffffu, aj, j);
      const double f = __shfl_sync(0xffffffffu, fj, j);
      const double l = __shfl_sync(0xffffffffu, lj, j);
      sum_abs = sum_abs + a;   // lookup.cpp:244-246
      w1 = w1 / f;             // top1_weight (lookup.cpp:185-189)
      logden = logden + l;     // lookup.cpp:102-109
    }
    double gzj = 0.0;
    for (int c = 0; c < p.nc; ++c) {
      const int64_t rec = (token * p.hl + k) * p.nc + c;
      const uint32_t code = p.codes[rec];
      const TT* row = T + ((int64_t)k * p.rows + code) * p.d_out;
      float part = 0.f;
      if constexpr (VEC == 8) {
        // bf16 rows, 16-byte loads: lane l owns columns 256 i + 8 l .. + 7
        for (int j = lane * 8; j < p.d_out; j += 256) {
          const float4 ga = *reinterpret_cast<const float4*>(gyr + j);
          const float4 gb = *reinterpret_cast<const float4*>(gyr + j + 4);
          const uint4 u = __ldg(reinterpret_cast<const uint4*>(row + j));
          part = fmaf(ga.x, __uint_as_float(u.x << 16), part);
          part = fmaf(ga.y, __uint_as_float(u.x & 0xffff0000u), part);
          part = fmaf(ga.z, __uint_as_float(u.y << 16), part);
          part = fmaf(ga.w, __uint_as_float(u.y & 0xffff0000u), part);
          part = fmaf(gb.x, __uint_as_float(u.z << 16), part);
          part = fmaf(gb.y, __uint_as_float(u.z & 0xffff0000u), part);
          part = fmaf(gb.z, __uint_as_float(u.w << 16), part);
          part = fmaf(gb.w, __uint_as_float(u.w & 0xffff0000u), part);
        }
      } else if constexpr (VEC == 4) {
        for (int j = lane * 4; j < p.d_out; j += 128) {
          const float4 g = *reinterpret_cast<const float4*>(gyr + j);
          float t0, t1, t2, t3;
          if constexpr (sizeof(TT) == 4) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(row + j));
            t0 = t.x; t1 = t.y; t2 = t.z; t3 = t.w;
          } else {
            const uint2 u = __ldg(reinterpret_cast<const uint2*>(row + j));
            t0 = __uint_as_float(u.x << 16); t1 = __uint_as_float(u.x & 0xffff0000u);
            t2 = __uint_as_float(u.y << 16); t3 = __uint_as_float(u.y & 0xffff0000u);
          }
          part = fmaf(g.x, t0, part);
          part = fmaf(g.y, t1, part);
          part = fmaf(g.z, t2, part);
          part = fmaf(g.w, t3, part);
        }
      } else {
        for (int j = lane; j < p.d_out; j += 32) part = fmaf(gyr[j], tload<TT>(row + j), part);
      }
      double gd = (double)part;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gd += __shfl_xor_sync(0xffffffffu, gd, o);
      // the record's weight and dot exactly as the forward (lookup.cpp:238-252)
      double dot = sum_abs, w = w1;
      if (p.nc > 1) {
        dot = 0.0;
        for (int j = 0; j < tau; ++j) {
          const double zz = __shfl_sync(0xffffffffu, zj, j);
          dot = dot + (((code >> j) & 1u) ? zz : -zz);   // code_dot (lookup.cpp:111-116)
        }
        w = exp(dot - logden);
      }
      if (lane < tau) {
        const double s = ((code >> lane) & 1u) ? 1.0 : -1.0;
        const double th = tanh_exact(zj);
        const double dcoeff = p.scaled ? w * (s * (1.0 + dot) - dot * th) : w * (s - th);
        gzj = gzj + gd * dcoeff;
      }
    }
    if (lane < tau) p.gz[token * p.code_width + (int64_t)(p.kb + k) * tau + lane] = gzj;
  }
  if (bad) atomicOr(p.flag, bad);
}

// KB1 in two passes (the default; bwd_gradz_kernel above stays for widths
// that are not a multiple of 4).
//
// KB1a bwd_gdot_kernel: gdot[record] = <grad_y_i, T_k[code]> for every
// record, one warp per token with the token's grad_y row in registers and
// TIF records' row segments in flight (the single-pass kernel waited for one
// row and one reduction per table).  Lane l owns columns c*128 + 4l .. +3
// and sums its fp32 products per record; every 32 records the per-lane
// partials are reduced across the warp in float64 with a transposed
// butterfly (31 exchanges for 32 sums instead of 5 per record), after which
// lane l holds record l's sum and the 32 results are stored coalesced.
template <typename TT, int MAXC, int TIF, int VEC = 4>
__global__ void __launch_bounds__(256, 2) bwd_gdot_kernel(BwdParams p, double* gdot) {
  // VEC columns per lane per chunk: 4 (fp32 rows, 16-byte loads; bf16 rows,
  // 8-byte loads) or 8 (bf16 rows, 16-byte loads) -- the same per-lane
  // column order as bwd_gradz_kernel<TT, VEC>
  static_assert(32 % TIF == 0, "TIF must divide 32");
  static_assert(VEC == 4 || (VEC == 8 && sizeof(TT) == 2), "VEC 8 is for bf16 rows");
  constexpr int CW = 32 * VEC;  // columns per chunk
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const TT* T = static_cast<const TT*>(p.T);
  const int R = p.hl * p.nc;
  int bad = 0;
  for (int64_t token = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; token < p.n;
       token += nwarps) {
    const float* gyr = p.gy + token * p.d_out;
    float g[MAXC][VEC];
    bool ok[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int j = c * CW + lane * VEC;
      ok[c] = j < p.d_out;
#pragma unroll
      for (int v = 0; v < VEC; v += 4) {
        const float4 q = ok[c] ? *reinterpret_cast<const float4*>(gyr + j + v) : make_float4(0.f, 0.f, 0.f, 0.f);
        g[c][v] = q.x; g[c][v + 1] = q.y; g[c][v + 2] = q.z; g[c][v + 3] = q.w;
        if (!isfinite(q.x) || !isfinite(q.y) || !isfinite(q.z) || !isfinite(q.w)) bad |= kFlagBwdInput;
      }
    }
    const uint32_t* cr = p.codes + token * R;
    for (int r32 = 0; r32 < R; r32 += 32) {
      // lane q of the warp loads code r32 + q; broadcast by shuffle
      const uint32_t mycode = r32 + lane < R ? __ldg(cr + r32 + lane) : 0u;
      float part[32];
#pragma unroll
      for (int q0 = 0; q0 < 32; q0 += TIF) {
        // raw rows in flight (bf16 VEC 8: packed, widened at the FMA)
        float t[sizeof(TT) == 2 && VEC == 8 ? 1 : TIF][MAXC][VEC];
        uint4 traw[sizeof(TT) == 2 && VEC == 8 ? TIF : 1][MAXC];
#pragma unroll
        for (int q = 0; q < TIF; ++q) {
          const int r = r32 + q0 + q;
          const uint32_t code = __shfl_sync(0xffffffffu, mycode, q0 + q);
          const int k = p.nc == 1 ? r : r / p.nc;
          const TT* row = T + ((int64_t)k * p.rows + code) * p.d_out + lane * VEC;
#pragma unroll
          for (int c = 0; c < MAXC; ++c) {
            const bool on = ok[c] && r < R;
            if constexpr (sizeof(TT) == 4) {
              const float4 u = on ? __ldg(reinterpret_cast<const float4*>(row + c * CW)) : make_float4(0.f, 0.f, 0.f, 0.f);
              t[q][c][0] = u.x; t[q][c][1] = u.y; t[q][c][2] = u.z; t[q][c][3] = u.w;
            } else if constexpr (VEC == 4) {
              const uint2 u = on ? __ldg(reinterpret_cast<const uint2*>(row + c * CW)) : make_uint2(0u, 0u);
              t[q][c][0] = __uint_as_float(u.x << 16); t[q][c][1] = __uint_as_float(u.x & 0xffff0000u);
              t[q][c][2] = __uint_as_float(u.y << 16); t[q][c][3] = __uint_as_float(u.y & 0xffff0000u);
            } else {
              traw[q][c] = on ? __ldg(reinterpret_cast<const uint4*>(row + c * CW)) : make_uint4(0u, 0u, 0u, 0u);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < TIF; ++q) {
          float acc = 0.f;
#pragma unroll
          for (int c = 0; c < MAXC; ++c) {
            if constexpr (sizeof(TT) == 2 && VEC == 8) {
              const uint32_t w4[4] = {traw[q][c].x, traw[q][c].y, traw[q][c].z, traw[q][c].w};
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                acc = fmaf(g[c][2 * h], __uint_as_float(w4[h] << 16), acc);
                acc = fmaf(g[c][2 * h + 1], __uint_as_float(w4[h] & 0xffff0000u), acc);
              }
            } else {
#pragma unroll
              for (int v = 0; v < VEC; ++v) acc = fmaf(g[c][v], t[q][c][v], acc);
            }
          }
          part[q0 + q] = acc;
        }
      }
      // transposed butterfly: after the step with offset s, the lanes with
      // bit s set hold the upper halves; lane l ends with record l's sum
      double v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const bool up = lane & 16;
        const double send = (double)(up ? part[i] : part[i + 16]);
        const double keep = (double)(up ? part[i + 16] : part[i]);
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
#pragma unroll
      for (int sft = 8; sft >= 1; sft >>= 1) {
#pragma unroll
        for (int i = 0; i < sft; ++i) {
          const bool up = lane & sft;
          const double send = up ? v[i] : v[i + sft];
          const double keep = up ? v[i + sft] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
        }
      }
      if (r32 + lane < R) gdot[token * R + r32 + lane] = v[0];
    }
  }
  if (bad) atomicOr(p.flag, bad);
}

// KB1b bwd_gz_kernel: one thread per (token, table): the straight-through
// gradient of the table's tau coordinates from the records' gdot, with the
// weight / dot / log-denominator folded in the reference's order exactly as
// bwd_gradz_kernel does (lookup.cpp:292-340) -- bit-identical to it.
// TAU > 0: compile-time code width (registers); 0: any tau <= 24.
template <int TAU>
__global__ void __launch_bounds__(256) bwd_gz_kernel(BwdParams p, const double* gdot) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= p.n * p.hl) return;
  const int64_t token = idx / p.hl;
  const int k = (int)(idx - token * p.hl);
  const int tau = TAU > 0 ? TAU : p.tau;
  const double* zk = p.z + token * p.code_width + (int64_t)(p.kb + k) * tau;
  double zv[TAU > 0 ? TAU : 24];
  if constexpr (TAU > 0 && TAU % 2 == 0) {
    // 16-byte loads (the table's tau coordinates are contiguous and 16-byte
    // aligned for even tau)
#pragma unroll
    for (int j = 0; j < TAU; j += 2) {
      const double2 q = *reinterpret_cast<const double2*>(zk + j);
      zv[j] = q.x;
      zv[j + 1] = q.y;
    }
  } else {
    for (int j = 0; j < tau; ++j) zv[j] = zk[j];
  }
  double sum_abs = 0.0, w1 = 1.0, logden = 0.0;
#pragma unroll
  for (int j = 0; j < tau; ++j) {
    const double zj = zv[j];
    const double aj = fabs(zj);
    sum_abs = sum_abs + aj;
    // 1 + exp(-2a) == 1.0 exactly for a >= 18.5: the division is then exact
    // and skipped (as the forward's top1 weight)
    if (aj < 18.5) w1 = w1 / (1.0 + exp(-2.0 * aj));
    if (p.nc > 1) logden = logden + (aj + log1p(exp(-2.0 * aj)));
  }
  double gzv[TAU > 0 ? TAU : 24];
#pragma unroll
  for (int j = 0; j < tau; ++j) gzv[j] = 0.0;
  for (int c = 0; c < p.nc; ++c) {
    const int64_t rec = (token * p.hl + k) * p.nc + c;
    const uint32_t code = p.codes[rec];
    const double gd = gdot[rec];
    double dot = sum_abs, w = w1;
    if (p.nc > 1) {
      dot = 0.0;
#pragma unroll
      for (int j = 0; j < tau; ++j) dot = dot + (((code >> j) & 1u) ? zv[j] : -zv[j]);
      w = exp(dot - logden);
    }
#pragma unroll
    for (int j = 0; j < tau; ++j) {
      const double sg = ((code >> j) & 1u) ? 1.0 : -1.0;
      const double th = tanh_exact(zv[j]);
      const double dcoeff = p.scaled ? w * (sg * (1.0 + dot) - dot * th) : w * (sg - th);
      gzv[j] = gzv[j] + gd * dcoeff;
    }
  }
  double* gz = p.gz + token * p.code_width + (int64_t)(p.kb + k) * tau;
  if constexpr (TAU > 0 && TAU % 2 == 0) {
#pragma unroll
    for (int j = 0; j < TAU; j += 2) *reinterpret_cast<double2*>(gz + j) = make_double2(gzv[j], gzv[j + 1]);
  } else {
    for (int j = 0; j < tau; ++j) gz[j] = gzv[j];
  }
}

// KB2a: deterministic ranks.  Thread (k, b) walks token block b in order
// (tokens ascending, neighbours ascending) and gives each record of table k
// its rank among the block's records of the same row; hist[k][b][code] ends
// as the block's count.
// token blocks of the rank pass: each thread's walk is a chain of dependent
// histogram updates, so more blocks = shorter chains (32 -> 128: c2 rank
// pass 0.47 -> ~0.12 ms) at hl * rows * kBwdBlocks * 4 bytes of scratch
constexpr int kBwdBlocks = 128;
__global__ void bwd_rank_kernel(BwdParams p, uint32_t* hist, uint32_t* rank) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (int64_t)p.hl * kBwdBlocks) return;
  const int k = int(tid % p.hl), b = int(tid / p.hl);
  const int64_t per = (p.n + kBwdBlocks - 1) / kBwdBlocks;
  const int64_t i0 = b * per, i1 = min(p.n, i0 + per);
  // hist layout [k][code][b]: a row's block counts are contiguous
  uint32_t* h = hist + (int64_t)k * p.rows * kBwdBlocks + b;
  for (int64_t i = i0; i < i1; ++i) {
    const int64_t rec0 = (i * p.hl + k) * p.nc;
    for (int c = 0; c < p.nc; ++c) {
      const uint32_t code = p.codes[rec0 + c];
      rank[rec0 + c] = h[(int64_t)code * kBwdBlocks]++;
    }
  }
}

// KB2b': per (table, code) row, one warp: exclusive scan of the row's
// kBwdBlocks block counts (contiguous, hist[k][code][b]) in place -- the
// block offsets -- and the row's total into offs.
__global__ void __launch_bounds__(256) bwd_block_offsets_kernel(BwdParams p, uint32_t* hist) {
  static_assert(kBwdBlocks % 32 == 0, "whole words per lane");
  constexpr int PL = kBwdBlocks / 32;  // counts per lane, consecutive
  const int lane = threadIdx.x & 31;
  const int64_t bin = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (bin >= (int64_t)p.hl * p.rows) return;
  uint32_t* hp = hist + bin * kBwdBlocks + lane * PL;
  uint32_t v[PL], tot = 0;
#pragma unroll
  for (int j = 0; j < PL; ++j) {
    v[j] = hp[j];
    tot += v[j];
  }
  uint32_t x = tot;  // inclusive scan of the lane totals
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  uint32_t run = x - tot;
#pragma unroll
  for (int j = 0; j < PL; ++j) {
    hp[j] = run;
    run += v[j];
  }
  if (lane == 31) p.offs[bin] = x;
}

// KB2b: exclusive scan of the row counts into row starts (one CTA).
__global__ void __launch_bounds__(1024) bwd_scan_kernel(BwdParams p) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t carry;
  const int64_t bins = (int64_t)p.hl * p.rows;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < bins; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const uint32_t v = i < bins ? p.offs[i] : 0u;
    // inclusive warp scan
    uint32_t x = v;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      warp_sums[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const uint32_t excl = carry + (wid > 0 ? warp_sums[wid - 1] : 0u) + x - v;
    if (i < bins) p.offs[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) p.offs[bins] = carry;
}

// KB2c: record ids into their row's slots, stable (tokens ascending).
__global__ void bwd_place_kernel(BwdParams p, const uint32_t* hist, const uint32_t* rank) {
  const int64_t total = p.n * p.hl * p.nc;
  const int64_t per = (p.n + kBwdBlocks - 1) / kBwdBlocks;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < total;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = r / ((int64_t)p.hl * p.nc);
    const int k = int((r / p.nc) % p.hl);
    const int b = int(i / per);
    const uint32_t code = p.codes[r];
    const uint32_t pos = p.offs[(int64_t)k * p.rows + code] +
                         hist[((int64_t)k * p.rows + code) * kBwdBlocks + b] + rank[r];
    p.list[pos] = uint32_t(r);
  }
}

// KB2d: one warp per (table, code) row: gT_row = sum coeff * grad_y_token.
// KB2e, d_out % 4 == 0: one warp per row with the whole row in registers
// (lane l owns columns c*128 + 4l .. +3), the row's records walked four at
// a time so four grad_y rows are in flight; per column the products are
// accumulated in record order exactly as bwd_gradT_kernel -- bit-identical.
template <int MAXC>
__global__ void __launch_bounds__(256) bwd_gradT4_kernel(BwdParams p, int parts) {
  // a row's columns are split into `parts` warps of MAXC chunks each (wide
  // rows would otherwise need > 128 registers); per column the order is the
  // same
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t bin = gw / parts;
  const int part = (int)(gw - bin * parts);
  const int64_t bins = (int64_t)p.hl * p.rows;
  if (bin >= bins) return;
  const uint32_t b0 = p.offs[bin], b1 = p.offs[bin + 1];
  const int per_tok = p.hl * p.nc;
  const int cbase = part * MAXC * 128;  // first column of this warp's part
  bool ok[MAXC];
  float4 acc[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    ok[c] = cbase + c * 128 + lane * 4 < p.d_out;
    acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (uint32_t e0 = b0; e0 < b1; e0 += 4) {
    float cf[4];
    const float* gyr[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t e = min(e0 + q, b1 - 1);
      const uint32_t rec = __ldg(p.list + e);
      cf[q] = e0 + q < b1 ? __ldg(p.coeff + rec) : 0.f;
      gyr[q] = p.gy + (int64_t)(rec / per_tok) * p.d_out + cbase + lane * 4;
    }
    float4 g[4][MAXC];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < MAXC; ++c)
        g[q][c] = ok[c] ? __ldg(reinterpret_cast<const float4*>(gyr[q] + c * 128))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (e0 + q >= b1) break;
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        acc[c].x = fmaf(cf[q], g[q][c].x, acc[c].x);
        acc[c].y = fmaf(cf[q], g[q][c].y, acc[c].y);
        acc[c].z = fmaf(cf[q], g[q][c].z, acc[c].z);
        acc[c].w = fmaf(cf[q], g[q][c].w, acc[c].w);
      }
    }
  }
  int bad = 0;
  float* out = p.gT + bin * p.d_out + cbase + lane * 4;
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    if (!ok[c]) continue;
    if (!isfinite(acc[c].x) || !isfinite(acc[c].y) || !isfinite(acc[c].z) || !isfinite(acc[c].w))
      bad |= kFlagBwdTables;
    *reinterpret_cast<float4*>(out + c * 128) = acc[c];
  }
  if (bad) atomicOr(p.flag, bad);
}

__global__ void __launch_bounds__(256) bwd_gradT_kernel(BwdParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t bin = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t bins = (int64_t)p.hl * p.rows;
  if (bin >= bins) return;
  const uint32_t b0 = p.offs[bin], b1 = p.offs[bin + 1];
  float* out = p.gT + bin * p.d_out;
  const int per_tok = p.hl * p.nc;
  int bad = 0;
  for (int j0 = 0; j0 < p.d_out; j0 += 32 * 8) {
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.f;
    for (uint32_t e = b0; e < b1; ++e) {
      const uint32_t rec = p.list[e];
      const float cf = p.coeff[rec];
      const float* gyr = p.gy + (int64_t)(rec / per_tok) * p.d_out;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = j0 + q * 32 + lane;
        if (j < p.d_out) acc[q] = fmaf(cf, gyr[j], acc[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = j0 + q * 32 + lane;
      if (j < p.d_out) {
        if (!isfinite(acc[q])) bad |= kFlagBwdTables;
        out[j] = acc[q];
      }
    }
  }
  if (bad) atomicOr(p.flag, bad);
}

// KB3 signflip: grad_x = first d_in of s_0 * H(s_1 * H(s_2 * H(g))), g = grad_z
// padded to D (projection.cpp:362-369).  p.signmask holds (0, s_2, s_1).
// LOGD > 0: compile-time transform width (all shared-memory geometry folds,
// as in hash_structured_kernel); NT / MINB: CTA size and residency.
template <int LOGE, int NT = 256, int MINB = 1, int LOGD = 0>
__global__ void __launch_bounds__(NT, MINB) proj_bwd_signflip_kernel(HashParams p, const double* gz,
                                                                const uint32_t* s0mask,
                                                                double* grad_x) {
  extern __shared__ double smem[];
  constexpr int E = 1 << LOGE;
  const int logD = LOGD > 0 ? LOGD : p.logD;
  const int tpt = LOGD > 0 ? (1 << (LOGD - LOGE)) : p.threads_per_token;
  const int slot = threadIdx.x / tpt;
  const int t = threadIdx.x - slot * tpt;
  const int64_t token = (int64_t)blockIdx.x * p.tokens_per_block + slot;
  const bool active = slot < p.tokens_per_block && token < p.n;
  const int D = 1 << logD;
  double* sm = smem + (size_t)slot * padded_len(D);
  int bad = 0;
  auto token_sync = [&]() {
    if (tpt <= 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(slot + 1), "r"(tpt) : "memory");
  };
  if (active)
    for (int a = t; a < D; a += tpt) {
      const double v = a < p.code_width ? gz[token * p.code_width + a] : 0.0;
      if (!isfinite(v)) bad |= kFlagBwdInput;
      sm[spos(a)] = v;
    }
  token_sync();
  int nph = 1;
  if constexpr (LOGE > 0) nph = (logD + LOGE - 1) / LOGE;
#pragma unroll 1
  for (int tr = 0; tr < 3; ++tr) {
    if (active) phase_smem<LOGE, LOGE, false, kPreSign>(sm, t, tpt, 0, p, tr, nullptr, bad, false);
    token_sync();
    const int nphc = LOGD > 0 ? (LOGD + LOGE - 1) / LOGE : nph;
#pragma unroll
    for (int ph = 1; ph < nphc; ++ph) {
      if (active) run_later_phase<LOGE>(sm, t, tpt, ph * LOGE, min(LOGE, logD - ph * LOGE), p, tr, bad, false);
      token_sync();
    }
  }
  if (active)
    for (int a = t; a < p.d_in; a += tpt) {
      double v = sm[spos(a)];
      v = flip_sign(v, __ldg(s0mask + (a >> 5)), a & 31);
      if (!isfinite(v)) bad |= kFlagBwdOutput;
      grad_x[token * p.d_in + a] = v;
    }
  if (bad) atomicOr(p.flag, bad);
}

// KB3 dense: C[m][nn] = sum_kk A(m, kk) * B(kk, nn), kk ascending from 0.0
// with separately rounded multiply and add -- the reference's loops for
// grad_x (j ascending) and grad_W (rows ascending), bit-identical.  8 x 8
// outputs per thread: 64 multiply-adds per 16 shared-memory operand loads,
// coalesced global staging for both layouts, and the next K slice loaded into
// registers while the current one is consumed (c2 dense backward 23.9 ->
// 16.7 ms against a 4 x 4-per-thread tile).  blockIdx.z selects a batch
// entry: A, B, C advance by sA, sB, sC elements.  64 threads own a 64 x 64 tile (thread (ty, tx): rows ty + 8i,
// columns tx + 8j, conflict-free shared-memory reads).
template <typename TA, bool TRANS_A, bool TRANS_B>
__global__ void __launch_bounds__(64, 4) gemm_f64_exact8_kernel(const TA* __restrict__ A, int lda,
                                                                const double* __restrict__ B, int ldb,
                                                                double* __restrict__ C, int ldc, int M,
                                                                int N, int K, int* flag,
                                                                int64_t sA = 0, int64_t sB = 0,
                                                                int64_t sC = 0, int a_bad = 0,
                                                                int c_bad = kFlagBwdOutput) {
  // a_bad / c_bad: flag bits raised by a non-finite A element / C output
  // (0: not checked)
  A += blockIdx.z * sA;
  B += blockIdx.z * sB;
  C += blockIdx.z * sC;
  int bad = 0;
  __shared__ double As[2][8][65];
  __shared__ double Bs[2][8][65];
  const int t = threadIdx.x;
  const int tx = t & 7, ty = t >> 3;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  // staging coordinates of this thread's 8 A and 8 B elements per K slice
  auto load_a = [&](int k0, double (&r)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int kk = TRANS_A ? i : (t & 7);
      const int mm = TRANS_A ? t : (t >> 3) + 8 * i;
      const int gm = m0 + mm, gk = k0 + kk;
      r[i] = (gm < M && gk < K) ? (double)(TRANS_A ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk])
                                : 0.0;
      if (a_bad && !isfinite(r[i])) bad |= a_bad;
    }
  };
  auto load_b = [&](int k0, double (&r)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int kk = TRANS_B ? (t & 7) : i;
      const int nn = TRANS_B ? (t >> 3) + 8 * i : t;
      const int gn = n0 + nn, gk = k0 + kk;
      r[i] = (gn < N && gk < K) ? (TRANS_B ? B[(int64_t)gn * ldb + gk] : B[(int64_t)gk * ldb + gn]) : 0.0;
    }
  };
  auto store = [&](int buf, const double (&ra)[8], const double (&rb)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      As[buf][TRANS_A ? i : (t & 7)][TRANS_A ? t : (t >> 3) + 8 * i] = ra[i];
      Bs[buf][TRANS_B ? (t & 7) : i][TRANS_B ? (t >> 3) + 8 * i : t] = rb[i];
    }
  };
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  double ra[8], rb[8];
  load_a(0, ra);
  load_b(0, rb);
  store(0, ra, rb);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += 8) {
    const bool more = k0 + 8 < K;
    if (more) {
      load_a(k0 + 8, ra);
      load_b(k0 + 8, rb);
    }
    const int kmax = min(8, K - k0);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      if (kk < kmax) {
        double a[8], b[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = As[buf][kk][ty + 8 * i];
#pragma unroll
        for (int j = 0; j < 8; ++j) b[j] = Bs[buf][kk][tx + 8 * j];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a[i], b[j]));
      }
    }
    if (more) {
      store(buf ^ 1, ra, rb);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gm = m0 + ty + 8 * i, gn = n0 + tx + 8 * j;
      if (gm < M && gn < N) {
        if (c_bad && !isfinite(acc[i][j])) bad |= c_bad;
        C[(int64_t)gm * ldc + gn] = acc[i][j];
      }
    }
  if (bad && flag) atomicOr(flag, bad);
}


// ---- stagewise kernels of the acdc / bh projection backward ----------------
// The stage vectors of all tokens live in [n x D] float64 arrays; every
// operation is the reference's, in its order (projection.cpp:216-245 forward,
// 322-360 backward).

// V[i][:] = pad(x_i) to D (projection.cpp:212-213)
__global__ void rows_pad_kernel(const float* __restrict__ x, int64_t n, int d_in, int D,
                                double* __restrict__ V) {
  const int64_t total = n * D;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / D;
    const int j = int(q - i * D);
    V[q] = j < d_in ? (double)x[i * d_in + j] : 0.0;
  }
}

// V[i][:] (or its first `cols`) from a [n x cols] float64 array, zero padded
__global__ void rows_load_kernel(const double* __restrict__ src, int64_t n, int cols, int D,
                                 double* __restrict__ V, int* flag) {
  const int64_t total = n * D;
  int bad = 0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / D;
    const int j = int(q - i * D);
    const double v = j < cols ? src[i * cols + j] : 0.0;
    if (!isfinite(v)) bad |= kFlagBwdInput;
    V[q] = v;
  }
  if (bad) atomicOr(flag, bad);
}

// out[i][:cols] = V[i][:cols]
__global__ void rows_store_kernel(const double* __restrict__ V, int64_t n, int cols, int D,
                                  double* __restrict__ out, int* flag) {
  const int64_t total = n * cols;
  int bad = 0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / cols;
    const double v = V[i * D + (q - i * cols)];
    if (!isfinite(v)) bad |= kFlagBwdOutput;
    out[q] = v;
  }
  if (bad) atomicOr(flag, bad);
}

// V[i][j] *= diag[j]
__global__ void rows_scale_kernel(double* __restrict__ V, int64_t n, int D,
                                  const double* __restrict__ diag) {
  const int64_t total = n * D;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x)
    V[q] = __dmul_rn(V[q], __ldg(diag + (q % D)));
}

// block_diag_apply (projection.hpp:101-119): out[g*b+c] = sum_r in[g*b+r] * B[g][r][c];
// TRANS: block_diag_apply_transposed (:122-137): out[g*b+r] = sum_c B[g][r][c] * in[g*b+c]
template <bool TRANS>
__global__ void rows_blockdiag_kernel(const double* __restrict__ in, double* __restrict__ out,
                                      int64_t n, int D, int b, const double* __restrict__ B) {
  const int64_t total = n * D;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / D;
    const int o = int(q - i * D);
    const int g = o / b, t = o - g * b;
    const double* src = in + i * D + (int64_t)g * b;
    const double* blk = B + (int64_t)g * b * b;
    double acc = 0.0;
    if (TRANS) {
      for (int c = 0; c < b; ++c) acc = __dadd_rn(acc, __dmul_rn(__ldg(blk + (int64_t)t * b + c), src[c]));
    } else {
      for (int r = 0; r < b; ++r) acc = __dadd_rn(acc, __dmul_rn(src[r], __ldg(blk + (int64_t)r * b + t)));
    }
    out[q] = acc;
  }
}

// The same exact GEMM with 32 x 32 tiles (4 x 4 outputs per thread, 64
// threads): four times the tiles of gemm_f64_exact8_kernel for GEMMs with few
// output tiles and a long sequential K (the bh parameter gradient: 32 blocks
// of 64 x 64 summed over all tokens).  Bit-identical sums.
template <typename TA, bool TRANS_A, bool TRANS_B>
__global__ void __launch_bounds__(64) gemm_f64_exact4_kernel(const TA* __restrict__ A, int lda,
                                                             const double* __restrict__ B, int ldb,
                                                             double* __restrict__ C, int ldc, int M,
                                                             int N, int K, int* flag, int64_t sA = 0,
                                                             int64_t sB = 0, int64_t sC = 0) {
  A += blockIdx.z * sA;
  B += blockIdx.z * sB;
  C += blockIdx.z * sC;
  int bad = 0;
  __shared__ double As[2][8][33];
  __shared__ double Bs[2][8][33];
  const int t = threadIdx.x;
  const int tx = t & 7, ty = t >> 3;
  const int m0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  auto load_a = [&](int k0, double (&r)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kk = TRANS_A ? (t >> 5) + 2 * i : (t & 7);
      const int mm = TRANS_A ? (t & 31) : (t >> 3) + 8 * i;
      const int gm = m0 + mm, gk = k0 + kk;
      r[i] = (gm < M && gk < K) ? (double)(TRANS_A ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk])
                                : 0.0;
    }
  };
  auto load_b = [&](int k0, double (&r)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kk = TRANS_B ? (t & 7) : (t >> 5) + 2 * i;
      const int nn = TRANS_B ? (t >> 3) + 8 * i : (t & 31);
      const int gn = n0 + nn, gk = k0 + kk;
      r[i] = (gn < N && gk < K) ? (TRANS_B ? B[(int64_t)gn * ldb + gk] : B[(int64_t)gk * ldb + gn]) : 0.0;
    }
  };
  auto store = [&](int buf, const double (&ra)[4], const double (&rb)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      As[buf][TRANS_A ? (t >> 5) + 2 * i : (t & 7)][TRANS_A ? (t & 31) : (t >> 3) + 8 * i] = ra[i];
      Bs[buf][TRANS_B ? (t & 7) : (t >> 5) + 2 * i][TRANS_B ? (t >> 3) + 8 * i : (t & 31)] = rb[i];
    }
  };
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  double ra[4], rb[4];
  load_a(0, ra);
  load_b(0, rb);
  store(0, ra, rb);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += 8) {
    const bool more = k0 + 8 < K;
    if (more) {
      load_a(k0 + 8, ra);
      load_b(k0 + 8, rb);
    }
    const int kmax = min(8, K - k0);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      if (kk < kmax) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[buf][kk][ty + 8 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kk][tx + 8 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a[i], b[j]));
      }
    }
    if (more) {
      store(buf ^ 1, ra, rb);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gm = m0 + ty + 8 * i, gn = n0 + tx + 8 * j;
      if (gm < M && gn < N) {
        if (!isfinite(acc[i][j])) bad |= kFlagBwdOutput;
        C[(int64_t)gm * ldc + gn] = acc[i][j];
      }
    }
  if (bad && flag) atomicOr(flag, bad);
}

// BT[k] = B[k]^T for nblk square b x b blocks (the bh backward multiplies by
// B_g^T through the coalesced non-transposed row kernel)
__global__ void blocks_transpose_kernel(const double* __restrict__ B, double* __restrict__ BT,
                                        int64_t nblk, int b) {
  const int64_t bb = (int64_t)b * b;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nblk * bb;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = q / bb;
    const int r = int((q - k * bb) / b), cc = int(q - k * bb - (int64_t)r * b);
    BT[k * bb + (int64_t)cc * b + r] = B[q];
  }
}

// out[j] = sum_i A[i][j] * G[i][j], i ascending from 0.0 (the reference's
// per-row accumulation of ga / gd, projection.cpp:345-356)
__global__ void __launch_bounds__(32) colsum_prod_kernel(const double* __restrict__ A,
                                                         const double* __restrict__ G, int64_t n, int D,
                                                         double* __restrict__ out) {
  // out[j] = sum_i A[i][j] * G[i][j], i ascending from 0.0 with separate
  // multiply and add (the reference's order).  Only the D columns are
  // independent, so each thread keeps the next U rows' operands in flight
  // (double-buffered registers) while it folds the current U in order.
  constexpr int U = 16;
  const int j = blockIdx.x * 32 + threadIdx.x;
  if (j >= D) return;
  double a[U], g[U], an[U], gn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    a[u] = u < n ? A[(int64_t)u * D + j] : 0.0;
    g[u] = u < n ? G[(int64_t)u * D + j] : 0.0;
  }
  double acc = 0.0;
  for (int64_t i0 = 0; i0 < n; i0 += U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + U + u;
      an[u] = i < n ? A[i * D + j] : 0.0;
      gn[u] = i < n ? G[i * D + j] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u < n) acc = __dadd_rn(acc, __dmul_rn(a[u], g[u]));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = an[u];
      g[u] = gn[u];
    }
  }
  out[j] = acc;
}

// in-place FWHT of every row (fwht.hpp:28-41), K1's phases in shared memory
template <int LOGE, int NT = 256, int MINB = 1, int LOGD = 0>
__global__ void __launch_bounds__(NT, MINB) rows_fwht_kernel(HashParams p, double* __restrict__ V) {
  extern __shared__ double smem[];
  const int tpt = LOGD > 0 ? (1 << (LOGD - LOGE)) : p.threads_per_token;
  const int slot = threadIdx.x / tpt;
  const int t = threadIdx.x - slot * tpt;
  const int64_t token = (int64_t)blockIdx.x * p.tokens_per_block + slot;
  const bool active = slot < p.tokens_per_block && token < p.n;
  const int logD = LOGD > 0 ? LOGD : p.logD;
  const int D = 1 << logD;
  double* sm = smem + (size_t)slot * padded_len(D);
  int bad = 0;
  auto token_sync = [&]() {
    if (tpt <= 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(slot + 1), "r"(tpt) : "memory");
  };
  if (active)
    for (int a = t; a < D; a += tpt) sm[spos(a)] = V[token * D + a];
  token_sync();
  int nph = 1;
  if constexpr (LOGE > 0) nph = (logD + LOGE - 1) / LOGE;
  if (active) phase_smem<LOGE, LOGE, false, kPreNone>(sm, t, tpt, 0, p, 0, nullptr, bad, false);
  token_sync();
  const int nphc = LOGD > 0 ? (LOGD + LOGE - 1) / LOGE : nph;
#pragma unroll
  for (int ph = 1; ph < nphc; ++ph) {
    if (active) run_later_phase<LOGE>(sm, t, tpt, ph * LOGE, min(LOGE, logD - ph * LOGE), p, 0, bad, false);
    token_sync();
  }
  if (active)
    for (int a = t; a < D; a += tpt) V[token * D + a] = sm[spos(a)];
}

}  // namespace lffn_gpu
