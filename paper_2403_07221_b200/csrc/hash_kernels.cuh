// hash_kernels.cuh -- K1: the fused hash stage (projection -> sign codes ->
// top-1 coefficients) for the structured projections, and the exact float64
// dense projection.
//
// Reference path being replaced (/root/reference/proj):
//   Projection::forward, signflip / acdc branches   projection.cpp:200-263
//   fwht_kernel (stage order half = 1, 2, 4, ...)    include/lookupffn/fwht.hpp:28-41
//   compute_codes / sign_code                         lookup.cpp:74-100
//   top1_weight, scaled numerator                     lookup.cpp:185-189, :241-253
//   lookup_hash_f32 + lookup_weights_f32              bench.cpp:115-180
//
// Numerics: the transform runs in float64 with exactly the reference's
// butterfly network (same pairs, same stage order, x+y / x-y operand order);
// the sign flips are exact (sign-bit XOR == multiply by +-1.0), so z is
// bit-identical to the reference's double Projection::forward.  Codes are
// therefore bit-exact; the coefficient differs from the reference only by
// the last-bit behaviour of the device exp().
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace lffn_gpu {

struct HashParams {
  const float* x;            // [n x d_in]
  int64_t n;
  int d_in;
  int D, logD;               // transform width (power of two) and log2
  int code_width;            // h * tau (projection d_out)
  int tau;
  int kb, ke;                // tables owned: [kb, ke)
  int scaled;                // scaled numerator (scaled / gelu-tau1)
  int n_transforms;          // signflip: 3; acdc: 2 * depth
  const uint32_t* signmask;  // signflip: n_transforms * ceil(D/32) words, bit set = -1
  const double* diag;        // acdc: n_transforms * D multipliers (else null)
  const double* z_in;        // dense: precomputed z [n x code_width] (else null)
  double* z_out;             // optional [n x code_width]
  uint32_t* codes;           // [n x (ke-kb)]
  float* coeff;              // [n x (ke-kb)]
  int* flag;
  int tokens_per_block;
  int threads_per_token;
};

// Padded shared-memory position: one spare double per 16 keeps both the
// contiguous (phase 0) and the strided (later phases) access patterns free
// of bank conflicts.
__device__ __forceinline__ int spos(int a) { return a + (a >> 4); }

__device__ __forceinline__ double flip_sign(double v, uint32_t bit) {
  // multiply by -1.0 when bit is set: exact, equal to the reference's
  // buf[j] *= sv[j] with sv = -1.0
  unsigned long long u = __double_as_longlong(v);
  u ^= (unsigned long long)bit << 63;
  return __longlong_as_double(u);
}

// One phase: B consecutive transform bits [lo, lo+B) applied to this
// thread's E = 2^LOGE elements held as E/2^B groups of 2^B.
template <int LOGE, int B>
__device__ __forceinline__ void butterfly_groups(double (&v)[1 << LOGE]) {
  constexpr int E = 1 << LOGE;
  constexpr int G = 1 << B;
#pragma unroll
  for (int grp = 0; grp < E / G; ++grp) {
#pragma unroll
    for (int half = 1; half < G; half <<= 1) {
#pragma unroll
      for (int blk = 0; blk < G; blk += 2 * half) {
#pragma unroll
        for (int j = blk; j < blk + half; ++j) {
          const double xx = v[grp * G + j];
          const double yy = v[grp * G + j + half];
          v[grp * G + j] = __dadd_rn(xx, yy);
          v[grp * G + j + half] = __dsub_rn(xx, yy);
        }
      }
    }
  }
}

// Element index of register slot r (group grp = r / G, member i = r % G) for
// thread t of a token in the phase with bits [lo, lo+B).
template <int B>
__device__ __forceinline__ int phase_index(int t, int tpt, int grp, int i, int lo) {
  const int g = t + grp * tpt;
  const int glow = g & ((1 << lo) - 1);
  const int ghigh = g >> lo;
  return glow | (i << lo) | (ghigh << (lo + B));
}

template <int LOGE, int B>
__device__ __forceinline__ void phase_smem(double* sm, int t, int tpt, int lo, bool first_of_tr,
                                           const HashParams& p, int tr) {
  constexpr int E = 1 << LOGE;
  constexpr int G = 1 << B;
  double v[E];
#pragma unroll
  for (int r = 0; r < E; ++r) v[r] = sm[spos(phase_index<B>(t, tpt, r / G, r % G, lo))];
  if (first_of_tr) {
    // phase 0 of a transform: lo == 0, B == LOGE, elements t*E .. t*E+E-1
    if (p.signmask) {
      const int words = (p.D + 31) >> 5;
      const int a0 = t * E;
      const uint32_t m = __ldg(p.signmask + tr * words + (a0 >> 5)) >> (a0 & 31);
#pragma unroll
      for (int r = 0; r < E; ++r) v[r] = flip_sign(v[r], (m >> r) & 1u);
    } else if (p.diag) {
      const double* dg = p.diag + (size_t)tr * p.D + t * E;
#pragma unroll
      for (int r = 0; r < E; ++r) v[r] = __dmul_rn(v[r], __ldg(dg + r));
    }
  }
  butterfly_groups<LOGE, B>(v);
#pragma unroll
  for (int r = 0; r < E; ++r) sm[spos(phase_index<B>(t, tpt, r / G, r % G, lo))] = v[r];
}

template <int LOGE>
__device__ __forceinline__ void run_phase(double* sm, int t, int tpt, int lo, int b,
                                          bool first_of_tr, const HashParams& p, int tr) {
  if constexpr (LOGE >= 4) { if (b == 4) { phase_smem<LOGE, 4>(sm, t, tpt, lo, first_of_tr, p, tr); return; } }
  if constexpr (LOGE >= 3) { if (b == 3) { phase_smem<LOGE, 3>(sm, t, tpt, lo, first_of_tr, p, tr); return; } }
  if constexpr (LOGE >= 2) { if (b == 2) { phase_smem<LOGE, 2>(sm, t, tpt, lo, first_of_tr, p, tr); return; } }
  if constexpr (LOGE >= 1) { if (b == 1) { phase_smem<LOGE, 1>(sm, t, tpt, lo, first_of_tr, p, tr); return; } }
  if (b == 0 && first_of_tr) phase_smem<LOGE, 0>(sm, t, tpt, lo, first_of_tr, p, tr);
}

// Codes + coefficient for one (token, table) from its tau soft-code
// coordinates (lookup.cpp:81-100, 185-189, 241-253).
__device__ __forceinline__ void code_and_coeff(const double* sm, int base, int tau, int scaled,
                                               uint32_t* code_out, float* coeff_out) {
  uint32_t code = 0;
  double w = 1.0, sum_abs = 0.0;
  for (int j = 0; j < tau; ++j) {
    const double zj = sm[spos(base + j)];
    if (zj >= 0.0) code |= (1u << j);
    const double a = fabs(zj);
    sum_abs = __dadd_rn(sum_abs, a);
    // 1 + exp(-2a) == 1.0 exactly once exp(-2a) <= 2^-53 (a >= 18.37):
    // dividing by 1.0 is then a no-op, so skipping the exp is exact.
    if (a < 18.5) w = __ddiv_rn(w, __dadd_rn(1.0, exp(-2.0 * a)));
  }
  *code_out = code;
  *coeff_out = (float)(scaled ? __dmul_rn(w, sum_abs) : w);
}

// K1 for structured projections (signflip, acdc) and the epilogue of the
// dense projection (z_in given): one CTA holds tokens_per_block token
// vectors of D doubles in shared memory; every phase loads 2^LOGE elements
// per thread, applies up to LOGE butterfly stages in registers and stores
// them back, so log2(D)/LOGE shared-memory round trips per transform.
template <int LOGE>
__global__ void __launch_bounds__(1024) hash_structured_kernel(HashParams p) {
  extern __shared__ double smem[];
  constexpr int E = 1 << LOGE;
  const int tpt = p.threads_per_token;
  const int slot = threadIdx.x / tpt;
  const int t = threadIdx.x - slot * tpt;
  const int64_t token = (int64_t)blockIdx.x * p.tokens_per_block + slot;
  const bool active = slot < p.tokens_per_block && token < p.n;
  const int D = p.D;
  double* sm = smem + (size_t)slot * (D + (D >> 4));
  int bad = 0;

  if (p.z_in) {
    // dense: z already computed; stage the token's z row into smem
    if (active)
      for (int a = t; a < p.code_width; a += tpt) sm[spos(a)] = p.z_in[token * p.code_width + a];
  } else if (active) {
    // pad x to D (projection.cpp:212-213), fp32 -> fp64 exactly
    const float* xr = p.x + token * (int64_t)p.d_in;
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int a = t * E + r;
      double v = 0.0;
      if (a < p.d_in) {
        const float xv = __ldg(xr + a);
        if (!isfinite(xv)) bad |= 1;
        v = (double)xv;
      }
      sm[spos(a)] = v;
    }
  }
  __syncthreads();

  if (!p.z_in) {
    int nph = 1;
    if constexpr (LOGE > 0) nph = (p.logD + LOGE - 1) / LOGE;
    for (int tr = 0; tr < p.n_transforms; ++tr) {
      for (int ph = 0; ph < nph; ++ph) {
        const int lo = ph * LOGE;
        const int b = min(LOGE, p.logD - lo);
        if (active) run_phase<LOGE>(sm, t, tpt, lo, b, ph == 0, p, tr);
        __syncthreads();
      }
    }
  }

  if (active) {
    // finiteness of the whole projection output (projection.cpp:264,
    // lookup.cpp:204) and the optional z copy-out
    for (int a = t; a < p.code_width; a += tpt) {
      const double zv = sm[spos(a)];
      if (!isfinite(zv)) bad |= 2;
      if (p.z_out) p.z_out[token * p.code_width + a] = zv;
    }
    const int hl = p.ke - p.kb;
    for (int k = p.kb + t; k < p.ke; k += tpt) {
      uint32_t code;
      float cf;
      code_and_coeff(sm, k * p.tau, p.tau, p.scaled, &code, &cf);
      p.codes[token * hl + (k - p.kb)] = code;
      p.coeff[token * hl + (k - p.kb)] = cf;
    }
  }
  if (bad) atomicOr(p.flag, bad);
}

// Exact float64 dense projection z = x W (projection.cpp:178-198): every
// output element is accumulated by one thread over k = 0..d_in-1 in order
// with separately rounded multiply and add (no FMA), which reproduces the
// reference's double result bit for bit.  64x64 output tile per CTA, 4x4
// per thread, x/W tiles staged through shared memory.
__global__ void __launch_bounds__(256) dense_proj_f64_kernel(const float* __restrict__ x,
                                                             const double* __restrict__ W,
                                                             double* __restrict__ z, int64_t n,
                                                             int d_in, int d_out, int* flag) {
  __shared__ double xs[16][64 + 1];
  __shared__ double ws[16][64];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t row0 = (int64_t)blockIdx.y * 64;
  const int col0 = blockIdx.x * 64;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  int bad = 0;
  for (int k0 = 0; k0 < d_in; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk = e & 15, r = e >> 4;
      const int64_t gr = row0 + r;
      double v = 0.0;
      if (gr < n && k0 + kk < d_in) {
        const float xv = x[gr * d_in + k0 + kk];
        if (!isfinite(xv)) bad |= 1;
        v = (double)xv;
      }
      xs[kk][r] = v;
    }
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int c = e & 63, kk = e >> 6;
      const int gc = col0 + c;
      ws[kk][c] = (k0 + kk < d_in && gc < d_out) ? W[(int64_t)(k0 + kk) * d_out + gc] : 0.0;
    }
    __syncthreads();
    const int kmax = min(16, d_in - k0);
    for (int kk = 0; kk < kmax; ++kk) {
      double xv[4], wv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = xs[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) wv[j] = ws[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(xv[i], wv[j]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gr = row0 + ty * 4 + i;
    if (gr >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gc = col0 + tx + 16 * j;
      if (gc < d_out) z[gr * d_out + gc] = acc[i][j];
    }
  }
  if (bad) atomicOr(flag, bad);
}

}  // namespace lffn_gpu
