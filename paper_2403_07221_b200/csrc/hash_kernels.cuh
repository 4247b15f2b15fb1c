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
//
// Data movement: each token's D-vector lives in shared memory (padded one
// double per 64).  A thread owns E = min(64, D) elements; a "phase" loads
// them, applies up to log2(E) consecutive butterfly stages in registers and
// stores them back, so a D = 2048 transform is two shared-memory round trips
// (bits 0-5, then bits 6-10) and D = 4096 is two as well.  Both access
// patterns (64 consecutive elements per thread; consecutive elements across
// threads) are bank-conflict free with the 65-double stride.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "checked.cuh"

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

constexpr int kMaxLogE = 6;

// Padded shared-memory position: two spare doubles per 64 elements.  A
// thread's 64 consecutive elements (phase 0) then start 66 doubles apart
// (16-byte aligned, conflict-free 128-bit accesses per quarter warp), and
// element pairs (a, a+1) stay adjacent for the later phases.
__device__ __forceinline__ int spos(int a) { return a + 2 * (a >> 6); }
__host__ __device__ constexpr int padded_len(int D) { return D + 2 * (D >> 6); }

// Multiply by -1.0 when bit `sh` of m is set -- exact, and equal to the
// reference's buf[j] *= sv[j] with sv = -1.0 (including 0.0 -> -0.0): the
// sign bit of the high word is XORed with the mask bit moved to bit 31.
__device__ __forceinline__ double flip_sign(double v, uint32_t m, int sh) {
  const int hi = __double2hiint(v) ^ (int)((m << (31 - sh)) & 0x80000000u);
  return __hiloint2double(hi, __double2loint(v));
}

// B consecutive transform bits applied to E/2^B register groups of 2^B.
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

// Shared-memory traffic of one phase over transform bits [lo, lo+B): the
// thread's E = 2^LOGE registers are J = E/2^B groups g = grp + J*t of 2^B
// elements a = glow | i << lo | ghigh << (lo+B) (glow = g mod 2^lo).  Every
// position is base[grp] + i * stride, and consecutive groups (grp, grp+1)
// are adjacent doubles, so the traffic is 128-bit LDS/STS pairs.
template <int LOGE, int B, bool STORE>
__device__ __forceinline__ void phase_io(double* sm, double (&v)[1 << LOGE], int t, int lo) {
  constexpr int E = 1 << LOGE;
  constexpr int G = 1 << B;
  constexpr int J = E / G;
  if (lo == 0) {
    // phase 0 (J == 1): elements t*E .. t*E + E-1, contiguous after padding
    if constexpr (J == 1) {
      double* q = sm + spos(t * E);
      if constexpr (E >= 2) {
#pragma unroll
        for (int i = 0; i < E; i += 2) {
          double2* d = reinterpret_cast<double2*>(q + i);
          if constexpr (STORE) *d = make_double2(v[i], v[i + 1]);
          else { const double2 w = *d; v[i] = w.x; v[i + 1] = w.y; }
        }
      } else {
        if constexpr (STORE) q[0] = v[0];
        else v[0] = q[0];
      }
    }
    return;
  }
  if (lo >= 6) {
    // the padding term is linear in i: position = base + i * stride
    const int stride = (1 << lo) + (1 << (lo - 5));
    if constexpr (J == 1) {
      const int glow = t & ((1 << lo) - 1);
      const int base = glow + 2 * (glow >> 6) + (t >> lo) * ((1 << (lo + B)) + (1 << (lo + B - 5)));
#pragma unroll
      for (int i = 0; i < G; ++i) {
        if constexpr (STORE) sm[base + i * stride] = v[i];
        else v[i] = sm[base + i * stride];
      }
    } else {
#pragma unroll
      for (int grp = 0; grp < J; grp += 2) {
        const int g = grp + J * t;
        const int glow = g & ((1 << lo) - 1);
        const int base = glow + 2 * (glow >> 6) + (g >> lo) * ((1 << (lo + B)) + (1 << (lo + B - 5)));
#pragma unroll
        for (int i = 0; i < G; ++i) {
          double2* d = reinterpret_cast<double2*>(sm + base + i * stride);
          if constexpr (STORE) *d = make_double2(v[grp * G + i], v[(grp + 1) * G + i]);
          else { const double2 w = *d; v[grp * G + i] = w.x; v[(grp + 1) * G + i] = w.y; }
        }
      }
    }
    return;
  }
  // 0 < lo < 6 (LOGE < 6 with several phases): generic positions
#pragma unroll
  for (int grp = 0; grp < J; ++grp) {
    const int g = grp + J * t;
    const int glow = g & ((1 << lo) - 1);
    const int ghigh = g >> lo;
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int pos = spos(glow | (i << lo) | (ghigh << (lo + B)));
      if constexpr (STORE) sm[pos] = v[grp * G + i];
      else v[grp * G + i] = sm[pos];
    }
  }
}

enum : int { kPreNone = 0, kPreSign = 1, kPreDiag = 2 };

// One phase over transform bits [lo, lo+B).  SRC_X: the token's inputs come
// straight from x (very first phase); PRE: the elementwise factor applied
// before a transform (signflip sign flip / acdc diagonal), phase 0 only.
template <int LOGE, int B, bool SRC_X, int PRE>
__device__ __forceinline__ void phase_smem(double* sm, int t, int tpt, int lo, const HashParams& p,
                                           int tr, const float* xr, int& bad, bool last) {
  constexpr int E = 1 << LOGE;
  constexpr int G = 1 << B;
  double v[E];
  if constexpr (SRC_X) {
    // pad x to D (projection.cpp:212-213), fp32 -> fp64 exactly (lo == 0:
    // this thread's elements are t*E .. t*E+E-1)
    if (t * E + E <= p.d_in && (p.d_in & 3) == 0) {
#pragma unroll
      for (int r = 0; r < E; r += 4) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(xr + t * E + r));
        if (!isfinite(f.x) || !isfinite(f.y) || !isfinite(f.z) || !isfinite(f.w)) bad |= 1;
        v[r] = (double)f.x;
        v[r + 1] = (double)f.y;
        v[r + 2] = (double)f.z;
        v[r + 3] = (double)f.w;
      }
    } else if (t * E >= p.d_in) {
      // all padding (projection.cpp:212-213): no loads, no checks -- keeps
      // the warp's threads past d_in out of the per-element path
#pragma unroll
      for (int r = 0; r < E; ++r) v[r] = 0.0;
    } else {
      // fully unrolled: a dynamic index would move v[] to local memory
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const int a = t * E + r;
        double xv = 0.0;
        if (a < p.d_in) {
          const float f = __ldg(xr + a);
          if (!isfinite(f)) bad |= 1;
          xv = (double)f;
        }
        v[r] = xv;
      }
    }
  } else {
    phase_io<LOGE, B, false>(sm, v, t, lo);
  }
  if constexpr (PRE == kPreSign) {
    const int words = (p.D + 31) >> 5;
    const uint32_t* mw = p.signmask + tr * words;
#pragma unroll
    for (int r0 = 0; r0 < E; r0 += 32) {
      const int a0 = t * E + r0;
      const uint32_t m = __ldg(mw + (a0 >> 5)) >> (a0 & 31);
#pragma unroll
      for (int r = r0; r < r0 + 32 && r < E; ++r) v[r] = flip_sign(v[r], m, r - r0);
    }
  } else if constexpr (PRE == kPreDiag) {
    const double* dg = p.diag + (size_t)tr * p.D + t * E;
#pragma unroll
    for (int r = 0; r < E; ++r) v[r] = __dmul_rn(v[r], __ldg(dg + r));
  }
  butterfly_groups<LOGE, B>(v);
  if (last && p.code_width == p.D) {
    // finiteness of the projection output (projection.cpp:264,
    // lookup.cpp:204) on the registers: some exponent field all ones
    uint32_t m = 0xffffffffu;
#pragma unroll
    for (int r = 0; r < E; ++r) m = min(m, (uint32_t)(__double2hiint(v[r]) & 0x7ff00000) ^ 0x7ff00000u);
    if (m == 0u) bad |= 2;
  }
  phase_io<LOGE, B, true>(sm, v, t, lo);
}

// Phase 0 of transform tr (bits [0, LOGE)) -- the pre-factor phase.
template <int LOGE, int PRE>
__device__ __forceinline__ void run_first_phase(double* sm, int t, int tpt, const HashParams& p,
                                                int tr, const float* xr, int& bad, bool last) {
  if (tr == 0) phase_smem<LOGE, LOGE, true, PRE>(sm, t, tpt, 0, p, tr, xr, bad, last);
  else phase_smem<LOGE, LOGE, false, PRE>(sm, t, tpt, 0, p, tr, xr, bad, last);
}

// Later phases (bits [lo, lo+b), b <= LOGE).
template <int LOGE>
__device__ __forceinline__ void run_later_phase(double* sm, int t, int tpt, int lo, int b,
                                                const HashParams& p, int tr, int& bad, bool last) {
  if constexpr (LOGE >= 6) { if (b == 6) { phase_smem<LOGE, 6, false, kPreNone>(sm, t, tpt, lo, p, tr, nullptr, bad, last); return; } }
  if constexpr (LOGE >= 5) { if (b == 5) { phase_smem<LOGE, 5, false, kPreNone>(sm, t, tpt, lo, p, tr, nullptr, bad, last); return; } }
  if constexpr (LOGE >= 4) { if (b == 4) { phase_smem<LOGE, 4, false, kPreNone>(sm, t, tpt, lo, p, tr, nullptr, bad, last); return; } }
  if constexpr (LOGE >= 3) { if (b == 3) { phase_smem<LOGE, 3, false, kPreNone>(sm, t, tpt, lo, p, tr, nullptr, bad, last); return; } }
  if constexpr (LOGE >= 2) { if (b == 2) { phase_smem<LOGE, 2, false, kPreNone>(sm, t, tpt, lo, p, tr, nullptr, bad, last); return; } }
  if constexpr (LOGE >= 1) { if (b == 1) { phase_smem<LOGE, 1, false, kPreNone>(sm, t, tpt, lo, p, tr, nullptr, bad, last); return; } }
}

// 1 + exp(-2a), kept out of line: it is needed only for |z| < 18.5 (rare
// for the unnormalised transforms), and inlining it per coordinate bloats
// the kernel past the instruction cache.
__device__ __noinline__ double one_plus_exp_m2(double a) { return __dadd_rn(1.0, exp(-2.0 * a)); }

// K1 for structured projections (signflip, acdc) and the epilogue of the
// dense projection (z_in given).
// KIND: kPreSign (signflip), kPreDiag (acdc), kPreNone (dense epilogue on z_in).
// LOGD > 0 fixes the transform width at compile time (with TR > 0 the
// transform count): every phase's shared-memory geometry then folds into
// constants, which removes most of the integer work around the butterflies.
template <int LOGE, int KIND, int NT = 256, int MINB = 1, int LOGD = 0, int TR = 0>
__global__ void __launch_bounds__(NT, MINB) hash_structured_kernel(HashParams p) {
  extern __shared__ double smem[];
  constexpr int E = 1 << LOGE;
  const int logD = LOGD > 0 ? LOGD : p.logD;
  const int ntr = TR > 0 ? TR : p.n_transforms;
  const int tpt = LOGD > 0 ? (1 << (LOGD - LOGE)) : p.threads_per_token;
  const int slot = threadIdx.x / tpt;
  const int t = threadIdx.x - slot * tpt;
  const int64_t token = (int64_t)blockIdx.x * p.tokens_per_block + slot;
  const bool active = slot < p.tokens_per_block && token < p.n;
  const int D = 1 << logD;
  double* sm = smem + (size_t)slot * padded_len(D);
  int bad = 0;

  // Only the threads of one token share its vector, so phases synchronise
  // per token: the warp when a token fits in one, else a named barrier.
  auto token_sync = [&]() {
    if (tpt <= 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(slot + 1), "r"(tpt) : "memory");
  };

  if constexpr (KIND == kPreNone) {
    // dense: z already computed; stage the token's z row into smem
    if (active)
      for (int a = t; a < p.code_width; a += tpt) sm[spos(a)] = p.z_in[token * p.code_width + a];
    token_sync();
  } else {
    const float* xr = p.x + token * (int64_t)p.d_in;
    int nph = 1;
    if constexpr (LOGE > 0) nph = (logD + LOGE - 1) / LOGE;
#pragma unroll 1
    for (int tr = 0; tr < ntr; ++tr) {
      const bool last_tr = tr == ntr - 1;
      if (active) run_first_phase<LOGE, KIND>(sm, t, tpt, p, tr, xr, bad, last_tr && nph == 1);
      token_sync();
      const int nphc = LOGD > 0 ? (LOGD + LOGE - 1) / LOGE : nph;
#pragma unroll
      for (int ph = 1; ph < nphc; ++ph) {
        const int lo = ph * LOGE;
        if (active)
          run_later_phase<LOGE>(sm, t, tpt, lo, min(LOGE, logD - lo), p, tr, bad,
                                last_tr && ph == nph - 1);
        token_sync();
      }
    }
  }

  if (active) {
    if (p.z_out || KIND == kPreNone || p.code_width != p.D) {
      // finiteness of the first h*tau outputs (projection.cpp:264,
      // lookup.cpp:204) when the registers did not cover exactly them, and
      // the optional z copy-out (coalesced)
      for (int a = t; a < p.code_width; a += tpt) {
        const double zv = sm[spos(a)];
        if (!isfinite(zv)) bad |= 2;
        if (p.z_out) p.z_out[token * p.code_width + a] = zv;
      }
    }
    // each table is finished by the thread whose element range holds its
    // first coordinate (neighbouring threads read 66 doubles apart: no bank
    // conflicts)
    const int tau = p.tau;
    const int hl = p.ke - p.kb;
    const int a_lo = t * E;
    const int a_hi = min(a_lo + E, p.code_width);
    // (a 64-coordinate integer fast path -- sign bits and |z| >= 18.5 from
    // the high words, exact path only for tables with a small |z| --
    // measured slower than this loop: c2 0.162 vs 0.150 ms)
    for (int k = max((a_lo + tau - 1) / tau, p.kb); k < p.ke && k * tau < a_hi; ++k) {
      const int base = k * tau;
      uint32_t code = 0;
      bool small = false;
      double sum_abs = 0.0;
#pragma unroll 4
      for (int j = 0; j < tau; ++j) {
        const double zj = sm[spos(base + j)];
        code |= (zj >= 0.0 ? 1u : 0u) << j;
        const double az = fabs(zj);
        small |= az < 18.5;
        sum_abs = __dadd_rn(sum_abs, az);
      }
      double w = 1.0;
      if (small) {
        // 1 + exp(-2a) == 1.0 exactly once exp(-2a) <= 2^-53 (a >= 18.37),
        // so only coordinates with a < 18.5 divide; same order as the
        // reference's w /= 1 + exp(-2|z_j|) (lookup.cpp:185-189)
        for (int j = 0; j < tau; ++j) {
          const double az = fabs(sm[spos(base + j)]);
          if (az < 18.5) w = __ddiv_rn(w, one_plus_exp_m2(az));
        }
      }
      LFFN_DCHECK(k - p.kb < hl && base + tau <= p.code_width);
      p.codes[token * hl + (k - p.kb)] = code;
      p.coeff[token * hl + (k - p.kb)] = (float)(p.scaled ? __dmul_rn(w, sum_abs) : w);
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
