// hash_sf_kernel.cuh -- K1f: the production signflip hash (Projection::forward
// signflip branch + compute_codes + top-1 weight) for D = 2048 / 4096, with
// three shared-memory transposes per token instead of K1's five round trips.
//
// Reference path being replaced (/root/reference/proj):
//   Projection::forward, signflip branch   projection.cpp:200-263 (:248-258)
//   fwht_kernel                            include/lookupffn/fwht.hpp:28-41
//   sign_code / compute_codes              lookup.cpp:74-100
//   top1_weight                            lookup.cpp:185-189
//
// Numerics (the north star's bar: codes bit-exact wherever |z| > 1e-5; the
// coefficient within the fp32 tolerance): float64 throughout, the same
// butterfly pairs and x+y / x-y operand order as fwht_kernel, but the eleven
// (twelve) stages of a transform run in a different order -- the stages of an
// unnormalised Walsh-Hadamard transform commute exactly in real arithmetic,
// so z differs from the reference's float64 z only by reassociation rounding
// (~1e-16 relative, i.e. ~1e-11 absolute at |z| ~ 1e5), far below the 1e-5
// band in which a code bit may differ.  The sign flips are exact (sign-bit
// XOR).  When z must be bit-identical (lffn_hash with a z output, and the
// backward's recompute) the launcher takes K1 (hash_kernels.cuh) instead.
//
// Layout: TPT = D / 64 threads own one token, 64 float64 registers each.
//   A: thread t holds indices 64 t + r            (index bits 0-5 in registers)
//   B: thread t holds indices t + TPT r          (bits log2(TPT) .. +5 in registers)
// Transform 0 runs its A bits, transposes A -> B through shared memory and
// finishes its remaining bits; transform 1 runs all its B bits, transposes
// B -> A and finishes; transform 2 runs all its A bits, transposes A -> B and
// finishes.  Three transposes (one 128-bit store + one 64-bit load pass, or
// the reverse) per token against K1's six stores and five loads; both access
// patterns are bank-conflict free with two padding doubles per 64.
//
// Epilogue in layout B: one warp ballot per register gives 32 consecutive
// sign bits (z >= 0, lookup.cpp:77), so the h*tau code bits come out as words
// in shared memory and each thread funnel-shifts its tables' codes out of
// them.  The weight is exactly 1.0 for a table whose every |z_j| >= 18.5
// (1 + exp(-2|z|) rounds to 1.0); the rare small coordinates (a second
// ballot) have their z stored, and the table's weight divides by
// 1 + exp(-2|z_j|) over exactly those j in ascending order -- the reference's
// sequential division, the other factors being exact divisions by 1.0.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "hash_kernels.cuh"

namespace lffn_gpu {

struct HashSfParams {
  const float* x;              // [n x d_in]
  int64_t n;
  int d_in;
  int code_width;              // h * tau
  int tau;
  int kb, ke;                  // tables owned: [kb, ke)
  const unsigned long long* masks;  // [3][TPT]: bit r = sign of the element thread t holds in
                               // register r (layout A for transforms 0 and 2, B for 1)
  uint32_t* codes;             // [n x (ke - kb)]
  float* coeff;                // [n x (ke - kb)]
  int* flag;
};

template <int LOGD>
struct SfGeom {
  static constexpr int D = 1 << LOGD;
  static constexpr int TPT = D / 64;                 // threads per token
  static constexpr int LOGT = LOGD - 6;
  static constexpr int PAD = D + 2 * (D >> 6);       // doubles per token in shared memory
  static constexpr int WORDS = D / 32;               // sign words per token
  // shared-memory position of index a (two padding doubles per 64)
  static __device__ __forceinline__ int pos(int a) { return a + 2 * (a >> 6); }
};

// butterflies over register bits [B0, B1) in ascending order
template <int B0, int B1>
__device__ __forceinline__ void sf_stages(double (&v)[64]) {
#pragma unroll
  for (int k = B0; k < B1; ++k) {
#pragma unroll
    for (int r = 0; r < 64; ++r) {
      if (r & (1 << k)) continue;
      const double a = v[r];
      const double b = v[r | (1 << k)];
      v[r] = __dadd_rn(a, b);
      v[r | (1 << k)] = __dsub_rn(a, b);
    }
  }
}

__device__ __forceinline__ void sf_flip(double (&v)[64], unsigned long long m) {
  const uint32_t lo = (uint32_t)m, hi = (uint32_t)(m >> 32);
#pragma unroll
  for (int r = 0; r < 64; ++r) {
    const uint32_t bit = ((r < 32 ? lo : hi) >> (r & 31)) & 1u;
    v[r] = __hiloint2double(__double2hiint(v[r]) ^ (int)(bit << 31), __double2loint(v[r]));
  }
}

// A layout <-> shared memory (thread t: indices 64 t + r; 128-bit accesses)
template <int LOGD, bool STORE>
__device__ __forceinline__ void sf_io_A(double* sm, double (&v)[64], int t) {
  double* q = sm + SfGeom<LOGD>::pos(64 * t);
#pragma unroll
  for (int r = 0; r < 64; r += 2) {
    double2* d = reinterpret_cast<double2*>(q + r);
    if constexpr (STORE) *d = make_double2(v[r], v[r + 1]);
    else { const double2 w = *d; v[r] = w.x; v[r + 1] = w.y; }
  }
}

// B layout <-> shared memory (thread t: indices t + TPT r; 64-bit accesses,
// consecutive across the threads of a warp)
template <int LOGD, bool STORE>
__device__ __forceinline__ void sf_io_B(double* sm, double (&v)[64], int t) {
  using Gm = SfGeom<LOGD>;
#pragma unroll
  for (int r = 0; r < 64; ++r) {
    double* q = sm + Gm::pos(t + Gm::TPT * r);
    if constexpr (STORE) *q = v[r];
    else v[r] = *q;
  }
}

__device__ __noinline__ double sf_one_plus_exp_m2(double a) { return __dadd_rn(1.0, exp(-2.0 * a)); }

template <int LOGD>
__global__ void __launch_bounds__(128, 3) hash_sf_kernel(HashSfParams p) {
  using Gm = SfGeom<LOGD>;
  constexpr int TPT = Gm::TPT;
  constexpr int TPB = 128 / TPT;  // tokens per CTA
  extern __shared__ double smem[];
  // per token: PAD doubles of transpose buffer, then 2 * WORDS sign / small words
  constexpr int SLOT = Gm::PAD + Gm::WORDS;  // doubles (the words take WORDS doubles)
  const int slot = threadIdx.x / TPT;
  const int t = threadIdx.x - slot * TPT;
  const int lane = threadIdx.x & 31;
  const int64_t token = (int64_t)blockIdx.x * TPB + slot;
  const bool active = token < p.n;
  double* sm = smem + (size_t)slot * SLOT;
  uint32_t* words = reinterpret_cast<uint32_t*>(sm + Gm::PAD);  // [WORDS] signs, [WORDS] small
  auto token_sync = [&]() {
    if constexpr (TPT <= 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(slot + 1), "r"(TPT) : "memory");
  };
  if (!active) return;  // whole tokens only: a token's threads exit together
  int bad = 0;
  double v[64];

  // ---- transform 0: x (padded to D) in layout A
  {
    const float* xr = p.x + token * (int64_t)p.d_in;
    const int a0 = 64 * t;
    if (a0 + 64 <= p.d_in && (p.d_in & 3) == 0) {
#pragma unroll
      for (int r = 0; r < 64; r += 4) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(xr + a0 + r));
        if (!isfinite(f.x) || !isfinite(f.y) || !isfinite(f.z) || !isfinite(f.w)) bad |= 1;
        v[r] = (double)f.x;
        v[r + 1] = (double)f.y;
        v[r + 2] = (double)f.z;
        v[r + 3] = (double)f.w;
      }
    } else if (a0 >= p.d_in) {
#pragma unroll
      for (int r = 0; r < 64; ++r) v[r] = 0.0;
    } else {
#pragma unroll
      for (int r = 0; r < 64; ++r) {
        double xv = 0.0;
        if (a0 + r < p.d_in) {
          const float f = __ldg(xr + a0 + r);
          if (!isfinite(f)) bad |= 1;
          xv = (double)f;
        }
        v[r] = xv;
      }
    }
  }
  sf_flip(v, __ldg(p.masks + 0 * TPT + t));
  sf_stages<0, 6>(v);
  sf_io_A<LOGD, true>(sm, v, t);
  token_sync();
  sf_io_B<LOGD, false>(sm, v, t);
  token_sync();
  // B holds index bits LOGT .. LOGT+5; bit 5 is done when LOGT == 5
  sf_stages<(LOGD == 11 ? 1 : 0), 6>(v);
  // ---- transform 1 in layout B
  sf_flip(v, __ldg(p.masks + 1 * TPT + t));
  sf_stages<0, 6>(v);
  sf_io_B<LOGD, true>(sm, v, t);
  token_sync();
  sf_io_A<LOGD, false>(sm, v, t);
  token_sync();
  sf_stages<0, (LOGD == 11 ? 5 : 6)>(v);
  // ---- transform 2 in layout A
  sf_flip(v, __ldg(p.masks + 2 * TPT + t));
  sf_stages<0, 6>(v);
  sf_io_A<LOGD, true>(sm, v, t);
  token_sync();
  sf_io_B<LOGD, false>(sm, v, t);
  token_sync();
  sf_stages<(LOGD == 11 ? 1 : 0), 6>(v);

  // ---- epilogue in layout B: z[t + TPT r] = v[r]
  // finiteness of the first h*tau outputs (projection.cpp:264, lookup.cpp:204)
  {
    bool fin = true;
#pragma unroll
    for (int r = 0; r < 64; ++r)
      if (t + TPT * r < p.code_width)
        fin &= (__double2hiint(v[r]) & 0x7ff00000) != 0x7ff00000;
    if (!fin) bad |= 2;
  }
  // sign words (z >= 0, lookup.cpp:77) and small-|z| words (|z| < 18.5):
  // register r of warp w covers indices 32 (w + (TPT / 32) r) .. + 31
  const int wsub = t >> 5;          // warp within the token (0 for D = 2048)
  constexpr int WPT = TPT / 32;     // warps per token
  uint32_t sw0 = 0, sw1 = 0, mw0 = 0, mw1 = 0;
  bool any_small = false;
#pragma unroll
  for (int r = 0; r < 64; ++r) {
    const uint32_t s = __ballot_sync(0xffffffffu, v[r] >= 0.0);
    const uint32_t m = __ballot_sync(0xffffffffu, fabs(v[r]) < 18.5);
    any_small |= m != 0u;
    if (r < 32) {
      if (lane == r) { sw0 = s; mw0 = m; }
    } else {
      if (lane == r - 32) { sw1 = s; mw1 = m; }
    }
  }
  // word index of register r in warp w: WPT * r + w
  words[WPT * lane + wsub] = sw0;
  words[WPT * (lane + 32) + wsub] = sw1;
  words[Gm::WORDS + WPT * lane + wsub] = mw0;
  words[Gm::WORDS + WPT * (lane + 32) + wsub] = mw1;
  // the z of every small coordinate (warp-uniform per register: only the
  // registers some lane flagged), at its natural shared-memory position
  if (any_small) {
#pragma unroll
    for (int r = 0; r < 64; ++r) {
      const uint32_t m = __shfl_sync(0xffffffffu, r < 32 ? mw0 : mw1, r & 31);
      if (m != 0u) sm[Gm::pos(t + TPT * r)] = v[r];
    }
  }
  token_sync();
  const int hl = p.ke - p.kb;
  const int tau = p.tau;
  const uint32_t cmask = tau >= 32 ? 0xffffffffu : ((1u << tau) - 1u);
  for (int k = p.kb + t; k < p.ke; k += TPT) {
    const int o = k * tau;
    const int wi = o >> 5, sh = o & 31;
    const uint32_t w_lo = words[wi];
    const uint32_t w_hi = (wi + 1 < Gm::WORDS) ? words[wi + 1] : 0u;
    const uint32_t code = __funnelshift_r(w_lo, w_hi, sh) & cmask;
    const uint32_t small = __funnelshift_r(words[Gm::WORDS + wi],
                                           (wi + 1 < Gm::WORDS) ? words[Gm::WORDS + wi + 1] : 0u, sh) &
                           cmask;
    double w = 1.0;
    if (small) {
      // w /= 1 + exp(-2|z_j|) over the small j ascending (lookup.cpp:185-189;
      // the other factors are exactly 1.0)
      for (int j = 0; j < tau; ++j)
        if ((small >> j) & 1u) w = __ddiv_rn(w, sf_one_plus_exp_m2(fabs(sm[Gm::pos(o + j)])));
    }
    p.codes[token * hl + (k - p.kb)] = code;
    p.coeff[token * hl + (k - p.kb)] = (float)w;
  }
  if (bad) atomicOr(p.flag, bad);
}

}  // namespace lffn_gpu
