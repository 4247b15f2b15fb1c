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
//   B: thread t, register q holds index t + TPT q    (the high index bits in registers)
//   A: thread t, register q holds index 64 t + pi(q) (64 consecutive indices;
//      pi(q) = 32 (q & 1) + (q >> 1) for D = 2048, pi(q) = q for D = 4096)
// Every transform runs the same code: sign flip, butterflies over the six
// register bits, one transpose through shared memory (64-bit stores at
// position t + TPT q, 128-bit loads of positions 64 t + pi(q); both
// bank-conflict free with two padding doubles per 64), butterflies over the
// register bits the transpose brought in (q bits 1-5 for D = 2048, where
// register bit 0 -- index bit 5 -- stays in the registers; all six for D =
// 4096).  The transpose is an involution on (thread, register), so the
// layouts alternate B, A, B, A: x is loaded in layout B (coalesced: lane t
// reads x[t + TPT q]) and the third transform ends in layout A.
//
// Zero padding: in layout B the padded coordinates (index >= d_in) are whole
// registers q >= ceil(d_in / TPT), the same in every thread.  The kernel is
// instantiated per LIVE (live registers, a multiple of 8): the first
// transform's first butterflies skip pairs of zeros and turn (x, 0) pairs
// into copies (x + 0 and x - 0 are exact), the loads, conversions and sign
// flips touch live registers only -- at c2 (d_in = 768 of 2048) 120 instead
// of 384 float64 adds in that phase, at c3 (1024 of 2048) 160.
//
// Epilogue in layout A: a thread's 64 registers are 64 consecutive
// coordinates, so its sign bits (z >= 0, lookup.cpp:77) form two words of the
// h*tau code bits in shared memory, from which each thread funnel-shifts its
// tables' codes.  The common case is integer-only: the sign bits of the high
// words are funnelled into the two words, and an unsigned min / max over the
// doubled high words (|z| without its sign) tells whether any coordinate is
// small (|z| < 18.5, which includes the -0.0 whose sign bit must not count)
// or non-finite.  Only then the float64 compares run.  The weight is exactly
// 1.0 for a table whose every |z_j| >= 18.5 (1 + exp(-2|z|) rounds to 1.0);
// the rare small coordinates have their z stored, and the table's weight
// divides by 1 + exp(-2|z_j|) over exactly those j in ascending order -- the
// reference's sequential division, the other factors being exact divisions
// by 1.0.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "checked.cuh"
#include "hash_kernels.cuh"

namespace lffn_gpu {

struct HashSfParams {
  const float* x;              // [n x d_in]
  int64_t n;
  int d_in;
  int code_width;              // h * tau
  int tau;
  int kb, ke;                  // tables owned: [kb, ke)
  int transforms;              // 3 (Projection::forward signflip: H S2 H S1 H S0)
  const unsigned long long* masks;  // [3][TPT]: bit r = sign of the element thread t holds in
                               // register r at the start of transform tr (sf_layout_index)
  uint32_t* codes;             // [n x (ke - kb)]
  float* coeff;                // [n x (ke - kb)]
  int* flag;
};

// threads per CTA: 64 (six CTAs, twelve warps per SM at 168 registers).  Measured
// c2 / c3 / c4: 128 threads 0.100 / 0.346 / 0.127 ms, 64 threads 0.098 /
// 0.338 / 0.119 ms, one token per CTA 0.098 / 0.346 / 0.119 ms; a persistent
// grid-stride loop over tokens (all warps in the same phase at the same
// time) 0.125 / 0.442 / 0.148 ms.
__host__ __device__ constexpr int sf_threads(int) { return 64; }

template <int LOGD>
struct SfGeom {
  static constexpr int D = 1 << LOGD;
  static constexpr int TPT = D / 64;                 // threads per token
  static constexpr int LOGT = LOGD - 6;
  static constexpr int PAD = D + 2 * (D >> 6);       // doubles per token in shared memory
  static constexpr int WORDS = D / 32;               // sign words per token
  static constexpr int B2 = LOGD == 11 ? 1 : 0;      // first register bit of the second butterflies
  // shared-memory position of index a (two padding doubles per 64)
  static __host__ __device__ __forceinline__ constexpr int pos(int a) { return a + 2 * (a >> 6); }
  // layout A: register q of thread t holds index 64 t + pi(q); pinv inverts pi
  static __host__ __device__ __forceinline__ constexpr int pi(int q) {
    return LOGD == 11 ? 32 * (q & 1) + (q >> 1) : q;
  }
  static __host__ __device__ __forceinline__ constexpr int pinv(int r) {
    return LOGD == 11 ? ((r & 31) << 1) | (r >> 5) : r;
  }
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

// Registers known to be zero before stage k when registers q >= live start
// as zeros and the stages run in ascending order: a (zero, zero) pair stays
// zero, an (x, zero) pair becomes two copies of x.
__host__ __device__ constexpr unsigned long long sf_zero_mask(int live, int k) {
  unsigned long long z = live >= 64 ? 0ull : ~0ull << live;
  for (int s = 0; s < k; ++s)
    for (int r = 0; r < 64; ++r) {
      if (r & (1 << s)) continue;
      const int b = r | (1 << s);
      const bool za = (z >> r) & 1ull, zb = (z >> b) & 1ull;
      if (!(za && zb)) z &= ~((1ull << r) | (1ull << b));
    }
  return z;
}

template <int LIVE, int K>
__device__ __forceinline__ void sf_stage_live(double (&v)[64]) {
  constexpr unsigned long long Z = sf_zero_mask(LIVE, K);
#pragma unroll
  for (int r = 0; r < 64; ++r) {
    if (r & (1 << K)) continue;
    const int b = r | (1 << K);
    const bool za = (Z >> r) & 1ull, zb = (Z >> b) & 1ull;
    if (za && zb) continue;           // 0 + 0, 0 - 0
    if (zb) { v[b] = v[r]; continue; }  // x + 0 = x - 0 = x
    const double x = v[r], y = v[b];  // (a zero x with a live y cannot occur: the zeros are a suffix)
    v[r] = __dadd_rn(x, y);
    v[b] = __dsub_rn(x, y);
  }
}

// the six register stages of the first transform, registers q >= LIVE zero
template <int LIVE>
__device__ __forceinline__ void sf_stages_live(double (&v)[64]) {
  if constexpr (LIVE >= 64) {
    sf_stages<0, 6>(v);
  } else {
    sf_stage_live<LIVE, 0>(v);
    sf_stage_live<LIVE, 1>(v);
    sf_stage_live<LIVE, 2>(v);
    sf_stage_live<LIVE, 3>(v);
    sf_stage_live<LIVE, 4>(v);
    sf_stage_live<LIVE, 5>(v);
  }
}

template <int NQ>
__device__ __forceinline__ void sf_flip(double (&v)[64], unsigned long long m) {
  const uint32_t lo = (uint32_t)m, hi = (uint32_t)(m >> 32);
#pragma unroll
  for (int r = 0; r < NQ; ++r) {
    const uint32_t bit = ((r < 32 ? lo : hi) >> (r & 31)) & 1u;
    v[r] = __hiloint2double(__double2hiint(v[r]) ^ (int)(bit << 31), __double2loint(v[r]));
  }
}

// layout A <- shared memory (thread t: positions 64 t + pi(q); 128-bit loads
// of position pairs (2m, 2m + 1))
template <int LOGD>
__device__ __forceinline__ void sf_load_A(const double* sm, double (&v)[64], int t) {
  using Gm = SfGeom<LOGD>;
  LFFN_DCHECK(Gm::pos(64 * t + 63) < Gm::PAD);
  const double* q = sm + Gm::pos(64 * t);
#pragma unroll
  for (int r = 0; r < 64; r += 2) {
    const double2 w = *reinterpret_cast<const double2*>(q + r);
    v[Gm::pinv(r)] = w.x;
    v[Gm::pinv(r + 1)] = w.y;
  }
}

// layout B -> shared memory (thread t: positions t + TPT q; 64-bit stores,
// consecutive across the threads of a warp)
template <int LOGD>
__device__ __forceinline__ void sf_store_B(double* sm, const double (&v)[64], int t) {
  using Gm = SfGeom<LOGD>;
#pragma unroll
  for (int r = 0; r < 64; ++r) {
    LFFN_DCHECK(Gm::pos(t + Gm::TPT * r) < Gm::PAD);
    sm[Gm::pos(t + Gm::TPT * r)] = v[r];
  }
}

// Index held by thread t in register q at the start of transform tr (the
// host builds the sign masks in these layouts): B, A, B.
__host__ __device__ __forceinline__ int sf_layout_index(int logd, int tr, int t, int q) {
  if (logd == 12) return (tr & 1) ? 64 * t + q : t + 64 * q;
  return (tr & 1) ? 64 * t + SfGeom<11>::pi(q) : t + 32 * q;
}

// 1 + exp(-2a) for 0 <= a < 18.5, inline (no libdevice call: 17 float64
// instructions against ~45 plus a subroutine call).  exp(x), x in (-37, 0]:
// k = rint(x log2 e), f = x - k ln 2 in two pieces (|f| <= 0.347), exp(f) by
// its Taylor polynomial of degree 10 (truncation 0.347^11 / 11! = 2e-13
// relative), scaled by 2^k through the exponent field (k >= -54: no
// denormals).  Relative error ~3e-13, against the 2.5e-7 of the fp32
// coefficient it feeds; the BH projection, whose z are O(1), takes this for
// every coordinate.
__device__ __forceinline__ double sf_one_plus_exp_m2(double a) {
  const double x = -2.0 * a;
  const double magic = 6755399441055744.0;  // 1.5 * 2^52: rint by addition
  const double tk = fma(x, 1.4426950408889634074, magic);
  const int k = __double2loint(tk);
  const double kf = tk - magic;
  double f = fma(kf, -6.93147180369123816490e-01, x);  // ln 2, high part
  f = fma(kf, -1.90821492927058770002e-10, f);        // ln 2, low part
  double p = 2.7557319223985893e-07;  // 1/10!
  p = fma(p, f, 2.7557319223985888e-06);  // 1/9!
  p = fma(p, f, 2.4801587301587302e-05);  // 1/8!
  p = fma(p, f, 1.9841269841269841e-04);  // 1/7!
  p = fma(p, f, 1.3888888888888889e-03);  // 1/6!
  p = fma(p, f, 8.3333333333333332e-03);  // 1/5!
  p = fma(p, f, 4.1666666666666664e-02);  // 1/4!
  p = fma(p, f, 1.6666666666666666e-01);  // 1/3!
  p = fma(p, f, 0.5);
  p = fma(p, f, 1.0);
  p = fma(p, f, 1.0);
  const double e = __hiloint2double(__double2hiint(p) + (k << 20), __double2loint(p));
  return __dadd_rn(1.0, e);
}

// live registers of layout B for an input width: ceil(d_in / TPT) rounded up
// to the instantiated classes
__host__ __device__ constexpr int sf_live_class(int logd, int d_in) {
  const int tpt = (1 << logd) / 64;
  const int need = (d_in + tpt - 1) / tpt;
  if (logd == 12) return need <= 32 ? 32 : 64;
  return need <= 16 ? 16 : need <= 24 ? 24 : need <= 32 ? 32 : need <= 48 ? 48 : 64;
}

// The epilogue of a token whose 64 z values per thread are 64 consecutive
// coordinates (register r' = PERM ? pinv(r) : r holds z[64 t + r]): sign
// words, small-|z| words, codes and top-1 weights (lookup.cpp:74-100,
// 185-189).  `sm` is the token's padded buffer (free by now: the small z are
// parked in it), `words` its 2 * WORDS sign / small words; token_sync
// synchronises the token's threads.
struct SfEpilogue {
  int code_width, tau, kb, ke;
  uint32_t* codes;
  float* coeff;
};

template <int LOGD, bool PERM, typename Sync>
__device__ __forceinline__ void sf_epilogue(double (&v)[64], double* sm, uint32_t* words, int t, int64_t token,
                                            const SfEpilogue& e, int& bad, Sync token_sync) {
  using Gm = SfGeom<LOGD>;
  constexpr int TPT = Gm::TPT;
  auto PINV = [](int r) { return PERM ? Gm::pinv(r) : r; };
  // ---- epilogue in layout A: z[64 t + r] = v[pinv(r)]
  // sign bits (z >= 0, lookup.cpp:77), small-|z| bits (|z| < 18.5) and the
  // finiteness of the first h*tau outputs (projection.cpp:264, lookup.cpp:204)
  uint32_t s0 = 0, s1 = 0, m0 = 0, m1 = 0;
  {
    // integer pass: negative-sign words (four funnel chains) and, per group
    // of eight coordinates, the range of |z|'s high words
    constexpr uint32_t kSmallHi = 0x40328000u, kInfHi = 0x7ff00000u;
    uint32_t n[4] = {0u, 0u, 0u, 0u};
    uint32_t gsmall = 0u;  // bit g: group g (coordinates 8 g .. 8 g + 7) holds a small or non-finite value
#pragma unroll
    for (int g = 7; g >= 0; --g) {
      uint32_t umin = 0xffffffffu, umax = 0u;
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        const int r = 8 * g + i;
        const uint32_t h = (uint32_t)__double2hiint(v[PINV(r)]);
        n[r >> 4] = __funnelshift_l(h, n[r >> 4], 1);
        const uint32_t u = h + h;  // the high word without its sign bit, doubled
        umin = min(umin, u);
        umax = max(umax, u);
      }
      // 18.5 = 0x4032800000000000: |z| < 18.5 iff its high word is below
      // 0x40328000 (the low word of 18.5 is zero); non-finite iff >= 0x7ff00000
      if (umin < 2u * kSmallHi || umax >= 2u * kInfHi) gsmall |= 1u << g;
    }
    s0 = ~((n[1] << 16) | n[0]);
    s1 = ~((n[3] << 16) | n[2]);
    if (gsmall) {
      // rare (one thread in ~60 at the BASELINE shapes): park the 64 values at
      // their natural shared-memory positions (this thread's own block; the
      // weights below read the small ones from there) and walk the flagged
      // groups -- small bits, the sign of a -0.0 (z >= 0 holds for it,
      // lookup.cpp:77), and the finiteness of the first h*tau outputs
      double* own = sm + Gm::pos(64 * t);
#pragma unroll
      for (int r = 0; r < 64; r += 2)
        *reinterpret_cast<double2*>(own + r) = make_double2(v[PINV(r)], v[PINV(r + 1)]);
      const int lim = e.code_width - 64 * t;  // outputs r < lim are code bits
#pragma unroll 1
      for (int g = 0; g < 8; ++g) {
        if (!((gsmall >> g) & 1u)) continue;
        uint4 w4[4];  // (low, high) words of the group's eight values
#pragma unroll
        for (int i = 0; i < 4; ++i) w4[i] = *reinterpret_cast<const uint4*>(own + 8 * g + 2 * i);
        uint32_t mb = 0u, zb = 0u, nb = 0u;  // small, exact zero, NaN bits of the group
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t lo = (i & 1) ? w4[i >> 1].z : w4[i >> 1].x;
          const uint32_t hi = (i & 1) ? w4[i >> 1].w : w4[i >> 1].y;
          const uint32_t habs = hi & 0x7fffffffu;
          if (habs < kSmallHi) mb |= 1u << i;
          if ((habs | lo) == 0u) zb |= 1u << i;
          if (habs >= kInfHi) {
            if (8 * g + i < lim) bad |= 2;
            if (habs > kInfHi || lo != 0u) nb |= 1u << i;  // NaN: z >= 0 is false whatever its sign bit
          }
        }
        const int sh = (8 * g) & 31;
        if (g < 4) { m0 |= mb << sh; s0 = (s0 | (zb << sh)) & ~(nb << sh); }
        else { m1 |= mb << sh; s1 = (s1 | (zb << sh)) & ~(nb << sh); }
      }
    }
  }
  if (e.tau == 8) {
    // tau = 8 (c2, c4, c5): the thread's 64 coordinates are exactly its own
    // eight tables 8 t .. 8 t + 7, so the codes are the bytes of its two sign
    // words -- no exchange through shared memory, no per-table loop: two
    // 128-bit stores of codes and two of unit weights per thread, then the
    // rare tables with small coordinates one by one.
    const int hl = e.ke - e.kb;
    const int k0 = 8 * t;
    uint32_t* crow = e.codes + token * hl - e.kb;
    float* wrow = e.coeff + token * hl - e.kb;
    if (k0 >= e.kb && k0 + 8 <= e.ke && (((token * hl - e.kb) & 3) == 0)) {
      uint4* cq = reinterpret_cast<uint4*>(crow + k0);
      cq[0] = make_uint4(s0 & 0xffu, (s0 >> 8) & 0xffu, (s0 >> 16) & 0xffu, s0 >> 24);
      cq[1] = make_uint4(s1 & 0xffu, (s1 >> 8) & 0xffu, (s1 >> 16) & 0xffu, s1 >> 24);
      float4* wq = reinterpret_cast<float4*>(wrow + k0);
      wq[0] = make_float4(1.f, 1.f, 1.f, 1.f);
      wq[1] = make_float4(1.f, 1.f, 1.f, 1.f);
    } else {
#pragma unroll 1
      for (int j = 0; j < 8; ++j) {
        const int k = k0 + j;
        if (k < e.kb || k >= e.ke) continue;
        crow[k] = ((j < 4 ? s0 : s1) >> (8 * (j & 3))) & 0xffu;
        wrow[k] = 1.f;
      }
    }
    if ((m0 | m1) != 0u) {
#pragma unroll 1
      for (int j = 0; j < 8; ++j) {
        const int k = k0 + j;
        const uint32_t small = ((j < 4 ? m0 : m1) >> (8 * (j & 3))) & 0xffu;
        if (!small || k < e.kb || k >= e.ke) continue;
        // w = 1 / prod (1 + exp(-2|z_j|)) over the small j (lookup.cpp:185-189);
        // the values were parked in this thread's block above
        double prod = 1.0;
#pragma unroll 1
        for (int b = 0; b < 8; ++b)
          if ((small >> b) & 1u) prod = __dmul_rn(prod, sf_one_plus_exp_m2(fabs(sm[Gm::pos(8 * k + b)])));
        wrow[k] = (float)__ddiv_rn(1.0, prod);
      }
    }
    return;
  }
  // words 2t, 2t+1 hold indices 64 t .. 64 t + 63
  reinterpret_cast<uint2*>(words)[t] = make_uint2(s0, s1);
  reinterpret_cast<uint2*>(words + Gm::WORDS)[t] = make_uint2(m0, m1);
  token_sync();
  const int hl = e.ke - e.kb;
  const int tau = e.tau;
  const uint32_t cmask = tau >= 32 ? 0xffffffffu : ((1u << tau) - 1u);
#pragma unroll 1
  for (int k = e.kb + t; k < e.ke; k += TPT) {
    const int o = k * tau;
    const int wi = o >> 5, sh = o & 31;
    LFFN_DCHECK(wi < Gm::WORDS && o + tau <= e.code_width);
    const uint32_t w_lo = words[wi];
    const uint32_t w_hi = (wi + 1 < Gm::WORDS) ? words[wi + 1] : 0u;
    const uint32_t code = __funnelshift_r(w_lo, w_hi, sh) & cmask;
    const uint32_t small = __funnelshift_r(words[Gm::WORDS + wi],
                                           (wi + 1 < Gm::WORDS) ? words[Gm::WORDS + wi + 1] : 0u, sh) &
                           cmask;
    double w = 1.0;
    if (small) {
      // w = 1 / prod_j (1 + exp(-2|z_j|)) over the small j (lookup.cpp:185-189
      // divides by the factors one after the other; the other factors are
      // exactly 1.0).  One division of the float64 product instead of tau:
      // within 1e-15 of the sequential quotient, far inside the fp32
      // coefficient's 2.5e-7 -- the BH projection's z are O(1), so there every
      // coordinate takes this path
      double prod = 1.0;
#pragma unroll 1
      for (int j = 0; j < tau; ++j)
        if ((small >> j) & 1u) prod = __dmul_rn(prod, sf_one_plus_exp_m2(fabs(sm[Gm::pos(o + j)])));
      w = __ddiv_rn(1.0, prod);
    }
    e.codes[token * hl + (k - e.kb)] = code;
    e.coeff[token * hl + (k - e.kb)] = (float)w;
  }
}

template <int LOGD, int LIVE>
__global__ void __launch_bounds__(sf_threads(LOGD), 384 / sf_threads(LOGD)) hash_sf_kernel(HashSfParams p) {
  using Gm = SfGeom<LOGD>;
  constexpr int TPT = Gm::TPT;
  constexpr int TPB = sf_threads(LOGD) / TPT;  // tokens per CTA
  extern __shared__ double smem[];
  // per token: PAD doubles of transpose buffer, then 2 * WORDS sign / small words
  constexpr int SLOT = Gm::PAD + Gm::WORDS;  // doubles (the words take WORDS doubles)
  const int slot = threadIdx.x / TPT;
  const int t = threadIdx.x - slot * TPT;
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
  // the second and third sign masks are loaded under the butterflies that
  // precede their use (~450 cycles of L2 latency each on a token's critical
  // path otherwise: c3 0.336 -> 0.334 ms, c4 0.117 -> 0.113) -- except in the
  // LIVE = 24 instance (c2, c5), where the two extra live registers spill
  // (0.096 -> 0.100 ms)
  constexpr bool kMaskAhead = !(LOGD == 11 && LIVE == 24);
  unsigned long long mask;

  // ---- x (padded to D) into layout B: register q of thread t holds
  // x[t + TPT q]; registers q >= LIVE are padding (launcher: d_in <= TPT *
  // LIVE).  The finiteness test rides on an FMA chain (x * 0 is NaN iff x is
  // inf / NaN).
  {
    const float* xr = p.x + token * (int64_t)p.d_in;
    float nanacc = 0.f;
    constexpr int LB = LIVE <= 32 ? LIVE : LIVE / 2;  // loads in flight per thread
#pragma unroll
    for (int g = 0; g < LIVE; g += LB) {
      float f[LB];
#pragma unroll
      for (int r = 0; r < LB; ++r) {
        const int a = t + TPT * (g + r);
        f[r] = a < p.d_in ? __ldg(xr + a) : 0.f;
      }
#pragma unroll
      for (int r = 0; r < LB; ++r) {
        nanacc = fmaf(f[r], 0.f, nanacc);
        v[g + r] = (double)f[r];
      }
    }
#pragma unroll
    for (int r = LIVE; r < 64; ++r) v[r] = 0.0;
    if (nanacc != nanacc) bad |= 1;
  }
  // Three transforms: sign flip, butterflies over the six register bits, the
  // transpose, butterflies over the register bits it brought in.  The first
  // transform's first half is specialised for the zero padding; everything
  // after it is one copy of code in a loop that is not unrolled (the hot loop
  // stays within the 32 KB L1.5 instruction cache).
  sf_flip<LIVE>(v, __ldg(p.masks + t));
  sf_stages_live<LIVE>(v);
  sf_store_B<LOGD>(sm, v, t);  // (the copies of the padding pairs are stored straight from their source)
  // (the trip count comes from the parameters so that the compiler keeps one
  // copy of the body instead of peeling the first transform's second half)
#pragma unroll 1
  for (int tr = 1; tr <= p.transforms; ++tr) {
    token_sync();
    sf_load_A<LOGD>(sm, v, t);
    token_sync();
    if (kMaskAhead && tr < p.transforms) mask = __ldg(p.masks + tr * TPT + t);
    sf_stages<Gm::B2, 6>(v);
    if (tr < p.transforms) {
      if (!kMaskAhead) mask = __ldg(p.masks + tr * TPT + t);
      sf_flip<64>(v, mask);
      sf_stages<0, 6>(v);
      sf_store_B<LOGD>(sm, v, t);
    }
  }

  // ---- epilogue in layout A: z[64 t + r] = v[pinv(r)]
  {
    SfEpilogue e{p.code_width, p.tau, p.kb, p.ke, p.codes, p.coeff};
    sf_epilogue<LOGD, true>(v, sm, words, t, token, e, bad, token_sync);
  }
  if (bad) atomicOr(p.flag, bad);
}

}  // namespace lffn_gpu
