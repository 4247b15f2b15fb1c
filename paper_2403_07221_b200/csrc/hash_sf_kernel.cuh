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
// Every transform runs the same code: sign flip, butterflies over the six
// index bits in the registers, one transpose through shared memory (64-bit
// stores in the B pattern, 128-bit loads in the A pattern; both bank-conflict
// free with two padding doubles per 64), butterflies over the bits the
// transpose brought into the registers.  The stages of a Walsh-Hadamard
// transform commute, so which bits sit in the registers may differ from
// transform to transform: x starts in a layout L0 chosen so that three
// transposes end in layout A (sf_start_index).  Three transposes per token
// against K1's six stores and five loads.
//
// Epilogue in layout A: a thread's 64 registers are 64 consecutive
// coordinates, so its sign bits (z >= 0, lookup.cpp:77) form two words of the
// h*tau code bits in shared memory, from which each thread funnel-shifts its
// tables' codes.  The weight is exactly 1.0 for a table whose every |z_j| >= 18.5
// (1 + exp(-2|z|) rounds to 1.0); the rare small coordinates (a second
// ballot) have their z stored, and the table's weight divides by
// 1 + exp(-2|z_j|) over exactly those j in ascending order -- the reference's
// sequential division, the other factors being exact divisions by 1.0.
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
  const unsigned long long* masks;  // [3][TPT]: bit r = sign of the element thread t holds in
                               // register r at the start of transform tr (sf_layout_index)
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
  LFFN_DCHECK(SfGeom<LOGD>::pos(64 * t + 63) < SfGeom<LOGD>::PAD);
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
    LFFN_DCHECK(Gm::pos(t + Gm::TPT * r) < Gm::PAD);
    double* q = sm + Gm::pos(t + Gm::TPT * r);
    if constexpr (STORE) *q = v[r];
    else v[r] = *q;
  }
}

// Index held by thread t in register r at the start (layout L0).  The
// transpose (store at index t + TPT r, load index 64 t' + r') maps layout L
// to L'(t', r') = L(r' mod TPT, (TPT/32) t' ... ) -- for D = 4096 it swaps t
// and r, for D = 2048 L'(l, r) = L(r & 31, 2 l + (r >> 5)).  L0 is chosen so
// that three transposes end in layout A (index 64 t + r):
//   D = 2048: L0 = 1024 (l & 1) + 32 (r >> 1) + 16 (r & 1) + (l >> 1)
//             L1 = 32 l + 1024 (r & 1) + (r >> 1),  L2 = l + 32 r (= B),  L3 = A
//   D = 4096: L0 = t + 64 r (= B), L1 = A, L2 = B, L3 = A
// Each transform's first butterflies cover the six index bits its layout
// holds in registers, the second ones the register bits that came from the
// threads (D = 2048: register bits 0-4; D = 4096: all six), i.e. every bit
// exactly once.  The host builds the sign masks in L0, L1, L2.
template <int LOGD>
__host__ __device__ __forceinline__ int sf_start_index(int t, int r) {
  if constexpr (LOGD == 11) return 1024 * (t & 1) + 32 * (r >> 1) + 16 * (r & 1) + (t >> 1);
  else return t + 64 * r;
}
__host__ __device__ __forceinline__ int sf_layout_index(int logd, int tr, int t, int r) {
  if (logd == 12) return (tr & 1) ? 64 * t + r : t + 64 * r;
  if (tr == 0) return sf_start_index<11>(t, r);
  if (tr == 1) return 32 * t + 1024 * (r & 1) + (r >> 1);
  if (tr == 2) return t + 32 * r;
  return 64 * t + r;
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

  // ---- x (padded to D) into the start layout L0 (below); the finiteness
  // test rides on an FMA chain (x * 0 is NaN iff x is inf / NaN)
  {
    const float* xr = p.x + token * (int64_t)p.d_in;
    float nanacc = 0.f;
#pragma unroll
    for (int g = 0; g < 64; g += 16) {
      float f[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int a = sf_start_index<LOGD>(t, g + r);
        f[r] = a < p.d_in ? __ldg(xr + a) : 0.f;
      }
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        nanacc = fmaf(f[r], 0.f, nanacc);
        v[g + r] = (double)f[r];
      }
    }
    if (nanacc != nanacc) bad |= 1;
  }
  // Three transforms with the same code: sign flip, butterflies over the six
  // register bits, the transpose (store in the B pattern, load in the A
  // pattern: it moves the value of thread / register (r' mod T, T' (...))
  // -- see sf_start_index), butterflies over the register bits the
  // transpose brought in from the threads.  The transpose permutes which
  // index bits sit in the registers so that every transform covers each of
  // its log2(D) bits exactly once, and three of them take the start layout
  // L0 to layout A.  The loop is not unrolled: one copy of the butterfly code
  // (the kernel stays within the 32 KB L1.5 instruction cache).
#pragma unroll 1
  for (int tr = 0; tr < 3; ++tr) {
    sf_flip(v, __ldg(p.masks + tr * TPT + t));
    sf_stages<0, 6>(v);
    sf_io_B<LOGD, true>(sm, v, t);
    token_sync();
    sf_io_A<LOGD, false>(sm, v, t);
    token_sync();
    sf_stages<0, (LOGD == 11 ? 5 : 6)>(v);
  }

  // ---- epilogue in layout A: z[64 t + r] = v[r]
  // sign bits (z >= 0, lookup.cpp:77), small-|z| bits (|z| < 18.5) and the
  // finiteness of the first h*tau outputs (projection.cpp:264, lookup.cpp:204)
  uint32_t s0 = 0, s1 = 0, m0 = 0, m1 = 0;
  bool fin = true;
#pragma unroll
  for (int r = 0; r < 64; ++r) {
    const uint32_t sb = v[r] >= 0.0 ? 1u : 0u;
    const uint32_t mb = fabs(v[r]) < 18.5 ? 1u : 0u;
    if (r < 32) { s0 |= sb << r; m0 |= mb << r; }
    else { s1 |= sb << (r - 32); m1 |= mb << (r - 32); }
    if (64 * t + r < p.code_width) fin &= (__double2hiint(v[r]) & 0x7ff00000) != 0x7ff00000;
  }
  if (!fin) bad |= 2;
  // words 2t, 2t+1 hold indices 64 t .. 64 t + 63
  reinterpret_cast<uint2*>(words)[t] = make_uint2(s0, s1);
  reinterpret_cast<uint2*>(words + Gm::WORDS)[t] = make_uint2(m0, m1);
  // the z of every small coordinate, at its natural shared-memory position
  if ((m0 | m1) != 0u) {
#pragma unroll
    for (int r = 0; r < 64; ++r)
      if ((((r < 32 ? m0 : m1) >> (r & 31)) & 1u) != 0u) sm[Gm::pos(64 * t + r)] = v[r];
  }
  token_sync();
  const int hl = p.ke - p.kb;
  const int tau = p.tau;
  const uint32_t cmask = tau >= 32 ? 0xffffffffu : ((1u << tau) - 1u);
  for (int k = p.kb + t; k < p.ke; k += TPT) {
    const int o = k * tau;
    const int wi = o >> 5, sh = o & 31;
    LFFN_DCHECK(wi < Gm::WORDS && o + tau <= p.code_width);
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
