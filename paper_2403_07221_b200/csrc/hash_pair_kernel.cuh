// hash_pair_kernel.cuh -- K1 specialised for transform widths D = 2048 and
// 4096 (BASELINE c2/c3/c5: D = 2048; c4: D = 4096).
//
// Same arithmetic as hash_structured_kernel (reference stage order, float64,
// exact sign flips: z bit-identical to projection.cpp:200-263), with half the
// registers per element in flight: a thread holds 32 doubles and the sixth
// bit of a 6-bit phase lives across the lane pair (t, t^1), so that stage is
// a 64-bit shuffle instead of a shared-memory round trip:
//   phase A  bits 0-5   elements 32t .. 32t+31 (contiguous), bits 0-4 in
//                       registers, bit 5 across the pair
//   phase B  bits 6-10  (D = 2048) all in registers, elements t + 64 i
//            bits 6-11  (D = 4096) bit 6 across the pair first, 7-11 in
//                       registers
// Two shared-memory round trips per transform, ~100 registers per thread,
// 6 CTAs (24 warps) per SM instead of 8-12 warps for the 64-element form.
#pragma once

#include "hash_kernels.cuh"

namespace lffn_gpu {

// Shared-memory position for the pair kernel: two spare doubles per 32, so
// phase A's 32-element runs start 34 doubles apart (conflict-free 128-bit
// accesses) and phase B's half warps read 16 consecutive elements.
__device__ __forceinline__ int ppos(int a) { return a + 2 * (a >> 5); }
__host__ __device__ constexpr int pair_padded_len(int D) { return D + 2 * (D >> 5); }

template <int L, int KIND>
__global__ void __launch_bounds__(128, 4) hash_pair_kernel(HashParams p) {
  static_assert(L == 11 || L == 12, "hash_pair_kernel: D must be 2048 or 4096");
  constexpr int D = 1 << L;
  constexpr int TPT = D / 32;       // threads per token: 64 or 128
  constexpr int TPB = 128 / TPT;    // tokens per CTA: 2 or 1
  extern __shared__ double smem[];
  const int slot = threadIdx.x / TPT;
  const int t = threadIdx.x % TPT;
  const int64_t token = (int64_t)blockIdx.x * TPB + slot;
  const bool active = token < p.n;  // whole warps share a token (TPT >= 64)
  double* sm = smem + (size_t)slot * pair_padded_len(D);
  int bad = 0;
  auto token_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(slot + 1), "r"(TPT) : "memory"); };
  // butterfly across a lane pair (lane ^ X): the lower lane keeps x + y,
  // the upper x - y, x being the lower lane's element (fwht.hpp:35-36)
  auto pair_stage = [&](double (&v)[32], int xmask, bool upper) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const double o = __shfl_xor_sync(0xffffffffu, v[i], xmask);
      v[i] = upper ? __dsub_rn(o, v[i]) : __dadd_rn(v[i], o);
    }
  };
  const int lane = threadIdx.x & 31;
  // phase B geometry: D = 2048 -> element t + 64 i; D = 4096 -> element
  // g | pb << 6 | i << 7 with g = 16 * warp + (lane & 15), pb = lane >> 4
  const int gB = (L == 11) ? t : 16 * (t >> 5) + (lane & 15);
  const int pbB = (L == 11) ? 0 : (lane >> 4);
  const int baseB = gB + 2 * (gB >> 5) + 68 * pbB;
  constexpr int strideB = (L == 11) ? 68 : 136;
  double v[32];
  const float* xr = p.x + token * (int64_t)p.d_in;

  for (int tr = 0; tr < p.n_transforms; ++tr) {
    const bool last_tr = tr == p.n_transforms - 1;
    // ---------------- phase A: bits 0-5, elements 32t .. 32t+31
    if (active) {
      if (tr == 0) {
        if (32 * t + 32 <= p.d_in && (p.d_in & 3) == 0) {
#pragma unroll
          for (int r = 0; r < 32; r += 4) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(xr + 32 * t + r));
            if (!isfinite(f.x) || !isfinite(f.y) || !isfinite(f.z) || !isfinite(f.w)) bad |= 1;
            v[r] = (double)f.x;
            v[r + 1] = (double)f.y;
            v[r + 2] = (double)f.z;
            v[r + 3] = (double)f.w;
          }
        } else {
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            const int a = 32 * t + r;
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
        const double2* q = reinterpret_cast<const double2*>(sm + ppos(32 * t));
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const double2 w = q[r];
          v[2 * r] = w.x;
          v[2 * r + 1] = w.y;
        }
      }
      if constexpr (KIND == kPreSign) {
        const uint32_t m = __ldg(p.signmask + tr * (D / 32) + t);
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = flip_sign(v[r], m, r);
      } else {
        const double* dg = p.diag + (size_t)tr * D + 32 * t;
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = __dmul_rn(v[r], __ldg(dg + r));
      }
      butterfly_groups<5, 5>(v);              // bits 0-4
      pair_stage(v, 1, (t & 1) != 0);         // bit 5 (lanes t, t^1)
      double2* q = reinterpret_cast<double2*>(sm + ppos(32 * t));
#pragma unroll
      for (int r = 0; r < 16; ++r) q[r] = make_double2(v[2 * r], v[2 * r + 1]);
    }
    token_sync();
    // ---------------- phase B: bits 6 .. L-1
    if (active) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = sm[baseB + strideB * i];
      if constexpr (L == 12) pair_stage(v, 16, pbB != 0);  // bit 6 (lanes l, l^16)
      butterfly_groups<5, 5>(v);                          // bits 6-10 / 7-11
      if (last_tr && p.code_width == D) {
        uint32_t mm = 0xffffffffu;
#pragma unroll
        for (int r = 0; r < 32; ++r)
          mm = min(mm, (uint32_t)(__double2hiint(v[r]) & 0x7ff00000) ^ 0x7ff00000u);
        if (mm == 0u) bad |= 2;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) sm[baseB + strideB * i] = v[i];
    }
    token_sync();
  }

  if (active) {
    if (p.z_out || p.code_width != D) {
      for (int a = t; a < p.code_width; a += TPT) {
        const double zv = sm[ppos(a)];
        if (!isfinite(zv)) bad |= 2;
        if (p.z_out) p.z_out[token * p.code_width + a] = zv;
      }
    }
    // tables whose first coordinate lies in this thread's 32 elements
    const int tau = p.tau;
    const int hl = p.ke - p.kb;
    const int a_lo = 32 * t;
    const int a_hi = min(a_lo + 32, p.code_width);
    for (int k = max((a_lo + tau - 1) / tau, p.kb); k < p.ke && k * tau < a_hi; ++k) {
      const int base = k * tau;
      uint32_t code = 0;
      bool small = false;
      double sum_abs = 0.0;
#pragma unroll 4
      for (int j = 0; j < tau; ++j) {
        const double zj = sm[ppos(base + j)];
        code |= (zj >= 0.0 ? 1u : 0u) << j;
        const double az = fabs(zj);
        small |= az < 18.5;
        sum_abs = __dadd_rn(sum_abs, az);
      }
      double w = 1.0;
      if (small) {
        for (int j = 0; j < tau; ++j) {
          const double az = fabs(sm[ppos(base + j)]);
          if (az < 18.5) w = __ddiv_rn(w, one_plus_exp_m2(az));
        }
      }
      p.codes[token * hl + (k - p.kb)] = code;
      p.coeff[token * hl + (k - p.kb)] = (float)(p.scaled ? __dmul_rn(w, sum_abs) : w);
    }
  }
  if (bad) atomicOr(p.flag, bad);
}

}  // namespace lffn_gpu
