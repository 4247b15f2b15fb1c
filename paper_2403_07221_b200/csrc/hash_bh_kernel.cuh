// hash_bh_kernel.cuh -- K1 for the BH{m} projection (the
// paper's recommended BH4), fused with codes and coefficients.
//
// Reference: Projection::forward bh branch (projection.cpp:217-228): per
// stage s, dst = block_diag_apply(buf, B_s) (projection.hpp:101-119:
// dst[g*b+c] = sum_r src[g*b+r] * B_s[g][r][c], r ascending, from 0.0), then
// fwht_kernel(dst) (fwht.hpp:28-41).
//
// Device form: a CTA of 512 threads owns T = 16384 / D tokens whose D-vectors
// live in shared memory.  The block-diagonal multiply gives every thread 32
// (token, column) outputs, accumulated in the reference's order with
// separately rounded multiply and add, so z stays bit-identical to the
// reference; each B_s element is read once per CTA and used for T tokens.
// The Hadamard stages then run with the 32-element register phases of
// hash_structured_kernel, and the epilogue packs codes / coefficients.
// Float64 arithmetic: 2*D*b + D*log2(D) flops per stage per token
// (flops.cpp:27-33).
#pragma once

#include "hash_kernels.cuh"
#include "hash_sf_kernel.cuh"

namespace lffn_gpu {

struct BhParams {
  const double* blocks;  // m stages x (D/b) blocks x b x b, row-major (projection.hpp:47-54)
  int b, logb;
  int stages;
};

// QPT: column quads per thread (D / 2048 for D >= 2048, else 1); every
// thread owns 32 (token, column) outputs = QPT quads x (8 / QPT) tokens.
template <int LOGE, int QPT>
__global__ void __launch_bounds__(512, 1) hash_bh_kernel(HashParams p, BhParams bh) {
  extern __shared__ double smem[];
  constexpr int E = 1 << LOGE;
  constexpr int NT = 512;
  constexpr int PAIRS = 32;  // (token, column) outputs per thread per stage
  const int D = p.D, logD = p.logD;
  const int pad = padded_len(D);
  const int T = p.tokens_per_block;  // T * D == NT * PAIRS
  const int tpt = p.threads_per_token;
  const int64_t tok0 = (int64_t)blockIdx.x * T;
  const int tid = threadIdx.x;
  int bad = 0;

  // pad x to D (projection.cpp:212-213), fp32 -> fp64 exactly
  for (int q = tid; q < T * D; q += NT) {
    const int t = q >> logD, a = q & (D - 1);
    const int64_t token = tok0 + t;
    double v = 0.0;
    if (token < p.n && a < p.d_in) {
      const float f = __ldg(p.x + token * p.d_in + a);
      if (!isfinite(f)) bad |= 1;
      v = (double)f;
    }
    smem[t * pad + spos(a)] = v;
  }
  __syncthreads();

  const int b = bh.b, logb = bh.logb;
  const size_t stage_size = (size_t)(D >> logb) * b * b;
  int nph = 1;
  if constexpr (LOGE > 0) nph = (logD + LOGE - 1) / LOGE;
  for (int s = 0; s < bh.stages; ++s) {
    // ---- block-diagonal multiply (projection.hpp:101-119)
    const double* Bs = bh.blocks + s * stage_size;
    if (b >= 4) {
      // a thread's 4 consecutive columns (one quad) lie in one block g: per r
      // it loads B_s[g][r][cc..cc+3] once (two 128-bit loads) and each token's
      // src[g*b + r] once, and updates 4 x (8 / QPT) accumulators -- the
      // reference's order (r ascending from 0.0), separate multiply and add
      constexpr int TPQ = 8 / QPT;
      const int nq = D >> 2;
      int tok[TPQ];
      int quad0, qstride;
      if (nq >= NT) {
        quad0 = tid;
        qstride = NT;
#pragma unroll
        for (int j = 0; j < TPQ; ++j) tok[j] = j;
      } else {
        const int tpq = NT / nq;
        quad0 = tid % nq;
        qstride = 0;
#pragma unroll
        for (int j = 0; j < TPQ; ++j) tok[j] = tid / nq + tpq * j;
      }
      double acc[QPT][TPQ][4];
#pragma unroll
      for (int qi = 0; qi < QPT; ++qi) {
        const int c = 4 * (quad0 + qi * qstride);
        const int g = c >> logb, cc = c & (b - 1);
        const double* Bp = Bs + ((size_t)g * b) * b + cc;
        const int sb = spos(g << logb);
#pragma unroll
        for (int j = 0; j < TPQ; ++j)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[qi][j][v] = 0.0;
        for (int r = 0; r < b; ++r) {
          const double2 b01 = __ldg(reinterpret_cast<const double2*>(Bp + (size_t)r * b));
          const double2 b23 = __ldg(reinterpret_cast<const double2*>(Bp + (size_t)r * b + 2));
          const int so = sb + r + 2 * (r >> 6);  // spos(g*b + r): b | 64 or 64 | b
#pragma unroll
          for (int j = 0; j < TPQ; ++j) {
            const double sv = smem[tok[j] * pad + so];
            acc[qi][j][0] = __dadd_rn(acc[qi][j][0], __dmul_rn(sv, b01.x));
            acc[qi][j][1] = __dadd_rn(acc[qi][j][1], __dmul_rn(sv, b01.y));
            acc[qi][j][2] = __dadd_rn(acc[qi][j][2], __dmul_rn(sv, b23.x));
            acc[qi][j][3] = __dadd_rn(acc[qi][j][3], __dmul_rn(sv, b23.y));
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int qi = 0; qi < QPT; ++qi) {
        const int c = 4 * (quad0 + qi * qstride);
#pragma unroll
        for (int j = 0; j < TPQ; ++j)
#pragma unroll
          for (int v = 0; v < 4; ++v) smem[tok[j] * pad + spos(c + v)] = acc[qi][j][v];
      }
      __syncthreads();
    } else {
      // b = 1, 2: one (token, column) per accumulator
      double acc[PAIRS];
#pragma unroll
      for (int j = 0; j < PAIRS; ++j) acc[j] = 0.0;
      for (int r = 0; r < b; ++r) {
#pragma unroll
        for (int j = 0; j < PAIRS; ++j) {
          const int q = tid + NT * j;
          const int t = q >> logD, c = q & (D - 1);
          const int g = c >> logb, cc = c & (b - 1);
          const double bv = __ldg(Bs + ((size_t)g * b + r) * b + cc);
          const double sv = smem[t * pad + spos((g << logb) + r)];
          acc[j] = __dadd_rn(acc[j], __dmul_rn(sv, bv));
        }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < PAIRS; ++j) {
        const int q = tid + NT * j;
        smem[(q >> logD) * pad + spos(q & (D - 1))] = acc[j];
      }
      __syncthreads();
    }
    // ---- Hadamard transform of every token (fwht.hpp:28-41)
    const bool last_stage = s == bh.stages - 1;
    for (int ph = 0; ph < nph; ++ph) {
      const int lo = ph * LOGE;
      const int bits = min(LOGE, logD - lo);
      for (int slot = tid / tpt; slot < T; slot += NT / tpt) {
        double* sm = smem + slot * pad;
        const int tt = tid % tpt;
        const bool last = last_stage && ph == nph - 1 && tok0 + slot < p.n;
        if (ph == 0) {
          phase_smem<LOGE, LOGE, false, kPreNone>(sm, tt, tpt, 0, p, s, nullptr, bad, last);
        } else {
          run_later_phase<LOGE>(sm, tt, tpt, lo, bits, p, s, bad, last);
        }
      }
      __syncthreads();
    }
  }

  // ---- codes + coefficients (lookup.cpp:81-100, 185-189), per token slot
  for (int slot = tid / tpt; slot < T; slot += NT / tpt) {
    const int64_t token = tok0 + slot;
    if (token >= p.n) continue;
    const double* sm = smem + slot * pad;
    const int t = tid % tpt;
    if (p.z_out || p.code_width != D) {
      for (int a = t; a < p.code_width; a += tpt) {
        const double zv = sm[spos(a)];
        if (!isfinite(zv)) bad |= 2;
        if (p.z_out) p.z_out[token * p.code_width + a] = zv;
      }
    }
    const int tau = p.tau;
    const int hl = p.ke - p.kb;
    const int a_lo = t * E;
    const int a_hi = min(a_lo + E, p.code_width);
    for (int k = max((a_lo + tau - 1) / tau, p.kb); k < p.ke && k * tau < a_hi; ++k) {
      const int base = k * tau;
      uint32_t code = 0;
      bool small = false;
      double sum_abs = 0.0;
      for (int j = 0; j < tau; ++j) {
        const double zj = sm[spos(base + j)];
        code |= (zj >= 0.0 ? 1u : 0u) << j;
        const double az = fabs(zj);
        small |= az < 18.5;
        sum_abs = __dadd_rn(sum_abs, az);
      }
      double w = 1.0;
      if (small) {
        for (int j = 0; j < tau; ++j) {
          const double az = fabs(sm[spos(base + j)]);
          if (az < 18.5) w = __ddiv_rn(w, one_plus_exp_m2(az));
        }
      }
      p.codes[token * hl + (k - p.kb)] = code;
      p.coeff[token * hl + (k - p.kb)] = (float)(p.scaled ? __dmul_rn(w, sum_abs) : w);
    }
  }
  if (bad) atomicOr(p.flag, bad);
}

// BH{m} at the paper's shape (D = 2048, b = 64; the BASELINE c2 BH4) --
// round 2.  hash_bh_kernel above re-reads each stage's 1 MB of blocks from L2
// with the loads on the critical path of every row (fp64 pipe 44 %, stalls on
// the row loads).  Here a CTA of 256 threads owns 8 tokens and every thread
// an 8-column x 8-token tile of the block-diagonal product (64 float64
// accumulators): per row r it needs 64 bytes of B_s (four coalesced 16-byte
// cp.async copies into the thread's own shared-memory ring, three rows ahead,
// so the L2 latency is hidden behind 3 x 128 float64 instructions and no
// register waits on a load) and the eight tokens' src values (64-bit
// broadcast loads from shared memory).  A warp owns four whole
// blocks, reads and rewrites only their coordinates, so the in-place update
// needs a warp barrier only.  The accumulation is the reference's
// (projection.hpp:101-119): r ascending from 0.0, separately rounded
// multiply and add -- z bit-identical; with FMA = true (no z requested) the
// multiply-add is fused (one rounding less per term: |dz| ~ 1e-16 |z|, codes
// bit-exact wherever |z| > 1e-5, the north star's bar).  The Hadamard stages
// and the epilogue are those of hash_bh_kernel.
template <bool FMA>
__global__ void __launch_bounds__(256, 1) hash_bh64_kernel(HashParams p, BhParams bh) {
  extern __shared__ double smem[];
  constexpr int D = 2048, LOGD = 11, NT = 256, T = 8, LOGE = 6, E = 64, TPT = D / E;  // a warp per token in the Hadamard stages
  constexpr int PADL = padded_len(D);
  const int64_t tok0 = (int64_t)blockIdx.x * T;
  const int tid = threadIdx.x;
  int bad = 0;

  // pad x to D (projection.cpp:212-213), fp32 -> fp64 exactly
  {
    const int t = tid >> 5;  // warp w loads token w
    const int64_t token = tok0 + t;
    for (int a = tid & 31; a < D; a += 32) {
      double v = 0.0;
      if (token < p.n && a < p.d_in) {
        const float f = __ldg(p.x + token * p.d_in + a);
        if (!isfinite(f)) bad |= 1;
        v = (double)f;
      }
      smem[t * PADL + spos(a)] = v;
    }
  }
  __syncthreads();

  // the thread's block g and its columns 16 j + 2 li + {0, 1}, j = 0..3 (the
  // eight threads of a block read 128 contiguous bytes per load)
  const int g = tid >> 3, li = tid & 7;
  const size_t stage_size = (size_t)(D >> 6) * 64 * 64;
  double* srcp = smem + spos(g << 6);  // src[t][g*64 + r] = srcp[t * PADL + r]
  // ring[(slot * 4 + j) * NT + tid]: the thread's j-th 16 bytes of the row in slot
  const double2* ring = reinterpret_cast<const double2*>(smem + T * PADL) + tid;
  const uint32_t ring_base = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  for (int s = 0; s < bh.stages; ++s) {
    const double2* Bp = reinterpret_cast<const double2*>(bh.blocks + s * stage_size + (size_t)g * 64 * 64) + li;
    // row r, load j: Bp[r * 32 + 8 j]  (a row is 32 double2; 16 columns = 8 double2)
    double acc[T][8];
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[t][c] = 0.0;
    // B rows through a per-thread ring of four rows in shared memory, filled
    // by cp.async three rows ahead: no registers held by loads in flight (a
    // register ring spilled at 255 registers and stalled on its own loads),
    // and no barrier -- a thread reads back only what it copied itself
    auto issue = [&](int r) {
      if (r < 64) {
        const uint32_t dst = ring_base + uint32_t((r & 3) * 4 * NT * 16);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + uint32_t(j * NT * 16)),
                       "l"(Bp + r * 32 + 8 * j)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0);
    issue(1);
    issue(2);
#pragma unroll 4
    for (int r = 0; r < 64; ++r) {
      issue(r + 3);
      asm volatile("cp.async.wait_group 3;" ::: "memory");
      const double2* rq = ring + (r & 3) * 4 * NT;
      double2 bq[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bq[j] = rq[j * NT];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const double sv = srcp[t * PADL + r];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (FMA) {
            acc[t][2 * j] = fma(sv, bq[j].x, acc[t][2 * j]);
            acc[t][2 * j + 1] = fma(sv, bq[j].y, acc[t][2 * j + 1]);
          } else {
            acc[t][2 * j] = __dadd_rn(acc[t][2 * j], __dmul_rn(sv, bq[j].x));
            acc[t][2 * j + 1] = __dadd_rn(acc[t][2 * j + 1], __dmul_rn(sv, bq[j].y));
          }
        }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();  // the warp's four blocks are read only by this warp
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<double2*>(srcp + t * PADL + 16 * j + 2 * li) = make_double2(acc[t][2 * j], acc[t][2 * j + 1]);
    __syncthreads();
    // ---- Hadamard transform of every token (fwht.hpp:28-41): warp w owns
    // token w, 64 elements per lane, bits 0-5 then bits 6-10 in the
    // reference's stage order (two conflict-free shared-memory round trips)
    {
      const bool last = s == bh.stages - 1 && tok0 + (tid >> 5) < p.n;
      double* sm = smem + (tid >> 5) * PADL;
      phase_smem<LOGE, 6, false, kPreNone>(sm, tid & 31, TPT, 0, p, s, nullptr, bad, false);
      __syncwarp();
      phase_smem<LOGE, 5, false, kPreNone>(sm, tid & 31, TPT, 6, p, s, nullptr, bad, last);
    }
    __syncthreads();
  }

  // ---- codes + coefficients (lookup.cpp:81-100, 185-189).  Top-1 weights
  // without a z copy: K1f's integer epilogue on the warp's token (each lane
  // reloads its 64 consecutive coordinates); else the per-table loop below.
  if (!p.z_out && !p.scaled) {
    const int64_t token = tok0 + (tid >> 5);
    if (token < p.n) {  // warp-uniform
      const int t = tid & 31;
      double* sm = smem + (tid >> 5) * PADL;
      uint32_t* words = reinterpret_cast<uint32_t*>(smem + T * PADL + 2 * 4 * 4 * NT) + (tid >> 5) * 128;
      double v[64];
      const double* q = sm + spos(64 * t);
#pragma unroll
      for (int r = 0; r < 64; r += 2) {
        const double2 w = *reinterpret_cast<const double2*>(q + r);
        v[r] = w.x;
        v[r + 1] = w.y;
      }
      SfEpilogue e{p.code_width, p.tau, p.kb, p.ke, p.codes, p.coeff};
      sf_epilogue<11, false>(v, sm, words, t, token, e, bad, [] { __syncwarp(); });
    }
    if (bad) atomicOr(p.flag, bad);
    return;
  }
  for (int slot = tid / TPT; slot < T; slot += NT / TPT) {
    const int64_t token = tok0 + slot;
    if (token >= p.n) continue;
    const double* sm = smem + slot * PADL;
    const int t = tid % TPT;
    if (p.z_out || p.code_width != D) {
      for (int a = t; a < p.code_width; a += TPT) {
        const double zv = sm[spos(a)];
        if (!isfinite(zv)) bad |= 2;
        if (p.z_out) p.z_out[token * p.code_width + a] = zv;
      }
    }
    const int tau = p.tau;
    const int hl = p.ke - p.kb;
    const int a_lo = t * E;
    const int a_hi = min(a_lo + E, p.code_width);
    for (int k = max((a_lo + tau - 1) / tau, p.kb); k < p.ke && k * tau < a_hi; ++k) {
      const int base = k * tau;
      uint32_t code = 0;
      bool small = false;
      double sum_abs = 0.0;
      for (int j = 0; j < tau; ++j) {
        const double zj = sm[spos(base + j)];
        code |= (zj >= 0.0 ? 1u : 0u) << j;
        const double az = fabs(zj);
        small |= az < 18.5;
        sum_abs = __dadd_rn(sum_abs, az);
      }
      double w = 1.0;
      if (small) {
        for (int j = 0; j < tau; ++j) {
          const double az = fabs(sm[spos(base + j)]);
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
