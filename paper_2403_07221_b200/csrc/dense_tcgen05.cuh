// dense_tcgen05.cuh -- K2: the dense projection z = x W on the 5th-gen
// tensor cores (accumulator in TMEM) with an fp32-faithful operand split --
// bf16 x3 (kind::f16, six products; the default when d_in % 8 == 0) or tf32
// hi / lo (kind::tf32, three products) -- fused with the code / coefficient
// epilogue.
//
// Reference: Projection::forward dense branch (projection.cpp:178-198) and
// lookup_hash_f32 dense (bench.cpp:122-129), compute_codes / top1_weight
// (lookup.cpp:81-100, 185-189).
//
// Numerics (tf32 split; the bf16 x3 split is the same idea with three bf16
// terms): x = x_hi + x_lo and W = W_hi + W_lo with *_hi = tf32(.) and
// *_lo = tf32(. - *_hi); D += x_hi W_hi + x_hi W_lo + x_lo W_hi accumulates in
// fp32 in TMEM.  The error (~1e-6 absolute at c2 scale, below the fp32 path
// of the reference itself) leaves codes bit-exact wherever |z| exceeds ~1e-5,
// the BASELINE.json criterion; the exact float64 kernel
// (dense_proj_f64_kernel) remains selectable.
//
// Tile: M = 128 tokens (TMEM lanes) x N = NT columns of z (NT a multiple of
// lcm(tau, 16), <= 128, so every tile holds whole tables) x K = 16 per stage.
// x is split into tf32 hi / lo once per call (dense_split_x_kernel), W once at
// context creation, so the main loop is pure TMA -> MMA: thread 0 keeps
// kStages stages of x_hi / x_lo / W_hi / W_lo tiles (SWIZZLE_64B, 32 KB per
// stage) in flight, thread 32 issues the stage's 6 tcgen05.mma and commits
// them to the stage's "empty" barrier.  96 KB of shared memory and 256 TMEM
// columns per CTA keep two CTAs resident per SM, so one CTA's epilogue runs
// under the other's main loop.  Epilogue: TMEM lane m = token m; each thread
// reads its token's z row (tcgen05.ld 32x32b) and packs the codes of the
// tables in the tile from registers.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cuda_bf16.h>

#include "hash_kernels.cuh"

namespace lffn_gpu {

struct DenseParams {
  const float* x;        // [n x d_in]
  const double* wt64;    // [ncols x d_in] float64 W^T of the slice (exact fixups)
  int64_t n;
  int d_in;
  int col_begin;         // first z column of the context's table slice (kb * tau)
  int ncols;             // columns of the slice ((ke - kb) * tau)
  int ntile;             // N of the MMA (multiple of 16 and of tau, <= 256)
  int tau;
  int scaled;
  double* z_out;         // optional [n x code_width] (slice columns only)
  int code_width;
  uint32_t* codes;       // [n x hl]
  float* coeff;          // [n x hl]
  int* flag;
  // |z| < fix_scale * ||x_t||_2 * ||w_c||_2 is recomputed exactly: a
  // rigorous bound on the split-precision chain error (dense_fix_scale)
  float fix_scale;
  const float* xnorm;    // [n] ||x_t||_2 (rounded up), written by the x split
  const float* wnorm;    // [ncols] ||W[:, c]||_2 of the slice (rounded up)
  uint2* fix_list;       // deferred exact recomputations {token, slice column}
  int* fix_count;        // entries appended (reset by dense_split_x_kernel)
  int fix_cap;           // capacity; a CTA that finds the list full fixes up inline
};

namespace umma {

constexpr int BM = 128;
constexpr int kRowBytes = 64;             // max bytes per operand row per stage

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t instr_desc_tf32(int m, int n) {
  uint32_t d = 0;
  d |= 1u << 4;                      // D format F32
  d |= 2u << 7;                      // A format TF32
  d |= 2u << 10;                     // B format TF32
  // a/b K-major (bits 15, 16 = 0), no negate, dense
  d |= uint32_t(n >> 3) << 17;       // N >> 3
  d |= uint32_t(m >> 4) << 24;       // M >> 4
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ uint32_t instr_desc_bf16(int m, int n) {
  uint32_t d = 0;
  d |= 1u << 4;                      // D format F32
  d |= 1u << 7;                      // A format BF16 (kind::f16)
  d |= 1u << 10;                     // B format BF16
  d |= uint32_t(n >> 3) << 17;       // N >> 3
  d |= uint32_t(m >> 4) << 24;       // M >> 4
  return d;
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n"
      ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

__device__ __forceinline__ float tf32_rn(float f) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(f));
  return __uint_as_float(r);
}

}  // namespace umma

// The tensor core accumulates with truncation, so the error of a long MMA
// chain grows linearly (3.2e-5 at c2 with one chain of 288 MMAs).  K is cut
// into kSegs segments accumulated in separate TMEM columns and summed in fp32
// round-to-nearest in the epilogue.  Every accumulation step truncates by at
// most 2^-23 of the running partial sum, which is bounded by
// sum_k |x_k w_k| <= ||x||_2 ||w_c||_2 (Cauchy-Schwarz), and the operand
// splits / the fp32 rounding of W add a few 2^-24 of the same sum, so
// |z - z_exact| <= fix_scale * ||x||_2 * ||w_c||_2 with
// fix_scale = (steps per segment + 48) * 2^-23 (dense_fix_scale); every z
// inside that band is recomputed exactly, so the codes are bit-exact for any
// input scale and width (c2: band ~6e-4 at ||x|| = 27.7, observed error
// 1.7e-5).
constexpr int kSegs = 2;
inline float dense_fix_scale(int d_in) {
  const int steps = ((d_in + 15) / 16) * 6 / kSegs + 48;
  return float(steps) * 1.1920929e-7f;  // 2^-23
}

// tcgen05.ld 32x32b.xN: N consecutive TMEM columns of this thread's lane
// (no wait; the caller issues tmem_wait_ld() once for a batch).
template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void tmem_ld<1>(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<2>(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
               : "=r"(r[0]), "=r"(r[1]) : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<4>(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<8>(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// TAU consecutive columns as power-of-two pieces (TAU <= 31)
template <int TAU>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[TAU]) {
  int off = 0;
  if constexpr ((TAU & 16) != 0) { tmem_ld<16>(taddr + off, r + off); off += 16; }
  if constexpr ((TAU & 8) != 0) { tmem_ld<8>(taddr + off, r + off); off += 8; }
  if constexpr ((TAU & 4) != 0) { tmem_ld<4>(taddr + off, r + off); off += 4; }
  if constexpr ((TAU & 2) != 0) { tmem_ld<2>(taddr + off, r + off); off += 2; }
  if constexpr ((TAU & 1) != 0) { tmem_ld<1>(taddr + off, r + off); }
}

// z[token][col] exactly as the reference computes it (projection.cpp:186-192):
// float64, k ascending, separately rounded multiply and add.  wt64 is the
// slice's W^T in float64 ([ncols][d_in], contiguous per column).
__device__ __noinline__ double exact_dot(const DenseParams& p, int64_t token, int col) {
  const float* xr = p.x + token * p.d_in;
  const double* wr = p.wt64 + (size_t)col * p.d_in;
  double acc = 0.0;
#pragma unroll 8
  for (int k = 0; k < p.d_in; ++k) acc = __dadd_rn(acc, __dmul_rn((double)__ldg(xr + k), __ldg(wr + k)));
  return acc;
}

// K-major SWIZZLE_64B tile geometry: a row of a stage tile is 64 bytes
// (16 tf32 or 32 bf16); 8-row atoms of 512 bytes.
constexpr int kTmemCols = 256;  // kSegs * NT (two CTAs per SM share the 512 columns)

// Operand splits.  kSplitTf32: x = x_hi + x_lo, W = W_hi + W_lo in tf32
// (kind::tf32, 8-wide K steps), products hi·hi + hi·lo + lo·hi.
// kSplitBf16x3: x = x0 + x1 + x2, W = w0 + w1 + w2 in bf16 (exact for
// normal fp32), kind::f16 with 16-wide K steps, products 00 + 01 + 10 + 02 +
// 11 + 20 -- 25% fewer operand bytes per K than the tf32 split.
// (bf16 x3 with 32-byte rows, SWIZZLE_32B, four 24 KB stages: main loop
// 41 us per CTA vs 26 us with 64-byte rows -- smaller TMA boxes are slower)
enum : int { kSplitTf32 = 0, kSplitBf16x3 = 1 };
template <int SPLIT>
struct SplitTraits;
template <>
struct SplitTraits<kSplitTf32> {
  static constexpr int P = 2, EB = 4, BK = 16, STAGES = 3, ROW = 64;
};
template <>
struct SplitTraits<kSplitBf16x3> {
  static constexpr int P = 3, EB = 2, BK = 32, STAGES = 2, ROW = 64;
};


struct DenseMaps {
  CUtensorMap x[3];  // x planes [max_tokens x d_in]
  CUtensorMap w[3];  // W^T planes [ncols x d_in]
};

// K-major swizzled smem descriptor: ROW = 64 (SWIZZLE_64B, layout 4) or 32
// (SWIZZLE_32B, layout 6) bytes per row, 8-row atoms.
template <int ROW>
__device__ __forceinline__ uint64_t smem_desc_sw(uint32_t addr) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);             // start address
  d |= uint64_t(1) << 16;                          // leading byte offset (unused for swizzled K-major)
  d |= uint64_t((8 * ROW) >> 4) << 32;             // stride byte offset: 8-row atom
  d |= uint64_t(1) << 46;                          // descriptor version (sm100)
  d |= uint64_t(ROW == 64 ? 4 : 6) << 61;          // layout type SWIZZLE_64B / SWIZZLE_32B
  return d;
}

__device__ __forceinline__ long long globaltimer_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// dynamic shared memory of one CTA for an N tile of ntile columns
inline size_t dense_smem_bytes(int ntile, int split) {
  int P, S, R;
  if (split == kSplitTf32) { P = SplitTraits<kSplitTf32>::P; S = SplitTraits<kSplitTf32>::STAGES; R = SplitTraits<kSplitTf32>::ROW; }
  else { P = SplitTraits<kSplitBf16x3>::P; S = SplitTraits<kSplitBf16x3>::STAGES; R = SplitTraits<kSplitBf16x3>::ROW; }
  return size_t(S) * size_t(P) * (size_t(umma::BM) + size_t(ntile)) * size_t(R) + 1024 + 128;
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(umma::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(umma::smem_u32(bar)), "r"(bytes) : "memory");
}

// 128 threads (4 warps), two CTAs per SM.  Thread 0 = TMA producer, thread
// 32 = MMA issuer (commits each stage to its "empty" barrier and, after the
// last, to "done"); then all four warps run the epilogue, thread = token row,
// one table (TAU columns, TAU a compile-time constant) at a time.
template <int TAU, int SPLIT>
__global__ void __launch_bounds__(128, 2)
    dense_tcgen05_kernel(const __grid_constant__ DenseMaps maps, DenseParams p) {
  using namespace umma;
  using TR = SplitTraits<SPLIT>;
  constexpr int P = TR::P, BK = TR::BK, kStages = TR::STAGES, ROW = TR::ROW;
  extern __shared__ __align__(1024) unsigned char dsm_raw[];
  unsigned char* dsm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~uintptr_t(1023));
  const int NT = p.ntile;
  const uint32_t a_bytes = BM * ROW;            // per plane
  const uint32_t b_bytes = uint32_t(NT) * ROW;  // per plane
  const uint32_t slot_bytes = P * (a_bytes + b_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + kStages * slot_bytes);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  // column tiles fastest: the CTAs sharing one x tile run together (x is read
  // from HBM once; the W tiles stay resident in L2)
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int c0 = blockIdx.x * NT;
  int bad = 0;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(kTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int q = 0; q < P; ++q) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.x[q])) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.w[q])) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int nk = (p.d_in + BK - 1) / BK;
  const int nseg = nk < kSegs ? nk : kSegs;  // K segments actually written
  const int64_t cta = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;

  if (tid == 0) {
    // producer: stage kc reuses the slot of stage kc - kStages once its MMAs completed
    const uint32_t tx_bytes = slot_bytes;
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % kStages;
      if (kc >= kStages) mbar_wait(&empty[s], uint32_t(((kc / kStages) - 1) & 1));
      unsigned char* st = dsm + s * slot_bytes;
      mbar_expect_tx(&full[s], tx_bytes);
#pragma unroll
      for (int q = 0; q < P; ++q) {
        tma_load_2d(smem_u32(st + q * a_bytes), &maps.x[q], kc * BK, int(m0), &full[s]);
        tma_load_2d(smem_u32(st + P * a_bytes + q * b_bytes), &maps.w[q], kc * BK, c0, &full[s]);
      }
    }
  } else if (tid == 32) {
    // MMA issuer: per 32-byte K step, tf32: D_seg += x_hi W_hi + x_hi W_lo +
    // x_lo W_hi; bf16x3: D_seg += x0 w0 + x0 w1 + x1 w0 + x0 w2 + x1 w1 + x2 w0
    const uint32_t idesc = SPLIT == kSplitTf32 ? instr_desc_tf32(BM, NT) : instr_desc_bf16(BM, NT);
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % kStages;
      mbar_wait(&full[s], uint32_t((kc / kStages) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int seg = (kc * nseg) / nk;
      const bool seg_first = (kc == 0) || ((kc - 1) * nseg) / nk != seg;
      const uint32_t acc_t = tmem + uint32_t(seg * NT);
      const uint32_t a0 = smem_u32(dsm + s * slot_bytes);
      const uint32_t b0 = a0 + P * a_bytes;
#pragma unroll
      for (int ks = 0; ks < ROW / 32; ++ks) {
        const uint32_t adv = uint32_t(ks) * 32;  // one MMA K step along the 64-byte swizzled row
        const uint32_t acc0 = (!seg_first || ks > 0) ? 1u : 0u;
        if constexpr (SPLIT == kSplitTf32) {
          mma_tf32(acc_t, smem_desc_sw<ROW>(a0 + adv), smem_desc_sw<ROW>(b0 + adv), idesc, acc0);
          mma_tf32(acc_t, smem_desc_sw<ROW>(a0 + adv), smem_desc_sw<ROW>(b0 + b_bytes + adv), idesc, 1u);
          mma_tf32(acc_t, smem_desc_sw<ROW>(a0 + a_bytes + adv), smem_desc_sw<ROW>(b0 + adv), idesc, 1u);
        } else {
          const uint32_t x0 = a0 + adv, x1 = x0 + a_bytes, x2 = x1 + a_bytes;
          const uint32_t w0 = b0 + adv, w1 = w0 + b_bytes, w2 = w1 + b_bytes;
          mma_bf16(acc_t, smem_desc_sw<ROW>(x0), smem_desc_sw<ROW>(w0), idesc, acc0);
          mma_bf16(acc_t, smem_desc_sw<ROW>(x0), smem_desc_sw<ROW>(w1), idesc, 1u);
          mma_bf16(acc_t, smem_desc_sw<ROW>(x1), smem_desc_sw<ROW>(w0), idesc, 1u);
          mma_bf16(acc_t, smem_desc_sw<ROW>(x0), smem_desc_sw<ROW>(w2), idesc, 1u);
          mma_bf16(acc_t, smem_desc_sw<ROW>(x1), smem_desc_sw<ROW>(w1), idesc, 1u);
          mma_bf16(acc_t, smem_desc_sw<ROW>(x2), smem_desc_sw<ROW>(w0), idesc, 1u);
        }
      }
      commit(&empty[s]);
    }
    commit(done);  // tracks completion of every MMA issued above
  }
  __syncwarp();
  mbar_wait(done, 0u);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---- epilogue: thread = token row m0 + 32*warp + lane (its TMEM lane)
  const int64_t token = m0 + tid;
  const bool live = token < p.n;
  const int hl = p.ncols / TAU;
  const uint32_t trow = tmem + (uint32_t(warp * 32) << 16);
  const int ntab = min(NT, p.ncols - c0) / TAU;
  const int k0 = c0 / TAU;
#pragma unroll 1
  for (int t = 0; t < ntab; ++t) {
    // the K-segment partial sums, combined in fp32 with round-to-nearest
    uint32_t r0[TAU], r1[TAU];
    tmem_ld_cols<TAU>(trow + uint32_t(t * TAU), r0);
    if (nseg > 1) tmem_ld_cols<TAU>(trow + uint32_t(NT + t * TAU), r1);
    tmem_wait_ld();
    float z[TAU];
#pragma unroll
    for (int q = 0; q < TAU; ++q)
      z[q] = nseg > 1 ? __fadd_rn(__uint_as_float(r0[q]), __uint_as_float(r1[q])) : __uint_as_float(r0[q]);
    // Near-zero z decide a code bit: they are recomputed exactly (float64,
    // the reference's order and rounding, projection.cpp:186-192) by
    // dense_fixup_kernel, which patches the code bit and z_out, so every code
    // is bit-exact.  Rare (|z| < 1e-4); appended to a list here.
    uint32_t fixmask = 0, forced = 0, forced_sign = 0;
    const float xn = live ? __ldg(p.xnorm + token) * p.fix_scale : 0.f;
#pragma unroll
    for (int q = 0; q < TAU; ++q)
      if (!(fabsf(z[q]) >= xn * __ldg(p.wnorm + c0 + t * TAU + q))) fixmask |= 1u << q;
    if (!live) fixmask = 0;
    if (fixmask) {
      const int cnt = __popc(fixmask);
      const int at = atomicAdd(p.fix_count, cnt);
      if (at + cnt <= p.fix_cap) {
        int i = at;
        for (uint32_t m = fixmask; m; m &= m - 1)
          p.fix_list[i++] = make_uint2(uint32_t(token), uint32_t(c0 + t * TAU + __ffs(m) - 1));
      } else {
        // list full (e.g. an all-zero projection): recompute inline
        for (uint32_t m = fixmask; m; m &= m - 1) {
          const int q = __ffs(m) - 1;
          const double zd = exact_dot(p, token, c0 + t * TAU + q);
          if (zd >= 0.0) forced_sign |= 1u << q;
          if (p.z_out) p.z_out[token * p.code_width + p.col_begin + c0 + t * TAU + q] = zd;
        }
        forced = fixmask;
      }
    }
    if (!live) continue;
    uint32_t code = 0;
    float den = 1.f, sum_abs = 0.f;
    bool finite = true;
#pragma unroll
    for (int q = 0; q < TAU; ++q) {
      const float zf = z[q];
      finite = finite && isfinite(zf);
      code |= (zf >= 0.f ? 1u : 0u) << q;
      const float a = fabsf(zf);
      sum_abs += a;
      // weight factors in fp32 (z itself carries ~1e-5 of tensor-core error)
      den *= a < 18.5f ? 1.f + __expf(-2.f * a) : 1.f;
    }
    code = (code & ~forced) | (forced_sign & forced);
    if (!finite) bad |= 2;
    if (p.z_out) {
#pragma unroll
      for (int q = 0; q < TAU; ++q)
        if (!((forced >> q) & 1u)) p.z_out[token * p.code_width + p.col_begin + c0 + t * TAU + q] = (double)z[q];
    }
    const float w = __frcp_rn(den);
    p.codes[token * hl + k0 + t] = code;
    p.coeff[token * hl + k0 + t] = p.scaled ? w * sum_abs : w;
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols)
                 : "memory");
  }
  if (bad) atomicOr(p.flag, bad);
}

// Per-call split of x into tf32 hi / lo operands (+ the finiteness check of
// the projection input, projection.cpp:172).
// ||v||_2 of one row by a warp (float64 sum of squares), rounded up so the
// fixup band stays a bound
__device__ __forceinline__ float warp_row_norm(double ss) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  return __double2float_ru(sqrt(ss) * (1.0 + 1e-12));
}

// x -> tf32 hi / lo planes (one warp per row) and ||x_t||_2
__global__ void dense_split_x_kernel(const float* __restrict__ x, int64_t n, int d_in,
                                     float* __restrict__ xhi, float* __restrict__ xlo,
                                     float* __restrict__ xnorm, int* flag, int* fix_count) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *fix_count = 0;  // for the GEMM launched next
  const int lane = threadIdx.x & 31;
  int bad = 0;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double ss = 0.0;
    for (int c = lane; c < d_in / 4; c += 32) {
      const int64_t i = row * (d_in / 4) + c;
      const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
      if (!isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w)) bad = 1;
      ss += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
      float4 h, l;
      h.x = umma::tf32_rn(v.x); l.x = umma::tf32_rn(v.x - h.x);
      h.y = umma::tf32_rn(v.y); l.y = umma::tf32_rn(v.y - h.y);
      h.z = umma::tf32_rn(v.z); l.z = umma::tf32_rn(v.z - h.z);
      h.w = umma::tf32_rn(v.w); l.w = umma::tf32_rn(v.w - h.w);
      reinterpret_cast<float4*>(xhi)[i] = h;
      reinterpret_cast<float4*>(xlo)[i] = l;
    }
    const float nr = warp_row_norm(ss);
    if (lane == 0) xnorm[row] = nr;
  }
  if (bad) atomicOr(flag, 1);
}

// Recomputation of the listed z inside the error band, one warp per entry:
// the lanes form the d_in products (coalesced loads, all in flight).  With a
// z output requested (SERIAL) they go to shared memory and lane 0 sums them
// in order -- float64, k ascending, separately rounded multiply and add,
// exactly as projection.cpp:186-192, so z is bit-identical; otherwise the
// warp sums them as a float64 tree (error ~1e-16 of the magnitudes, far
// below the 1e-5 band in which the north star lets a code bit differ), 31
// lanes no longer waiting on lane 0's 768-step chain.  Patches the code bit
// (atomics: several entries can share a code word) and z_out.  (One thread
// per entry with its own serial chain measured slower: 84 vs 46 us at c2.)
constexpr int kFixupWarps = 4;
template <bool SERIAL>
__global__ void __launch_bounds__(32 * kFixupWarps) dense_fixup_kernel(DenseParams p) {
  extern __shared__ double fix_prod[];  // SERIAL: [kFixupWarps][d_in]
  const int lane = threadIdx.x & 31;
  double* prod = fix_prod + size_t(threadIdx.x >> 5) * p.d_in;
  const int cnt = min(*p.fix_count, p.fix_cap);
  const int hl = p.ncols / p.tau;
  for (int i = blockIdx.x * kFixupWarps + (threadIdx.x >> 5); i < cnt; i += gridDim.x * kFixupWarps) {
    const uint2 e = p.fix_list[i];
    const int64_t token = e.x;
    const int col = int(e.y);
    const float* xr = p.x + token * p.d_in;
    const double* wr = p.wt64 + (size_t)col * p.d_in;
    double acc = 0.0;
    if constexpr (SERIAL) {
      for (int k = lane; k < p.d_in; k += 32) prod[k] = __dmul_rn((double)__ldg(xr + k), __ldg(wr + k));
      __syncwarp();
      if (lane == 0) {
#pragma unroll 16
        for (int k = 0; k < p.d_in; ++k) acc = __dadd_rn(acc, prod[k]);
      }
      __syncwarp();
    } else {
      for (int k = lane; k < p.d_in; k += 32) acc = fma((double)__ldg(xr + k), __ldg(wr + k), acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    }
    if (lane == 0) {
      unsigned int* word = reinterpret_cast<unsigned int*>(p.codes + token * hl + col / p.tau);
      const unsigned int bit = 1u << (col % p.tau);
      if (acc >= 0.0) atomicOr(word, bit);
      else atomicAnd(word, ~bit);
      if (p.z_out) p.z_out[token * p.code_width + p.col_begin + col] = acc;
    }
  }
}

// bf16x3 split: v = v0 + v1 + v2 exactly (normal fp32), each bf16 RN.
__device__ __forceinline__ void split_bf16x3(float v, __nv_bfloat16& b0, __nv_bfloat16& b1,
                                             __nv_bfloat16& b2) {
  b0 = __float2bfloat16_rn(v);
  const float r1 = v - __bfloat162float(b0);
  b1 = __float2bfloat16_rn(r1);
  b2 = __float2bfloat16_rn(r1 - __bfloat162float(b1));
}

// x -> bf16 x3 planes (one warp per row) and ||x_t||_2
__global__ void dense_split_x_bf16x3_kernel(const float* __restrict__ x, int64_t n, int d_in,
                                            __nv_bfloat16* __restrict__ x0,
                                            __nv_bfloat16* __restrict__ x1,
                                            __nv_bfloat16* __restrict__ x2,
                                            float* __restrict__ xnorm, int* flag,
                                            int* fix_count) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *fix_count = 0;  // for the GEMM launched next
  const int lane = threadIdx.x & 31;
  int bad = 0;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double ss = 0.0;
    for (int c = lane; c < d_in / 4; c += 32) {
      const int64_t i = row * (d_in / 4) + c;
      const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
      if (!isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w)) bad = 1;
      ss += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
      __nv_bfloat16 a[4], b[4], c3[4];
      split_bf16x3(v.x, a[0], b[0], c3[0]);
      split_bf16x3(v.y, a[1], b[1], c3[1]);
      split_bf16x3(v.z, a[2], b[2], c3[2]);
      split_bf16x3(v.w, a[3], b[3], c3[3]);
      reinterpret_cast<uint2*>(x0)[i] = *reinterpret_cast<const uint2*>(a);
      reinterpret_cast<uint2*>(x1)[i] = *reinterpret_cast<const uint2*>(b);
      reinterpret_cast<uint2*>(x2)[i] = *reinterpret_cast<const uint2*>(c3);
    }
    const float nr = warp_row_norm(ss);
    if (lane == 0) xnorm[row] = nr;
  }
  if (bad) atomicOr(flag, 1);
}

__global__ void dense_split_weights_bf16x3_kernel(const double* __restrict__ W, int d_in,
                                                  int code_width, int col_begin, int ncols,
                                                  __nv_bfloat16* __restrict__ w0,
                                                  __nv_bfloat16* __restrict__ w1,
                                                  __nv_bfloat16* __restrict__ w2,
                                                  double* __restrict__ wt64) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)ncols * d_in) return;
  const int col = int(i / d_in), k = int(i % d_in);
  const double wd = W[(int64_t)k * code_width + col_begin + col];
  wt64[i] = wd;
  split_bf16x3((float)wd, w0[i], w1[i], w2[i]);
}

// One-time split of W (d_in x ncols slice, row-major, float64) into the
// transposed tf32 hi / lo operands.
__global__ void dense_split_weights_kernel(const double* __restrict__ W, int d_in, int code_width,
                                           int col_begin, int ncols, float* __restrict__ wt_hi,
                                           float* __restrict__ wt_lo, double* __restrict__ wt64) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)ncols * d_in) return;
  const int col = int(i / d_in), k = int(i % d_in);
  const double wd = W[(int64_t)k * code_width + col_begin + col];
  wt64[i] = wd;
  const float w = (float)wd;
  const float hi = umma::tf32_rn(w);
  wt_hi[i] = hi;
  wt_lo[i] = umma::tf32_rn(w - hi);
}

}  // namespace lffn_gpu
