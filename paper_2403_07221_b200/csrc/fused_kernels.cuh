// fused_kernels.cuh -- K13 (opt-in, LFFN_OPT_FUSED = 1): hash and gather of
// the forward in one persistent, warp-specialised kernel (signflip
// projection, D = 2048, top-1 codes).
//
// Reference path: Projection::forward signflip branch (projection.cpp:200-263)
// -> compute_codes / top1_weight (lookup.cpp:74-100, 185-189) -> the gather
// of forward_impl (lookup.cpp:223-268) / lookup_gather_f32 (bench.cpp:182-194).
//
// Idea: the gather is bound by L2 latency x bytes in flight and leaves most
// issue slots idle, the hash by the fp64 pipe / shared memory; running them
// on the same SM at once could hide the hash.  Measured (c2
// 16384 tokens): slower than the two kernels (1.01 vs 0.82 ms).  Both
// phases want the register file: the gather needs ~16 warps x 128 registers
// of row segments in flight (12 gather warps: 0.81 ms for the walk alone),
// and the hash needs ~4 warps of 64-thread tokens to keep up (0.49 ms
// alone).  Kept for A/B and as the base of a shared-memory-staged gather.
//
// Streaming hooks (unused by default): with `ready` set, a token of chunk c
// is hashed only once ready[c] is non-zero, and after its y row is stored
// the warp bumps done[c] (release).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gather_kernels.cuh"
#include "hash_kernels.cuh"

namespace lffn_gpu {

constexpr int kFlagStreamDev = 64;  // = kFlagStream (lffn_internal.h)

struct FusedParams {
  HashParams h;
  GatherParams g;           // codes / coeff unused (records stay in shared memory)
  int parts;                // column parts per token (walked in turn by the warp)
  const volatile int* ready;  // streaming: per-chunk ready flags (null = all ready)
  int* done;                // streaming: per-chunk finished-token counters
  int64_t chunk_tokens;     // streaming: tokens per chunk
  int64_t spin_limit;       // streaming: give up (flag 8) after this many polls
  int debug_mode;           // tuning: 1 = hash only (no table walk), 2 = walk only (synthetic codes)
};

// (code, coefficient) of table k from the z row in shared memory: the
// reference's sign_code (lookup.cpp:74-79, LSB = coordinate 0, z >= 0 -> 1)
// and top1_weight (lookup.cpp:185-189), exactly as hash_structured_kernel.
__device__ __forceinline__ void fused_table_record(const double* sm, int base, int tau, bool scaled,
                                                   uint32_t& code, float& coeff) {
  code = 0;
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
  coeff = (float)(scaled ? __dmul_rn(w, sum_abs) : w);
}

}  // namespace lffn_gpu

namespace lffn_gpu {
namespace fws {

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
// bounded wait: false after `limit` polls (the caller flags the error)
__device__ __forceinline__ bool bar_wait(uint64_t* b, uint32_t parity, int64_t limit) {
  for (int64_t i = 0; i < limit; ++i) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok) : "r"(su32(b)), "r"(parity) : "memory");
    if (ok) return true;
  }
  return false;
}

}  // namespace fws

// Warp-specialised fused forward: per SM one CTA of 16 warps.  HP pairs of
// hash warps (64 threads per token, 32 float64 coordinates per thread, three
// register phases per D = 2048 transform -- half the registers of K1's
// 64-element phases) write each token's (code, coeff) records into a ring of
// R shared-memory slots; the other 16 - 2*HP warps are gather warps that
// take the tokens round-robin and walk the tables from the slot, keeping
// TIF tables' row segments in flight.  Full / empty mbarriers per slot
// order the ring.  The gather warps never stop issuing row loads for hash
// work, and the hash runs in the issue slots the latency-bound gather
// leaves idle.  Each CTA owns a contiguous token range.
// GWT > 0: that many gather warps (else 16 - 2 HP); ANS > 0: the gather warps
// stage their rows in shared memory (AsyncWalk, ANS stages of one table)
// instead of registers, which leaves the register file to the hash warps.
template <typename TT, int TAU, int MAXC, int HP, int R, int GWT = 0, int ANS = 0>
__global__ void __launch_bounds__(32 * (2 * HP + (GWT > 0 ? GWT : 16 - 2 * HP)), 1)
    fused_ws_kernel(FusedParams fp) {
  extern __shared__ __align__(16) unsigned char fws_smem[];
  constexpr int LOGE = 5;
  constexpr int E = 1 << LOGE;
  constexpr int LOGD = 11;
  constexpr int D = 1 << LOGD;
  constexpr int TPT = D / E;            // 64 threads per token
  constexpr int KMAX = E / TAU + 1;
  constexpr int GW = GWT > 0 ? GWT : 16 - 2 * HP;  // gather warps
  constexpr int VEC = Raw<TT>::VEC;
  constexpr int CHUNK = 32 * VEC;
  constexpr int TIF = 4;
  const HashParams& p = fp.h;
  const GatherParams& g = fp.g;
  const int hl = p.ke - p.kb;
  const int rec_slot = ((hl * 8 + 15) / 16) * 16;  // bytes per ring slot
  uint64_t* full = reinterpret_cast<uint64_t*>(fws_smem);
  uint64_t* empty = full + R;
  double* zbuf = reinterpret_cast<double*>(fws_smem + 16 * R);
  unsigned char* ring = fws_smem + 16 * R + (size_t)HP * padded_len(D) * sizeof(double);

  const int64_t per = (p.n + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per;
  const int64_t rem = p.n - t0;
  const int64_t cnt = rem <= 0 ? 0 : (rem < per ? rem : per);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int64_t kLimit = int64_t(1) << 26;
  int bad = 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < R; ++s) {
      fws::bar_init(full + s, 1);
      fws::bar_init(empty + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp < 2 * HP) {
    // ---------------- hash pairs
    const int q = warp >> 1;
    const int t = threadIdx.x - q * TPT;  // 0..63
    double* sm = zbuf + (size_t)q * padded_len(D);
    auto pair_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(q + 1), "r"(TPT) : "memory"); };
    for (int64_t j = q; j < cnt; j += HP) {
      const int64_t token = t0 + j;
      const int slot = (int)(j % R);
      const uint32_t use = (uint32_t)(j / R);
      if (fp.ready) {
        const int64_t ch = token / fp.chunk_tokens;
        int64_t polls = 0;
        while (fp.ready[ch] == 0) {
          if (++polls > fp.spin_limit) { bad |= kFlagStreamDev; break; }
          __nanosleep(256);
        }
        __threadfence();
      }
      const float* xr = p.x + token * (int64_t)p.d_in;
#pragma unroll 1
      for (int tr = 0; tr < (fp.debug_mode == 2 ? 0 : 3); ++tr) {
        run_first_phase<LOGE, kPreSign>(sm, t, TPT, p, tr, xr, bad, false);
        pair_sync();
        phase_smem<LOGE, LOGE, false, kPreNone>(sm, t, TPT, LOGE, p, tr, nullptr, bad, false);
        pair_sync();
        phase_smem<LOGE, LOGD - 2 * LOGE, false, kPreNone>(sm, t, TPT, 2 * LOGE, p, tr, nullptr, bad,
                                                           tr == 2 && p.code_width == D);
        pair_sync();
      }
      if (p.code_width != D) {
        for (int a = t; a < p.code_width; a += TPT)
          if (!isfinite(sm[spos(a)])) bad |= 2;
      }
      // the slot's previous token must have been consumed
      if (use > 0 && !fws::bar_wait(empty + slot, (use - 1) & 1, kLimit)) bad |= kFlagStreamDev;
      uint2* rec = reinterpret_cast<uint2*>(ring + (size_t)slot * rec_slot);
      const int a_lo = t * E;
      const int a_hi = min(a_lo + E, p.code_width);
      const int k0 = max((a_lo + TAU - 1) / TAU, p.kb);
#pragma unroll
      for (int i = 0; i < KMAX; ++i) {
        const int k = k0 + i;
        if (k < p.ke && k * TAU < a_hi) {
          uint32_t code;
          float w;
          if (fp.debug_mode == 2) {
            code = (uint32_t)((token * 2654435761u + k * 40503u) >> 7) & ((1u << TAU) - 1u);
            w = 1.0f;
          } else {
            fused_table_record(sm, k * TAU, TAU, p.scaled != 0, code, w);
          }
          rec[k - p.kb] = make_uint2(code, __float_as_uint(w));
        }
      }
      pair_sync();  // records complete, z free for the next token
      if (t == 0) fws::bar_arrive(full + slot);
    }
  } else {
    // ---------------- gather warps
    const int gw = warp - 2 * HP;
    const int nchunks = (g.d_out + CHUNK - 1) / CHUNK;
    if constexpr (ANS > 0) {
      using Wk = AsyncWalk<TT, MAXC, 1, ANS>;
      uint4* gring = reinterpret_cast<uint4*>(ring + (size_t)R * rec_slot) + (size_t)gw * ANS * Wk::STAGE;
      const TT* T = reinterpret_cast<const TT*>(g.T);
      const int64_t tstride = (int64_t)g.rows * g.d_out;
      for (int64_t j = gw; j < cnt; j += GW) {
        const int64_t token = t0 + j;
        const int slot = (int)(j % R);
        const uint32_t use = (uint32_t)(j / R);
        if (!fws::bar_wait(full + slot, use & 1, kLimit)) bad |= kFlagStreamDev;
        const uint2* rec = reinterpret_cast<const uint2*>(ring + (size_t)slot * rec_slot);
        float* yr = g.y + token * g.d_out;
        for (int part = 0; part < fp.parts; ++part) {
          const int c0 = part * MAXC;
          bool ok[MAXC];
#pragma unroll
          for (int c = 0; c < MAXC; ++c)
            ok[c] = (c0 + c < nchunks) && (c0 * CHUNK + lane * VEC + c * CHUNK < g.d_out);
          float acc[MAXC][VEC];
#pragma unroll
          for (int c = 0; c < MAXC; ++c)
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[c][v] = 0.f;
          if (fp.debug_mode != 1)
            Wk::walk(gring, T + c0 * CHUNK, tstride, g.d_out, hl, lane, ok, acc,
                     [&](int k) { return rec[k].x; }, [&](int k) { return __uint_as_float(rec[k].y); });
#pragma unroll
          for (int c = 0; c < MAXC; ++c) {
            if (!ok[c]) continue;
            const int col = (c0 + c) * CHUNK + lane * VEC;
#pragma unroll
            for (int v = 0; v < VEC; v += 4) {
              const float4 o = make_float4(acc[c][v], acc[c][v + 1], acc[c][v + 2], acc[c][v + 3]);
              if (!isfinite(o.x) || !isfinite(o.y) || !isfinite(o.z) || !isfinite(o.w)) bad |= 4;
              *reinterpret_cast<float4*>(yr + col + v) = o;
            }
          }
        }
        __syncwarp();
        if (lane == 0) fws::bar_arrive(empty + slot);
      }
    } else {
    const TT* T = reinterpret_cast<const TT*>(g.T);
    const int64_t tstride = (int64_t)g.rows * g.d_out;
    for (int64_t j = gw; j < cnt; j += GW) {
      const int64_t token = t0 + j;
      const int slot = (int)(j % R);
      const uint32_t use = (uint32_t)(j / R);
      if (!fws::bar_wait(full + slot, use & 1, kLimit)) bad |= kFlagStreamDev;
      const uint4* rec4 = reinterpret_cast<const uint4*>(ring + (size_t)slot * rec_slot);
      float* yr = g.y + token * g.d_out;
      for (int part = 0; part < fp.parts; ++part) {
        const int c0 = part * MAXC;
        const int colbase = c0 * CHUNK + lane * VEC;
        bool ok[MAXC];
#pragma unroll
        for (int c = 0; c < MAXC; ++c) ok[c] = (c0 + c < nchunks) && (colbase + c * CHUNK < g.d_out);
        float acc[MAXC][VEC];
#pragma unroll
        for (int c = 0; c < MAXC; ++c)
#pragma unroll
          for (int v = 0; v < VEC; ++v) acc[c][v] = 0.f;
        uint4 r01 = rec4[0], r23 = rec4[1];
        for (int kg = 0; kg < (fp.debug_mode == 1 ? 0 : hl); kg += 4) {
          uint4 n01 = r01, n23 = r23;
          if (kg + 4 < hl) {
            n01 = rec4[(kg + 4) / 2];
            n23 = rec4[(kg + 4) / 2 + 1];
          }
          const uint32_t code4[4] = {r01.x, r01.z, r23.x, r23.z};
          const float w4[4] = {__uint_as_float(r01.y), __uint_as_float(r01.w), __uint_as_float(r23.y),
                               __uint_as_float(r23.w)};
          uint4 raw[TIF][MAXC];
#pragma unroll
          for (int qq = 0; qq < TIF; ++qq) {
            const TT* rp = T + (int64_t)(kg + qq) * tstride + (int64_t)code4[qq] * g.d_out + colbase;
#pragma unroll
            for (int c = 0; c < MAXC; ++c)
              raw[qq][c] = ok[c] ? Raw<TT>::load(rp + c * CHUNK) : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
          for (int qq = 0; qq < TIF; ++qq)
#pragma unroll
            for (int c = 0; c < MAXC; ++c) Raw<TT>::fma(acc[c], w4[qq], raw[qq][c]);
          r01 = n01;
          r23 = n23;
        }
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
          if (!ok[c]) continue;
          const int col = colbase + c * CHUNK;
#pragma unroll
          for (int v = 0; v < VEC; v += 4) {
            const float4 o = make_float4(acc[c][v], acc[c][v + 1], acc[c][v + 2], acc[c][v + 3]);
            if (!isfinite(o.x) || !isfinite(o.y) || !isfinite(o.z) || !isfinite(o.w)) bad |= 4;
            *reinterpret_cast<float4*>(yr + col + v) = o;
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        fws::bar_arrive(empty + slot);  // records read: the slot may be refilled
        if (fp.done) {
          __threadfence_system();
          atomicAdd(fp.done + token / fp.chunk_tokens, 1);
        }
      }
    }
    }
  }
  if (bad) atomicOr(p.flag, bad);
}

}  // namespace lffn_gpu
