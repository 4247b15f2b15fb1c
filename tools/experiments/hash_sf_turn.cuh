// hash_sf_turn.cuh -- EXPERIMENT (not built into liblffn_gpu.so): K1f as one
// persistent CTA of twelve warps per SM whose float64 phases take turns
// through a per-scheduler lock in shared memory, with clock64() laps around
// the phases of one warp.
//
// Measured on B200 (tools/hash_turns.py while it was wired in as
// LFFN_OPT_HASH_EXACT = 2; c2 / c3, ms):
//   hash_sf_kernel (64-thread CTAs, 12 warps per SM)      0.096 / 0.336
//   this kernel, no lock, 12 / 8 / 4 warps per SM          0.113 / 0.399, 0.127 / 0.453, 0.186 / 0.668
//   lock per scheduler (warp & 3), spinning or with pauses 0.25-0.27 / 0.99-1.06
//   lock per warp / 3                                      0.317 / 1.217
// The lock makes it 2.3x slower: a warp that waits for the pipe gives up the
// overlap of its own load / transpose / epilogue phases with nothing gained,
// because the float64 phases are less than half of a token's time.  Cycles
// per token of one warp alone on its scheduler (c2, 4 warps per SM): x load
// and conversion 1500-2000, first butterflies 700 (of which ~450 the sign-mask
// load), three transposes 2400-2700, the other butterflies 5100-5500 (1728
// float64 adds: 3 cycles each including the flips and two more mask loads),
// epilogue and codes 4300-4800 -- 14.7 k cycles, 5.5 k of them on the float64
// pipe; with three warps per scheduler the phases stretch to 2400 / 1100 /
// 4200 / 9500 / 6700.  The pipe is 60 % busy because a token spends most of
// its time outside it, not because the warps collide on it.
//
// To rebuild: include after hash_sf_kernel.cuh in lffn_gpu.cu, launch one
// 384-thread CTA per SM with 12 * (PAD + WORDS) * 8 + 16 bytes of dynamic
// shared memory; HashSfParams needs an `unsigned ahead_ns` field (0: no lock,
// 1: lock per warp / 3, 2: spin, 3-999: pause in ns, >= 1000: no lock,
// >= 2000: print the laps) and sf_epilogue a trailing `long long* dbg` lap
// array.
#pragma once

#include <cstdio>

#include "hash_sf_kernel.cuh"

namespace lffn_gpu {

// K1f with the float64 phases taking turns (D = 2048).  One CTA of twelve
// warps per SM (a token per warp, the warps walking the tokens with a grid
// stride); the three warps of a scheduler (warp & 3) pass a lock in shared
// memory around so that one of them at a time runs a butterfly phase at the
// full rate of the scheduler's float64 pipe while the other two load,
// transpose or pack codes.  Without the lock, warps that share the pipe slow
// each other down, leave their float64 phases together and then all sit in
// load / transpose / epilogue phases with the pipe idle (it is 60 % busy in
// hash_sf_kernel, and the kernel runs slower on L2-resident inputs than on
// cold ones: less jitter, more lock-step).
template <int LIVE>
__global__ void __launch_bounds__(384, 1) hash_sf_turn_kernel(HashSfParams p) {
  constexpr int LOGD = 11;
  using Gm = SfGeom<LOGD>;
  constexpr int TPT = Gm::TPT;
  extern __shared__ double smem[];
  constexpr int SLOT = Gm::PAD + Gm::WORDS;
  const int slot = threadIdx.x >> 5;
  const int t = threadIdx.x & 31;
  double* sm = smem + (size_t)slot * SLOT;
  uint32_t* words = reinterpret_cast<uint32_t*>(sm + Gm::PAD);
  int* lock = reinterpret_cast<int*>(smem + 12 * SLOT) + (p.ahead_ns == 1 ? slot / 3 : (slot & 3));
  const bool locking = p.ahead_ns != 0 && p.ahead_ns < 1000;  // (>= 1000: no lock; >= 2000: print phase cycles)
  if (threadIdx.x < 4) reinterpret_cast<int*>(smem + 12 * SLOT)[threadIdx.x] = 0;
  __syncthreads();
  auto acquire = [&]() {
    if (!locking) return;
    if (t == 0) {
      while (atomicCAS(lock, 0, 1) != 0) {
        if (p.ahead_ns > 2) __nanosleep(p.ahead_ns);
      }
    }
    __syncwarp();
  };
  auto release = [&]() {
    if (!locking) return;
    __syncwarp();
    if (t == 0) atomicExch(lock, 0);
  };
  auto token_sync = [] { __syncwarp(); };
  int bad = 0;
  long long tm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long em[4] = {0, 0, 0, 0};
  long long t0 = clock64();
  int ntok = 0;
  auto lap = [&](int i) { const long long t1 = clock64(); tm[i] += t1 - t0; t0 = t1; };
  const int nw = blockDim.x >> 5;
#pragma unroll 1
  for (int64_t token = (int64_t)blockIdx.x * nw + slot; token < p.n; token += (int64_t)gridDim.x * nw) {
    double v[64];
    t0 = clock64();
    ++ntok;
    {
      const float* xr = p.x + token * (int64_t)p.d_in;
      float nanacc = 0.f;
      constexpr int LB = LIVE <= 32 ? LIVE : LIVE / 2;
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
    lap(0);
    sf_flip<LIVE>(v, __ldg(p.masks + t));
    acquire();
    sf_stages_live<LIVE>(v);
    release();
    lap(1);
    sf_store_B<LOGD>(sm, v, t);
#pragma unroll 1
    for (int tr = 1; tr <= p.transforms; ++tr) {
      token_sync();
      sf_load_A<LOGD>(sm, v, t);
      token_sync();
      lap(2);
      acquire();
      sf_stages<Gm::B2, 6>(v);
      if (tr < p.transforms) {
        sf_flip<64>(v, __ldg(p.masks + tr * TPT + t));
        sf_stages<0, 6>(v);
        release();
        lap(3);
        sf_store_B<LOGD>(sm, v, t);
      } else {
        release();
        lap(3);
      }
    }
    {
      SfEpilogue e{p.code_width, p.tau, p.kb, p.ke, p.codes, p.coeff};
      sf_epilogue<LOGD, true>(v, sm, words, t, token, e, bad, token_sync, em);
    }
    token_sync();  // the words and small z are read; the buffer may be rewritten
    lap(4);
  }
  if (blockIdx.x == 3 && threadIdx.x == 0 && p.ahead_ns >= 2000)
    printf("tokens %d per token: load+convert %lld | T1a %lld | transposes %lld | butterflies %lld | epilogue+codes %lld (integer pass %lld, rare %lld, words %lld, code loop %lld)\n", ntok,
           tm[0] / ntok, tm[1] / ntok, tm[2] / ntok, tm[3] / ntok, tm[4] / ntok, em[0] / ntok, em[1] / ntok, em[2] / ntok, em[3] / ntok);
  if (bad) atomicOr(p.flag, bad);
}

}  // namespace lffn_gpu
