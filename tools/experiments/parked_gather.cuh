// parked_gather.cuh -- EXPERIMENT (not built into liblffn_gpu.so): the
// persistent row gather with several tokens per warp in rotation, the idle
// tokens' accumulators parked in shared memory, so a stack larger than L2 is
// streamed from HBM once per park x (resident warps) tokens.
//
// Measured on B200 (tools/gather_sweep.py with LFFN_OPT_GATHER_VARIANT =
// 1000 * park + window while it was wired in; ncu in profiles/r2_parked_gather.md):
//   c3 (268 MB bf16 stack): DRAM reads per launch 5.47 GB -> 3.34 GB (park 2,
//   16-table windows) -> 2.70 GB (park 4), L2 hit rate 52 % -> 69 % -> 75 %,
//   but time 1.08 ms -> 1.20-1.26 ms -> 1.32 ms: the L2 lookups per launch do
//   not change (669 M -> 687 M sectors, 142 M of them arriving over the
//   die-to-die fabric) and the plain walk already runs at the L2's lookup
//   ceiling (620 sectors / ns); the extra loop state costs +34 % instructions.
//   c2 fp32: 0.637 ms plain, 0.715 ms for this loop with park = 1, 0.695 ms
//   with park = 2 .. 4 (32-table windows).
// Conclusion: c3's gather is bound by the L2 lookup rate, not by its HBM
// re-reads; fewer HBM bytes per launch do not make it faster.
//
// To rebuild the experiment: include this header after gather_kernels.cuh in
// lffn_gpu.cu and launch with 8 * (park - 1) * MAXC * VEC / 4 * 32 * 16 +
// 8 * 2 * park * 8 bytes of dynamic shared memory, nk % window == 0.
//
// Reference: lookup_gather_f32 (bench.cpp:182-194), forward_impl's gather
// loop (lookup.cpp:223-268).
#pragma once

#include "gather_kernels.cuh"

namespace lffn_gpu {

// Parked-accumulator walk (round 2): the persistent row kernel with `park`
// tokens per warp in rotation.  The table walk is cut into windows of
// `window` tables; a warp walks window w for each of its tokens in turn,
// keeping the active token's fp32 accumulators in registers and the others'
// parked in shared memory (one 128-bit store + load per lane and chunk at a
// switch), then moves to window w + 1.  All resident warps therefore work
// inside the same few windows of the stack for park x as long, and a stack
// larger than L2 is streamed from HBM once per park x (resident warps)
// tokens instead of once per (resident warps) tokens -- without the
// register cost of several tokens' accumulators (the token-blocked walk,
// measured slower) and without a round trip of partial y through L2 (the
// table-group walk, measured slower).  Per token the tables are still
// accumulated in ascending (or, on reversed rounds, descending) order in one
// fp32 register chain, so y equals the plain walk's for the same direction.
//
// Rotation: window w visits the batch's tokens in the order (-w) mod nb,
// (-w) + 1, ...; the token at position 0 is the one the previous window left
// in the registers, and the token at position i >= 1 is swapped in from slot
// i - 1, which receives the accumulators of position i - 1: nb - 1 slots.
// Shared memory per warp: (park - 1) x MAXC x VEC x 32 floats, then per-slot
// (token, part) words.
template <typename TT, int MAXC, int MINB, bool PM>
__global__ void __launch_bounds__(256, MINB)
    gather_row_parked_kernel(GatherParams p, int warps_per_token, int park, int window) {
  constexpr int VEC = Raw<TT>::VEC;
  constexpr int CHUNK = 32 * VEC;
  constexpr int Q4 = MAXC * VEC / 4;  // float4 per lane per accumulator set
  constexpr int TIF = 4;
  extern __shared__ __align__(16) unsigned char park_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float4* slots = reinterpret_cast<float4*>(park_raw) + (size_t)wib * (park - 1) * Q4 * 32 + lane;
  int64_t* slot_tok = reinterpret_cast<int64_t*>(park_raw + (size_t)8 * (park - 1) * Q4 * 32 * sizeof(float4)) +
                      wib * 2 * park;
  int64_t* slot_part = slot_tok + park;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nchunks = (p.d_out + CHUNK - 1) / CHUNK;
  const TT* T = reinterpret_cast<const TT*>(p.T);
  const int64_t tstride = (int64_t)p.rows * p.d_out;
  const int64_t nitems = p.n * warps_per_token;
  const int nwin = p.nk / window;  // launcher: nk % window == 0, window % 4 == 0
  const int gpw = window >> 2;     // 4-table record groups per window
  int bad = 0;
  for (int64_t base = gwarp; base < nitems; base += nwarps * park) {
    const int64_t left = (nitems - base + nwarps - 1) / nwarps;
    const int nb = left < park ? (int)left : park;
    __syncwarp();
    if (lane < nb) {
      const int64_t item = base + (int64_t)lane * nwarps;
      int64_t token, part;
      if constexpr (PM) {
        part = item / p.n;
        token = item - part * p.n;
      } else {
        token = item / warps_per_token;
        part = item - token * warps_per_token;
      }
      slot_tok[lane] = token;
      slot_part[lane] = part;
    }
    __syncwarp();
    const bool rev = p.reverse_odd_rounds && ((base / (nwarps * park)) & 1);
    // first table of record group g of window w (reversed batches walk the
    // groups from the end, the four tables of a group ascending)
    auto kg_of = [&](int w, int g) {
      const int k = w * window + 4 * g;
      return rev ? p.nk - 4 - k : k;
    };
    float acc[MAXC][VEC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[c][v] = 0.f;
    const int kstep = rev ? -4 : 4;
    int j = 0;
    int64_t tok = slot_tok[0];
    int64_t roff = tok * p.ld;  // record offset of the segment's token
    int colbase = (int)slot_part[0] * MAXC * CHUNK + lane * VEC;
    uint4 cc = __ldg(reinterpret_cast<const uint4*>(p.codes + roff + kg_of(0, 0)));
    float4 ww = __ldg(reinterpret_cast<const float4*>(p.coeff + roff + kg_of(0, 0)));
    for (int w = 0; w < nwin; ++w) {
      const int kbase = kg_of(w, 0);
      for (int i = 0; i < nb; ++i) {
        // the segment after this one: the next token of this window, or the
        // token left in the registers (this one's last position) in window w + 1
        int i2 = i + 1, w2 = w, j2 = (j + 1 == nb) ? 0 : j + 1;
        if (i2 == nb) {
          i2 = 0;
          w2 = w + 1;
          j2 = j;
        }
        const bool more = w2 < nwin;
        const int64_t tok2 = more ? slot_tok[j2] : tok;
        const int64_t roff2 = tok2 * p.ld;
        const int64_t next_first = roff2 + (more ? kg_of(w2, 0) : 0);
        for (int g = 0; g < gpw; ++g) {
          const int kg = kbase + kstep * g;
          uint4 cn = cc;
          float4 wn = ww;
          if (g + 1 < gpw || more) {
            const int64_t off = (g + 1 < gpw) ? roff + kg + kstep : next_first;
            cn = __ldg(reinterpret_cast<const uint4*>(p.codes + off));
            wn = __ldg(reinterpret_cast<const float4*>(p.coeff + off));
          }
          const uint32_t code4[4] = {cc.x, cc.y, cc.z, cc.w};
          const float w4[4] = {ww.x, ww.y, ww.z, ww.w};
          const bool fastw = p.bf16w && coeffs_bf16_exact<4>(w4);
          uint4 raw[TIF][MAXC];
#pragma unroll
          for (int q = 0; q < TIF; ++q) {
            LFFN_DCHECK(code4[q] < (uint32_t)p.rows && kg + q < p.nk && kg + q >= 0);
            const TT* rp = T + (kg + q) * tstride + (int64_t)code4[q] * p.d_out + colbase;
#pragma unroll
            for (int c = 0; c < MAXC; ++c)
              raw[q][c] = (colbase + c * CHUNK < p.d_out) ? Raw<TT>::load(rp + c * CHUNK) : make_uint4(0u, 0u, 0u, 0u);
          }
          if (sizeof(TT) == 2 && fastw) {
#pragma unroll
            for (int q = 0; q < TIF; ++q)
#pragma unroll
              for (int c = 0; c < MAXC; ++c)
                Raw<TT>::fma_bf16w(acc[c], (uint16_t)(__float_as_uint(w4[q]) >> 16), raw[q][c]);
          } else {
#pragma unroll
            for (int q = 0; q < TIF; ++q)
#pragma unroll
              for (int c = 0; c < MAXC; ++c) Raw<TT>::fma(acc[c], w4[q], raw[q][c]);
          }
          cc = cn;
          ww = wn;
        }
        // segment (w, i) of token j is done
        if (w == nwin - 1) {
          float* yr = p.y + tok * p.d_out;
#pragma unroll
          for (int c = 0; c < MAXC; ++c) {
            const int col = colbase + c * CHUNK;
            if (col < p.d_out) {
              if (p.accumulate) {
#pragma unroll
                for (int v = 0; v < VEC; v += 4) {
                  const float4 a = *reinterpret_cast<const float4*>(yr + col + v);
                  acc[c][v] += a.x; acc[c][v + 1] += a.y; acc[c][v + 2] += a.z; acc[c][v + 3] += a.w;
                }
              }
#pragma unroll
              for (int v = 0; v < VEC; ++v)
                if (!isfinite(acc[c][v])) bad = 4;
#pragma unroll
              for (int v = 0; v < VEC; v += 4)
                *reinterpret_cast<float4*>(yr + col + v) =
                    make_float4(acc[c][v], acc[c][v + 1], acc[c][v + 2], acc[c][v + 3]);
            }
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[c][v] = 0.f;
          }
        } else if (w == 0 && i < nb - 1) {
          LFFN_DCHECK(i < park - 1);
#pragma unroll
          for (int c = 0; c < MAXC; ++c)
#pragma unroll
            for (int v = 0; v < VEC; v += 4) {
              slots[(size_t)(i * Q4 + c * (VEC / 4) + v / 4) * 32] =
                  make_float4(acc[c][v], acc[c][v + 1], acc[c][v + 2], acc[c][v + 3]);
              acc[c][v] = acc[c][v + 1] = acc[c][v + 2] = acc[c][v + 3] = 0.f;
            }
        }
        if (more && w2 > 0 && i2 > 0) {
          // position i2 of a later window: its accumulators wait in slot
          // i2 - 1, which takes those of position i2 - 1 (just walked)
          LFFN_DCHECK(i2 - 1 < park - 1);
#pragma unroll
          for (int c = 0; c < MAXC; ++c)
#pragma unroll
            for (int v = 0; v < VEC; v += 4) {
              float4* s = slots + (size_t)((i2 - 1) * Q4 + c * (VEC / 4) + v / 4) * 32;
              const float4 in = *s;
              *s = make_float4(acc[c][v], acc[c][v + 1], acc[c][v + 2], acc[c][v + 3]);
              acc[c][v] = in.x; acc[c][v + 1] = in.y; acc[c][v + 2] = in.z; acc[c][v + 3] = in.w;
            }
        }
        if (more) {
          j = j2;
          tok = tok2;
          roff = roff2;
          colbase = (int)slot_part[j2] * MAXC * CHUNK + lane * VEC;
        }
      }
    }
  }
  (void)nchunks;
  if (bad) atomicOr(p.flag, bad);
}

}  // namespace lffn_gpu
