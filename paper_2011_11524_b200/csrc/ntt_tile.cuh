// Shared-memory column transforms for sm_100a.
//
// A "tile" is W independent columns of length R = 2^LOGR held in shared memory.
// tile_dif runs the reference's Gentleman-Sande DIF on every column (natural
// order in, bit-reversed out; reference ntt.cpp:29-50) and tile_dit the
// Cooley-Tukey DIT (bit-reversed in, natural out, unscaled; ntt.cpp:52-73).
// The radix-2 stages are grouped into register-resident rounds of up to three
// stages (radix-8 blocks): each thread loads 8 elements of one column, runs the
// stages in registers, and writes back — one shared-memory round trip per three
// stages instead of per stage.
//
// Twiddles come from a shared table tw[k] = omega_R^k (k < R/2) in Shoup form;
// the stage with span M uses omega_M^j = tw[j * R / M] exactly like the
// reference's flat stage slices (ntt.hpp:10-19). The column -> (prime, table)
// mapping is a functor so one tile can carry both primes.
#pragma once
#include "modarith.cuh"

namespace dmg {

// Row-major [r][w] with an XOR swizzle on the column so that both row-wise
// (S >= W passes) and column-wise (S == 1 pass) global<->shared copies are
// bank-conflict free.
template <int W>
struct SwizzledRows {
  __device__ __forceinline__ int operator()(int r, int w) const { return r * W + (w ^ (r & (W - 1))); }
};
// Column-major [w][r] (each column contiguous): used by the one-CTA-per-product kernel.
template <int LOGR>
struct ContigColumns {
  __device__ __forceinline__ int operator()(int r, int w) const { return (w << LOGR) + r; }
};

// Same prime and table for every column.
struct UniformField {
  u64 pv;
  const TwPair* t;
  __device__ __forceinline__ u64 p(int) const { return pv; }
  __device__ __forceinline__ const TwPair* tw(int) const { return t; }
};

// One register round of DIF covering spans 2^MLOG down to 2^(MLOG-E+1).
template <int LOGR, int MLOG, int E, int W, class L, class F>
__device__ __forceinline__ void dif_round(u64* s, const L& idx, const F& fld, int tid, int nt) {
  constexpr int R = 1 << LOGR, NE = 1 << E, STRIDE = 1 << (MLOG - E);
  constexpr int NG = (R >> E) * W;
  for (int g = tid; g < NG; g += nt) {
    const int w = g % W;
    const int q = g / W;
    const int j0 = q & (STRIDE - 1);
    const int base = ((q >> (MLOG - E)) << MLOG) + j0;
    const u64 p = fld.p(w);
    const TwPair* tw = fld.tw(w);
    u64 v[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) v[i] = s[idx(base + i * STRIDE, w)];
#pragma unroll
    for (int st = 0; st < E; ++st) {
      const int half = NE >> (st + 1);
      const int mlog = MLOG - st;  // span of this stage is 2^mlog
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        if (i & half) continue;
        const int j = (j0 + i * STRIDE) & ((1 << (mlog - 1)) - 1);
        bfly_dif(v[i], v[i + half], tw[j << (LOGR - mlog)], p);
      }
    }
#pragma unroll
    for (int i = 0; i < NE; ++i) s[idx(base + i * STRIDE, w)] = v[i];
  }
}

// One register round of DIT covering spans 2^(ALOG+1) up to 2^(ALOG+E).
template <int LOGR, int ALOG, int E, int W, class L, class F>
__device__ __forceinline__ void dit_round(u64* s, const L& idx, const F& fld, int tid, int nt) {
  constexpr int R = 1 << LOGR, NE = 1 << E, STRIDE = 1 << ALOG;
  constexpr int NG = (R >> E) * W;
  for (int g = tid; g < NG; g += nt) {
    const int w = g % W;
    const int q = g / W;
    const int j0 = q & (STRIDE - 1);
    const int base = ((q >> ALOG) << (ALOG + E)) + j0;
    const u64 p = fld.p(w);
    const TwPair* tw = fld.tw(w);
    u64 v[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) v[i] = s[idx(base + i * STRIDE, w)];
#pragma unroll
    for (int st = 0; st < E; ++st) {
      const int d = 1 << st;
      const int mlog = ALOG + st + 1;
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        if (i & d) continue;
        const int j = (j0 + i * STRIDE) & ((1 << (mlog - 1)) - 1);
        bfly_dit(v[i], v[i + d], tw[j << (LOGR - mlog)], p);
      }
    }
#pragma unroll
    for (int i = 0; i < NE; ++i) s[idx(base + i * STRIDE, w)] = v[i];
  }
}

template <int LOGR, int MLOG, int W, class L, class F>
__device__ __forceinline__ void dif_rounds(u64* s, const L& idx, const F& fld, int tid, int nt) {
  if constexpr (MLOG > 0) {
    constexpr int E = MLOG >= 3 ? 3 : MLOG;
    dif_round<LOGR, MLOG, E, W>(s, idx, fld, tid, nt);
    __syncthreads();
    dif_rounds<LOGR, MLOG - E, W>(s, idx, fld, tid, nt);
  }
}

template <int LOGR, int ALOG, int W, class L, class F>
__device__ __forceinline__ void dit_rounds(u64* s, const L& idx, const F& fld, int tid, int nt) {
  if constexpr (ALOG < LOGR) {
    constexpr int E = (LOGR - ALOG) >= 3 ? 3 : (LOGR - ALOG);
    dit_round<LOGR, ALOG, E, W>(s, idx, fld, tid, nt);
    __syncthreads();
    dit_rounds<LOGR, ALOG + E, W>(s, idx, fld, tid, nt);
  }
}

// Full column transforms. Caller must __syncthreads() before (data and table
// resident); both end with a barrier (none when LOGR == 0: identity).
template <int LOGR, int W, class L, class F>
__device__ __forceinline__ void tile_dif(u64* s, const L& idx, const F& fld, int tid, int nt) {
  dif_rounds<LOGR, LOGR, W>(s, idx, fld, tid, nt);
}
template <int LOGR, int W, class L, class F>
__device__ __forceinline__ void tile_dit(u64* s, const L& idx, const F& fld, int tid, int nt) {
  dit_rounds<LOGR, 0, W>(s, idx, fld, tid, nt);
}

__device__ __forceinline__ int bitrev(int x, int bits) { return bits ? int(__brev(unsigned(x)) >> (32 - bits)) : 0; }

}  // namespace dmg
