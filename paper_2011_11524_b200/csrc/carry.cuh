// Device helpers for decimal recovery: CRT (reference decimal.cpp:136-152),
// base-B digit split, and the parallel form of the reference's sequential carry
// recurrence (decimal.cpp:154-189).
//
// Parallel carry: every coefficient c_i < p1 p2 < 2^126 < B^3 splits into three
// base-B digits (d0, d1, d2). The product's value is sum_k s_k B^k with
// s_k = d0[k] + d1[k-1] + d2[k-2] <= 3(B-1), so a carry entering limb k is in
// {0, 1, 2} and leaves in {0, 1, 2}. Each limb is a map {0,1,2} -> {0,1,2}
// (6 bits: output for input c at bits [2c, 2c+1]); maps compose associatively,
// so the carries are an ordered scan over maps.
#pragma once
#include "modarith.cuh"

namespace dmg {

constexpr unsigned kIdentityMap = 0x24u;  // c -> c

__device__ __forceinline__ unsigned map_apply(unsigned m, unsigned c) { return (m >> (2 * c)) & 3u; }
// Every map here is monotone (limb maps are, and composition keeps it), so out(0) == out(2)
// means a constant map c -> k (0x15 k). Limb sums sit within 2 of a band edge (B or 2B) with
// probability ~4/B, so nearly every limb map and every composed aggregate is constant:
// DMG_MAP_FAST takes those through a short path and keeps the general bit-field code for
// the rest (the branch is taken by whole warps almost always).
#ifndef DMG_MAP_FAST
#define DMG_MAP_FAST 1
#endif
__device__ __forceinline__ unsigned map_compose_full(unsigned later, unsigned earlier) {
  return map_apply(later, earlier & 3u) | (map_apply(later, (earlier >> 2) & 3u) << 2) |
         (map_apply(later, (earlier >> 4) & 3u) << 4);
}
// later o earlier
__device__ __forceinline__ unsigned map_compose(unsigned later, unsigned earlier) {
#if DMG_MAP_FAST
  if ((later & 3u) == (later >> 4)) return later;  // constant later map
#endif
  return map_compose_full(later, earlier);
}
__device__ __forceinline__ unsigned limb_map_full(u64 s, u64 B) {
  unsigned m = 0;
#pragma unroll
  for (unsigned c = 0; c < 3; ++c) {
    const u64 v = s + c;
    m |= (unsigned(v >= B) + unsigned(v >= 2 * B)) << (2 * c);
  }
  return m;
}
__device__ __forceinline__ unsigned limb_map(u64 s, u64 B) {
#if DMG_MAP_FAST
  // s in [B - 2, B) or [2B - 2, 2B): the carry-in decides; else the constant map of s's band
  if (s - (B - 2) >= 2 && s - (2 * B - 2) >= 2) return (unsigned(s >= B) + unsigned(s >= 2 * B)) * 0x15u;
#endif
  return limb_map_full(s, B);
}

// m = a1 + p1 * REDC_{p2}(r~, (a2 - a1) mod p2) < p1 p2.
__device__ __forceinline__ void crt2(u64 a1, u64 a2, u64 p1, u64 p2, u64 p2p, u64 r_tilde, u64& lo, u64& hi) {
  const u64 diff = mod_sub(a2, a1, p2);
  const u64 q = mont_mul(r_tilde, diff, p2, p2p);
  const u64 l = p1 * q;
  hi = __umul64hi(p1, q);
  lo = l + a1;
  hi += lo < l ? 1ull : 0ull;
}

// c = d0 + d1 B + d2 B^2 (each < B), for c < B^3.
// d2 = floor(c / B^2) from a double-precision estimate (error <= 1 for c < 2^126,
// corrected exactly in 128-bit arithmetic), then (d1, d0) from one 2-by-1 reciprocal
// division of the remainder (< B^2, so the quotient fits one word; reference
// udiv_2by1, decimal.hpp:106-121).
__device__ __forceinline__ void split3(const DivB& d, u64 lo, u64 hi, u64& d0, u64& d1, u64& d2) {
  const double cd = __ull2double_rn(hi) * 18446744073709551616.0 + __ull2double_rn(lo);
  long long q = (long long)(cd * d.inv_b2);
  if (q < 0) q = 0;
  // r = c - q B^2 (two's-complement 128-bit)
  u64 tlo = (u64)q * d.b2lo;
  u64 thi = __umul64hi((u64)q, d.b2lo) + (u64)q * d.b2hi;
  u64 rlo = lo - tlo;
  u64 rhi = hi - thi - (lo < tlo ? 1ull : 0ull);
  // the estimate is off by at most one either way: one predicated correction each
  if ((long long)rhi < 0) {  // r < 0: q was one too large
    --q;
    const u64 s = rlo + d.b2lo;
    rhi += d.b2hi + (s < rlo ? 1ull : 0ull);
    rlo = s;
  }
  if (rhi > d.b2hi || (rhi == d.b2hi && rlo >= d.b2lo)) {  // r >= B^2: q one too small
    ++q;
    rhi -= d.b2hi + (rlo < d.b2lo ? 1ull : 0ull);
    rlo -= d.b2lo;
  }
  d2 = (u64)q;
  // r < B^2: r = d1 B + d0 with d1 < B < 2^64 — one normalized 2-by-1 step
  const unsigned sh = d.shift;
  const u64 n1 = sh ? (rhi << sh) | (rlo >> (64 - sh)) : rhi;
  const u64 n0 = rlo << sh;
  u64 r;
  udiv_2by1(n1, n0, d.d_norm, d.recip, d1, r);
  d0 = r >> sh;
}

__device__ __forceinline__ bool above_cap(u64 lo, u64 hi, u64 cap_lo, u64 cap_hi) {
  return hi > cap_hi || (hi == cap_hi && lo > cap_lo);
}

__device__ __forceinline__ unsigned decimal_len(u64 v) {
  unsigned n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}

// x < 10^8 -> its 8 ASCII digits, most significant in the lowest byte (SWAR:
// 4+4 digit lanes, then pairs, then single digits via reciprocal multiplies).
__device__ __forceinline__ u64 ascii8(unsigned x) {
  const unsigned hi4 = x / 10000u, lo4 = x - hi4 * 10000u;
  const u64 y = (u64)hi4 | ((u64)lo4 << 32);
  const u64 z = ((y * 5243) >> 19) & 0x0000007F0000007Full;  // lane / 100 (exact below 43699)
  const u64 w = z | ((y - z * 100) << 16);
  const u64 t = ((w * 103) >> 10) & 0x000F000F000F000Full;   // lane / 10 (exact below 179)
  return (t | ((w - t * 10) << 8)) | 0x3030303030303030ull;
}

// Write the `len` least-significant decimal digits of v (zero padded) to out[0..len).
// (Measured: a SWAR ascii8-based variant with predicated byte stores was slower here —
// the byte stores, not the divisions, dominate.)
__device__ __forceinline__ void write_digits(char* out, u64 v, unsigned len) {
  // split at 10^9 so the digit loop runs on 32-bit values
  unsigned lo = unsigned(v % 1000000000ull);
  unsigned hi = unsigned(v / 1000000000ull);
  int pos = int(len) - 1;
  for (int k = 0; k < 9 && pos >= 0; ++k, --pos) {
    out[pos] = char('0' + lo % 10u);
    lo /= 10u;
  }
  for (; pos >= 0; --pos) {
    out[pos] = char('0' + hi % 10u);
    hi /= 10u;
  }
}

// ---- eight limbs of a fixed width BE (14..17) as one text run, SWAR ----
// Text bytes are accumulated in registers (all offsets compile-time after unrolling) as
// 2 BE 32-bit words, then stored at the run's byte offset with funnel shifts: 2 BE word
// stores plus at most 6 byte stores instead of 8 BE byte stores and per-digit divisions.
struct TextAcc {
  u64 acc = 0;  // pending bytes, the first at the lowest byte
  int n = 0;    // pending byte count (< 4 between pushes)
  int nw = 0;   // words emitted
};
template <int NW>
__device__ __forceinline__ void text_push(TextAcc& t, unsigned (&W)[NW], unsigned x, int bytes) {
  t.acc |= (u64)x << (8 * t.n);
  t.n += bytes;
  if (t.n >= 4) {
    W[t.nw++] = unsigned(t.acc);
    t.acc >>= 32;
    t.n -= 4;
  }
}
template <int NW>
__device__ __forceinline__ void text_push8(TextAcc& t, unsigned (&W)[NW], u64 x, int bytes) {  // bytes <= 8
  if (bytes > 4) {
    text_push(t, W, unsigned(x), 4);
    text_push(t, W, unsigned(x >> 32), bytes - 4);
  } else {
    text_push(t, W, unsigned(x), bytes);
  }
}

// NL limbs of width BE (highest first) as one text run of NL BE bytes at dst (any alignment):
// the text is built in registers as 32-bit words, stored as aligned words (funnel shifts) with
// the partial words at both ends (shared with the neighbouring runs) byte by byte.
template <int BE, int NL>
__device__ __forceinline__ void print_run(char* dst, const u64 (&v)[NL]) {
  static_assert(BE >= 14 && BE <= 17, "limb width");
  constexpr int TB = NL * BE, NWF = TB / 4, REM = TB % 4;
  unsigned W[NWF + 2];
  TextAcc t;
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const u64 q = v[j] / 100000000ull;  // the digits above the low 8
    const unsigned lo8 = unsigned(v[j] - q * 100000000ull);
    if constexpr (BE == 17) {
      const unsigned d = unsigned(q / 100000000ull);
      text_push(t, W, 0x30u + d, 1);
      text_push8(t, W, ascii8(unsigned(q - (u64)d * 100000000ull)), 8);
    } else {
      text_push8(t, W, ascii8(unsigned(q)) >> (8 * (16 - BE)), BE - 8);
    }
    text_push8(t, W, ascii8(lo8), 8);
  }
  const unsigned tail = unsigned(t.acc);  // the last REM bytes
  const int ph = int(reinterpret_cast<unsigned long long>(dst) & 3);
  unsigned* aw = reinterpret_cast<unsigned*>(dst - ph);
  if (ph == 0) {
#pragma unroll
    for (int i = 0; i < NWF; ++i) aw[i] = W[i];
    for (int b = 0; b < REM; ++b) dst[4 * NWF + b] = char(tail >> (8 * b));
  } else {
    const int sh = 8 * ph;
    for (int b = 0; b < 4 - ph; ++b) dst[b] = char(W[0] >> (8 * b));
#pragma unroll
    for (int i = 1; i < NWF; ++i) aw[i] = __funnelshift_l(W[i - 1], W[i], sh);
    // the last ph bytes of W[NWF - 1], then the REM tail bytes
    const u64 rest = (u64)(W[NWF - 1] >> (32 - sh)) | ((u64)tail << sh);
    char* e = dst + (4 * NWF - ph);
    for (int b = 0; b < ph + REM; ++b) e[b] = char(rest >> (8 * b));
  }
}
template <int BE>
__device__ __forceinline__ void print_run8(char* dst, const u64 (&v)[8]) {
  print_run<BE, 8>(dst, v);
}

// Copy len bytes from shared s to global g with 16-byte stores in the aligned middle.
// Requires (g mod 16) == (s mod 16): callers place the staged text at that offset.
__device__ __forceinline__ void cta_store_bytes(char* g, const char* s, unsigned len, int tid, int nt) {
  unsigned head = unsigned((16 - (reinterpret_cast<unsigned long long>(g) & 15)) & 15);
  if (head > len) head = len;
  for (unsigned i = tid; i < head; i += nt) g[i] = s[i];
  const unsigned nvec = (len - head) / 16;
  const uint4* sv = reinterpret_cast<const uint4*>(s + head);
  uint4* gv = reinterpret_cast<uint4*>(g + head);
  for (unsigned i = tid; i < nvec; i += nt) gv[i] = sv[i];
  for (unsigned i = head + nvec * 16 + tid; i < len; i += nt) g[i] = s[i];
}

// Byte offset of limb k in the most-significant-first output (to_decimal layout,
// reference decimal.cpp:120-134): the top limb unpadded first, then lambda digits each.
__device__ __forceinline__ unsigned long long limb_pos(unsigned long long k, unsigned long long top, unsigned top_len,
                                                       unsigned be) {
  return k == top ? 0 : top_len + (top - 1 - k) * be;
}

// Exclusive ordered scan of maps across a block of NT threads (NT multiple of 32).
// Returns the composition of all earlier threads' maps; *total gets the block composition.
template <int NT>
__device__ __forceinline__ unsigned block_scan_maps(unsigned m, unsigned* smem_warp, unsigned* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned inc = m;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned o = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc = map_compose(inc, o);
  }
  unsigned exc = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) exc = kIdentityMap;
  if (lane == 31) smem_warp[wid] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned acc = kIdentityMap;
    for (int w = 0; w < NT / 32; ++w) {
      const unsigned t = smem_warp[w];
      smem_warp[w] = acc;  // exclusive prefix of warp w
      acc = map_compose(t, acc);
    }
    smem_warp[NT / 32] = acc;
  }
  __syncthreads();
  const unsigned pre = map_compose(exc, smem_warp[wid]);
  if (total) *total = smem_warp[NT / 32];
  __syncthreads();
  return pre;
}

}  // namespace dmg
