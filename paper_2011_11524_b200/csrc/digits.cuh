// ASCII digits -> integers with SWAR arithmetic, from text staged in shared memory
// (the pack step, reference decimal.cpp:102-118). Used by k_pack and k_small.
//
// 32-bit lanes throughout: a limb's <= 20 digits are five 4-digit groups taken from the
// right out of an 8-byte-aligned window with funnel shifts, each converted by two
// multiply-add steps (one IMAD each on 32-bit words, where 64-bit SWAR needs 3-4 per
// multiply and multi-instruction variable shifts).
#pragma once
#include "modarith.cuh"

namespace dmg {

// 4 bytes of shared memory at any byte offset (buf 4-aligned, readable 4 bytes past).
__device__ __forceinline__ unsigned smem_bytes4(const char* buf, int pos) {
  const unsigned* w = reinterpret_cast<const unsigned*>(buf + (pos & ~3));
  return __funnelshift_r(w[0], w[1], (pos & 3) * 8);
}

// Value of 4 ASCII digits (first byte most significant) whose first `skip` bytes are
// treated as '0'; flags any byte outside '0'..'9'.
__device__ __forceinline__ unsigned swar4(unsigned x, int skip, unsigned& bad) {
  const unsigned keep = skip >= 4 ? 0u : (0xFFFFFFFFu << (8 * skip));
  x = (x & keep) | (0x30303030u & ~keep);
  // per byte b: high bit of b (non-ASCII), of b + 0x46 (b > '9'), or clear in
  // (b | 0x80) - 0x30 (b < '0'); no carry or borrow crosses a byte for ASCII bytes
  bad |= (x | (x + 0x46464646u) | ~((x | 0x80808080u) - 0x30303030u)) & 0x80808080u;
  x &= 0x0F0F0F0Fu;
  x = (x * 10u + (x >> 8)) & 0x00FF00FFu;  // bytes 0, 2: 10 d0 + d1, 10 d2 + d3
  return (x * 100u + (x >> 16)) & 0xFFFFu;
}

// Digits buf[s, s + n), n <= 4 NG, as an integer (NG 4-digit groups from the right; NG = 4
// covers lambda <= 16, NG = 5 lambda = 17). buf must be 8-byte aligned and readable from
// 23 bytes before s to 8 bytes past s + n.
//
// WINDOW (k_pack): the 16 bytes ending at the limb's end are read as one 8-byte-aligned
// window of three 8-byte loads and shifted into place with selects and funnel
// shifts, so each group sits in a fixed register: half the shared-memory wavefronts of
// one 4-byte funnel-shifted read per group, and k_pack's bank conflicts 34.7M -> 0.7M
// (config 4). !WINDOW (k_small): the per-group reads; in k_small the window measured
// 0.4% slower on config 2 (re-checked with the 3-load window: +0.45%).
template <int NG = 5, bool WINDOW = true>
__device__ __forceinline__ u64 parse_digits(const char* buf, int s, int n, unsigned& bad) {
  static_assert(NG == 4 || NG == 5, "4 or 5 groups");
  unsigned g[5] = {0, 0, 0, 0, 0};
  constexpr int NS = NG < 4 ? NG : 4;  // SWAR groups; with NG = 5 the fifth holds <= 1 digit
  if constexpr (NG == 5) {
    // n <= 17 leaves the fifth group's first 20 - n >= 3 bytes before s: it is the single
    // digit buf[s] when n == 17, else 0
    const unsigned c = n >= 17 ? unsigned((unsigned char)buf[s]) - '0' : 0u;
    bad |= c > 9 ? 0x80u : 0u;
    g[4] = c;
  }
  if constexpr (!WINDOW) {
    const int e = s + n;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int skip = 4 * (k + 1) - n;  // bytes of the group before s
      g[k] = skip < 4 ? swar4(smem_bytes4(buf, e - 4 * (k + 1)), skip < 0 ? 0 : skip, bad) : 0u;
    }
  } else {
    constexpr int BYTES = 4 * NS, NQ = (BYTES + 14) / 8;  // window: BYTES + up to 7 bytes of offset
    const int st = s + n - BYTES;                          // first byte of the NS groups
    const int a0 = st & ~7;
    const int o = st - a0;  // 0..7
    const uint2* wp = reinterpret_cast<const uint2*>(buf + a0);
    unsigned w[2 * NQ];
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      const uint2 q = wp[i];
      w[2 * i] = q.x;
      w[2 * i + 1] = q.y;
    }
    const bool up = o >= 4;
    const int sh = (o & 3) * 8;
#pragma unroll
    for (int k = 0; k < NS; ++k) {  // group k from the right = word NS - 1 - k of the window
      const int j = NS - 1 - k;
      const unsigned lo = up ? w[j + 1] : w[j], hi = up ? w[j + 2] : w[j + 1];
      const int skip = 4 * (k + 1) - n;  // bytes of the group before s
      g[k] = skip < 4 ? swar4(__funnelshift_r(lo, hi, sh), skip < 0 ? 0 : skip, bad) : 0u;
    }
  }
  const unsigned lo8 = g[1] * 10000u + g[0], hi8 = g[3] * 10000u + g[2];
  const u64 v = (u64)hi8 * 100000000ull + lo8;
  return NG == 5 ? v + (u64)g[4] * 10000000000000000ull : v;
}

}  // namespace dmg
