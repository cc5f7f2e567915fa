// ASCII digits -> integers with SWAR arithmetic, from text staged in shared memory
// (the pack step, reference decimal.cpp:102-118). Used by k_pack and k_small.
#pragma once
#include "modarith.cuh"

namespace dmg {

// 8 bytes of shared memory at any byte offset (buf 8-aligned, readable 8 bytes past).
__device__ __forceinline__ u64 smem_bytes8(const char* buf, int pos) {
  const u64* w = reinterpret_cast<const u64*>(buf + (pos & ~7));
  const int sh = (pos & 7) * 8;
  return sh ? (w[0] >> sh) | (w[1] << (64 - sh)) : w[0];
}

// Value of 8 ASCII digits (first byte most significant) whose first `skip` bytes are
// treated as '0'; flags any non-digit byte.
__device__ __forceinline__ u64 swar8(u64 x, int skip, unsigned& bad) {
  const u64 keep = skip >= 8 ? 0 : (~0ull << (8 * skip));
  x = (x & keep) | (0x3030303030303030ull & ~keep);
  bad |= ((x & 0xF0F0F0F0F0F0F0F0ull) != 0x3030303030303030ull) |
         ((((x & 0x0F0F0F0F0F0F0F0Full) + 0x0606060606060606ull) & 0xF0F0F0F0F0F0F0F0ull) != 0);
  x &= 0x0F0F0F0F0F0F0F0Full;
  x = (x * 2561) >> 8;                                    // pairs: 10 d0 + d1
  x = ((x & 0x00FF00FF00FF00FFull) * 6553601) >> 16;     // quads
  x = ((x & 0x0000FFFF0000FFFFull) * 42949672960001ull) >> 32;  // 8 digits
  return x;
}

// Digits buf[s, s + n), n <= 24, as an integer (three 8-digit chunks from the right).
__device__ __forceinline__ u64 parse_digits(const char* buf, int s, int n, unsigned& bad) {
  const int e = s + n;
  u64 v = swar8(smem_bytes8(buf, e - 8), n >= 8 ? 0 : 8 - n, bad);
  if (n > 8) v += swar8(smem_bytes8(buf, e - 16), n >= 16 ? 0 : 16 - n, bad) * 100000000ull;
  if (n > 16) v += swar8(smem_bytes8(buf, e - 24), 24 - n, bad) * 10000000000000000ull;
  return v;
}

}  // namespace dmg
