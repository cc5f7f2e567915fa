// 63-bit prime-field arithmetic for sm_100a, built on 32-bit IMAD chains.
//
// Values are plain residues in [0, p); p < 2^63 (reference montgomery.hpp:9-17,
// words.hpp:29-78). Two multiplication forms are used:
//  * Shoup: x * w mod p for a fixed factor w with precomputed
//    w' = floor(w 2^64 / p). One high product, two low products. Used for
//    every root-of-unity factor (tables hold (w, w') pairs).
//  * Montgomery REDC (R = 2^64), reference montgomery.hpp:26-39, for
//    data x data products (pointwise spectra, CRT inner product).
// Both produce canonical [0, p) results, so every transform value is the same
// field element the reference computes (its tables hold Montgomery forms, whose
// REDC against plain data yields plain products — ntt.hpp:14-19).
#pragma once
#include <cstdint>

namespace dmg {

typedef unsigned long long u64;

// 16-byte aligned so a pair is one 128-bit load (LDG.E.128 / LDS.128), not two 64-bit ones.
struct __align__(16) TwPair {  // Shoup form of one root-of-unity factor
  u64 w, wp;
};

// Because p < 2^63, a value in [-p, p) is unambiguous as a signed 64-bit word:
// corrections test the sign bit (reference words.hpp:38-45, adjust_signed).
#ifndef DMG_CORR_FMA
#define DMG_CORR_FMA 0
#endif
#ifndef DMG_CORR_PRED32
#define DMG_CORR_PRED32 1
#endif
__device__ __forceinline__ u64 adjust_signed(u64 t, u64 p) {
#if DMG_CORR_FMA
  // t + s p with the sign bit s = hi(t) >> 31 taken as mul.hi(hi(t), 2) and s p added by
  // mad.wide / mad.lo: ptxas emits IMAD.HI + IMAD.WIDE + IMAD (FMA pipe) + IADD3 + IADD3.X
  // instead of ISETP + IADD3 + IADD3.X + 2 SEL (all ALU pipe, the transforms' binding pipe).
  asm("{\n\t.reg .u32 tl, th, s, pl, ph;\n\t"
      "mov.b64 {tl, th}, %0;\n\t"
      "mov.b64 {pl, ph}, %1;\n\t"
      "mul.hi.u32 s, th, 2;\n\t"
      "mad.wide.u32 %0, s, pl, %0;\n\t"
      "mov.b64 {tl, th}, %0;\n\t"
      "mad.lo.u32 th, s, ph, th;\n\t"
      "mov.b64 %0, {tl, th};\n\t}"
      : "+l"(t)
      : "l"(p));
#elif DMG_CORR_PRED32
  // 32-bit halves: the low add is predicated in place, ptxas selects only the high word
  // (ISETP + @P IADD3 + IADD3.X + SEL: 4 instructions after the subtraction, not 5).
  // Measured against the 64-bit predicated form below: config 3 -2.9%, config 4 -0.4%.
  // (The FMA-pipe form above, on every site or only after Shoup products, was 5-16% slower:
  // the transforms are issue-bound and IMAD.WIDE is the costlier slot.)
  asm("{\n\t.reg .u32 tl, th, pl, ph;\n\t.reg .pred n;\n\t"
      "mov.b64 {tl, th}, %0;\n\t"
      "mov.b64 {pl, ph}, %1;\n\t"
      "setp.lt.s32 n, th, 0;\n\t"
      "@n add.cc.u32 tl, tl, pl;\n\t"
      "@n addc.u32 th, th, ph;\n\t"
      "mov.b64 %0, {tl, th};\n\t}"
      : "+l"(t)
      : "l"(p));
#else
  // sign test + predicated add (ptxas emits ISETP + IADD3 + 2 SEL) rather than the
  // mask form SHF + 2 LOP3 + IADD3 + IADD3.X: measured 0.6% (config 2) and 1.8%
  // (config 4) faster on B200.
  asm("{\n\t.reg .pred n;\n\tsetp.lt.s64 n, %0, 0;\n\t@n add.u64 %0, %0, %1;\n\t}" : "+l"(t) : "l"(p));
#endif
  return t;
}
// The same correction on the FMA pipe: s = sign bit by IMAD.HI, t += s p by IMAD.WIDE + IMAD.
__device__ __forceinline__ u64 adjust_fma(u64 t, u64 p) {
  asm("{\n\t.reg .u32 tl, th, s, pl, ph;\n\t"
      "mov.b64 {tl, th}, %0;\n\t"
      "mov.b64 {pl, ph}, %1;\n\t"
      "mul.hi.u32 s, th, 2;\n\t"
      "mad.wide.u32 %0, s, pl, %0;\n\t"
      "mov.b64 {tl, th}, %0;\n\t"
      "mad.lo.u32 th, s, ph, th;\n\t"
      "mov.b64 %0, {tl, th};\n\t}"
      : "+l"(t)
      : "l"(p));
  return t;
}
#ifndef DMG_SHOUP_CORR_FMA
#define DMG_SHOUP_CORR_FMA 0
#endif
__device__ __forceinline__ u64 mod_add(u64 a, u64 b, u64 p) { return adjust_signed(a + b - p, p); }
__device__ __forceinline__ u64 mod_sub(u64 a, u64 b, u64 p) { return adjust_signed(a - b, p); }

// x in [0, 2^64), w < p: returns x w mod p in [0, p).
// (Measured on B200: folding -q p as q (2^64 - p) plus an explicit predicated
// select was 3% slower than letting ptxas schedule this form. Rejected too: for primes
// == 1 mod 2^32 writing q p as q_lo + (q_lo p_hi + q_hi) 2^32 — ptxas kept the same
// IMAD.WIDE count and the transforms slowed down.)
#ifndef DMG_SHOUP_FOLD
#define DMG_SHOUP_FOLD 0
#endif
__device__ __forceinline__ u64 shoup_mul(u64 x, u64 w, u64 wp, u64 p) {
#if DMG_SHOUP_FOLD
  // p = 2^63 - c with c < 2^32 (both production primes): r - p = x w - (q + 1) p
  // = x w + (q + 1) c + (q + 1) 2^63 mod 2^64, with (q + 1) 2^63 = (q_lo + 1) 2^63: one wide and
  // four plain 32-bit multiply-adds instead of the full q p product and its negation
  const u64 q = __umul64hi(x, wp);
  const unsigned c = 0u - unsigned(p);
  u64 r;
  asm("{\n\t.reg .u32 xl, xh, wl, wh, ql, qh, rl, rh;\n\t.reg .u64 k, tt;\n\t"
      "mov.b64 {xl, xh}, %1;\n\t"
      "mov.b64 {wl, wh}, %2;\n\t"
      "mov.b64 {ql, qh}, %3;\n\t"
      "cvt.u64.u32 k, %4;\n\t"
      "add.u64 k, k, 0x8000000000000000;\n\t"
      "mad.wide.u32 tt, ql, %4, k;\n\t"
      "mad.wide.u32 tt, xl, wl, tt;\n\t"
      "mov.b64 {rl, rh}, tt;\n\t"
      "mad.lo.u32 rh, xl, wh, rh;\n\t"
      "mad.lo.u32 rh, xh, wl, rh;\n\t"
      "mad.lo.u32 rh, qh, %4, rh;\n\t"
      "mad.lo.u32 rh, ql, 0x80000000, rh;\n\t"
      "mov.b64 %0, {rl, rh};\n\t}"
      : "=l"(r)
      : "l"(x), "l"(w), "l"(q), "r"(c));
  return adjust_signed(r, p);
#else
  u64 q = __umul64hi(x, wp);
  u64 r = x * w - q * p;  // exact, r < 2p
#if DMG_SHOUP_CORR_FMA
  return adjust_fma(r - p, p);
#else
  return adjust_signed(r - p, p);
#endif
#endif
}
__device__ __forceinline__ u64 shoup_mul(u64 x, TwPair t, u64 p) { return shoup_mul(x, t.w, t.wp, p); }

// REDC(a b) = a b 2^-64 mod p for a b < p 2^64 (one operand may lie in [0, 2p)).
__device__ __forceinline__ u64 mont_mul(u64 a, u64 b, u64 p, u64 pp) {
  u64 lo = a * b, hi = __umul64hi(a, b);
  u64 m = lo * pp;
  // lo + lo(m p) == 0 mod 2^64: the carry out of the low word is (lo != 0).
  u64 r = hi + __umul64hi(m, p) + (lo != 0 ? 1ull : 0ull);  // r < 2p
  return adjust_signed(r - p, p);
}

// Goldilocks prime 2^64 - 2^32 + 1 with its Solinas reduction (2^64 = 2^32 - 1,
// 2^96 = -1): the reference's third modmul benchmark variant (montgomery.hpp:60-77).
// Not on the product path (the production primes are < 2^63); bench / self-test only.
constexpr u64 kSolinasPrime = 0xffffffff00000001ull;
__device__ __forceinline__ u64 solinas_mul(u64 a, u64 b) {
  const u64 lo = a * b, hi = __umul64hi(a, b);
  const u64 hh = hi >> 32, hl = hi & 0xffffffffull;
  u64 t = lo - hh;  // lo - hh mod p: on a borrow, add p = subtract 2^32 - 1 mod 2^64
  if (lo < hh) t -= 0xffffffffull;
  const u64 m = hl * 0xffffffffull;  // hl (2^32 - 1)
  u64 r = t + m;
  if (r < m) r += 0xffffffffull;  // carry out of 2^64 = 2^32 - 1
  if (r >= kSolinasPrime) r -= kSolinasPrime;
  return r;
}

// Shoup product left in [0, 2p) (no final correction), for consumers that accept it.
__device__ __forceinline__ u64 shoup_mul_lazy(u64 x, TwPair t, u64 p) {
  u64 q = __umul64hi(x, t.wp);
  return x * t.w - q * p;
}

// Gentleman-Sande butterfly (reference ntt.cpp:42-47): (u + v, (u - v) w).
__device__ __forceinline__ void bfly_dif(u64& u, u64& v, TwPair t, u64 p) {
  u64 a = mod_add(u, v, p);
  v = shoup_mul(u - v + p, t, p);  // u - v + p in [1, 2p)
  u = a;
}
__device__ __forceinline__ void bfly_dif1(u64& u, u64& v, u64 p) {  // factor 1 (j = 0 peel)
  u64 a = mod_add(u, v, p);
  v = mod_sub(u, v, p);
  u = a;
}
// Cooley-Tukey butterfly (reference ntt.cpp:65-70): (u + v w, u - v w).
__device__ __forceinline__ void bfly_dit(u64& u, u64& v, TwPair t, u64 p) {
  u64 w = shoup_mul(v, t, p);
  v = mod_sub(u, w, p);
  u = mod_add(u, w, p);
}
__device__ __forceinline__ void bfly_dit1(u64& u, u64& v, u64 p) {
  u64 w = v;
  v = mod_sub(u, w, p);
  u = mod_add(u, w, p);
}

// Lazy butterflies of a final stage: outputs in [0, 2p) instead of [0, p), for a consumer that
// accepts any input below 2p (a Shoup product, or one operand of a REDC product against a
// canonical one). p < 2^63, so 2p - 1 still fits the word; nothing uses these values as
// inputs of another add or subtract.
__device__ __forceinline__ void bfly_dif_lz(u64& u, u64& v, TwPair t, u64 p) {
  const u64 a = u + v;
  v = shoup_mul_lazy(u - v + p, t, p);
  u = a;
}
__device__ __forceinline__ void bfly_dif1_lz(u64& u, u64& v, u64 p) {
  const u64 a = u + v;
  v = u - v + p;
  u = a;
}
__device__ __forceinline__ void bfly_dit_lz(u64& u, u64& v, TwPair t, u64 p) {
  const u64 w = shoup_mul(v, t, p);
  v = u - w + p;
  u = u + w;
}
__device__ __forceinline__ void bfly_dit1_lz(u64& u, u64& v, u64 p) {
  const u64 w = v;
  v = u - w + p;
  u = u + w;
}
// Cooley-Tukey butterfly with per-output laziness: LU / LV leave u + v w / u - v w in [0, 2p)
// (for outputs that the next stage only multiplies). v may be anything below 2^64 (it is
// multiplied first); u must be canonical.
template <bool LU, bool LV>
__device__ __forceinline__ void bfly_dit_m(u64& u, u64& v, TwPair t, u64 p) {
  const u64 w = shoup_mul(v, t, p);
  v = LV ? u - w + p : mod_sub(u, w, p);
  u = LU ? u + w : mod_add(u, w, p);
}
template <bool LU, bool LV>
__device__ __forceinline__ void bfly_dit1_m(u64& u, u64& v, u64 p) {  // factor 1: v canonical
  const u64 w = v;
  v = LV ? u - w + p : mod_sub(u, w, p);
  u = LU ? u + w : mod_add(u, w, p);
}
// [0, 2p) -> [0, p)
__device__ __forceinline__ u64 reduce_2p(u64 a, u64 p) { return adjust_signed(a - p, p); }

// ---- two-word division by the constant limb base B = 10^lambda ----
// Restates the reciprocal scheme of reference decimal.hpp:93-146 (make_div_by_const,
// udiv_2by1, divmod_base) for the device.
struct DivB {
  u64 base, d_norm, recip;
  unsigned shift;
  u64 b2lo, b2hi;  // B^2 as a 128-bit value
  double inv_b2;   // 1 / B^2
};

__device__ __forceinline__ void udiv_2by1(u64 u1, u64 u0, u64 d, u64 v, u64& q, u64& r) {
  // t = v u1 + (u1 + 1) 2^64 + u0
  u64 tlo = v * u1, thi = __umul64hi(v, u1);
  u64 q0 = tlo + u0;
  u64 q1 = thi + u1 + 1 + (q0 < tlo ? 1ull : 0ull);
  u64 rr = u0 - q1 * d;
  if (rr > q0) {
    --q1;
    rr += d;
  }
  if (rr >= d) {
    ++q1;
    rr -= d;
  }
  q = q1;
  r = rr;
}

// (hi 2^64 + lo) = q B + r with q returned as (qhi, qlo). Requires the quotient to fit two words.
__device__ __forceinline__ u64 divmod_base(const DivB& d, u64 lo, u64 hi, u64& qlo, u64& qhi) {
  const unsigned sh = d.shift;
  u64 n0, n1, n2;
  if (sh == 0) {
    n0 = lo;
    n1 = hi;
    n2 = 0;
  } else {
    n0 = lo << sh;
    n1 = (hi << sh) | (lo >> (64 - sh));
    n2 = hi >> (64 - sh);
  }
  u64 rmid, rlo;
  udiv_2by1(n2, n1, d.d_norm, d.recip, qhi, rmid);
  udiv_2by1(rmid, n0, d.d_norm, d.recip, qlo, rlo);
  return rlo >> sh;
}

}  // namespace dmg
