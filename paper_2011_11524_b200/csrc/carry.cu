// Decimal recovery for one large product: CRT + digit split + chunk maps,
// chunk-carry scan + top-limb detection, then carry application fused with the
// ASCII formatting (reference recover_digits decimal.cpp:154-189 and
// to_decimal decimal.cpp:120-134).
#include "carry.cuh"
#include "kernels.cuh"

namespace dmg {

namespace {

// Chunk of CH = PERC NTC limbs per CTA of NTC threads; each thread composes the maps of
// PERC consecutive limbs, moved as one PERC-byte word. Large products: 256 threads x 8
// limbs. Small products: 512-limb chunks as 256 threads x 2 limbs (more CTAs and short
// per-thread chains: the kernels are latency-bound there), and the chunk scan folds into
// the emit kernel.
constexpr int PER = 8;
constexpr int CH = kCarryChunk;  // chunk of the large-product and sharded paths
constexpr int NT = kCarryThreads;
static_assert(CH == NT * PER, "chunk = threads x 8 limbs");
constexpr int PER_SMALL = 2;
constexpr int NT_SMALL = kCarryChunkSmall / PER_SMALL;

template <int PERC> struct MapWord;  // PERC one-byte limb maps as one integer
template <> struct MapWord<8> { typedef unsigned long long type; };
template <> struct MapWord<4> { typedef unsigned type; };
template <> struct MapWord<2> { typedef unsigned short type; };
template <> struct MapWord<1> { typedef unsigned char type; };

// Local coefficient i (global k_off + i); i = -2, -1 are the previous rank's halo.
__device__ __forceinline__ void coeff_digits(const CarryArgs& a, long long i, u64& d0, u64& d1, u64& d2) {
  d0 = d1 = d2 = 0;
  if (i < -2 || (i >= 0 && (unsigned long long)i >= a.n)) return;
  const u64 r1 = i < 0 ? a.halo1[i + 2] : a.z1[i];
  const u64 r2 = i < 0 ? a.halo2[i + 2] : a.z2[i];
  u64 lo, hi;
  crt2(r1, r2, a.p1, a.p2, a.p2_prime, a.r_tilde, lo, hi);
  if (above_cap(lo, hi, a.coeff_cap_lo, a.coeff_cap_hi)) atomicOr(a.err, kErrCoeffBound);
  split3(a.div, lo, hi, d0, d1, d2);
}

// Phase 2 (one block of NTB threads): exclusive scan of chunk maps -> chunk carry-ins (stored
// in place), then the top limb, its digit count and the output length. Reads bypass L1
// (__ldcg): in the last-block form the other CTAs' writes are only ordered through L2.
template <int NTB, int CHC>
__device__ __forceinline__ void scan_chunks_top(const CarryArgs& a, unsigned nchunks, unsigned* wsm, u64* zc) {
  // With the split's in-chunk prefix maps (a.pm), a candidate top limb's carry-in is its
  // prefix applied to its chunk's carry-in: its sum and prefix do not depend on the chunk
  // scan, so threads 0 and 1 load them first and their L2 latency overlaps the scan (the
  // small-product chain ends in this one CTA: config 1 split 12.6 us under ncu, 60% idle SMs).
  const bool fast = a.pm != nullptr;
  u64 sk = 0;
  unsigned pk = 0;
  if (fast && threadIdx.x < 2) {
    const unsigned long long k = a.top_candidates[threadIdx.x];
    sk = __ldcg(a.s + k);
    pk = __ldcg(a.pm + k);
  }
  const unsigned per = (nchunks + NTB - 1) / NTB;
  const unsigned c0 = threadIdx.x * per;
  unsigned agg = kIdentityMap;
  for (unsigned c = c0; c < c0 + per && c < nchunks; ++c) agg = map_compose(__ldcg(a.maps + c), agg);
  unsigned pre = block_scan_maps<NTB>(agg, wsm, nullptr);
  unsigned carry = map_apply(pre, 0);
  for (unsigned c = c0; c < c0 + per && c < nchunks; ++c) {
    const unsigned m = __ldcg(a.maps + c);
    a.maps[c] = carry;  // chunk carry-in
    carry = map_apply(m, carry);
  }
  __syncthreads();
  __threadfence_block();
  const u64 B = a.div.base;
  if (fast) {
    if (threadIdx.x < 2) {
      const unsigned long long k = a.top_candidates[threadIdx.x];
      u64 v = sk + map_apply(pk, a.maps[k / CHC]);
      v -= (v >= B ? B : 0);
      v -= (v >= B ? B : 0);
      zc[threadIdx.x] = v;
    }
    __syncthreads();
  } else {
    // z at the two candidate top limbs: carry-in of the chunk, then the maps of
    // the limbs before the candidate inside its chunk.
    for (int t = 0; t < 2; ++t) {
      const unsigned long long k = a.top_candidates[t];
      const unsigned long long cs = k / CHC * CHC;
      unsigned m = kIdentityMap;
      const unsigned long long len = k - cs;  // ordered contiguous segments, one per thread
      const unsigned long long seg = (len + NTB - 1) / NTB;
      const unsigned long long j0 = cs + threadIdx.x * seg;
      for (unsigned long long j = j0; j < j0 + seg && j < k; ++j) m = map_compose(limb_map(__ldcg(a.s + j), B), m);
      block_scan_maps<NTB>(m, wsm, &m);
      if (threadIdx.x == 0) {
        const unsigned cin = a.maps[k / CHC];
        const unsigned c = map_apply(m, cin);
        u64 v = __ldcg(a.s + k) + c;
        v -= (v >= B ? B : 0);
        v -= (v >= B ? B : 0);
        zc[t] = v;
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    unsigned long long top;
    u64 z;
    if (zc[1] != 0) {
      top = a.top_candidates[1];
      z = zc[1];
    } else if (zc[0] != 0) {
      top = a.top_candidates[0];
      z = zc[0];
    } else {
      top = 0;
      z = 0;
    }
    const unsigned len = decimal_len(z);
    a.meta[0] = top;
    a.meta[1] = len;
    a.meta[2] = len + top * a.base_exp;
  }
}

// Per-limb in-chunk exclusive prefix maps (a.pm, one byte per limb): `pre` is the composition
// of the earlier threads' limbs, m8 this thread's PERC limb maps; the emit then applies
// pm[k] to the chunk's carry-in instead of recomputing every limb's map and scanning again.
template <int PERC, class Word>
__device__ __forceinline__ void store_prefix_maps(unsigned char* pm, unsigned long long first, unsigned pre,
                                                  unsigned long long m8) {
  unsigned long long out = 0;
  unsigned c = pre;
#pragma unroll
  for (int j = 0; j < PERC; ++j) {
    out |= (unsigned long long)c << (8 * j);
    c = map_compose(unsigned(m8 >> (8 * j)) & 63u, c);
  }
  *reinterpret_cast<Word*>(pm + first) = Word(out);
}

// Phase 1: s_k for the chunk's limbs and the chunk's composed transfer map.
// Coefficients are read and limb sums written in coalesced order (loc = j NT + tid);
// each limb's 6-bit transfer map goes to shared memory as a byte, and each thread
// then composes the maps of PERC consecutive limbs (one PERC-byte shared load).
// FROM_S: the limb sums are already in a.s (the general small-base recovery); only the maps.
// LASTSCAN (small products): the last CTA to finish (a.ticket) runs phase 2 itself, so the
// chain is split -> emit with no one-block scan launch in between (which, like an emit that
// re-derived every chunk carry-in and the top limb per CTA, cost config 1 several us).
template <int NTC, int PERC, bool FROM_S = false, bool LASTSCAN = false>
__global__ void __launch_bounds__(NTC) k_carry_split(CarryArgs a) {
  pdl_wait();
  constexpr int CHC = NTC * PERC;
  typedef typename MapWord<PERC>::type Word;
  __shared__ u64 d1s[FROM_S ? 1 : CHC + 2], d2s[FROM_S ? 1 : CHC + 2];
  __shared__ __align__(8) unsigned char mp[CHC];
  __shared__ unsigned wsm[NTC / 32 + 1];
  const unsigned long long k0 = (unsigned long long)blockIdx.x * CHC;
  const unsigned long long K = a.n + (a.tail ? 2 : 0);
  const u64 B = a.div.base;
  if constexpr (FROM_S) {
#pragma unroll
    for (int j = 0; j < PERC; ++j) {
      const int loc = j * NTC + threadIdx.x;
      const unsigned long long k = k0 + loc;
      mp[loc] = (unsigned char)(k < K ? limb_map(a.s[k], B) : kIdentityMap);
    }
  } else {
    u64 d0r[PERC];
#pragma unroll
    for (int j = 0; j < PERC; ++j) {
      const int loc = j * NTC + threadIdx.x;
      u64 d0, d1, d2;
      coeff_digits(a, (long long)(k0 + loc), d0, d1, d2);
      d0r[j] = d0;
      d1s[loc + 2] = d1;
      d2s[loc + 2] = d2;
    }
    if (threadIdx.x < 2) {
      u64 d0, d1, d2;
      coeff_digits(a, (long long)k0 - 2 + threadIdx.x, d0, d1, d2);
      d1s[threadIdx.x] = d1;
      d2s[threadIdx.x] = d2;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < PERC; ++j) {
      const int loc = j * NTC + threadIdx.x;
      const unsigned long long k = k0 + loc;
      const u64 s = d0r[j] + d1s[loc + 1] + d2s[loc];
      if (k < K) a.s[k] = s;
      mp[loc] = (unsigned char)(k < K ? limb_map(s, B) : kIdentityMap);
    }
  }
  __syncthreads();
  const unsigned long long m8 = reinterpret_cast<const Word*>(mp)[threadIdx.x];
  unsigned agg = kIdentityMap;
#pragma unroll
  for (int j = 0; j < PERC; ++j) agg = map_compose(unsigned(m8 >> (8 * j)) & 63u, agg);
  unsigned total;
  const unsigned pre = block_scan_maps<NTC>(agg, wsm, &total);
  if (threadIdx.x == 0) a.maps[blockIdx.x] = total;
  if (a.pm) store_prefix_maps<PERC, Word>(a.pm, k0 + threadIdx.x * PERC, pre, m8);
  if constexpr (LASTSCAN) {
    __shared__ unsigned is_last;
    __shared__ u64 zc[2];
    __threadfence();  // this CTA's limb sums and chunk map, before its ticket
    __syncthreads();
    if (threadIdx.x == 0) is_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (is_last) {
      __threadfence();
      scan_chunks_top<NTC, CHC>(a, gridDim.x, wsm, zc);
      if (threadIdx.x == 0) *a.ticket = 0;  // ready for the next product
    }
  }
}

template <int CHC>
__global__ void __launch_bounds__(1024) k_carry_scan(CarryArgs a, unsigned nchunks) {
  pdl_wait();
  __shared__ unsigned wsm[1024 / 32 + 1];
  __shared__ u64 zc[2];
  scan_chunks_top<1024, CHC>(a, nchunks, wsm, zc);
}

// Phase 3: apply carries and print each limb at its place in the output string.
// The chunk's digits are staged in shared memory and stored as 16-byte vectors.
template <int NTC, int PERC>
__global__ void __launch_bounds__(NTC) k_carry_emit(CarryArgs a) {
  pdl_wait();
  constexpr int CHC = NTC * PERC;
  typedef typename MapWord<PERC>::type Word;
  __shared__ unsigned wsm[NTC / 32 + 1];
  __shared__ __align__(16) char buf[CHC * 17 + 32];
  __shared__ __align__(8) unsigned char mp[CHC];  // limb maps, then limb carry-ins
  const unsigned long long cbase = (unsigned long long)blockIdx.x * CHC;
  const unsigned long long top = a.meta[0];
  const unsigned top_len = unsigned(a.meta[1]);
  if (a.k_off + cbase > top) return;  // nothing of this chunk is printed (uniform per block)
  const unsigned chunk_cin = a.maps[blockIdx.x];
  const unsigned long long K = a.n + (a.tail ? 2 : 0);
  const u64 B = a.div.base;
  unsigned long long cin8 = 0;
  if (a.pm) {
    // the split stored every limb's in-chunk prefix map: carry-in = prefix applied to the
    // chunk's carry-in (no limb maps, no block scan here)
    const unsigned long long p8 = *reinterpret_cast<const Word*>(a.pm + cbase + threadIdx.x * PERC);
#pragma unroll
    for (int j = 0; j < PERC; ++j)
      cin8 |= (unsigned long long)map_apply(unsigned(p8 >> (8 * j)) & 63u, chunk_cin) << (8 * j);
  } else {
    // coalesced limb sums (loc = j NTC + tid); their maps to shared memory
    u64 s[PERC];
#pragma unroll
    for (int j = 0; j < PERC; ++j) {
      const unsigned long long k = cbase + j * NTC + threadIdx.x;
      s[j] = k < K ? a.s[k] : 0;
      mp[j * NTC + threadIdx.x] = (unsigned char)limb_map(s[j], B);
    }
    __syncthreads();
    // each thread: PERC consecutive limbs -> composed map -> block scan -> per-limb carry-ins
    unsigned long long m8 = reinterpret_cast<const Word*>(mp)[threadIdx.x];
    unsigned agg = kIdentityMap;
#pragma unroll
    for (int j = 0; j < PERC; ++j) agg = map_compose(unsigned(m8 >> (8 * j)) & 63u, agg);
    const unsigned pre = block_scan_maps<NTC>(agg, wsm, nullptr);  // ends with a barrier
    unsigned c = map_apply(pre, chunk_cin);
#pragma unroll
    for (int j = 0; j < PERC; ++j) {
      cin8 |= (unsigned long long)c << (8 * j);
      c = map_apply(unsigned(m8 >> (8 * j)) & 63u, c);
    }
  }
  reinterpret_cast<Word*>(mp)[threadIdx.x] = Word(cin8);
  __syncthreads();
  const unsigned be = a.base_exp;
  // global limb range printed by this chunk: [gbase, ghi]
  const unsigned long long gbase = a.k_off + cbase;
  const unsigned long long last_local = (cbase + CHC < K ? cbase + CHC : K) - 1;
  const unsigned long long ghi = a.k_off + last_local < top ? a.k_off + last_local : top;
  const unsigned long long start = limb_pos(ghi, top, top_len, be);
  const unsigned long long end = limb_pos(gbase, top, top_len, be) + (gbase == top ? top_len : be);
  char* g = a.out + start;
  char* sb = buf + (reinterpret_cast<unsigned long long>(g) & 15);
  // digits: each thread prints PERC consecutive limbs (a contiguous PERC lambda-byte run)
  const unsigned long long* sg = reinterpret_cast<const unsigned long long*>(a.s);
  // fast path: 8 full-width limbs below the top one -> one 8 lambda-byte run built in registers
  // (SWAR) and stored as 32-bit words; the chunk holding the top limb (or a lambda < 14 tail)
  // prints limb by limb. Both paths end at the block's one barrier below.
  const unsigned long long kg0 = a.k_off + cbase + threadIdx.x * PERC;
  if (PERC == 8 && kg0 + 7 < top && be >= 14) {
    u64 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // text order: the highest limb first
      const int loc = threadIdx.x * PERC + 7 - j;
      u64 x = sg[cbase + loc] + mp[loc];
      if (x >= B) x -= B;
      if (x >= B) x -= B;
      v[j] = x;
    }
    char* dst = sb + (limb_pos(kg0 + 7, top, top_len, be) - start);
    switch (be) {
      case 14: print_run8<14>(dst, v); break;
      case 15: print_run8<15>(dst, v); break;
      case 16: print_run8<16>(dst, v); break;
      default: print_run8<17>(dst, v); break;
    }
  } else {
#pragma unroll
    for (int j = 0; j < PERC; ++j) {
      const int loc = threadIdx.x * PERC + j;
      const unsigned long long k = cbase + loc, kg = a.k_off + k;
      if (kg > ghi) break;
      u64 v = sg[k] + mp[loc];  // re-read from L1/L2 (this block just streamed it)
      if (v >= B) v -= B;
      if (v >= B) v -= B;
      write_digits(sb + (limb_pos(kg, top, top_len, be) - start), v, kg == top ? top_len : be);
    }
  }
  __syncthreads();
  cta_store_bytes(g, sb, unsigned(end - start), threadIdx.x, NTC);
}

// ---- sharded product: the rank's carry-in comes from the other ranks ----

// Exclusive prefix maps of the chunks (in place in maps[]) and the rank's composed map.
__global__ void __launch_bounds__(1024) k_carry_prefix(CarryArgs a, unsigned nchunks, unsigned* rank_map) {
  __shared__ unsigned wsm[1024 / 32 + 1];
  const unsigned per = (nchunks + 1023) / 1024;
  const unsigned c0 = threadIdx.x * per;
  unsigned agg = kIdentityMap;
  for (unsigned c = c0; c < c0 + per && c < nchunks; ++c) agg = map_compose(a.maps[c], agg);
  unsigned total;
  unsigned pre = block_scan_maps<1024>(agg, wsm, &total);
  for (unsigned c = c0; c < c0 + per && c < nchunks; ++c) {
    const unsigned m = a.maps[c];
    a.maps[c] = pre;  // maps of all earlier chunks of this rank
    pre = map_compose(m, pre);
  }
  if (threadIdx.x == 0) *rank_map = total;
}

// z (the final limb value) at the candidate top limbs this rank owns.
__global__ void __launch_bounds__(1024) k_carry_probe(CarryArgs a, unsigned rank_cin, u64* z) {
  __shared__ unsigned wsm[1024 / 32 + 1];
  const u64 B = a.div.base;
  const unsigned long long K = a.n + (a.tail ? 2 : 0);
  for (int t = 0; t < 2; ++t) {
    const unsigned long long kg = a.top_candidates[t];
    const bool mine = kg >= a.k_off && kg - a.k_off < K;  // uniform across the block
    if (!mine) {
      if (threadIdx.x == 0) z[t] = ~0ull;
      continue;
    }
    const unsigned long long k = kg - a.k_off, cs = k / CH * CH;
    const unsigned long long len = k - cs, seg = (len + 1023) / 1024;
    const unsigned long long j0 = cs + threadIdx.x * seg;
    unsigned m = kIdentityMap;
    for (unsigned long long j = j0; j < j0 + seg && j < k; ++j) m = map_compose(limb_map(a.s[j], B), m);
    block_scan_maps<1024>(m, wsm, &m);
    if (threadIdx.x == 0) {
      const unsigned c = map_apply(m, map_apply(a.maps[k / CH], rank_cin));
      u64 v = a.s[k] + c;
      v -= (v >= B ? B : 0);
      v -= (v >= B ? B : 0);
      z[t] = v;
    }
    __syncthreads();
  }
}

__global__ void k_carry_cin(unsigned* maps, unsigned nchunks, unsigned rank_cin) {
  const unsigned c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nchunks) maps[c] = map_apply(maps[c], rank_cin);
}

// ---- inverse radix-3 pass fused with CRT and the digit split (large N = 3 S) ----

// Coefficient k (0 <= k < 3 S) from the last inverse power-of-two pass's output: the inverse
// radix-3 butterfly of column s = k mod S (reference three_row_inverse_columns,
// conv.cpp:129-147, as k_radix3_inv computes it) for both primes, output row g = k / S.
__device__ __forceinline__ void r3inv_load(const Radix3Args& r, unsigned long long s, u64 x[2][3]) {
#pragma unroll
  for (int pr = 0; pr < 2; ++pr) {
#pragma unroll
    for (int g = 0; g < 3; ++g) x[pr][g] = r.src[pr][g * r.S + s];
  }
}
// (the inputs are only multiplied before the length-3 DFT: they may be lazy, [0, 2p))
// PRE: the merged twiddles omega_{3 R1}^{-f r} from r.pinv, one Shoup product
// per element; else the factorised lo * hi.
template <bool PRE>
__device__ __forceinline__ void r3inv_from(const Radix3Args& r, unsigned long long s, const u64 x[2][3],
                                           u64 out[2][3]) {
  const unsigned long long L = 1ull << r.lbits, H = r.hrow;
  const unsigned long long sl = s & (L - 1), sh = s >> r.lbits;
#pragma unroll
  for (int pr = 0; pr < 2; ++pr) {
    const u64 p = r.p[pr];
    u64 y0, y1, y2;
    if constexpr (PRE) {
      const TwPair* __restrict__ pv = r.pinv[pr] + (s >> r.pre_shift);
      y0 = shoup_mul(x[pr][0], pv[0], p);
      y1 = shoup_mul(x[pr][1], pv[r.pre_rows], p);
      y2 = shoup_mul(x[pr][2], pv[2 * r.pre_rows], p);
    } else {
      const TwPair* __restrict__ lo = r.lo[pr];
      const TwPair* __restrict__ hi = r.hi[pr];
      y0 = shoup_mul(x[pr][0], hi[sh], p);  // lo[0][.] = 1
      y1 = shoup_mul(shoup_mul(x[pr][1], lo[L + sl], p), hi[H + sh], p);
      y2 = shoup_mul(shoup_mul(x[pr][2], lo[2 * L + sl], p), hi[2 * H + sh], p);
    }
    const u64 t = shoup_mul(mod_sub(y1, y2, p), r.lam[pr], p);
    out[pr][0] = mod_add(mod_add(y0, y1, p), y2, p);
    out[pr][1] = mod_add(mod_sub(y0, y2, p), t, p);
    out[pr][2] = mod_sub(mod_sub(y0, y1, p), t, p);
  }
}
template <bool PRE>
__device__ __forceinline__ void r3inv_column(const Radix3Args& r, unsigned long long s, u64 out[2][3]) {
  u64 x[2][3];
  r3inv_load(r, s, x);
  r3inv_from<PRE>(r, s, x, out);
}

__device__ __forceinline__ void coeff_split(const CarryArgs& a, u64 r1, u64 r2, bool check, u64& d0, u64& d1,
                                            u64& d2) {
  u64 lo, hi;
  crt2(r1, r2, a.p1, a.p2, a.p2_prime, a.r_tilde, lo, hi);
  if (check && above_cap(lo, hi, a.coeff_cap_lo, a.coeff_cap_hi)) atomicOr(a.err, kErrCoeffBound);
  split3(a.div, lo, hi, d0, d1, d2);
}

// d1, d2 of coefficient k (k < 0: zero)
template <bool PRE>
__device__ __forceinline__ void coeff_d12(const CarryArgs& a, const Radix3Args& r, long long k, u64& d1, u64& d2) {
  d1 = d2 = 0;
  if (k < 0) return;
  u64 c[2][3];
  const unsigned long long g = (unsigned long long)k / r.S;
  r3inv_column<PRE>(r, (unsigned long long)k - g * r.S, c);
  u64 d0;
  coeff_split(a, g == 0 ? c[0][0] : (g == 1 ? c[0][1] : c[0][2]), g == 0 ? c[1][0] : (g == 1 ? c[1][1] : c[1][2]),
              false, d0, d1, d2);
}

// CTA b (< S / CH) takes columns [b CH, (b + 1) CH) and produces the limb sums and chunk maps of
// the three chunks g S / CH + b (g = 0, 1, 2); the coefficient k's own digit d0 meets d1 of
// k - 1 and d2 of k - 2 through warp shuffles, with the warp edges (and the chunk's two halo
// coefficients) in shared memory. The last CTA (a.tail) forms the two trailing limbs N, N + 1.
// Replaces k_radix3_inv + k_carry_split: the natural-order coefficients never touch HBM.
template <bool PRE>
__global__ void __launch_bounds__(NT) k_carry_split_r3(CarryArgs a, Radix3Args r) {
  pdl_wait();
  constexpr int NW = NT / 32;
  __shared__ u64 e1[3][PER * NW + 1], e2a[3][PER * NW + 1], e2b[3][PER * NW + 1];
  __shared__ __align__(8) unsigned char mp[3][CH];
  __shared__ unsigned wsm[NT / 32 + 1];
  const unsigned long long S = r.S, N = 3 * S;
  const u64 B = a.div.base;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (blockIdx.x == S / CH) {  // tail chunk N / CH: limbs N, N + 1 (K = N + 2)
    if (tid == 0) {
      u64 d1a, d2a, d1b, d2b;
      coeff_d12<PRE>(a, r, (long long)N - 1, d1a, d2a);
      coeff_d12<PRE>(a, r, (long long)N - 2, d1b, d2b);
      const u64 sN = d1a + d2b, sN1 = d2a;
      a.s[N] = sN;
      a.s[N + 1] = sN1;
      a.maps[N / CH] = map_compose(limb_map(sN1, B), limb_map(sN, B));
      if (a.pm) {  // in-chunk prefixes of the tail chunk's two limbs
        a.pm[N] = (unsigned char)kIdentityMap;
        a.pm[N + 1] = (unsigned char)limb_map(sN, B);
      }
    }
    return;
  }
  const unsigned long long s0 = (unsigned long long)blockIdx.x * CH;
  if (tid < 6) {  // halo: coefficients k0 - 1 and k0 - 2 of each group's chunk
    const int g = tid >> 1, which = tid & 1;
    u64 d1, d2;
    coeff_d12<PRE>(a, r, (long long)(g * S + s0) - 1 - which, d1, d2);
    if (which == 0) {
      e1[g][0] = d1;
      e2b[g][0] = d2;
    } else {
      e2a[g][0] = d2;
    }
  }
  // round j + 1's six inputs are loaded while round j computes
  u64 xin[2][3];
  r3inv_load(r, s0 + tid, xin);
#pragma unroll 1
  for (int j = 0; j < PER; ++j) {
    const unsigned long long s = s0 + j * NT + tid;
    u64 c[2][3];
    {
      u64 cur[2][3];
#pragma unroll
      for (int q = 0; q < 6; ++q) cur[q / 3][q % 3] = xin[q / 3][q % 3];
      if (j + 1 < PER) r3inv_load(r, s + NT, xin);
      r3inv_from<PRE>(r, s, cur, c);
    }
    u64 d0[3], d1[3], d2[3];
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      coeff_split(a, c[0][g], c[1][g], true, d0[g], d1[g], d2[g]);
      if (lane == 31) {
        e1[g][1 + j * NW + w] = d1[g];
        e2b[g][1 + j * NW + w] = d2[g];
      } else if (lane == 30) {
        e2a[g][1 + j * NW + w] = d2[g];
      }
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      u64 p1 = __shfl_up_sync(0xffffffffu, d1[g], 1);
      u64 p2 = __shfl_up_sync(0xffffffffu, d2[g], 2);
      const int prev = j * NW + w;  // edge slot of the previous warp (0: the halo)
      if (lane == 0) {
        p1 = e1[g][prev];
        p2 = e2a[g][prev];
      } else if (lane == 1) {
        p2 = e2b[g][prev];
      }
      const u64 sum = d0[g] + p1 + p2;
      a.s[g * S + s] = sum;
      mp[g][j * NT + tid] = (unsigned char)limb_map(sum, B);
    }
  }
  __syncthreads();
  // each group's chunk map: PER consecutive limbs per thread, then a block scan
#pragma unroll
  for (int g = 0; g < 3; ++g) {
    const unsigned long long m8 = reinterpret_cast<const unsigned long long*>(mp[g])[tid];
    unsigned agg = kIdentityMap;
#pragma unroll
    for (int j = 0; j < PER; ++j) agg = map_compose(unsigned(m8 >> (8 * j)) & 63u, agg);
    unsigned total;
    const unsigned pre = block_scan_maps<NT>(agg, wsm, &total);
    if (tid == 0) a.maps[(g * S + s0) / CH] = total;
    if (a.pm) store_prefix_maps<PER, unsigned long long>(a.pm, g * S + s0 + tid * PER, pre, m8);
  }
}

// ---- general recovery for small forced bases (lambda < 14) ----

// Coefficient i = sum_j d_j B^j (D digits; the reference's recover_digits, decimal.cpp:154-189,
// carries the whole 128-bit value instead); digit j is added into the limb sum s[i + j].
__global__ void k_carry_scatter(CarryArgs a, int D) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < a.n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    u64 lo, hi;
    crt2(a.z1[i], a.z2[i], a.p1, a.p2, a.p2_prime, a.r_tilde, lo, hi);
    if (above_cap(lo, hi, a.coeff_cap_lo, a.coeff_cap_hi)) atomicOr(a.err, kErrCoeffBound);
    for (int j = 0; j < D && (lo | hi); ++j) {
      u64 qlo, qhi;
      const u64 d = divmod_base(a.div, lo, hi, qlo, qhi);
      if (d) atomicAdd(&a.s[i + j], (unsigned long long)d);
      lo = qlo;
      hi = qhi;
    }
  }
}

// t_k = s_k mod B + floor(s_{k-1} / B): the value sum s_k B^k is unchanged.
__global__ void k_carry_normalize(const u64* __restrict__ s, u64* __restrict__ t, unsigned long long K, u64 B) {
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < K;
       k += (unsigned long long)gridDim.x * blockDim.x)
    t[k] = s[k] % B + (k ? s[k - 1] / B : 0);
}

}  // namespace

int launch_carry_general(const CarryArgs& a0, int D, int rounds, u64* tmp, unsigned long long K, cudaStream_t st) {
  CarryArgs a = a0;
  int launched = 0;
  cudaMemsetAsync(a.s, 0, K * sizeof(u64), st);
  {
    const unsigned long long b = (a.n + 255) / 256;
    k_carry_scatter<<<unsigned(b < 148ull * 16 ? (b ? b : 1) : 148ull * 16), 256, 0, st>>>(a, D);
    ++launched;
  }
  prof_mark("k_carry_scatter", st, double(a.n), double(a.n) * 16 + double(K) * 8);
  u64* src = a.s;
  u64* dst = tmp;
  for (int r = 0; r < rounds; ++r) {
    const unsigned long long b = (K + 255) / 256;
    k_carry_normalize<<<unsigned(b < 148ull * 16 ? b : 148ull * 16), 256, 0, st>>>(src, dst, K, a.div.base);
    ++launched;
    u64* t = src;
    src = dst;
    dst = t;
  }
  if (src != a.s) cudaMemcpyAsync(a.s, src, K * sizeof(u64), cudaMemcpyDeviceToDevice, st);
  // the {0,1,2} scan over K limbs: n' + 2 = K with the sums already in s
  a.n = K - 2;
  a.tail = 1;
  const unsigned nchunks = unsigned((K + CH - 1) / CH);
  launch_pdl(k_carry_split<NT, PER, true>, dim3(nchunks), dim3(NT), 0, st, a);
  launch_pdl(k_carry_scan<CH>, dim3(1), dim3(1024), 0, st, a, nchunks);
  launch_pdl(k_carry_emit<NT, PER>, dim3(nchunks), dim3(NT), 0, st, a);
  prof_mark("k_carry_general_scan_emit", st, 0, double(K) * 16);
  return launched + 3;
}

template <int PERL>
static int launch_carry_large(const CarryArgs& a, unsigned long long K, cudaStream_t st) {
  constexpr int CHL = NT * PERL;
  const unsigned nchunks = unsigned((K + CHL - 1) / CHL);
  const double n = double(a.n), k = double(K);
  launch_pdl(k_carry_split<NT, PERL>, dim3(nchunks), dim3(NT), 0, st, a);
  prof_mark("k_carry_split", st, n, 16 * n + 8 * k);
  launch_pdl(k_carry_scan<CHL>, dim3(1), dim3(1024), 0, st, a, nchunks);
  prof_mark("k_carry_scan", st, 0, 8.0 * nchunks);
  launch_pdl(k_carry_emit<NT, PERL>, dim3(nchunks), dim3(NT), 0, st, a);
  prof_mark("k_carry_emit", st, 0, 8 * k + k * a.base_exp);
  return 3;
}

int launch_carry_r3(const CarryArgs& a, const Radix3Args& r, cudaStream_t st) {
  const unsigned long long N = 3 * r.S, K = N + 2;
  const unsigned nchunks = unsigned((K + CH - 1) / CH);  // S / CH column blocks + the tail chunk
  const double n = double(N), k = double(K);
  launch_pdl(r.pinv[0] ? k_carry_split_r3<true> : k_carry_split_r3<false>, dim3(unsigned(r.S / CH + 1)), dim3(NT), 0,
             st, a, r);
  prof_mark("k_carry_split_r3", st, 2.0 * 6.0 * r.S + n, 16 * n + 8 * k);
  launch_pdl(k_carry_scan<CH>, dim3(1), dim3(1024), 0, st, a, nchunks);
  prof_mark("k_carry_scan", st, 0, 8.0 * nchunks);
  launch_pdl(k_carry_emit<NT, PER>, dim3(nchunks), dim3(NT), 0, st, a);
  prof_mark("k_carry_emit", st, 0, 8 * k + k * a.base_exp);
  return 3;
}

bool carry_r3_fusable(unsigned long long S) { return S % CH == 0 && (3 * S + 2 + CH - 1) / CH >= 2 * 148; }

int launch_carry(const CarryArgs& a, cudaStream_t st) {
  const unsigned long long K = a.n + (a.tail ? 2 : 0);
  const unsigned nchunks = unsigned((K + CH - 1) / CH);
  if (nchunks < 2 * 148) {  // small product: 512-limb chunks, no separate scan
    const unsigned ns = unsigned((K + kCarryChunkSmall - 1) / kCarryChunkSmall);
    const double n = double(a.n), k = double(K);
    launch_pdl(k_carry_split<NT_SMALL, PER_SMALL, false, true>, dim3(ns), dim3(NT_SMALL), 0, st, a);
    prof_mark("k_carry_split_small", st, n, 16 * n + 8 * k);
    launch_pdl(k_carry_emit<NT_SMALL, PER_SMALL>, dim3(ns), dim3(NT_SMALL), 0, st, a);
    prof_mark("k_carry_emit_small", st, 0, 8 * k + k * a.base_exp);
    return 2;
  }
  // large products are throughput-bound: 8 limbs per thread (4 and 2 measured 0.7-4% slower)
  return launch_carry_large<PER>(a, K, st);
}

void launch_carry_shard_begin(const CarryArgs& a, unsigned* rank_map_dev, cudaStream_t st) {
  const unsigned long long K = a.n + (a.tail ? 2 : 0);
  const unsigned nchunks = unsigned((K + CH - 1) / CH);
  k_carry_split<NT, PER><<<nchunks, NT, 0, st>>>(a);
  k_carry_prefix<<<1, 1024, 0, st>>>(a, nchunks, rank_map_dev);
}

void launch_carry_shard_probe(const CarryArgs& a, unsigned rank_cin, u64* z_dev, cudaStream_t st) {
  k_carry_probe<<<1, 1024, 0, st>>>(a, rank_cin, z_dev);
}

void launch_carry_shard_emit(const CarryArgs& a, unsigned rank_cin, cudaStream_t st) {
  const unsigned long long K = a.n + (a.tail ? 2 : 0);
  const unsigned nchunks = unsigned((K + CH - 1) / CH);
  k_carry_cin<<<(nchunks + 255) / 256, 256, 0, st>>>(a.maps, nchunks, rank_cin);
  k_carry_emit<NT, PER><<<nchunks, NT, 0, st>>>(a);
}

}  // namespace dmg
