// Column transforms for sm_100a, built from register-resident radix-8 rounds.
//
// A column of R = 2^LOGR words runs the reference's Gentleman-Sande DIF
// (natural order in, bit-reversed out; reference ntt.cpp:29-50) or Cooley-Tukey
// DIT (bit-reversed in, natural out, unscaled; ntt.cpp:52-73). The radix-2
// stages are grouped into rounds of up to three stages: a thread holds the 8
// (or 4, 2) elements of one group in registers and runs the round's stages
// there, so memory (shared or global) is touched once per round, not per stage.
//
// Schedules: DIF takes the remainder round first and ends with full radix-8
// rounds; DIT starts with radix-8 rounds and ends with the remainder. Hence the
// last DIF round and the first DIT round act on the same groups (8 consecutive
// positions), which lets a pass run DIF -> pointwise -> DIT in registers.
//
// Twiddles come from a shared table tw[tw_index(k)] = omega_R^k (k < R/2) in Shoup form;
// the stage with span M uses omega_M^j = tw[j * R / M] like the reference's flat
// stage slices (ntt.hpp:10-19). A radix-8 group needs 7 distinct factors, each
// loaded once; in rounds with stride 1 the j = 0 factors are 1 and skipped
// (the reference's peel, ntt.cpp:39-41).
//
// Bank conflicts: a half-warp's 16 u64 accesses must hit 16 distinct 8-byte
// slots. Row-major tiles (16 columns) map threads column-fastest, so a
// half-warp reads one 128 B row. Column-major tiles map threads along the
// column and XOR-swizzle the in-column index (r ^ ((r >> 3) & 15)), which makes
// every round of these schedules conflict-free (checked offline for R = 2^4..2^11).
// The 16-byte twiddle loads conflict too unless the table is swizzled: a column-major
// warp spans 32 groups, so a middle round reads tw[(j0 + k STRIDE) << s] for 8 values
// of j0, and the strides 4, 8, 16 put all 8 entries in 1-2 of the 8 sixteen-byte bank
// slots (up to 8-way). Column-major kernels therefore store tables at tw_slot(k), which
// XORs the low 3 bits with bits 3-5 ^ 6-8: conflict-free for every round of R = 2^7..2^9
// (simulated offline; ncu counters in DESIGN.md §2). Row-major warps span only 2 groups,
// so their few conflicts are cheaper than the swizzle's index arithmetic: SWZ = false.
#pragma once
#include "modarith.cuh"

namespace dmg {

__device__ __forceinline__ int tw_slot(int k) { return k ^ (((k >> 3) ^ (k >> 6)) & 7); }
template <bool SWZ>
__device__ __forceinline__ int tw_index(int k) { return SWZ ? tw_slot(k) : k; }

// ---- round schedules ----
template <int LOGR>
struct Sched {
  static constexpr int rem = LOGR % 3;
  // DIF: the round starting at span 2^MLOG has e_dif(MLOG) stages
  static constexpr int e_dif(int mlog) { return (mlog == LOGR && rem) ? rem : (mlog < 3 ? mlog : 3); }
  // DIT: the round starting after ALOG stages has e_dit(ALOG) stages
  static constexpr int e_dit(int alog) { return (LOGR - alog == rem && rem) ? rem : (LOGR - alog < 3 ? LOGR - alog : 3); }
  static constexpr int first_e = LOGR < 3 ? LOGR : 3;  // last DIF round == first DIT round
};

// ---- register stages ----
// DIF stages of one group: elements v[i] at positions base + i * STRIDE, STRIDE = 2^(MLOG-E),
// j0 = base mod STRIDE. Spans 2^MLOG down to 2^(MLOG-E+1).
// LZ: the last stage's outputs stay in [0, 2p) (modarith.cuh lazy butterflies) for a consumer
// that accepts them (the inter-pass twiddle, the pointwise REDC).
template <int LOGR, int MLOG, int E, bool SWZ, bool LZ = false>
__device__ __forceinline__ void dif_regs(u64 (&v)[1 << E], int j0, const TwPair* tw, u64 p) {
  constexpr int NE = 1 << E, STRIDE = 1 << (MLOG - E);
#pragma unroll
  for (int st = 0; st < E; ++st) {
    const int half = NE >> (st + 1);
    const int mlog = MLOG - st;  // span 2^mlog
    TwPair t[NE / 2];
#pragma unroll
    for (int k = 0; k < half; ++k)
      if (!(STRIDE == 1 && k == 0)) t[k] = tw[tw_index<SWZ>((j0 + k * STRIDE) << (LOGR - mlog))];
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      if (i & half) continue;
      const bool lz = LZ && st == E - 1;
      if (STRIDE == 1 && (i & (half - 1)) == 0) {  // j = 0: factor 1 (reference ntt.cpp:39-41 peel)
        if (lz)
          bfly_dif1_lz(v[i], v[i + half], p);
        else
          bfly_dif1(v[i], v[i + half], p);
      } else if (lz) {
        bfly_dif_lz(v[i], v[i + half], t[i & (half - 1)], p);
      } else {
        bfly_dif(v[i], v[i + half], t[i & (half - 1)], p);
      }
    }
  }
}

// DIT stages of one group: positions base + i * STRIDE, STRIDE = 2^ALOG; spans 2^(ALOG+1)..2^(ALOG+E).
template <int LOGR, int ALOG, int E, bool SWZ, bool LZ = false>
__device__ __forceinline__ void dit_regs(u64 (&v)[1 << E], int j0, const TwPair* tw, u64 p) {
  constexpr int NE = 1 << E, STRIDE = 1 << ALOG;
#pragma unroll
  for (int st = 0; st < E; ++st) {
    const int d = 1 << st;
    const int mlog = ALOG + st + 1;
    TwPair t[NE / 2];
#pragma unroll
    for (int k = 0; k < d; ++k)
      if (!(STRIDE == 1 && k == 0)) t[k] = tw[tw_index<SWZ>((j0 + k * STRIDE) << (LOGR - mlog))];
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      if (i & d) continue;
      // Outputs that the next stage of this group only multiplies stay lazy ([0, 2p)): both
      // outputs of a pair whose bit st + 1 is set are v inputs of stage st + 1, except the u
      // output when its consumer is the j = 0 peel (no multiplication). The last stage's
      // outputs leave the group: lazy only if the pass's consumer allows it (LZ).
      const bool last = st == E - 1;
      const bool is_v = !last && (i & (2 * d)) != 0;
      const bool peel = STRIDE == 1 && (i & (d - 1)) == 0;
      const bool next_peel = STRIDE == 1 && (i & (2 * d - 1)) == 0;
      const bool lu = last ? LZ : (is_v && !next_peel);
      const bool lv = last ? LZ : is_v;
      // (j = 0: factor 1, reference ntt.cpp:62-64 peel)
      if (lu && lv) {
        if (peel) bfly_dit1_m<true, true>(v[i], v[i + d], p);
        else bfly_dit_m<true, true>(v[i], v[i + d], t[i & (d - 1)], p);
      } else if (lv) {
        if (peel) bfly_dit1_m<false, true>(v[i], v[i + d], p);
        else bfly_dit_m<false, true>(v[i], v[i + d], t[i & (d - 1)], p);
      } else {
        if (peel) bfly_dit1(v[i], v[i + d], p);
        else bfly_dit(v[i], v[i + d], t[i & (d - 1)], p);
      }
    }
  }
}

// Group geometry of a round: group q (0 <= q < R >> E) covers positions base + i * STRIDE.
template <int MLOG, int E>
__device__ __forceinline__ void dif_group(int q, int& j0, int& base) {
  constexpr int STRIDE = 1 << (MLOG - E);
  j0 = q & (STRIDE - 1);
  base = ((q >> (MLOG - E)) << MLOG) + j0;
}
template <int ALOG, int E>
__device__ __forceinline__ void dit_group(int q, int& j0, int& base) {
  constexpr int STRIDE = 1 << ALOG;
  j0 = q & (STRIDE - 1);
  base = ((q >> ALOG) << (ALOG + E)) + j0;
}

// ---- shared-memory layouts ----
// Row-major [r][W]: threads column-fastest, a half-warp reads one 128 B row.
template <int W>
struct Rows {
  static constexpr bool kColumnFastest = true;
  __device__ __forceinline__ int operator()(int r, int w) const { return r * W + w; }
};

__device__ __forceinline__ int col_swizzle(int r) { return r ^ ((r >> 3) & 15); }

// Column-major [w][r] (each column contiguous, swizzled inside), threads along the column.
template <int LOGR>
struct ContigColumns {
  static constexpr bool kColumnFastest = false;
  __device__ __forceinline__ int operator()(int r, int w) const { return (w << LOGR) + col_swizzle(r); }
};

// Same prime and table for every column; SWZ: the table is stored at tw_slot(k).
template <bool SWZ>
struct UniformField {
  static constexpr bool kSwz = SWZ;
  u64 pv;
  const TwPair* t;
  __device__ __forceinline__ u64 p(int) const { return pv; }
  __device__ __forceinline__ const TwPair* tw(int) const { return t; }
};

template <bool COLFAST, int NQ, int W>
__device__ __forceinline__ void group_of(int g, int& w, int& q) {
  if constexpr (COLFAST) {
    w = g % W;
    q = g / W;
  } else {
    q = g % NQ;
    w = g / NQ;
  }
}

// ---- shared-memory rounds ----
// pre (first round only, may be nullptr): input row r is multiplied by pre[r] first.
template <int LOGR, int MLOG, int E, int W, class L, class F>
__device__ __forceinline__ void dif_round_smem(u64* s, const L& idx, const F& fld, int tid, int nt,
                                               const TwPair* pre = nullptr) {
  constexpr int NE = 1 << E, STRIDE = 1 << (MLOG - E), NQ = (1 << LOGR) >> E;
  for (int g = tid; g < NQ * W; g += nt) {
    int w, q, j0, base;
    group_of<L::kColumnFastest, NQ, W>(g, w, q);
    dif_group<MLOG, E>(q, j0, base);
    u64 v[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) v[i] = s[idx(base + i * STRIDE, w)];
    if (pre) {
#pragma unroll
      for (int i = 0; i < NE; ++i) v[i] = shoup_mul(v[i], pre[base + i * STRIDE], fld.p(w));
    }
    dif_regs<LOGR, MLOG, E, F::kSwz>(v, j0, fld.tw(w), fld.p(w));
#pragma unroll
    for (int i = 0; i < NE; ++i) s[idx(base + i * STRIDE, w)] = v[i];
  }
}

template <int LOGR, int ALOG, int E, int W, class L, class F>
__device__ __forceinline__ void dit_round_smem(u64* s, const L& idx, const F& fld, int tid, int nt) {
  constexpr int NE = 1 << E, STRIDE = 1 << ALOG, NQ = (1 << LOGR) >> E;
  for (int g = tid; g < NQ * W; g += nt) {
    int w, q, j0, base;
    group_of<L::kColumnFastest, NQ, W>(g, w, q);
    dit_group<ALOG, E>(q, j0, base);
    u64 v[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) v[i] = s[idx(base + i * STRIDE, w)];
    dit_regs<LOGR, ALOG, E, F::kSwz>(v, j0, fld.tw(w), fld.p(w));
#pragma unroll
    for (int i = 0; i < NE; ++i) s[idx(base + i * STRIDE, w)] = v[i];
  }
}

// DIF rounds whose first span is 2^MLOG, down to (but excluding) span 2^STOP.
template <int LOGR, int MLOG, int STOP, int W, class L, class F>
__device__ __forceinline__ void dif_rounds_smem(u64* s, const L& idx, const F& fld, int tid, int nt,
                                                const TwPair* pre = nullptr) {
  if constexpr (MLOG > STOP) {
    constexpr int E = Sched<LOGR>::e_dif(MLOG);
    dif_round_smem<LOGR, MLOG, E, W>(s, idx, fld, tid, nt, pre);
    __syncthreads();
    dif_rounds_smem<LOGR, MLOG - E, STOP, W>(s, idx, fld, tid, nt);
  }
}
// DIT rounds starting after ALOG stages, up to (but excluding) the round starting at STOP.
template <int LOGR, int ALOG, int STOP, int W, class L, class F>
__device__ __forceinline__ void dit_rounds_smem(u64* s, const L& idx, const F& fld, int tid, int nt) {
  if constexpr (ALOG < STOP) {
    constexpr int E = Sched<LOGR>::e_dit(ALOG);
    dit_round_smem<LOGR, ALOG, E, W>(s, idx, fld, tid, nt);
    __syncthreads();
    dit_rounds_smem<LOGR, ALOG + E, STOP, W>(s, idx, fld, tid, nt);
  }
}

// Full column transforms in shared memory. Caller must __syncthreads() before;
// both end with a barrier (none when LOGR == 0: identity).
template <int LOGR, int W, class L, class F>
__device__ __forceinline__ void tile_dif(u64* s, const L& idx, const F& fld, int tid, int nt) {
  dif_rounds_smem<LOGR, LOGR, 0, W>(s, idx, fld, tid, nt);
}
template <int LOGR, int W, class L, class F>
__device__ __forceinline__ void tile_dit(u64* s, const L& idx, const F& fld, int tid, int nt) {
  dit_rounds_smem<LOGR, 0, LOGR, W>(s, idx, fld, tid, nt);
}

__device__ __forceinline__ int bitrev(int x, int bits) { return bits ? int(__brev(unsigned(x)) >> (32 - bits)) : 0; }

}  // namespace dmg
