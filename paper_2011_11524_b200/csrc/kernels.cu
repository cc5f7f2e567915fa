// Hot-path kernels for the decimal multiplier (sm_100a).
//
// Transform passes. A length-N transform (N = 2^k or 3*2^k) is a sequence of
// passes over the array viewed as [G][R][S]: each pass runs length-R column DFTs
// (stride S) for every (g, s), then multiplies output frequency f by
// omega_{R S}^{f s} — the decimation-in-frequency step the reference's six-step
// and three-row shapes perform (conv.cpp:72-87, :109-125), generalised to any
// number of passes so every tile fits shared memory. Columns are read as
// 128 B row segments (16 adjacent columns) so the reference's explicit
// transpositions (conv.cpp:30-38) become strided addressing.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

#include <cuda.h>

#include "kernels.cuh"
#include "digits.cuh"
#include "engine.hpp"
#include "ntt_tile.cuh"

namespace dmg {

namespace {

constexpr int W = kTileW;
constexpr int NT = kPassThreads;

// bit reversal of a compile-time index (unrolled register groups)
constexpr int crev(int i, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
  return r;
}

// Tile geometry. Row passes (S >= 16): one group g, 16 adjacent columns s0..s0+15;
// element (r, w) at g R S + r S + s0 + w. Column passes (S == 1): 16 adjacent
// groups, each a contiguous run of R words; element (r, w) at (c0 + w) R + r.
template <int LOGR, bool ROWS, int TW>
struct Geom {
  unsigned long long base, s0;
  unsigned long long S, tw_col;
  int logS, tw_logS, tw_lb;
  __device__ __forceinline__ Geom(const PassArgs& a) {
    const unsigned long long tile = blockIdx.x / a.np;
    S = a.S;
    logS = a.logS;
    tw_logS = a.tw_logS;
    tw_lb = a.tw_lbits;
    if (ROWS) {
      // group-fastest tile order: the G groups share the twiddle rows T[f][s0..s0+15],
      // so consecutive CTAs reuse them from L2 instead of re-streaming them from HBM
      const unsigned long long g = tile % a.G;
      s0 = (tile / a.G) * TW;
      base = (g << (LOGR + a.logS)) + s0;
    } else {
      const unsigned long long c0 = tile * TW;
      s0 = 0;
      base = c0 << LOGR;
    }
    tw_col = a.tw_off + s0;
  }
  __device__ __forceinline__ unsigned long long at(int r, int w) const {
    return ROWS ? base + ((unsigned long long)r << logS) + w : base + ((unsigned long long)w << LOGR) + r;
  }
  // inter-pass twiddle omega_M^{f s} for the element at row r (frequency bitrev(r) after DIF)
  __device__ __forceinline__ const TwPair& tw(const TwPair* T, int r, int w) const {
    return T[((unsigned long long)bitrev(r, LOGR) << tw_logS) + tw_col + w];
  }
  // v omega_M^{f s}: one Shoup product with the full R x S table, or two with the factorised
  // tables lo[f][s mod 2^lb] * hi[f][s >> lb] (tw_lb > 0; hi carries the scale)
  // (FACT is a template parameter: a runtime branch here split the unrolled 8-element groups
  // into separate blocks and cost the R = 512 passes 5-28%)
  // The same for the 2^E elements base + i of one register group (base = q 2^E, STRIDE 1):
  // f_i = bitrev(base + i) = bitrev(i, E) 2^(LOGR - E) + bitrev(q, LOGR - E), so every row pointer
  // is one per-group base plus a compile-time multiple of a per-kernel stride (the per-element
  // bit reversal, shift and 64-bit index sum cost ~10 instructions per element in the epilogue).
  template <int E, bool FACT>
  __device__ __forceinline__ void twist_group(u64 (&v)[1 << E], const TwPair* T, const TwPair* Hi, int q, int w,
                                              u64 p) const {
    const unsigned long long f0 = (unsigned long long)bitrev(q, LOGR - E);
    const unsigned long long s = tw_col + w;
    if constexpr (!FACT) {
      const TwPair* t0 = T + (f0 << tw_logS) + s;
      const unsigned long long fs = 1ull << (LOGR - E + tw_logS);
#pragma unroll
      for (int i = 0; i < (1 << E); ++i) v[i] = shoup_mul(v[i], t0[(unsigned long long)crev(i, E) * fs], p);
    } else {
      const TwPair* l0 = T + (f0 << tw_lb) + (s & ((1ull << tw_lb) - 1));
      const TwPair* h0 = Hi + (f0 << (tw_logS - tw_lb)) + (s >> tw_lb);
      const unsigned long long fl = 1ull << (LOGR - E + tw_lb), fh = 1ull << (LOGR - E + tw_logS - tw_lb);
#pragma unroll
      for (int i = 0; i < (1 << E); ++i) {
        const unsigned long long k = (unsigned long long)crev(i, E);
        v[i] = shoup_mul(shoup_mul(v[i], l0[k * fl], p), h0[k * fh], p);
      }
    }
  }
  // element stride between consecutive rows of the tile
  __device__ __forceinline__ unsigned long long row_stride() const { return ROWS ? (1ull << logS) : 1ull; }
  template <bool FACT>
  __device__ __forceinline__ u64 twist(u64 v, const TwPair* T, const TwPair* Hi, int r, int w, u64 p) const {
    const unsigned long long f = (unsigned long long)bitrev(r, LOGR);
    if constexpr (!FACT) {
      return shoup_mul(v, T[(f << tw_logS) + tw_col + w], p);
    } else {
      const unsigned long long s = tw_col + w;
      v = shoup_mul(v, T[(f << tw_lb) + (s & ((1ull << tw_lb) - 1))], p);
      return shoup_mul(v, Hi[(f << (tw_logS - tw_lb)) + (s >> tw_lb)], p);
    }
  }
};

template <int LOGR, bool ROWS, int TW>
using TileLayout = typename std::conditional<ROWS, Rows<TW>, ContigColumns<LOGR>>::type;

// Threads of a pass CTA: one 8-element register group per thread, 32..256.
constexpr int pass_threads(int logr, int tw) {
  return ((1 << logr) * tw / 8) < 32 ? 32 : (((1 << logr) * tw / 8) > NT ? NT : ((1 << logr) * tw / 8));
}

// Twiddle tables of column-major tiles are swizzled (ntt_tile.cuh); row-major ones are not.
#ifndef DMG_PASS_NOSWZ
template <bool ROWS>
constexpr bool kSwzTables = !ROWS;
#else
template <bool ROWS>
constexpr bool kSwzTables = false;
#endif

// Tiles are staged HBM -> SMEM by one burst of cp.async before the first round (every load
// in flight at once) instead of the first round reading HBM into registers. Measured (A/B,
// DMG_STAGE_MASK bits): 1 forward row tiles (config 3 -2.1%, 4 -1.3%, 5 -1.3%); 2 inverse
// row tiles (config 4 a further -0.8%); 4 column tiles of the forward and fused passes —
// only the narrow 4-column tiles gain (config 1 -2.4%); full 16-column ones lose 1%
// (configs 3-5), so they keep the direct first round.
#ifndef DMG_STAGE_MASK
#define DMG_STAGE_MASK 7
#endif
template <bool ROWS, int TW>
constexpr bool kStageFwd = ROWS ? (DMG_STAGE_MASK & 1) != 0 : ((DMG_STAGE_MASK & 4) != 0 && TW < kTileW);
template <bool ROWS>
constexpr bool kStageInv = ROWS && (DMG_STAGE_MASK & 2) != 0;

// Full-width row tiles (16 columns: R row segments of 128 B, dense [r][16] in shared memory)
// are staged by the TMA unit instead: the array is a 2-D tensor {S, G R} of u64 (row pitch
// 8 S bytes), the tile a box {16, min(R, 256)} at (s0, g R) -- one or two
// cp.async.bulk.tensor.2d instructions from one thread per CTA (against 16 cp.async plus
// index arithmetic from every thread), completion counted in bytes on an mbarrier that
// every thread waits on. (Per-row cp.async.bulk copies are no substitute: UBLKCP takes
// uniform-register addresses, so per-thread rows compile to a 32-step loop per warp.)
// DMG_BULK_ROWS=0 keeps the cp.async burst (A/B).
#ifndef DMG_BULK_ROWS
#define DMG_BULK_ROWS 1
#endif
// DMG_BULK_NARROW=1: the 4-column tiles of small transforms too (32-byte box rows); measured
// neutral (config 1 39 us either way), so they keep the cp.async burst
#ifndef DMG_BULK_NARROW
#define DMG_BULK_NARROW 0
#endif
template <bool ROWS, int TW>
constexpr bool kBulkRows = ROWS && (TW == kTileW || DMG_BULK_NARROW != 0) && DMG_BULK_ROWS != 0;
constexpr int kBoxRows = 256;  // TMA box dimensions are at most 256

__device__ __forceinline__ void mbar_init(u64* bar, unsigned count) {
  const unsigned b = unsigned(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");  // visible to the async proxy
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, unsigned bytes) {
  const unsigned b = unsigned(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, unsigned parity) {
  const unsigned b = unsigned(__cvta_generic_to_shared(bar));
  unsigned done;
  do {
    asm volatile(
        "{\n\t.reg .pred ok;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 ok, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, ok;\n\t}"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
  } while (!done);
}

// The same tiles leave through the TMA unit: the last round writes its results back into the
// tile in shared memory (same positions it read) and one thread stores the box to the output
// tensor, instead of 8 strided 8-byte global stores per register group (config 4 32.89 ->
// 32.35 ms, config 5 314.9 -> 308.7 ms). DMG_BULK_STORE=0 keeps the direct stores (A/B).
#ifndef DMG_BULK_STORE
#define DMG_BULK_STORE 1
#endif
#ifndef DMG_FUSED_BULK_X
#define DMG_FUSED_BULK_X 1
#endif
#ifndef DMG_FUSED_BULK_Y
#define DMG_FUSED_BULK_Y 1
#endif
#ifndef DMG_FUSED_BULK_OUT
#define DMG_FUSED_BULK_OUT 1
#endif
template <int LOGR, int TW>
__device__ __forceinline__ void store_rows_tma(const u64* sm, const void* map, unsigned long long s0,
                                               unsigned long long row0) {
  constexpr int R = 1 << LOGR, BR = R < kBoxRows ? R : kBoxRows;
#pragma unroll
  for (int h = 0; h < R / BR; ++h) {
    const unsigned sa = unsigned(__cvta_generic_to_shared(sm + h * BR * TW));
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map),
                 "r"(int(s0)), "r"(int(row0) + h * BR), "r"(sa)
                 : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the CTA's shared memory outlives the reads
}

// The tile's inter-pass twiddle rows T[f][s0 .. s0 + 16) (16 pairs = 256 bytes per row, all R
// rows) pulled towards L2 by the TMA unit: the table is a 2-D tensor {2 S' u64, rows}, the
// rows a box {32, min(R, 256)} -- one or two prefetch instructions from one thread instead of
// four prefetch.global.L2 per thread (DMG_TMA_TWPF=0 keeps those). DMG_TMA_TWPF_FWD_GROUP: the
// forward pass over per-group tables (pass 1 of N = 3 * 2^k), which the per-thread loop did
// not pay for: 0 none, 1 at kernel entry, 2 after the first round.
#ifndef DMG_TMA_TWPF
#define DMG_TMA_TWPF 1
#endif
#ifndef DMG_TMA_TWPF_FWD_GROUP
#define DMG_TMA_TWPF_FWD_GROUP 0
#endif
#ifndef DMG_TMA_TWPF_INV_SHARED
#define DMG_TMA_TWPF_INV_SHARED 0
#endif
template <int LOGR>
__device__ __forceinline__ void prefetch_tw_rows_tma(const void* map, unsigned long long col, unsigned long long row0) {
  constexpr int R = 1 << LOGR, BR = R < kBoxRows ? R : kBoxRows;
#pragma unroll
  for (int h = 0; h < R / BR; ++h)
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(int(2 * col)),
                 "r"(int(row0) + h * BR)
                 : "memory");
}

// Thread 0 of the CTA: arm the barrier and issue the tile's TMA copies (rows row0 .. row0 + R
// of the tensor, columns s0 .. s0 + 16). Everyone else meets it at the next __syncthreads and
// then waits on the barrier's phase 0.
// table != nullptr (DMG_BULK_TABLE): the pass's butterfly table (R / 2 pairs, stored linearly
// for row-major tiles) rides on the same barrier as one more bulk copy, instead of a load and a
// shared store per thread.
#ifndef DMG_BULK_TABLE
#define DMG_BULK_TABLE 1
#endif
template <int LOGR, int TW>
__device__ __forceinline__ void stage_rows_tma(u64* sm, const void* map, unsigned long long s0,
                                               unsigned long long row0, u64* bar, TwPair* tw_dst = nullptr,
                                               const TwPair* table = nullptr) {
  constexpr int R = 1 << LOGR, BR = R < kBoxRows ? R : kBoxRows;
  constexpr unsigned kTableBytes = unsigned((R / 2) * sizeof(TwPair));
  mbar_init(bar, 1);
  mbar_expect_tx(bar, unsigned(R * TW * sizeof(u64)) + (table ? kTableBytes : 0u));
  const unsigned b = unsigned(__cvta_generic_to_shared(bar));
  if (table)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     unsigned(__cvta_generic_to_shared(tw_dst))),
                 "l"(table), "r"(kTableBytes), "r"(b)
                 : "memory");
#pragma unroll
  for (int h = 0; h < R / BR; ++h) {
    const unsigned sa = unsigned(__cvta_generic_to_shared(sm + h * BR * TW));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(sa), "l"(map), "r"(int(s0)), "r"(int(row0) + h * BR), "r"(b)
        : "memory");
  }
}

// Issue the async copy of a tile into its shared layout: 16-byte chunks of the row segments
// for row-major tiles; 8-byte words for swizzled columns (the swizzle may swap a 16-byte
// pair), consecutive threads on consecutive rows of a column (coalesced). The caller waits
// (cp.async.wait_all) and synchronises.
template <int LOGR, bool ROWS, int TW, int NTK, class Gm, class Lay>
__device__ __forceinline__ void stage_tile(u64* sm, const u64* src, const Gm& G, const Lay& L, int tid) {
  constexpr int R = 1 << LOGR;
  if constexpr (ROWS) {
    constexpr int CH = TW / 2;  // 16-byte chunks per row segment
    for (int i = tid; i < R * CH; i += NTK) {
      const int r = i / CH, c = (i % CH) * 2;
      const unsigned sa = unsigned(__cvta_generic_to_shared(&sm[L(r, c)]));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src + G.at(r, c)) : "memory");
    }
  } else {
    for (int i = tid; i < R * TW; i += NTK) {
      const int w = i >> LOGR, r = i & (R - 1);
      const unsigned sa = unsigned(__cvta_generic_to_shared(&sm[L(r, w)]));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src + G.at(r, w)) : "memory");
    }
  }
}

template <int LOGR, int NTK, bool SWZ>
__device__ __forceinline__ void load_table(TwPair* dst, const TwPair* src) {
  for (int i = threadIdx.x; i < (1 << LOGR) / 2; i += NTK) dst[tw_index<SWZ>(i)] = src[i];
}

template <int LOGR, bool ROWS, int E, int TW>
__device__ __forceinline__ void group_coords(int g, int& w, int& q) {
  group_of<ROWS, ((1 << LOGR) >> E), TW>(g, w, q);
}

// Minimum resident CTAs per SM requested from ptxas (launch bounds), measured per shape:
//  * R = 256: tiles use 34 KB of shared memory, so registers limit occupancy; capping them
//    at 64 (4 CTAs/SM) is 1-2% faster on configs 3-5 than ptxas's own choice (80: 3 CTAs);
//  * R = 512, 16-column tiles (68 KB, at most 3 CTAs/SM): 3 (DMG_FWD_MINB9) for the forward
//    pass; the fused/inverse ones below;
//  * R = 512, 4-column tiles (small transforms, config 1): 3;
//  * smaller radices: ptxas's default (0 = unspecified). NB an explicit 1 is not the
//    default: it let ptxas double the registers of the R = 128 passes (6 -> 4 CTAs/SM,
//    config 5 +2.6%).
// R = 512 forward row passes: 3 CTAs/SM (<= 85 registers). The grouped epilogue addressing
// (Geom::twist_group) let ptxas grow an unconstrained kernel to 106 registers (2 CTAs/SM);
// capped, config 4's forward passes run 13.30 -> 12.75 ms.
#ifndef DMG_FWD_MINB9
#define DMG_FWD_MINB9 3
#endif
#ifndef DMG_GROUP_PREFETCH
#define DMG_GROUP_PREFETCH 0
#endif
#ifndef DMG_INV_GROUP_PREFETCH
#define DMG_INV_GROUP_PREFETCH 1
#endif
constexpr int pass_min_blocks(int logr, int tw) {
  return logr == 9 ? (tw == kTileW ? DMG_FWD_MINB9 : 3) : (logr == 8 ? 4 : 0);
}

// Forward pass: column DIFs, then the inter-pass twiddle omega_M^{f s} (row passes).
// Full-width row tiles arrive and leave by TMA (stage_rows_tma / store_rows_tma); narrow
// tiles are staged by cp.async; column tiles read HBM into the first round's registers. All
// but the TMA-stored tiles write HBM from the last round's registers.
template <int LOGR, bool ROWS, int TW, bool FACT = false>
__global__ void __launch_bounds__(pass_threads(LOGR, TW), pass_min_blocks(LOGR, TW)) k_pass_fwd(const __grid_constant__ PassArgs a, const __grid_constant__ TileMaps maps) {
  // at entry: a wait placed after the table loads kept the compiler from hoisting the
  // first round's HBM loads above that barrier (config 5 +5%)
  pdl_wait();
  constexpr int R = 1 << LOGR, NTK = pass_threads(LOGR, TW);
  constexpr int E1 = Sched<LOGR>::e_dif(LOGR), EL = Sched<LOGR>::first_e;
  extern __shared__ __align__(128) u64 sm[];
  TwPair* tw = reinterpret_cast<TwPair*>(sm + R * TW);
  const int pr = int(blockIdx.x % a.np), tid = threadIdx.x;
  const u64 p = a.p[pr];
  const u64* src = blockIdx.y ? a.src_b[pr] : a.src[pr];  // blockIdx.y: the second operand
  u64* dst = blockIdx.y ? a.dst_b[pr] : a.dst[pr];
  const Geom<LOGR, ROWS, TW> G(a);
  const unsigned long long grp = ROWS ? (blockIdx.x / a.np) % a.G : 0;  // group of a row tile
  const TwPair* __restrict__ T = a.pass_tw[pr] + grp * a.tw_gstride;
  const TwPair* __restrict__ Hi = a.pass_hi[pr] + grp * a.hi_gstride;
  // (the launcher encodes the table maps for the launches whose tiles move by TMA)
  constexpr bool TWPF = ROWS && !FACT && DMG_TMA_TWPF != 0 && kBulkRows<ROWS, TW> && kStageFwd<ROWS, TW> && LOGR > E1;
  if constexpr (ROWS && !FACT) if (DMG_GROUP_PREFETCH || a.tw_gstride == 0) {
    // The twiddles are applied in the epilogue, after the DIF; start pulling the tile's
    // rows T[f][s0 .. s0 + TW) (TW pairs = TW * 16 bytes each) into L2 now so those
    // loads hit L2 instead of DRAM (large-S passes stream a table of N / 3 .. N pairs).
    if constexpr (TWPF) {
      if (tid == 0) prefetch_tw_rows_tma<LOGR>(&maps.m[8 + pr], G.tw_col, a.tw_gstride ? grp << LOGR : 0);
    } else {
      constexpr int LINES = TW * 16 / 128 > 0 ? TW * 16 / 128 : 1;
      for (int i = tid; i < R * LINES; i += NTK) {
        const TwPair* row = &G.tw(T, i / LINES, 0) + (i % LINES) * 8;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(row));
      }
    }
  }
  if constexpr (TWPF && DMG_TMA_TWPF_FWD_GROUP == 1)
    if (a.tw_gstride != 0 && tid == 0) prefetch_tw_rows_tma<LOGR>(&maps.m[8 + pr], G.tw_col, grp << LOGR);
  const TileLayout<LOGR, ROWS, TW> L;
  constexpr bool BULK = kBulkRows<ROWS, TW> && kStageFwd<ROWS, TW> && LOGR > E1;
  u64* bar = sm + R * TW + R;  // after the tile and the R / 2 table pairs
  if constexpr (BULK) {
    constexpr bool TBL = false;  // forward passes: neutral at R = 512, +2.7% at R = 256
    if (tid == 0)
      stage_rows_tma<LOGR, TW>(sm, &maps.m[blockIdx.y * 2 + pr], G.s0, grp << LOGR, bar, tw,
                               TBL ? a.dft_fwd[pr] : nullptr);
    if constexpr (!TBL) load_table<LOGR, NTK, kSwzTables<ROWS>>(tw, a.dft_fwd[pr]);
  } else if constexpr (kStageFwd<ROWS, TW> && LOGR > E1) {
    stage_tile<LOGR, ROWS, TW, NTK>(sm, src, G, L, tid);
  }
  if constexpr (!BULK) load_table<LOGR, NTK, kSwzTables<ROWS>>(tw, a.dft_fwd[pr]);
  if constexpr (!BULK && kStageFwd<ROWS, TW> && LOGR > E1) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if constexpr (BULK) mbar_wait(bar, 0);
  pdl_trigger_mid();
  if constexpr (TWPF && DMG_TMA_TWPF_FWD_GROUP == 2)  // once the tile has arrived
    if (a.tw_gstride != 0 && tid == 0) prefetch_tw_rows_tma<LOGR>(&maps.m[8 + pr], G.tw_col, grp << LOGR);
  // merged radix-3 twiddles: column input r of radix-3 row g times omega_{3 R}^{g r}, in the
  // first round (a separate shared-memory sweep cost config 4's two launches +1.1 ms)
  const TwPair* pre = (ROWS && a.pre[pr] && grp) ? a.pre[pr] + grp * R : nullptr;
  if constexpr (LOGR == E1) {  // one round: HBM -> registers -> HBM
    for (int g = tid; g < (R >> E1) * TW; g += NTK) {
      int w, q, j0, base;
      group_coords<LOGR, ROWS, E1, TW>(g, w, q);
      dif_group<LOGR, E1>(q, j0, base);
      u64 v[1 << E1];
#pragma unroll
      for (int i = 0; i < (1 << E1); ++i) v[i] = src[G.at(base + i, w)];
      dif_regs<LOGR, LOGR, E1, kSwzTables<ROWS>, ROWS>(v, j0, tw, p);  // lazy: twiddled next
      if constexpr (ROWS) G.template twist_group<E1, FACT>(v, T, Hi, q, w, p);
      u64* d = dst + G.at(base, w);
      const unsigned long long es = G.row_stride();
#pragma unroll
      for (int i = 0; i < (1 << E1); ++i) d[i * es] = v[i];
    }
    return;
  } else {
    if constexpr (kStageFwd<ROWS, TW>) {
      dif_rounds_smem<LOGR, LOGR, EL, TW>(sm, L, UniformField<kSwzTables<ROWS>>{p, tw}, tid, NTK, pre);
    } else {
      constexpr int ST1 = 1 << (LOGR - E1);
      for (int g = tid; g < (R >> E1) * TW; g += NTK) {
        int w, q, j0, base;
        group_coords<LOGR, ROWS, E1, TW>(g, w, q);
        dif_group<LOGR, E1>(q, j0, base);
        u64 v[1 << E1];
#pragma unroll
        for (int i = 0; i < (1 << E1); ++i) v[i] = src[G.at(base + i * ST1, w)];
        dif_regs<LOGR, LOGR, E1, kSwzTables<ROWS>>(v, j0, tw, p);
#pragma unroll
        for (int i = 0; i < (1 << E1); ++i) sm[L(base + i * ST1, w)] = v[i];
      }
      __syncthreads();
      dif_rounds_smem<LOGR, LOGR - E1, EL, TW>(sm, L, UniformField<kSwzTables<ROWS>>{p, tw}, tid, NTK);
    }
    for (int g = tid; g < (R >> EL) * TW; g += NTK) {
      int w, q, j0, base;
      group_coords<LOGR, ROWS, EL, TW>(g, w, q);
      dif_group<EL, EL>(q, j0, base);
      u64 v[1 << EL];
#pragma unroll
      for (int i = 0; i < (1 << EL); ++i) v[i] = sm[L(base + i, w)];
      dif_regs<LOGR, EL, EL, kSwzTables<ROWS>, ROWS>(v, 0, tw, p);  // lazy: twiddled next
      if constexpr (ROWS) G.template twist_group<EL, FACT>(v, T, Hi, q, w, p);
      if constexpr (BULK && DMG_BULK_STORE) {
#pragma unroll
        for (int i = 0; i < (1 << EL); ++i) sm[L(base + i, w)] = v[i];
      } else {
        u64* d = dst + G.at(base, w);
        const unsigned long long es = G.row_stride();
#pragma unroll
        for (int i = 0; i < (1 << EL); ++i) d[i * es] = v[i];
      }
    }
    if constexpr (BULK && DMG_BULK_STORE) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async proxy
      __syncthreads();
      if (tid == 0) store_rows_tma<LOGR, TW>(sm, &maps.m[4 + blockIdx.y * 2 + pr], G.s0, grp << LOGR);
    }
  }
}

// Inverse pass: conjugate inter-pass twiddle (row passes; carries the convolution
// scale on the first inverse pass), then column DITs.
// R = 512 inverse row passes capped at 80 registers (3 CTAs/SM, like the forward pass) instead
// of ptxas's 96 (2 CTAs/SM): config 4 inverse passes 7.56 -> 7.08 ms, no spills.
#ifndef DMG_INV_MINB9
#define DMG_INV_MINB9 3
#endif
constexpr int pass_inv_min_blocks(int logr, int tw) {
  return (logr == 9 && tw == kTileW) ? DMG_INV_MINB9 : pass_min_blocks(logr, tw);
}
template <int LOGR, bool ROWS, int TW, bool FACT = false, bool LZO = false>
__global__ void __launch_bounds__(pass_threads(LOGR, TW), pass_inv_min_blocks(LOGR, TW)) k_pass_inv(const __grid_constant__ PassArgs a, const __grid_constant__ TileMaps maps) {
  // at entry: a wait placed after the table loads kept the compiler from hoisting the
  // first round's HBM loads above that barrier (config 5 +5%)
  pdl_wait();
  constexpr int R = 1 << LOGR, NTK = pass_threads(LOGR, TW);
  constexpr int E1 = Sched<LOGR>::first_e;
  constexpr int EL = Sched<LOGR>::rem ? Sched<LOGR>::rem : E1;  // last DIT round
  constexpr int AL = LOGR - EL;                                   // its starting stage
  extern __shared__ __align__(128) u64 sm[];
  TwPair* tw = reinterpret_cast<TwPair*>(sm + R * TW);
  const int pr = int(blockIdx.x % a.np), tid = threadIdx.x;
  const u64 p = a.p[pr];
  const u64* src = a.src[pr];
  u64* dst = a.dst[pr];
  const unsigned long long grp = ROWS ? (blockIdx.x / a.np) % a.G : 0;  // group of a row tile
  const TwPair* __restrict__ T = a.pass_tw[pr] + grp * a.tw_gstride;
  const TwPair* __restrict__ Hi = a.pass_hi[pr] + grp * a.hi_gstride;
  const TwPair sc = a.final_scale[pr];
  const Geom<LOGR, ROWS, TW> G(a);
  const TileLayout<LOGR, ROWS, TW> L;
#if DMG_TMA_TWPF_INV_SHARED
  // tables shared by the pass's groups too, now that the prefetch costs one thread two
  // instructions (as a per-thread loop it lost on configs 3 and 5)
  if constexpr (ROWS && !FACT && DMG_TMA_TWPF != 0 && kBulkRows<ROWS, TW> && kStageInv<ROWS> && LOGR > E1)
    if (a.tw_gstride == 0 && tid == 0) prefetch_tw_rows_tma<LOGR>(&maps.m[8 + pr], G.tw_col, 0);
#endif
#if DMG_INV_GROUP_PREFETCH
  if constexpr (ROWS && !FACT) if (a.tw_gstride != 0) {
    // per-group tables (pass 1 after a merged radix-3 pass) stream from HBM with no reuse
    // across tiles: start them towards L2 before the tile's own loads
    if constexpr (DMG_TMA_TWPF != 0 && kBulkRows<ROWS, TW> && kStageInv<ROWS> && LOGR > E1) {
      if (tid == 0) prefetch_tw_rows_tma<LOGR>(&maps.m[8 + pr], G.tw_col, grp << LOGR);
    } else {
      constexpr int LINES = TW * 16 / 128 > 0 ? TW * 16 / 128 : 1;
      for (int i = tid; i < R * LINES; i += NTK) {
        const TwPair* row = &G.tw(T, i / LINES, 0) + (i % LINES) * 8;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(row));
      }
    }
  }
#endif
  constexpr bool STAGE = kStageInv<ROWS> && LOGR > E1;
  constexpr bool BULK = STAGE && kBulkRows<ROWS, TW>;
  u64* bar = sm + R * TW + R;  // after the tile and the R / 2 table pairs
  if constexpr (BULK) {
    // R = 512 only: the inverse pass 5.83 -> 5.62 ms on config 4; R = 256 passes lose 3%
    constexpr bool TBL = DMG_BULK_TABLE != 0 && !kSwzTables<ROWS> && LOGR >= 9;
    if (tid == 0)
      stage_rows_tma<LOGR, TW>(sm, &maps.m[pr], G.s0, grp << LOGR, bar, tw, TBL ? a.dft_inv[pr] : nullptr);
    if constexpr (!TBL) load_table<LOGR, NTK, kSwzTables<ROWS>>(tw, a.dft_inv[pr]);
  } else if constexpr (STAGE) {
    stage_tile<LOGR, ROWS, TW, NTK>(sm, src, G, L, tid);
  }
  if constexpr (!BULK) load_table<LOGR, NTK, kSwzTables<ROWS>>(tw, a.dft_inv[pr]);
  if constexpr (STAGE && !BULK) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if constexpr (BULK) mbar_wait(bar, 0);
  pdl_trigger_mid();
  for (int g = tid; g < (R >> E1) * TW; g += NTK) {
    int w, q, j0, base;
    group_coords<LOGR, ROWS, E1, TW>(g, w, q);
    dit_group<0, E1>(q, j0, base);
    u64 v[1 << E1];
    if constexpr (STAGE) {
#pragma unroll
      for (int i = 0; i < (1 << E1); ++i) v[i] = sm[L(base + i, w)];
    } else {
      const u64* s0 = src + G.at(base, w);
      const unsigned long long es = G.row_stride();
#pragma unroll
      for (int i = 0; i < (1 << E1); ++i) v[i] = s0[i * es];
    }
    if constexpr (ROWS) G.template twist_group<E1, FACT>(v, T, Hi, q, w, p);
    dit_regs<LOGR, 0, E1, kSwzTables<ROWS>, LZO && LOGR == E1>(v, 0, tw, p);
#pragma unroll
    for (int i = 0; i < (1 << E1); ++i) {
      if constexpr (LOGR == E1) {
        if (a.has_final_scale) v[i] = shoup_mul(v[i], sc, p);
        dst[G.at(base + i, w)] = v[i];
      } else {
        sm[L(base + i, w)] = v[i];
      }
    }
  }
  if constexpr (LOGR > E1) {
    __syncthreads();
    dit_rounds_smem<LOGR, E1, AL, TW>(sm, L, UniformField<kSwzTables<ROWS>>{p, tw}, tid, NTK);
    constexpr int STL = 1 << AL;
    for (int g = tid; g < (R >> EL) * TW; g += NTK) {
      int w, q, j0, base;
      group_coords<LOGR, ROWS, EL, TW>(g, w, q);
      dit_group<AL, EL>(q, j0, base);
      u64 v[1 << EL];
#pragma unroll
      for (int i = 0; i < (1 << EL); ++i) v[i] = sm[L(base + i * STL, w)];
      dit_regs<LOGR, AL, EL, kSwzTables<ROWS>, LZO>(v, j0, tw, p);
#pragma unroll
      for (int i = 0; i < (1 << EL); ++i) {
        if (a.has_final_scale) v[i] = shoup_mul(v[i], sc, p);
        if constexpr (BULK && DMG_BULK_STORE)
          sm[L(base + i * STL, w)] = v[i];
        else
          dst[G.at(base + i * STL, w)] = v[i];
      }
    }
    if constexpr (BULK && DMG_BULK_STORE) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async proxy
      __syncthreads();
      if (tid == 0) store_rows_tma<LOGR, TW>(sm, &maps.m[4 + pr], G.s0, grp << LOGR);
    }
  }
}

// Last forward pass (S == 1) of one operand fused with the pointwise REDC
// product against the other operand's finished spectrum (reference
// conv.cpp:205-208, :299-305) and the first inverse pass. The last DIF round
// and the first DIT round act on the same 8-element groups, so DIF -> pointwise
// -> DIT happens in registers.
// TWO: a.other holds the first operand BEFORE its last forward pass (not its spectrum); the
// CTA stages that tile too and runs its whole DIF in shared memory, so the first operand's
// last pass needs no launch (and its spectrum no HBM round trip): the standalone column pass
// ran at ~0.5 instructions per cycle against the fused kernel's ~0.66.
// (Two tiles of R = 256 x 16 take 64 KB: three CTAs per SM by shared memory, so TWO
// kernels get the 85 registers of a 3-CTA bound instead of R = 256's 64.)
constexpr int fused_min_blocks(int logr, int tw, bool two) {
  return two && logr == 8 && tw == kTileW ? 3 : pass_min_blocks(logr, tw);
}
template <int LOGR, int TW, bool LZO = false, bool TWO = false>
__global__ void __launch_bounds__(pass_threads(LOGR, TW), fused_min_blocks(LOGR, TW, TWO)) k_pass_fused(PassArgs a) {
  // at entry: a wait placed after the table loads kept the compiler from hoisting the
  // first round's HBM loads above that barrier (config 5 +5%)
  pdl_wait();
  constexpr int R = 1 << LOGR, NTK = pass_threads(LOGR, TW);
  constexpr int E1 = Sched<LOGR>::e_dif(LOGR), EM = Sched<LOGR>::first_e;
  constexpr int EL = Sched<LOGR>::rem ? Sched<LOGR>::rem : EM;
  constexpr int AL = LOGR - EL;
  extern __shared__ __align__(128) u64 sm[];
  u64* smx = sm + R * TW;  // TWO: the first operand's tile
  TwPair* twf = reinterpret_cast<TwPair*>(sm + (TWO ? 2 : 1) * R * TW);
  TwPair* twi = twf + R / 2;
  const int pr = int(blockIdx.x % a.np), tid = threadIdx.x;
  const u64 p = a.p[pr], pp = a.pp[pr];
  const u64* src = a.src[pr];
  const u64* oth = a.other[pr];
  u64* dst = a.dst[pr];
  const TwPair sc = a.final_scale[pr];
  const Geom<LOGR, false, TW> G(a);
  const ContigColumns<LOGR> L;
  constexpr bool STAGE = kStageFwd<false, TW> && LOGR > EM;
  // TWO, full-width tiles: the first operand's tile (one contiguous run of R * TW words) comes
  // in by a single bulk copy into the still unused y region, unswizzled; its first DIF round
  // reads it from there and writes the swizzled layout into smx (DMG_FUSED_BULK_X=0: the
  // 8-byte cp.async burst straight into the swizzled layout).
  constexpr bool XBULK = TWO && !STAGE && LOGR > E1 && DMG_FUSED_BULK_X != 0;
  // The operand's own tile the same way (DMG_FUSED_BULK_Y): copied unswizzled into its region
  // -- for TWO once the first operand's first round has left it, so the copy runs under that
  // operand's remaining rounds -- and re-laid out in place by the first round (all reads,
  // a barrier, then the swizzled writes) instead of that round reading HBM into registers.
  constexpr bool YBULK = !STAGE && LOGR > E1 && TW == kTileW && DMG_FUSED_BULK_Y != 0 && (!TWO || XBULK) &&
                         ((R >> E1) % 32) == 0 && (1 << (LOGR - E1)) >= 16;  // (the re-layout's hazard analysis)
  // ... and the results leave the same way (DMG_FUSED_BULK_OUT): the last DIT round writes
  // them unswizzled into the tile's region (same hazard analysis, its stride is 2^AL) and one
  // thread stores the contiguous run.
  constexpr bool OBULK = YBULK && DMG_FUSED_BULK_OUT != 0 && LOGR > EM && (((R >> EL) % 32) == 0) && (1 << AL) >= 16;
  u64* bar = sm + (TWO ? 2 : 1) * R * TW + 2 * R;  // after the tiles and both tables
  auto bulk_tile = [&](const u64* g) {  // thread 0: one bulk copy of the contiguous tile into sm
    mbar_expect_tx(bar, unsigned(R * TW * sizeof(u64)));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     unsigned(__cvta_generic_to_shared(sm))),
                 "l"(g + G.at(0, 0)), "r"(unsigned(R * TW * sizeof(u64))), "r"(unsigned(__cvta_generic_to_shared(bar)))
                 : "memory");
  };
  if constexpr (STAGE) stage_tile<LOGR, false, TW, NTK>(sm, src, G, L, tid);
  if constexpr (XBULK || YBULK) {
    if (tid == 0) {
      mbar_init(bar, 1);
      bulk_tile(XBULK ? oth : src);
    }
  }
  if constexpr (TWO && !XBULK) stage_tile<LOGR, false, TW, NTK>(smx, oth, G, L, tid);
  load_table<LOGR, NTK, kSwzTables<false>>(twf, a.dft_fwd[pr]);
  load_table<LOGR, NTK, kSwzTables<false>>(twi, a.dft_inv[pr]);
  if constexpr (STAGE || (TWO && !XBULK)) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if constexpr (XBULK || YBULK) mbar_wait(bar, 0);
  pdl_trigger_mid();
  if constexpr (XBULK) {
    constexpr int ST1 = 1 << (LOGR - E1);
    for (int g = tid; g < (R >> E1) * TW; g += NTK) {
      int w, q, j0, base;
      group_coords<LOGR, false, E1, TW>(g, w, q);
      dif_group<LOGR, E1>(q, j0, base);
      u64 v[1 << E1];
#pragma unroll
      for (int i = 0; i < (1 << E1); ++i) v[i] = sm[(w << LOGR) + base + i * ST1];
      dif_regs<LOGR, LOGR, E1, kSwzTables<false>>(v, j0, twf, p);
#pragma unroll
      for (int i = 0; i < (1 << E1); ++i) smx[L(base + i * ST1, w)] = v[i];
    }
    __syncthreads();
    if constexpr (YBULK) {
      if (tid == 0) {  // the y region is free again: its tile comes in under the rounds below
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bulk_tile(src);
      }
    }
    dif_rounds_smem<LOGR, LOGR - E1, 0, TW>(smx, L, UniformField<kSwzTables<false>>{p, twf}, tid, NTK);
  } else if constexpr (TWO) {
    tile_dif<LOGR, TW>(smx, L, UniformField<kSwzTables<false>>{p, twf}, tid, NTK);
  }
  if constexpr (STAGE) {
    dif_rounds_smem<LOGR, LOGR, EM, TW>(sm, L, UniformField<kSwzTables<false>>{p, twf}, tid, NTK);
  } else if constexpr (YBULK) {
    // In-place re-layout: the swizzle permutes positions inside aligned 16-element blocks of a
    // column; a group's elements are >= 32 apart (one per block), and the 16 groups that share
    // a set of blocks are 16 adjacent lanes of one warp in the same iteration (lanes run along
    // the column, (R >> E1) is a multiple of 32). So a warp-level barrier between a group's
    // reads and its writes is enough.
    static_assert(((R >> E1) % 32) == 0 && (1 << (LOGR - E1)) >= 16, "re-layout hazard analysis");
    constexpr int ST1 = 1 << (LOGR - E1);
    if constexpr (TWO) mbar_wait(bar, 1);
    for (int g = tid; g < (R >> E1) * TW; g += NTK) {
      int w, q, j0, base;
      group_coords<LOGR, false, E1, TW>(g, w, q);
      dif_group<LOGR, E1>(q, j0, base);
      u64 v[1 << E1];
#pragma unroll
      for (int i = 0; i < (1 << E1); ++i) v[i] = sm[(w << LOGR) + base + i * ST1];
      __syncwarp();
      dif_regs<LOGR, LOGR, E1, kSwzTables<false>>(v, j0, twf, p);
#pragma unroll
      for (int i = 0; i < (1 << E1); ++i) sm[L(base + i * ST1, w)] = v[i];
    }
    __syncthreads();
    dif_rounds_smem<LOGR, LOGR - E1, EM, TW>(sm, L, UniformField<kSwzTables<false>>{p, twf}, tid, NTK);
  } else if constexpr (LOGR > EM) {
    constexpr int ST1 = 1 << (LOGR - E1);
    for (int g = tid; g < (R >> E1) * TW; g += NTK) {
      int w, q, j0, base;
      group_coords<LOGR, false, E1, TW>(g, w, q);
      dif_group<LOGR, E1>(q, j0, base);
      u64 v[1 << E1];
#pragma unroll
      for (int i = 0; i < (1 << E1); ++i) v[i] = src[G.at(base + i * ST1, w)];
      dif_regs<LOGR, LOGR, E1, kSwzTables<false>>(v, j0, twf, p);
#pragma unroll
      for (int i = 0; i < (1 << E1); ++i) sm[L(base + i * ST1, w)] = v[i];
    }
    __syncthreads();
    dif_rounds_smem<LOGR, LOGR - E1, EM, TW>(sm, L, UniformField<kSwzTables<false>>{p, twf}, tid, NTK);
  }
  for (int g = tid; g < (R >> EM) * TW; g += NTK) {
    int w, q, j0, base;
    group_coords<LOGR, false, EM, TW>(g, w, q);
    dit_group<0, EM>(q, j0, base);
    u64 v[1 << EM];
#pragma unroll
    for (int i = 0; i < (1 << EM); ++i) v[i] = LOGR > EM ? sm[L(base + i, w)] : src[G.at(base + i, w)];
    // the last DIF stage stays lazy ([0, 2p)): REDC takes a b < p 2^64 with the other factor
    // canonical (the other operand's spectrum, or the reduced copy when squaring)
    dif_regs<LOGR, EM, EM, kSwzTables<false>, true>(v, 0, twf, p);
#pragma unroll
    for (int i = 0; i < (1 << EM); ++i) {
      const u64 o = TWO ? smx[L(base + i, w)] : (oth ? oth[G.at(base + i, w)] : reduce_2p(v[i], p));
      v[i] = mont_mul(v[i], o, p, pp);
    }
    dit_regs<LOGR, 0, EM, kSwzTables<false>, LZO && LOGR == EM>(v, 0, twi, p);
#pragma unroll
    for (int i = 0; i < (1 << EM); ++i) {
      if constexpr (LOGR == EM) {
        if (a.has_final_scale) v[i] = shoup_mul(v[i], sc, p);
        dst[G.at(base + i, w)] = v[i];
      } else {
        sm[L(base + i, w)] = v[i];
      }
    }
  }
  if constexpr (LOGR > EM) {
    __syncthreads();
    dit_rounds_smem<LOGR, EM, AL, TW>(sm, L, UniformField<kSwzTables<false>>{p, twi}, tid, NTK);
    constexpr int STL = 1 << AL;
    for (int g = tid; g < (R >> EL) * TW; g += NTK) {
      int w, q, j0, base;
      group_coords<LOGR, false, EL, TW>(g, w, q);
      dit_group<AL, EL>(q, j0, base);
      u64 v[1 << EL];
#pragma unroll
      for (int i = 0; i < (1 << EL); ++i) v[i] = sm[L(base + i * STL, w)];
      dit_regs<LOGR, AL, EL, kSwzTables<false>, LZO>(v, j0, twi, p);
      if constexpr (OBULK) __syncwarp();  // every lane has read its group: un-swizzle in place
#pragma unroll
      for (int i = 0; i < (1 << EL); ++i) {
        if (a.has_final_scale) v[i] = shoup_mul(v[i], sc, p);
        if constexpr (OBULK)
          sm[(w << LOGR) + base + i * STL] = v[i];
        else
          dst[G.at(base + i * STL, w)] = v[i];
      }
    }
    if constexpr (OBULK) {
      // the tile is one contiguous run of R * TW words in the output too: one bulk store
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + G.at(0, 0)),
                     "r"(unsigned(__cvta_generic_to_shared(sm))), "r"(unsigned(R * TW * sizeof(u64)))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    }
  }
}

// Radix-3 pass (reference three_row_forward_columns conv.cpp:109-125, with the
// length-3 DFT written with one multiplication: omega_3^2 = -1 - omega_3).
__global__ void k_radix3_fwd(Radix3Args a) {
  pdl_wait();
  const int pr = blockIdx.y;  // select, not index: keeps the parameter block out of local memory
  const u64 p = pr ? a.p[1] : a.p[0];
  const unsigned long long S = a.S;
  const u64* src = pr ? a.src[1] : a.src[0];
  u64* dst = pr ? a.dst[1] : a.dst[0];
  const TwPair* __restrict__ lo = pr ? a.lo[1] : a.lo[0];
  const TwPair* __restrict__ hi = pr ? a.hi[1] : a.hi[0];
  const TwPair lam = pr ? a.lam[1] : a.lam[0];
  const unsigned long long L = 1ull << a.lbits, H = a.hrow;
  for (unsigned long long s = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; s < S;
       s += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long sg = ((s >> a.cb) << a.sb) + a.off + (s & ((1ull << a.cb) - 1));  // global column
    const unsigned long long sl = sg & (L - 1), sh = sg >> a.lbits;
    const u64 x0 = src[s], x1 = src[S + s], x2 = src[2 * S + s];
    const u64 t = shoup_mul(mod_sub(x1, x2, p), lam, p);
    const u64 y0 = mod_add(mod_add(x0, x1, p), x2, p);
    const u64 y1 = mod_add(mod_sub(x0, x2, p), t, p);
    const u64 y2 = mod_sub(mod_sub(x0, x1, p), t, p);
    dst[s] = y0;
    if (a.notw) {  // the twiddles are pass 1's (merged)
      dst[S + s] = y1;
      dst[2 * S + s] = y2;
    } else {
      dst[S + s] = shoup_mul(shoup_mul(y1, lo[L + sl], p), hi[H + sh], p);
      dst[2 * S + s] = shoup_mul(shoup_mul(y2, lo[2 * L + sl], p), hi[2 * H + sh], p);
    }
  }
}

// Inverse radix-3 pass (conv.cpp:129-147): twiddle (with the convolution scale
// folded into the hi table when this is the first inverse pass) then length-3 IDFT*.
__global__ void k_radix3_inv(Radix3Args a) {
  pdl_wait();
  const int pr = blockIdx.y;  // select, not index: keeps the parameter block out of local memory
  const u64 p = pr ? a.p[1] : a.p[0];
  const unsigned long long S = a.S;
  const u64* src = pr ? a.src[1] : a.src[0];
  u64* dst = pr ? a.dst[1] : a.dst[0];
  const TwPair* __restrict__ lo = pr ? a.lo[1] : a.lo[0];
  const TwPair* __restrict__ hi = pr ? a.hi[1] : a.hi[0];
  const TwPair lam = pr ? a.lam[1] : a.lam[0];
  const unsigned long long L = 1ull << a.lbits, H = a.hrow;
  for (unsigned long long s = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; s < S;
       s += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long sg = ((s >> a.cb) << a.sb) + a.off + (s & ((1ull << a.cb) - 1));  // global column
    const unsigned long long sl = sg & (L - 1), sh = sg >> a.lbits;
    u64 y0, y1, y2;
    if (const TwPair* __restrict__ pv = pr ? a.pinv[1] : a.pinv[0]) {  // merged: omega_{3 R1}^{-f r} scale
      const unsigned long long r = sg >> a.pre_shift;
      y0 = shoup_mul(src[s], pv[r], p);
      y1 = shoup_mul(src[S + s], pv[a.pre_rows + r], p);
      y2 = shoup_mul(src[2 * S + s], pv[2 * a.pre_rows + r], p);
    } else {
      y0 = shoup_mul(src[s], hi[sh], p);  // lo[0][.] = 1
      y1 = shoup_mul(shoup_mul(src[S + s], lo[L + sl], p), hi[H + sh], p);
      y2 = shoup_mul(shoup_mul(src[2 * S + s], lo[2 * L + sl], p), hi[2 * H + sh], p);
    }
    const u64 t = shoup_mul(mod_sub(y1, y2, p), lam, p);
    dst[s] = mod_add(mod_add(y0, y1, p), y2, p);
    dst[S + s] = mod_add(mod_sub(y0, y2, p), t, p);
    dst[2 * S + s] = mod_sub(mod_sub(y0, y1, p), t, p);
  }
}

// ---- table generation (plan time) ----

__device__ u64 mont_pow_dev(u64 base_mont, u64 e, u64 one_mont, u64 p, u64 pp) {
  u64 r = one_mont;
  while (e) {
    if (e & 1) r = mont_mul(r, base_mont, p, pp);
    base_mont = mont_mul(base_mont, base_mont, p, pp);
    e >>= 1;
  }
  return r;
}

struct GenArgs {
  TwPair* out;
  u64 root_mont, one_mont, scale_mont;  // Montgomery forms
  u64 p, pp, d_norm, recip;
  unsigned shift;
  int R, f_off;
  unsigned long long S, M, f_mul, f_add;
};

__global__ void k_gen_table(GenArgs g) {
  const unsigned long long total = (unsigned long long)g.R * g.S;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long f = i / g.S + g.f_off, s = i % g.S;
    const unsigned long long fe = (g.f_mul * f + g.f_add) % g.M;
    const unsigned long long e = (unsigned long long)(((unsigned __int128)fe * s) % g.M);  // exponent of the root
    u64 w = mont_pow_dev(g.root_mont, e, g.one_mont, g.p, g.pp);
    w = mont_mul(w, g.scale_mont, g.p, g.pp);  // Montgomery form of omega^e * scale
    w = mont_mul(w, 1, g.p, g.pp);             // plain
    u64 q, r;
    udiv_2by1(w << g.shift, 0, g.d_norm, g.recip, q, r);  // w' = floor(w 2^64 / p)
    g.out[i] = TwPair{w, q};
  }
}

// ---- elementwise kernels ----

// pack (reference decimal.cpp:102-118): limb t holds digits
// [nd - (t+1) lambda, nd - t lambda) of the most-significant-first string.
// A CTA packs kPackLimbs consecutive limbs: their digit span (<= 17 kPackLimbs bytes,
// contiguous in the string) is staged in shared memory with 16-byte loads, then
// each thread parses its lambda digits 8 at a time (SWAR).
constexpr int kPackLimbs = 256;
constexpr int kPackBuf = kPackLimbs * 17 + 96;

// Staging half of the pack of the kPackLimbs consecutive limbs starting at t0 (block-uniform):
// their digit span is copied into buf (kPackBuf bytes of shared memory, 16-byte aligned) with
// 16-byte vector loads. Returns the string position of buf[32] (the span's aligned start),
// or a value > nd when the block is past the last limb (all zero). The caller syncs, then
// pack_parse reads each thread's limb.
template <bool ASYNC = false>
__device__ __forceinline__ long long pack_stage(const char* __restrict__ d, unsigned long long nd, unsigned be,
                                                unsigned long long t0, char* smem) {
  char* buf = smem + 32;  // parse_digits may read up to 24 bytes before a limb and 8 past it
  // digit span of limbs [t0, min(t0 + kPackLimbs, nl)): [lo, hi)
  const long long hi = (long long)nd - (long long)(t0 * be);
  if (hi <= 0) return (long long)nd + 1;  // block-uniform: zero padding to the transform length
  const long long lo = hi - (long long)kPackLimbs * be > 0 ? hi - (long long)kPackLimbs * be : 0;
  // 16-byte vectors aligned in the ADDRESS space; string position x lands at buf[x - lo + o]
  const int o = int((reinterpret_cast<unsigned long long>(d) + (unsigned long long)lo) & 15);
  const long long g0 = lo - o;  // string position of buf[0] (may be < 0)
  const int nvec = int((o + (hi - lo) + 15) / 16);
  for (int v = threadIdx.x; v < nvec; v += kPackLimbs) {
    const long long g = g0 + 16LL * v;
    if (g >= 0 && g + 16 <= (long long)nd) {
      if constexpr (ASYNC) {  // cp.async: the copy proceeds while the block computes
        const unsigned sa = unsigned(__cvta_generic_to_shared(buf + 16 * v));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(d + g) : "memory");
      } else {
        reinterpret_cast<uint4*>(buf)[v] = *reinterpret_cast<const uint4*>(d + g);
      }
    } else {  // head or tail: byte loads inside the string only
      for (int b = 0; b < 16; ++b) buf[v * 16 + b] = (g + b >= 0 && g + b < (long long)nd) ? d[g + b] : '0';
    }
  }
  return g0;
}

// Limb t0 + threadIdx.x (0 past the string's last limb) from a span staged by pack_stage.
// Raises kErrLeadingZero in *err and ORs the non-digit flag of its bytes into bad.
template <int NG, bool LEAD = true>
__device__ __forceinline__ u64 pack_parse(const char* __restrict__ d, unsigned long long nd, unsigned be,
                                          unsigned long long t0, const char* smem, long long g0, unsigned* err,
                                          unsigned& bad) {
  if (g0 > (long long)nd) return 0;
  const unsigned long long nl = (nd + be - 1) / be;
  const unsigned long long t = t0 + threadIdx.x;
  if (t >= nl) return 0;
  const long long end = (long long)nd - (long long)(t * be);
  const long long begin = end > (long long)be ? end - (long long)be : 0;
  const u64 limb = parse_digits<NG>(smem + 32, int(begin - g0), int(end - begin), bad);
  if (LEAD && begin == 0 && nd > 1 && d[0] == '0') atomicOr(err, kErrLeadingZero);
  return limb;
}

// LEAD: d is the whole operand (its leading zero is an error); false for a rank's compacted
// digit slices (multi.cu), whose first digit may be 0.
// blockIdx.y == 1: the second operand of a two-operand launch (d2, nd2 -> limbs2, unsharded).
template <bool ROWMAP, int NG, bool LEAD = true>
__global__ void __launch_bounds__(kPackLimbs) k_pack(const char* __restrict__ d, unsigned long long nd, unsigned be,
                                                     u64* __restrict__ limbs, unsigned long long total, unsigned* err,
                                                     int row_bits, unsigned long long row_stride,
                                                     unsigned long long off, const char* __restrict__ d2,
                                                     unsigned long long nd2, u64* __restrict__ limbs2) {
  pdl_wait();
  if (blockIdx.y) {
    d = d2;
    nd = nd2;
    limbs = limbs2;
  }
  __shared__ __align__(16) char smem[kPackBuf];
  const unsigned long long rmask = row_bits >= 63 ? ~0ull : (1ull << row_bits) - 1;
  unsigned bad = 0;
  for (unsigned long long i0 = (unsigned long long)blockIdx.x * kPackLimbs; i0 < total;
       i0 += (unsigned long long)gridDim.x * kPackLimbs) {
    // local limbs i0 .. i0 + 255 are global limbs t0 .. t0 + 255 (rows hold >= 256 limbs);
    // unsharded (ROWMAP false): the identity
    const unsigned long long t0 = ROWMAP ? (i0 >> row_bits) * row_stride + off + (i0 & rmask) : i0;
    const long long g0 = pack_stage(d, nd, be, t0, smem);
    __syncthreads();
    const u64 limb = pack_parse<NG, LEAD>(d, nd, be, t0, smem, g0, err, bad);
    __syncthreads();
    const unsigned long long li = i0 + threadIdx.x;
    if (li < total) limbs[li] = limb;
  }
  if (bad) atomicOr(err, kErrBadDigit);
}

// Pack fused with the forward radix-3 pass (reference three_row_forward_columns,
// conv.cpp:109-125) for N = 3 S: column s takes limbs s, S + s, 2 S + s straight from the
// digit string (three staged spans), runs the length-3 DFT and the twiddles omega_N^{f s}
// (factorised lo * hi as in k_radix3_fwd) for both primes, and writes pass 0's output.
// The packed limbs never touch HBM (the separate pack wrote 8 B and the radix-3 pass read
// them back per limb).
// The block's three spans are staged with 16-byte loads; in span-local coordinates column c's
// limb always ends at byte (kR3Cols - c) lambda, so the parse needs no 64-bit index
// arithmetic (only the block holding the string's head clips). Rows past the last limb are
// skipped block-uniformly (config 4's y fills one of the three rows, x two).
// (Rejected: double-buffered cp.async staging of the spans and twiddles, 4.48 / 5.74 ms for the
// two config-4 launches vs 4.32 single-buffered.)
// CB = kR3Cols columns per block, two per thread (c = t, t + 256): the per-iteration work
// (span bounds, staging set-up, barriers) is shared by two columns and the two columns'
// arithmetic interleaves.
constexpr int kR3Cols = 2 * kPackLimbs;
constexpr int kR3Buf = kR3Cols * 17 + 96;

// Limb of column c of a block whose row span ends at string position hi (exclusive).
template <int NG>
__device__ __forceinline__ u64 r3_row_limb(const char* __restrict__ d, unsigned long long nd, long long hi,
                                           unsigned be, const char* buf, int c, unsigned* err, unsigned& bad) {
  const long long base = hi - (long long)kR3Cols * be;  // string position of span byte 0
  const int o = int((reinterpret_cast<unsigned long long>(d) + (unsigned long long)base) & 15);
  const int e = (kR3Cols - c) * int(be);  // limb end, span-local
  int b = e - int(be);
  if (base < 0) {  // the string's head: limbs may be short or absent
    const int b0 = int(-base);
    if (e <= b0) return 0;
    if (b < b0) b = b0;
    const u64 v = parse_digits<NG>(buf + 32, o + b, e - b, bad);
    if (b == b0 && nd > 1 && d[0] == '0') atomicOr(err, kErrLeadingZero);  // the most significant limb
    return v;
  }
  if (base + b == 0 && nd > 1 && d[0] == '0') atomicOr(err, kErrLeadingZero);
  return parse_digits<NG>(buf + 32, o + b, int(be), bad);
}
__device__ __forceinline__ void r3_row_stage(const char* __restrict__ d, unsigned long long nd, long long hi,
                                             unsigned be, char* buf) {
  const long long base = hi - (long long)kR3Cols * be;
  const int o = int((reinterpret_cast<unsigned long long>(d) + (unsigned long long)base) & 15);
  const char* g0 = d + (base - o);  // 16-byte aligned in the address space
  const int nvec = (o + kR3Cols * int(be) + 15) >> 4;
  // vectors [vlo, vhi) lie wholly inside the string; the few others go byte by byte
  const long long first = base - o;
  const int vlo = first >= 0 ? 0 : int((-first + 15) >> 4);
  const long long room = (long long)nd - first;
  const int vhi = room >= 16LL * nvec ? nvec : (room < 16 ? 0 : int(room >> 4));
  uint4* dst = reinterpret_cast<uint4*>(buf + 32);
  for (int v = threadIdx.x; v < nvec; v += kPackLimbs) {
    if (v >= vlo && v < vhi) {
      dst[v] = reinterpret_cast<const uint4*>(g0)[v];
    } else {
      const long long g = first + 16LL * v;
      char* db = buf + 32 + 16 * v;
      for (int k = 0; k < 16; ++k) db[k] = (g + k >= 0 && g + k < (long long)nd) ? d[g + k] : '0';
    }
  }
}

template <int NG>
__global__ void __launch_bounds__(kPackLimbs) k_pack_radix3(const char* __restrict__ d, unsigned long long nd,
                                                           unsigned be, Radix3Args a, unsigned* err) {
  pdl_wait();
  __shared__ __align__(16) char smem[3][kR3Buf];
  const unsigned long long S = a.S, L = 1ull << a.lbits, H = a.hrow;
  const unsigned long long nl = (nd + be - 1) / be;  // limbs of the string
  const long long SB = (long long)(S * be);           // digits per row of limbs
  unsigned bad = 0;
  for (unsigned long long s0 = (unsigned long long)blockIdx.x * kR3Cols; s0 < S;
       s0 += (unsigned long long)gridDim.x * kR3Cols) {
    bool live[3];
    long long hi[3];
    hi[0] = (long long)nd - (long long)(s0 * be);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      if (j) hi[j] = hi[j - 1] - SB;
      live[j] = j * S + s0 < nl;  // the block's first limb of row j
      if (live[j]) r3_row_stage(d, nd, hi[j], be, smem[j]);
    }
    __syncthreads();
    u64 x[2][3];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = threadIdx.x + h * kPackLimbs;
      const unsigned long long s = s0 + c;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        x[h][j] = 0;
        // limbs past the string's end inside a live block: its last block may be partial
        if (live[j] && j * S + s < nl) x[h][j] = r3_row_limb<NG>(d, nd, hi[j], be, smem[j], c, err, bad);
      }
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const unsigned long long s = s0 + threadIdx.x + h * kPackLimbs;
      if (s >= S) continue;
      const unsigned long long sl = s & (L - 1), sh = s >> a.lbits;
#pragma unroll
      for (int pr = 0; pr < 2; ++pr) {
        const u64 p = a.p[pr];
        const TwPair lam = a.lam[pr];
        const TwPair* __restrict__ lo = a.lo[pr];
        const TwPair* __restrict__ hiw = a.hi[pr];
        u64* dst = a.dst[pr] + s;
        // limbs are < 10^17 < p: canonical residues of both primes
        const u64 t = shoup_mul(mod_sub(x[h][1], x[h][2], p), lam, p);
        const u64 y0 = mod_add(mod_add(x[h][0], x[h][1], p), x[h][2], p);
        const u64 y1 = mod_add(mod_sub(x[h][0], x[h][2], p), t, p);
        const u64 y2 = mod_sub(mod_sub(x[h][0], x[h][1], p), t, p);
        dst[0] = y0;
        if (a.notw) {  // the twiddles are pass 1's (merged)
          dst[S] = y1;
          dst[2 * S] = y2;
        } else {
          dst[S] = shoup_mul(shoup_mul(y1, lo[L + sl], p), hiw[H + sh], p);
          dst[2 * S] = shoup_mul(shoup_mul(y2, lo[2 * L + sl], p), hiw[2 * H + sh], p);
        }
      }
    }
  }
  if (bad) atomicOr(err, kErrBadDigit);
}

// Column-sharded pack for rows narrower than one 256-limb block: one limb per thread.
__global__ void k_pack_rows(const char* __restrict__ d, unsigned long long nd, unsigned be, u64* __restrict__ limbs,
                            unsigned long long total, unsigned* err, int row_bits, unsigned long long row_stride,
                            unsigned long long off) {
  const unsigned long long nl = (nd + be - 1) / be;
  const unsigned long long rmask = (1ull << row_bits) - 1;
  unsigned bad = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long t = (i >> row_bits) * row_stride + off + (i & rmask);
    u64 limb = 0;
    if (t < nl) {
      const long long end = (long long)nd - (long long)(t * be);
      const long long begin = end > (long long)be ? end - (long long)be : 0;
      for (long long j = begin; j < end; ++j) {
        const unsigned c = (unsigned char)d[j] - '0';
        bad |= c > 9;
        limb = limb * 10 + c;
      }
      if (begin == 0 && nd > 1 && d[0] == '0') atomicOr(err, kErrLeadingZero);
    }
    limbs[i] = limb;
  }
  if (bad) atomicOr(err, kErrBadDigit);
}

// [peer][row][c] <-> [row][peer][c]: the all-to-all block layout vs contiguous segments.
// Segment <-> block reorder around the all-to-alls of the sharded product: the data is
// peers x rows blocks of `width` contiguous words (width = the column-block width Bc, a
// power of two >= 16), permuted as whole blocks. Work is split into tiles of up to 1024
// 16-byte vectors inside a block: one division per tile, 16-byte loads and stores (an
// element-wise version spent three 64-bit divisions per word).
__global__ void k_block_reorder(const u64* __restrict__ src, u64* __restrict__ dst, unsigned long long peers,
                                unsigned long long rows, unsigned long long width, int to_segments) {
  const unsigned long long nvec = width / 2, tile = nvec < 1024 ? nvec : 1024, tpb = nvec / tile;
  const unsigned long long ntiles = peers * rows * tpb;
  for (unsigned long long u = blockIdx.x; u < ntiles; u += gridDim.x) {
    const unsigned long long b = u / tpb, off = (u - b * tpb) * tile;
    unsigned long long sb;
    if (to_segments) {  // destination [row][peer], source [peer][row]
      sb = (b % peers) * rows + b / peers;
    } else {  // destination [peer][row], source [row][peer]
      sb = (b % rows) * peers + b / rows;
    }
    const uint4* s4 = reinterpret_cast<const uint4*>(src + sb * width) + off;
    uint4* d4 = reinterpret_cast<uint4*>(dst + b * width) + off;
    for (unsigned long long i = threadIdx.x; i < tile; i += blockDim.x) d4[i] = s4[i];
  }
}

__global__ void k_pointwise(u64* a, const u64* b, unsigned long long n, u64 p, u64 pp) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    a[i] = mont_mul(a[i], b[i], p, pp);
}

__global__ void k_mont_scale(u64* a, unsigned long long n, u64 f, u64 p, u64 pp) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    a[i] = mont_mul(a[i], f, p, pp);
}

__global__ void k_gather(const u64* src, u64* dst, const unsigned long long* map, unsigned long long n) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    dst[i] = src[map[i]];
}

__global__ void k_validate(const char* __restrict__ d, unsigned long long n, unsigned* err) {
  unsigned bad = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    bad |= unsigned((unsigned char)d[i] - '0') > 9u;
  if (bad) atomicOr(err, kErrBadDigit);
  if (blockIdx.x == 0 && threadIdx.x == 0 && n > 1 && d[0] == '0') atomicOr(err, kErrLeadingZero);
}

int grid_for(unsigned long long n, int threads) {
  unsigned long long b = (n + threads - 1) / threads;
  const unsigned long long cap = 148ull * 16;
  return int(b < 1 ? 1 : (b > cap ? cap : b));
}

// One-time (per device) opt-in to the large dynamic shared-memory carve-out for kernel fn.
template <auto FN>
void set_smem(int bytes) {
  static unsigned long long done = 0;  // one bit per device, one flag set per kernel instantiation
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !(done >> dev & 1)) {
    cudaFuncSetAttribute((const void*)FN, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done |= 1ull << dev;
  }
}

// blockIdx.x = tile * np + prime: both primes of a tile run back to back, so a shared
// source (the packed limbs of pass 0) is read from HBM once and from L2 the second time.
template <auto FN, int TW, int NTK>
void launch_pass_kernel(const PassArgs& a, unsigned long long ncols, int np, int smem, cudaStream_t st) {
  set_smem<FN>(smem);
  PassArgs b = a;
  b.np = np;
  launch_pdl(FN, dim3(unsigned((ncols + TW - 1) / TW * np), a.nops > 1 ? 2 : 1), dim3(NTK), size_t(smem), st, b);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link against libcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// The {S, rows} u64 tensor over base with the row-tile box {16, min(R, 256)}.
void encode_row_map(unsigned char (&out)[128], const u64* base, unsigned long long S, unsigned long long rows,
                    int logR, int tw);

// The twiddle table of a row pass as a {2 S' u64, rows} tensor with the box {32, min(R, 256)}
// (16 pairs of one row): Sp = pairs per table row, rows = R times the number of per-group tables.
void encode_table_map(unsigned char (&out)[128], const TwPair* table, unsigned long long Sp, unsigned long long rows,
                      int logR) {
  encode_row_map(out, reinterpret_cast<const u64*>(table), 2 * Sp, rows, logR, 2 * kTileW);
}

void encode_row_map(unsigned char (&out)[128], const u64* base, unsigned long long S, unsigned long long rows,
                    int logR, int tw) {
  static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap size");
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) throw CudaError("cuTensorMapEncodeTiled: driver entry point not found");
  CUtensorMap m;
  const cuuint64_t dims[2] = {S, rows};
  const cuuint64_t strides[1] = {S * sizeof(u64)};
  const cuuint32_t box[2] = {cuuint32_t(tw), cuuint32_t(std::min(1 << logR, kBoxRows))};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult rc = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<u64*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(rc)) + ")");
  std::memcpy(out, &m, sizeof m);
}

// Forward / inverse passes: the same launch plus the tiles' tensor maps (full-width row tiles
// of multi-round radices are staged by TMA; other shapes ignore the maps).
template <auto FN, int TW, int NTK>
void launch_pass_kernel_maps(const PassArgs& a, unsigned long long ncols, int np, int smem, bool tma, int logR,
                             cudaStream_t st) {
  set_smem<FN>(smem);
  PassArgs b = a;
  b.np = np;
  TileMaps maps;
  if (tma) {
    const unsigned long long rows = a.G << logR;
    for (int pr = 0; pr < np; ++pr) {
      encode_row_map(maps.m[pr], a.src[pr], a.S, rows, logR, TW);
      if (a.nops > 1) encode_row_map(maps.m[2 + pr], a.src_b[pr], a.S, rows, logR, TW);
      if (DMG_BULK_STORE) {
        encode_row_map(maps.m[4 + pr], a.dst[pr], a.S, rows, logR, TW);
        if (a.nops > 1) encode_row_map(maps.m[6 + pr], a.dst_b[pr], a.S, rows, logR, TW);
      }
      if (DMG_TMA_TWPF && TW == kTileW && a.pass_tw[pr] && !a.tw_lbits)
        encode_table_map(maps.m[8 + pr], a.pass_tw[pr], 1ull << a.tw_logS,
                         (a.tw_gstride ? a.G : 1ull) << logR, logR);
    }
  }
  launch_pdl(FN, dim3(unsigned((ncols + TW - 1) / TW * np), a.nops > 1 ? 2 : 1), dim3(NTK), size_t(smem), st, b, maps);
}

// Tile width: 16 columns (128 B row segments) normally; 4 when a pass would otherwise
// launch fewer than two CTAs per SM (small transforms, e.g. config 1's N = 2^17 has
// 16 tiles of 512 x 16 per prime), trading segment length for parallelism.
constexpr int kNarrowW = 4;
inline bool narrow_tiles(int logR, unsigned long long ncols, int np) {
  return logR >= 5 && (ncols / W) * (unsigned long long)np < 2ull * 148;
}

template <int LOGR, int TW>
void pass_fwd_w(const PassArgs& a, unsigned long long ncols, int np, cudaStream_t st) {
  constexpr int NTK = pass_threads(LOGR, TW);
  const int sm = (1 << LOGR) * TW * 8 + (1 << LOGR) / 2 * 16 + 16;  // tile, table, mbarrier
  constexpr bool TMA = kBulkRows<true, TW> && kStageFwd<true, TW> && LOGR > Sched<LOGR>::e_dif(LOGR);
  if (a.S > 1 && a.tw_lbits)
    launch_pass_kernel_maps<k_pass_fwd<LOGR, true, TW, true>, TW, NTK>(a, ncols, np, sm, TMA, LOGR, st);
  else if (a.S > 1)
    launch_pass_kernel_maps<k_pass_fwd<LOGR, true, TW>, TW, NTK>(a, ncols, np, sm, TMA, LOGR, st);
  else
    launch_pass_kernel_maps<k_pass_fwd<LOGR, false, TW>, TW, NTK>(a, ncols, np, sm, false, LOGR, st);
}
template <int LOGR, int TW>
void pass_inv_w(const PassArgs& a, unsigned long long ncols, int np, cudaStream_t st) {
  constexpr int NTK = pass_threads(LOGR, TW);
  const int sm = (1 << LOGR) * TW * 8 + (1 << LOGR) / 2 * 16 + 16;  // tile, table, mbarrier
  constexpr bool TMA = kBulkRows<true, TW> && kStageInv<true> && LOGR > Sched<LOGR>::first_e;
  if (a.S > 1 && a.tw_lbits && a.lazy_out)
    launch_pass_kernel_maps<k_pass_inv<LOGR, true, TW, true, true>, TW, NTK>(a, ncols, np, sm, TMA, LOGR, st);
  else if (a.S > 1 && a.tw_lbits)
    launch_pass_kernel_maps<k_pass_inv<LOGR, true, TW, true>, TW, NTK>(a, ncols, np, sm, TMA, LOGR, st);
  else if (a.S > 1 && a.lazy_out)
    launch_pass_kernel_maps<k_pass_inv<LOGR, true, TW, false, true>, TW, NTK>(a, ncols, np, sm, TMA, LOGR, st);
  else if (a.S > 1)
    launch_pass_kernel_maps<k_pass_inv<LOGR, true, TW>, TW, NTK>(a, ncols, np, sm, TMA, LOGR, st);
  else
    launch_pass_kernel_maps<k_pass_inv<LOGR, false, TW>, TW, NTK>(a, ncols, np, sm, false, LOGR, st);
}
template <int LOGR, int TW>
void pass_fused_w(const PassArgs& a, unsigned long long ncols, int np, cudaStream_t st) {
  constexpr int NTK = pass_threads(LOGR, TW);
  const int sm = (1 << LOGR) * TW * 8 * (a.two ? 2 : 1) + (1 << LOGR) * 16 + 16;  // tiles, tables, mbarrier
  if (a.two) {
    if (a.lazy_out)
      launch_pass_kernel<k_pass_fused<LOGR, TW, true, true>, TW, NTK>(a, ncols, np, sm, st);
    else
      launch_pass_kernel<k_pass_fused<LOGR, TW, false, true>, TW, NTK>(a, ncols, np, sm, st);
  } else if (a.lazy_out)
    launch_pass_kernel<k_pass_fused<LOGR, TW, true>, TW, NTK>(a, ncols, np, sm, st);
  else
    launch_pass_kernel<k_pass_fused<LOGR, TW>, TW, NTK>(a, ncols, np, sm, st);
}

template <int LOGR>
void pass_fwd_t(const PassArgs& a, unsigned long long ncols, int np, cudaStream_t st) {
  if constexpr (LOGR >= 5) {
    if (narrow_tiles(LOGR, ncols, np)) return pass_fwd_w<LOGR, kNarrowW>(a, ncols, np, st);
  }
  pass_fwd_w<LOGR, W>(a, ncols, np, st);
}
template <int LOGR>
void pass_inv_t(const PassArgs& a, unsigned long long ncols, int np, cudaStream_t st) {
  if constexpr (LOGR >= 5) {
    if (narrow_tiles(LOGR, ncols, np)) return pass_inv_w<LOGR, kNarrowW>(a, ncols, np, st);
  }
  pass_inv_w<LOGR, W>(a, ncols, np, st);
}
template <int LOGR>
void pass_fused_t(const PassArgs& a, unsigned long long ncols, int np, cudaStream_t st) {
  if constexpr (LOGR >= 5) {
    if (narrow_tiles(LOGR, ncols, np)) return pass_fused_w<LOGR, kNarrowW>(a, ncols, np, st);
  }
  pass_fused_w<LOGR, W>(a, ncols, np, st);
}

}  // namespace

#define DMG_DISPATCH_LOGR(fn, logR, ...)  \
  switch (logR) {                          \
    case 1: fn<1>(__VA_ARGS__); break;     \
    case 2: fn<2>(__VA_ARGS__); break;     \
    case 3: fn<3>(__VA_ARGS__); break;     \
    case 4: fn<4>(__VA_ARGS__); break;     \
    case 5: fn<5>(__VA_ARGS__); break;     \
    case 6: fn<6>(__VA_ARGS__); break;     \
    case 7: fn<7>(__VA_ARGS__); break;     \
    case 8: fn<8>(__VA_ARGS__); break;     \
    case 9: fn<9>(__VA_ARGS__); break;     \
    default: break;                        \
  }

void launch_pass_fwd(int logR, const PassArgs& a, unsigned long long ncols, int np, cudaStream_t st) {
  DMG_DISPATCH_LOGR(pass_fwd_t, logR, a, ncols, np, st);
}
void launch_pass_inv(int logR, const PassArgs& a, unsigned long long ncols, int np, cudaStream_t st) {
  DMG_DISPATCH_LOGR(pass_inv_t, logR, a, ncols, np, st);
}
void launch_pass_fused(int logR, const PassArgs& a, unsigned long long ncols, int np, cudaStream_t st) {
  DMG_DISPATCH_LOGR(pass_fused_t, logR, a, ncols, np, st);
}

void launch_radix3(bool inverse, const Radix3Args& a, int np, cudaStream_t st) {
  const int g = grid_for(a.S, 256);
  if (inverse)
    launch_pdl(k_radix3_inv, dim3(g, np), dim3(256), 0, st, a);
  else
    launch_pdl(k_radix3_fwd, dim3(g, np), dim3(256), 0, st, a);
}

void launch_gen_pass_table(TwPair* out, u64 root_mont, u64 scale_mont, int R, int /*logR*/, unsigned long long S,
                           u64 p, u64 recip, cudaStream_t st, unsigned long long order, int f_off,
                           unsigned long long f_mul, unsigned long long f_add) {
  GenArgs g;
  g.f_off = f_off;
  g.f_mul = f_mul;
  g.f_add = f_add;
  g.out = out;
  g.root_mont = root_mont;
  g.scale_mont = scale_mont;
  g.p = p;
  u64 inv = p;
  for (int i = 0; i < 6; ++i) inv *= 2 - p * inv;
  g.pp = 0 - inv;
  g.one_mont = u64(((unsigned __int128)1 << 64) % p);
  g.shift = __builtin_clzll(p);
  g.d_norm = p << g.shift;
  g.recip = recip;
  g.R = R;
  g.S = S;
  g.M = order ? order : (unsigned long long)(R + f_off) * S * f_mul;  // order of the root (exponents mod M)
  k_gen_table<<<grid_for((unsigned long long)R * S, 256), 256, 0, st>>>(g);
}

void launch_pack(const char* digits, unsigned long long nd, unsigned be, u64* limbs, unsigned long long total,
                 unsigned* err, cudaStream_t st, int row_bits, unsigned long long row_stride,
                 unsigned long long off, bool lead_check) {
  const char* nd2 = nullptr;
  if (row_bits < 8)
    k_pack_rows<<<grid_for(total, 256), 256, 0, st>>>(digits, nd, be, limbs, total, err, row_bits, row_stride, off);
  else if (!lead_check)
    launch_pdl(be > 16 ? k_pack<false, 5, false> : k_pack<false, 4, false>, dim3(grid_for(total, 256)), dim3(256), 0,
               st, digits, nd, be, limbs, total, err, row_bits, row_stride, off, nd2, 0ull, (u64*)nullptr);
  else
    launch_pdl(row_bits >= 63 ? (be > 16 ? k_pack<false, 5> : k_pack<false, 4>)
                              : (be > 16 ? k_pack<true, 5> : k_pack<true, 4>),
               dim3(grid_for(total, 256)), dim3(256), 0, st, digits, nd, be, limbs, total, err, row_bits, row_stride,
               off, nd2, 0ull, (u64*)nullptr);
}
void launch_pack2(const char* dx, unsigned long long nx, u64* limbs_x, const char* dy, unsigned long long ny,
                  u64* limbs_y, unsigned be, unsigned long long total, unsigned* err, cudaStream_t st) {
  launch_pdl(be > 16 ? k_pack<false, 5> : k_pack<false, 4>, dim3(grid_for(total, 256), 2), dim3(256), 0, st, dx, nx, be,
             limbs_x, total, err, 63, 0ull, 0ull, dy, ny, limbs_y);
}
void launch_pack_radix3(const char* digits, unsigned long long nd, unsigned be, const Radix3Args& a, unsigned* err,
                        cudaStream_t st) {
  auto fn = be > 16 ? k_pack_radix3<5> : k_pack_radix3<4>;
  launch_pdl(fn, dim3(grid_for(a.S, kR3Cols)), dim3(kPackLimbs), 0, st, digits, nd, be, a, err);
}
void launch_block_reorder(const u64* src, u64* dst, unsigned long long peers, unsigned long long rows,
                          unsigned long long width, bool to_segments, cudaStream_t st) {
  const unsigned long long nvec = width / 2, tile = nvec < 1024 ? nvec : 1024;
  const unsigned long long ntiles = peers * rows * (nvec / tile);
  k_block_reorder<<<unsigned(ntiles < 148ull * 16 ? ntiles : 148ull * 16), 256, 0, st>>>(src, dst, peers, rows, width,
                                                                                          to_segments ? 1 : 0);
}
void launch_validate(const char* d, unsigned long long n, unsigned* err, cudaStream_t st) {
  k_validate<<<grid_for(n, 256), 256, 0, st>>>(d, n, err);
}
void launch_pointwise(u64* a, const u64* b, unsigned long long n, u64 p, u64 pp, cudaStream_t st) {
  k_pointwise<<<grid_for(n, 256), 256, 0, st>>>(a, b, n, p, pp);
}
void launch_mont_scale(u64* a, unsigned long long n, u64 f, u64 p, u64 pp, cudaStream_t st) {
  k_mont_scale<<<grid_for(n, 256), 256, 0, st>>>(a, n, f, p, pp);
}
void launch_gather(const u64* src, u64* dst, const unsigned long long* map, unsigned long long n, cudaStream_t st) {
  k_gather<<<grid_for(n, 256), 256, 0, st>>>(src, dst, map, n);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DECMUL_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace dmg
