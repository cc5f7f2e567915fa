// One product per CTA, end to end in shared memory: pack -> forward transforms
// (both primes, both operands) -> pointwise REDC -> inverse -> CRT -> carry
// scan -> ASCII. HBM sees only the digits in and the digits out.
//
// Replaces, for transform lengths that fit one SM (N <= 3 * 2^10 or 2^11), the
// whole reference multiply (decimal.cpp:191-216): pack :102-118, the
// three-row / direct convolution conv.cpp:149-166, :292-309, crt2 :148-152,
// recover_digits :154-189 and to_decimal :120-134.
//
// Shared layout: arrays (X mod p1, X mod p2, Y mod p1, Y mod p2) of N words, each
// a set of NR rows of C = 2^LOGC words; element (array a, logical index i) lives
// at a N + (i & ~(C-1)) + col_swizzle(i & (C-1)) (ContigColumns, conflict-free).
#include "carry.cuh"
#include "digits.cuh"
#include "kernels.cuh"
#include "ntt_tile.cuh"

namespace dmg {

namespace {

#ifdef DMG_PHASE_TIMING
// Diagnostic build only (make PHASE_TIMING=1): cycles per k_small phase summed over CTAs.
__device__ unsigned long long g_phase_cycles[12];
#define DMG_PHASE(i)                                         \
  do {                                                       \
    __syncthreads();                                         \
    if (threadIdx.x == 0) {                                  \
      const long long t_ = clock64();                        \
      atomicAdd(&g_phase_cycles[i], (unsigned long long)(t_ - t_phase)); \
      t_phase = t_;                                          \
    }                                                        \
  } while (0)
#else
#define DMG_PHASE(i) \
  do {               \
  } while (0)
#endif

#ifndef DMG_SMALL_TW_PREFETCH
#define DMG_SMALL_TW_PREFETCH 1
#endif
constexpr int NT = 256;  // 8 warps, 3 CTAs/SM at <= 85 registers; measured fastest of 192/256/320/384(x3) and 512(x2)

struct SmallField {
  static constexpr bool kSwz = true;  // tables stored at tw_slot(k) (ntt_tile.cuh)
  u64 p0, p1;
  const TwPair* t0;
  const TwPair* t1;
  int nr;  // rows per array
  __device__ __forceinline__ int q(int w) const { return (w / nr) & 1; }
  __device__ __forceinline__ u64 p(int w) const { return q(w) ? p1 : p0; }
  __device__ __forceinline__ const TwPair* tw(int w) const { return q(w) ? t1 : t0; }
};

template <int LOGC, int THREE, int SQ>
struct SmallCfg {
  static constexpr int C = 1 << LOGC;
  static constexpr int NR = THREE ? 3 : 1;
  static constexpr int N = NR * C;
  static constexpr int NOPER = SQ ? 1 : 2;
  static constexpr int W = 2 * NOPER * NR;          // columns (rows of length C) in the forward tile
  static constexpr int NARR = 2 * NOPER < 3 ? 3 : 2 * NOPER;  // arrays of N words (3 needed for digits)
  static constexpr int KL = N + 2;                  // limbs after carry
  static constexpr int KPT = (KL + NT - 1) / NT;    // limbs per thread
  static constexpr int TBL = C / 2 > 0 ? C / 2 : 1;
  // data arrays, or (after the carry) limbs + staged text (<= 17 digits per limb)
  static constexpr size_t raw_bytes = size_t(NARR) * N * 8 > size_t(KL) * 8 + size_t(N) * 17 + 64
                                          ? size_t(NARR) * N * 8
                                          : size_t(KL) * 8 + size_t(N) * 17 + 64;
  static constexpr size_t data_bytes = (raw_bytes + 15) / 16 * 16;  // twiddle tables follow, 16 B aligned
  static constexpr size_t smem = data_bytes + 4 * size_t(TBL) * 16;
};

template <int LOGC>
__device__ __forceinline__ int phys(int i) {  // logical index -> swizzled offset inside one array
  return (i & ~((1 << LOGC) - 1)) + col_swizzle(i & ((1 << LOGC) - 1));
}

// arrays: 0 = X mod p1, 1 = X mod p2, 2 = Y mod p1, 3 = Y mod p2 (each N words).
template <int LOGC, int THREE, int SQ>
__global__ void __launch_bounds__(NT, 3) k_small(SmallArgs a) {
  using Cfg = SmallCfg<LOGC, THREE, SQ>;
  constexpr int C = Cfg::C, N = Cfg::N, NR = Cfg::NR;
  extern __shared__ __align__(16) u64 sm[];
  TwPair* tf0 = reinterpret_cast<TwPair*>(reinterpret_cast<char*>(sm) + Cfg::data_bytes);
  TwPair* tf1 = tf0 + Cfg::TBL;
  TwPair* ti0 = tf1 + Cfg::TBL;
  TwPair* ti1 = ti0 + Cfg::TBL;
  __shared__ unsigned wsm[NT / 32 + 1];
  __shared__ unsigned long long meta[3];
  const int tid = threadIdx.x;
  const unsigned prod = blockIdx.x;
  const unsigned be = a.base_exp;
#ifdef DMG_PHASE_TIMING
  long long t_phase = clock64();
#endif
  const u64 p0 = a.p[0], p1 = a.p[1];

  for (int i = tid; i < C / 2; i += NT) {
    const int k = tw_slot(i);  // swizzled table (ntt_tile.cuh)
    tf0[k] = a.dft_fwd[0][i];
    tf1[k] = a.dft_fwd[1][i];
    ti0[k] = a.dft_inv[0][i];
    ti1[k] = a.dft_inv[1][i];
  }
  // ---- pack (decimal.cpp:102-118) ----
  const char* dxs = a.xs + prod * a.x_stride;
  const char* dys = a.ys + prod * a.y_stride;
  // Fast path: both digit strings land in shared memory in one burst of 16-byte
  // cp.async copies (all in flight at once) into the y arrays, which are not written
  // yet; x parses from there into its arrays, y's limbs wait in registers across one
  // barrier. Strings whose aligned spans do not fit take the direct per-limb loads.
  const unsigned long long ax0 = reinterpret_cast<unsigned long long>(dxs) & ~15ull;
  const unsigned long long ay0 = reinterpret_cast<unsigned long long>(dys) & ~15ull;
  const int nxv = int((reinterpret_cast<unsigned long long>(dxs) + a.nx + 15 - ax0) / 16);
  const int nyv = Cfg::NOPER > 1 ? int((reinterpret_cast<unsigned long long>(dys) + a.ny + 15 - ay0) / 16) : 0;
  constexpr int kRegion = (Cfg::NOPER > 1 ? 2 : 1) * N * 8;  // bytes of the y arrays (array 2 when squaring)
  bool fused3 = false;  // the radix-3 column pass already ran on the packed limbs
  if (32 + 16 * (nxv + nyv) + 48 + 16 <= kRegion) {
    char* xb = reinterpret_cast<char*>(sm + 2 * N) + 32;  // xb[k] = byte at address ax0 + k
    char* yb = xb + 16 * nxv + 48;
    constexpr int LPT = (N + NT - 1) / NT;  // limbs per thread
    // C = 2 NT (config 2: 3 x 512 at 256 threads): a thread's limbs t = tid + j NT are the
    // three limbs s, s + C, s + 2C of its columns s = tid and tid + NT, so the radix-3
    // column pass runs on them in registers (no limb store and reload).
    constexpr bool kFuse3 = THREE && C == 2 * NT && LPT == 6;
#if DMG_SMALL_TW_PREFETCH
    // the radix-3 twiddles of the thread's two columns (both primes, rows 1 and 2; the same
    // for x and y) are loaded with the digits, so their L2 latency hides behind the copies
    TwPair tw3[2][2][2];
    if constexpr (kFuse3) {
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int f = 1; f <= 2; ++f) tw3[cc][q][f - 1] = a.r3_fwd[q][f * C + tid + cc * NT];
    }
#endif
    for (int v = tid; v < nxv + nyv; v += NT) {
      const bool isx = v < nxv;
      char* dst = isx ? xb + 16 * v : yb + 16 * (v - nxv);
      const char* src = reinterpret_cast<const char*>(isx ? ax0 + 16ull * v : ay0 + 16ull * (v - nxv));
      const unsigned saddr = unsigned(__cvta_generic_to_shared(dst));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(src) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    DMG_PHASE(8);  // tables + digit loads
    unsigned bad = 0;
    auto r3_columns = [&](const u64* lim, int first_arr) {
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int sc = tid + cc * NT;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const u64 p = q ? p1 : p0;
          const TwPair* T = a.r3_fwd[q];
          u64* x = sm + (first_arr + q) * N + col_swizzle(sc);
          const u64 x0 = lim[cc], x1 = lim[cc + 2], x2 = lim[cc + 4];
          const u64 t = shoup_mul(mod_sub(x1, x2, p), a.lam[q], p);
#if DMG_SMALL_TW_PREFETCH
          const TwPair w1 = tw3[cc][q][0], w2 = tw3[cc][q][1];
          (void)T;
#else
          const TwPair w1 = T[C + sc], w2 = T[2 * C + sc];
#endif
          x[0] = mod_add(mod_add(x0, x1, p), x2, p);
          x[C] = shoup_mul(mod_add(mod_sub(x0, x2, p), t, p), w1, p);
          x[2 * C] = shoup_mul(mod_sub(mod_sub(x0, x1, p), t, p), w2, p);
        }
      }
    };
    u64 xlimb[LPT], ylimb[LPT];
    for (int o = 0; o < Cfg::NOPER; ++o) {
      const long long nd = (long long)(o ? a.ny : a.nx);
      const long long nl = (nd + be - 1) / be;
      const char* b = o ? yb : xb;
      const int sh = int(reinterpret_cast<unsigned long long>(o ? dys : dxs) - (o ? ay0 : ax0));
#pragma unroll
      for (int j = 0; j < LPT; ++j) {
        const int t = tid + j * NT;
        u64 limb = 0;
        if (t < nl) {
          const long long end = nd - (long long)t * be, begin = end > (long long)be ? end - (long long)be : 0;
          limb = parse_digits<5, false>(b, sh + int(begin), int(end - begin), bad);
        }
        if (o == 0) {
          xlimb[j] = limb;
          if (!kFuse3 && t < N) {
            const int ph = phys<LOGC>(t);
            sm[ph] = limb;
            sm[N + ph] = limb;
          }
        } else {
          ylimb[j] = limb;
        }
      }
      if (tid == 0 && nd > 1 && b[sh] == '0') atomicOr(a.err, kErrLeadingZero);
      if (o == 0) {
        if constexpr (kFuse3) r3_columns(xlimb, 0);
        DMG_PHASE(9);  // parse x
      }
    }
    if (bad) atomicOr(a.err, kErrBadDigit);
    if constexpr (Cfg::NOPER > 1) {
      __syncthreads();  // the staged text is dead: y's arrays may be written
      if constexpr (kFuse3) {
        r3_columns(ylimb, 2);
      } else {
#pragma unroll
        for (int j = 0; j < LPT; ++j) {
          const int t = tid + j * NT;
          if (t < N) {
            const int ph = phys<LOGC>(t);
            sm[2 * N + ph] = ylimb[j];
            sm[3 * N + ph] = ylimb[j];
          }
        }
      }
    }
    fused3 = kFuse3;
  } else {
    for (int o = 0; o < Cfg::NOPER; ++o) {
      const char* d = o ? dys : dxs;
      const unsigned long long nd = o ? a.ny : a.nx;
      const long long nl = (long long)((nd + be - 1) / be);
      unsigned bad = 0;
      for (int t = tid; t < N; t += NT) {
        u64 limb = 0;
        if (t < nl) {
          const long long end = (long long)nd - (long long)t * be;
          const long long begin = end > (long long)be ? end - (long long)be : 0;
          // fixed trip count, predicated: the <= 17 byte loads issue back to back
#pragma unroll
          for (int j = 0; j < 17; ++j) {
            if (begin + j < end) {
              const unsigned c = (unsigned char)d[begin + j] - '0';
              bad |= c > 9;
              limb = limb * 10 + c;
            }
          }
        }
        const int ph = phys<LOGC>(t);
        sm[(2 * o) * N + ph] = limb;
        sm[(2 * o + 1) * N + ph] = limb;
      }
      if (bad) atomicOr(a.err, kErrBadDigit);
      if (tid == 0 && nd > 1 && d[0] == '0') atomicOr(a.err, kErrLeadingZero);
    }
  }
  __syncthreads();
  DMG_PHASE(0);  // pack
  // ---- forward: radix-3 columns (conv.cpp:109-125), then rows ----
  if (THREE && !fused3) {
    for (int i = tid; i < 2 * Cfg::NOPER * C; i += NT) {
      const int arr = i / C, s = i % C, q = arr & 1;
      const u64 p = q ? p1 : p0;
      u64* x = sm + arr * N + col_swizzle(s);
      const TwPair* T = a.r3_fwd[q];
      const u64 x0 = x[0], x1 = x[C], x2 = x[2 * C];
      const u64 t = shoup_mul(mod_sub(x1, x2, p), a.lam[q], p);
      x[0] = mod_add(mod_add(x0, x1, p), x2, p);
      x[C] = shoup_mul(mod_add(mod_sub(x0, x2, p), t, p), T[C + s], p);
      x[2 * C] = shoup_mul(mod_sub(mod_sub(x0, x1, p), t, p), T[2 * C + s], p);
    }
    __syncthreads();
  }
  DMG_PHASE(1);  // radix-3 forward
  tile_dif<LOGC, Cfg::W>(sm, ContigColumns<LOGC>(), SmallField{p0, p1, tf0, tf1, NR}, tid, NT);
  DMG_PHASE(2);  // forward rows
  // ---- pointwise REDC (conv.cpp:205-208); squaring reuses X. X and Y share the
  // same swizzle, so physical offsets pair the same spectrum index. ----
  for (int i = tid; i < 2 * N; i += NT) {
    const int q = i / N;
    const u64 v = sm[i];
    sm[i] = mont_mul(v, SQ ? v : sm[2 * N + i], q ? p1 : p0, a.pp[q]);
  }
  __syncthreads();
  DMG_PHASE(3);  // pointwise
  tile_dit<LOGC, 2 * NR>(sm, ContigColumns<LOGC>(), SmallField{p0, p1, ti0, ti1, NR}, tid, NT);
  if constexpr (THREE) {
    for (int i = tid; i < 2 * C; i += NT) {
      const int q = i / C, s = i % C;
      const u64 p = q ? p1 : p0;
      u64* x = sm + q * N + col_swizzle(s);
      const TwPair* T = a.r3_inv[q];
      const u64 y0 = shoup_mul(x[0], T[s], p);
      const u64 y1 = shoup_mul(x[C], T[C + s], p);
      const u64 y2 = shoup_mul(x[2 * C], T[2 * C + s], p);
      const u64 t = shoup_mul(mod_sub(y1, y2, p), a.lam_inv[q], p);
      x[0] = mod_add(mod_add(y0, y1, p), y2, p);
      x[C] = mod_add(mod_sub(y0, y2, p), t, p);
      x[2 * C] = mod_sub(mod_sub(y0, y1, p), t, p);
    }
  } else {
    for (int i = tid; i < 2 * N; i += NT) {
      const int q = i / N;
      sm[i] = shoup_mul(sm[i], a.scale[q], q ? p1 : p0);
    }
  }
  __syncthreads();
  DMG_PHASE(4);  // inverse (rows + radix-3)
  // ---- CRT + digit split (decimal.cpp:148-152, bounds :174-180), per physical slot ----
  u64* D0 = sm;
  u64* D1 = sm + N;
  u64* D2 = sm + 2 * N;
  for (int i = tid; i < N; i += NT) {
    u64 lo, hi, d0, d1, d2;
    crt2(D0[i], D1[i], p0, p1, a.pp[1], a.r_tilde, lo, hi);
    if (above_cap(lo, hi, a.coeff_cap_lo, a.coeff_cap_hi)) atomicOr(a.err, kErrCoeffBound);
    split3(a.div, lo, hi, d0, d1, d2);
    D0[i] = d0;
    D1[i] = d1;
    D2[i] = d2;
  }
  __syncthreads();
  DMG_PHASE(5);  // CRT + split
  // ---- carry scan over limbs k < N + 2 (logical order) ----
  const u64 B = a.div.base;
  u64 s[Cfg::KPT];
  unsigned agg = kIdentityMap;
  const int k0 = tid * Cfg::KPT;
#pragma unroll
  for (int j = 0; j < Cfg::KPT; ++j) {
    const int k = k0 + j;
    u64 v = 0;
    if (k < Cfg::KL) {
      if (k < N) v += D0[phys<LOGC>(k)];
      if (k >= 1 && k - 1 < N) v += D1[phys<LOGC>(k - 1)];
      if (k >= 2 && k - 2 < N) v += D2[phys<LOGC>(k - 2)];
    }
    s[j] = v;
    agg = map_compose(limb_map(v, B), agg);
  }
  const unsigned pre = block_scan_maps<NT>(agg, wsm, nullptr);  // ends with a barrier
  unsigned c = map_apply(pre, 0);
  u64* Z = sm;  // D arrays are dead after the barrier inside the scan
#pragma unroll
  for (int j = 0; j < Cfg::KPT; ++j) {
    const int k = k0 + j;
    u64 v = s[j] + c;
    unsigned q = 0;
    if (v >= B) { v -= B; ++q; }
    if (v >= B) { v -= B; ++q; }
    c = q;
    if (k < Cfg::KL) Z[k] = v;
  }
  __syncthreads();
  if (tid == 0) {
    const unsigned long long dsum = a.nx + a.ny;
    const unsigned long long chi = (dsum - 1) / be, clo = dsum >= 2 ? (dsum - 2) / be : 0;
    unsigned long long top = 0;
    u64 z = 0;
    if (chi < (unsigned long long)Cfg::KL && Z[chi] != 0) {
      top = chi;
      z = Z[chi];
    } else if (clo < (unsigned long long)Cfg::KL && Z[clo] != 0) {
      top = clo;
      z = Z[clo];
    }
    const unsigned len = decimal_len(z);
    meta[0] = top;
    meta[1] = len;
    meta[2] = len + top * be;
    a.out_lens[prod] = meta[2];
  }
  __syncthreads();
  DMG_PHASE(6);  // carry scan
  // ---- to_decimal: stage the text in shared memory, store 16-byte vectors ----
  const unsigned long long top = meta[0];
  const unsigned top_len = unsigned(meta[1]);
  char* out = a.outs + prod * a.out_stride;
  // text = out (mod 16) for cta_store_bytes, from the 16-byte aligned sm + KL + (KL & 1) (at
  // most the old round-down's offset); plain pointer arithmetic keeps the shared address
  // space visible to the compiler (STS/LDS, not generic stores)
  char* text = reinterpret_cast<char*>(sm + Cfg::KL + (Cfg::KL & 1)) + 16 +
               int(reinterpret_cast<unsigned long long>(out) & 15);
  for (int k = tid; k <= (int)top; k += NT)
    write_digits(text + limb_pos(k, top, top_len, be), Z[k], (unsigned long long)k == top ? top_len : be);
  __syncthreads();
  cta_store_bytes(out, text, unsigned(meta[2]), tid, NT);
  DMG_PHASE(7);  // digits out
}

template <int LOGC, int THREE, int SQ>
bool run_small(const SmallArgs& a, cudaStream_t st) {
  using Cfg = SmallCfg<LOGC, THREE, SQ>;
  static unsigned long long done = 0;  // per device (the attribute is per device)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return false;
  if (!(done >> dev & 1)) {
    if (cudaFuncSetAttribute((const void*)k_small<LOGC, THREE, SQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(Cfg::smem)) != cudaSuccess)
      return false;
    done |= 1ull << dev;
  }
  if (a.count == 0) {  // occupancy query (see small_resident_ctas)
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_small<LOGC, THREE, SQ>, NT, Cfg::smem) != cudaSuccess)
      return false;
    *a.out_lens = (unsigned long long)n;
    return true;
  }
  k_small<LOGC, THREE, SQ><<<a.count, NT, Cfg::smem, st>>>(a);
  return true;
}

template <int LOGC, int THREE>
bool run_small_sq(const SmallArgs& a, cudaStream_t st) {
  return a.squaring ? run_small<LOGC, THREE, 1>(a, st) : run_small<LOGC, THREE, 0>(a, st);
}

}  // namespace

int small_max_logc(int three) { return three ? 10 : 11; }

int small_resident_ctas(int logc, int three, int squaring) {
  unsigned long long n = 0;
  SmallArgs a{};
  a.logc = logc;
  a.three = three;
  a.squaring = squaring;
  a.count = 0;
  a.out_lens = &n;  // host pointer: the count == 0 branch writes the occupancy here
  return launch_small(a, nullptr) ? int(n) : 0;
}

bool launch_small(const SmallArgs& a, cudaStream_t st) {
  if (a.three) {
    switch (a.logc) {
      case 0: return run_small_sq<0, 1>(a, st);
      case 1: return run_small_sq<1, 1>(a, st);
      case 2: return run_small_sq<2, 1>(a, st);
      case 3: return run_small_sq<3, 1>(a, st);
      case 4: return run_small_sq<4, 1>(a, st);
      case 5: return run_small_sq<5, 1>(a, st);
      case 6: return run_small_sq<6, 1>(a, st);
      case 7: return run_small_sq<7, 1>(a, st);
      case 8: return run_small_sq<8, 1>(a, st);
      case 9: return run_small_sq<9, 1>(a, st);
      case 10: return run_small_sq<10, 1>(a, st);
      default: return false;
    }
  }
  switch (a.logc) {
    case 1: return run_small_sq<1, 0>(a, st);
    case 2: return run_small_sq<2, 0>(a, st);
    case 3: return run_small_sq<3, 0>(a, st);
    case 4: return run_small_sq<4, 0>(a, st);
    case 5: return run_small_sq<5, 0>(a, st);
    case 6: return run_small_sq<6, 0>(a, st);
    case 7: return run_small_sq<7, 0>(a, st);
    case 8: return run_small_sq<8, 0>(a, st);
    case 9: return run_small_sq<9, 0>(a, st);
    case 10: return run_small_sq<10, 0>(a, st);
    case 11: return run_small_sq<11, 0>(a, st);
    default: return false;
  }
}

}  // namespace dmg

#ifdef DMG_PHASE_TIMING
extern "C" int decmul_gpu_debug_phase_cycles(unsigned long long* out) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, dmg::g_phase_cycles, sizeof dmg::g_phase_cycles) != cudaSuccess) return 1;
  unsigned long long z[12] = {0};
  return cudaMemcpyToSymbol(dmg::g_phase_cycles, z, sizeof z) == cudaSuccess ? 0 : 1;
}
#endif
