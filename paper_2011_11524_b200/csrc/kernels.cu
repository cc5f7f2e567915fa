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
#include <cstdio>

#include "kernels.cuh"
#include "ntt_tile.cuh"

namespace dmg {

namespace {

constexpr int W = kTileW;
constexpr int NT = kPassThreads;

struct TileGeom {
  bool rows;  // S >= W: tile = one group, 16 adjacent columns; else S == 1: 16 adjacent groups
  unsigned long long base, s0;
  int logS;
  template <int LOGR>
  __device__ __forceinline__ void at(int i, int& r, int& w, unsigned long long& addr) const {
    if (rows) {
      r = i >> kTileLogW;
      w = i & (W - 1);
      addr = base + ((unsigned long long)r << logS) + w;
    } else {
      w = i >> LOGR;
      r = i & ((1 << LOGR) - 1);
      addr = base + i;
    }
  }
};

template <int LOGR>
__device__ __forceinline__ TileGeom tile_geom(const PassArgs& a) {
  TileGeom t;
  const unsigned long long c0 = (unsigned long long)blockIdx.x * W;
  t.rows = a.S > 1;
  t.logS = a.logS;
  if (t.rows) {
    const unsigned long long g = c0 >> a.logS;
    t.s0 = c0 & (a.S - 1);
    t.base = (g << (LOGR + a.logS)) + t.s0;
  } else {
    t.s0 = 0;
    t.base = c0 << LOGR;
  }
  return t;
}

template <int LOGR>
__device__ __forceinline__ void load_table(TwPair* dst, const TwPair* src) {
  for (int i = threadIdx.x; i < (1 << LOGR) / 2; i += NT) dst[i] = src[i];
}

template <int LOGR>
__global__ void __launch_bounds__(NT) k_pass_fwd(PassArgs a) {
  constexpr int R = 1 << LOGR;
  extern __shared__ u64 sm[];
  TwPair* tw = reinterpret_cast<TwPair*>(sm + R * W);
  const int pr = blockIdx.y, tid = threadIdx.x;
  const u64 p = a.p[pr];
  const u64* src = a.src[pr];
  u64* dst = a.dst[pr];
  load_table<LOGR>(tw, a.dft_fwd[pr]);
  const TileGeom t = tile_geom<LOGR>(a);
  const SwizzledRows<W> L;
  for (int i = tid; i < R * W; i += NT) {
    int r, w;
    unsigned long long addr;
    t.at<LOGR>(i, r, w, addr);
    sm[L(r, w)] = src[addr];
  }
  __syncthreads();
  tile_dif<LOGR, W>(sm, L, UniformField{p, tw}, tid, NT);
  const TwPair* __restrict__ T = a.pass_tw[pr];
  for (int i = tid; i < R * W; i += NT) {
    int r, w;
    unsigned long long addr;
    t.at<LOGR>(i, r, w, addr);
    u64 v = sm[L(r, w)];
    if (t.rows) v = shoup_mul(v, T[((unsigned long long)bitrev(r, LOGR) << t.logS) + t.s0 + w], p);
    dst[addr] = v;
  }
}

template <int LOGR>
__global__ void __launch_bounds__(NT) k_pass_inv(PassArgs a) {
  constexpr int R = 1 << LOGR;
  extern __shared__ u64 sm[];
  TwPair* tw = reinterpret_cast<TwPair*>(sm + R * W);
  const int pr = blockIdx.y, tid = threadIdx.x;
  const u64 p = a.p[pr];
  const u64* src = a.src[pr];
  u64* dst = a.dst[pr];
  load_table<LOGR>(tw, a.dft_inv[pr]);
  const TileGeom t = tile_geom<LOGR>(a);
  const SwizzledRows<W> L;
  const TwPair* __restrict__ T = a.pass_tw[pr];
  for (int i = tid; i < R * W; i += NT) {
    int r, w;
    unsigned long long addr;
    t.at<LOGR>(i, r, w, addr);
    u64 v = src[addr];
    if (t.rows) v = shoup_mul(v, T[((unsigned long long)bitrev(r, LOGR) << t.logS) + t.s0 + w], p);
    sm[L(r, w)] = v;
  }
  __syncthreads();
  tile_dit<LOGR, W>(sm, L, UniformField{p, tw}, tid, NT);
  for (int i = tid; i < R * W; i += NT) {
    int r, w;
    unsigned long long addr;
    t.at<LOGR>(i, r, w, addr);
    u64 v = sm[L(r, w)];
    if (a.has_final_scale) v = shoup_mul(v, a.final_scale[pr], p);
    dst[addr] = v;
  }
}

// Last forward pass (S == 1) of one operand fused with the pointwise REDC
// product against the other operand's finished spectrum (reference
// conv.cpp:205-208, :299-305) and the first inverse pass (DIT of the same
// contiguous groups).
template <int LOGR>
__global__ void __launch_bounds__(NT) k_pass_fused(PassArgs a) {
  constexpr int R = 1 << LOGR;
  extern __shared__ u64 sm[];
  TwPair* twf = reinterpret_cast<TwPair*>(sm + R * W);
  TwPair* twi = twf + R / 2;
  const int pr = blockIdx.y, tid = threadIdx.x;
  const u64 p = a.p[pr], pp = a.pp[pr];
  const u64* src = a.src[pr];
  const u64* oth = a.other[pr];
  u64* dst = a.dst[pr];
  load_table<LOGR>(twf, a.dft_fwd[pr]);
  load_table<LOGR>(twi, a.dft_inv[pr]);
  const TileGeom t = tile_geom<LOGR>(a);
  const SwizzledRows<W> L;
  for (int i = tid; i < R * W; i += NT) {
    int r, w;
    unsigned long long addr;
    t.at<LOGR>(i, r, w, addr);
    sm[L(r, w)] = src[addr];
  }
  __syncthreads();
  tile_dif<LOGR, W>(sm, L, UniformField{p, twf}, tid, NT);
  for (int i = tid; i < R * W; i += NT) {
    int r, w;
    unsigned long long addr;
    t.at<LOGR>(i, r, w, addr);
    const int k = L(r, w);
    const u64 v = sm[k];
    sm[k] = mont_mul(v, oth ? oth[addr] : v, p, pp);
  }
  __syncthreads();
  tile_dit<LOGR, W>(sm, L, UniformField{p, twi}, tid, NT);
  for (int i = tid; i < R * W; i += NT) {
    int r, w;
    unsigned long long addr;
    t.at<LOGR>(i, r, w, addr);
    u64 v = sm[L(r, w)];
    if (a.has_final_scale) v = shoup_mul(v, a.final_scale[pr], p);
    dst[addr] = v;
  }
}

// Radix-3 pass (reference three_row_forward_columns conv.cpp:109-125, with the
// length-3 DFT written with one multiplication: omega_3^2 = -1 - omega_3).
__global__ void k_radix3_fwd(Radix3Args a) {
  const int pr = blockIdx.y;
  const u64 p = a.p[pr];
  const unsigned long long S = a.S;
  const u64* src = a.src[pr];
  u64* dst = a.dst[pr];
  const TwPair* __restrict__ T = a.tw[pr];
  for (unsigned long long s = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; s < S;
       s += (unsigned long long)gridDim.x * blockDim.x) {
    const u64 x0 = src[s], x1 = src[S + s], x2 = src[2 * S + s];
    const u64 t = shoup_mul(mod_sub(x1, x2, p), a.lam[pr], p);
    const u64 y0 = mod_add(mod_add(x0, x1, p), x2, p);
    const u64 y1 = mod_add(mod_sub(x0, x2, p), t, p);
    const u64 y2 = mod_sub(mod_sub(x0, x1, p), t, p);
    dst[s] = y0;
    dst[S + s] = shoup_mul(y1, T[S + s], p);
    dst[2 * S + s] = shoup_mul(y2, T[2 * S + s], p);
  }
}

// Inverse radix-3 pass (conv.cpp:129-147): twiddle (with the convolution scale
// folded into the table when this is the first inverse pass) then length-3 IDFT*.
__global__ void k_radix3_inv(Radix3Args a) {
  const int pr = blockIdx.y;
  const u64 p = a.p[pr];
  const unsigned long long S = a.S;
  const u64* src = a.src[pr];
  u64* dst = a.dst[pr];
  const TwPair* __restrict__ T = a.tw[pr];
  for (unsigned long long s = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; s < S;
       s += (unsigned long long)gridDim.x * blockDim.x) {
    const u64 y0 = shoup_mul(src[s], T[s], p);
    const u64 y1 = shoup_mul(src[S + s], T[S + s], p);
    const u64 y2 = shoup_mul(src[2 * S + s], T[2 * S + s], p);
    const u64 t = shoup_mul(mod_sub(y1, y2, p), a.lam[pr], p);
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
  int R;
  unsigned long long S, M;
};

__global__ void k_gen_table(GenArgs g) {
  const unsigned long long total = (unsigned long long)g.R * g.S;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long f = i / g.S, s = i % g.S;
    const unsigned long long e = (f * s) % g.M;  // exponent of omega_M (root_mont may be omega^-1)
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
__global__ void k_pack(const char* __restrict__ d, unsigned long long nd, unsigned be, u64* __restrict__ limbs,
                       unsigned long long total, unsigned* err) {
  const unsigned long long nl = (nd + be - 1) / be;
  for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < total;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    u64 limb = 0;
    if (t < nl) {
      const long long end = (long long)nd - (long long)(t * be);
      const long long begin = end > (long long)be ? end - (long long)be : 0;
      unsigned bad = 0;
      for (long long i = begin; i < end; ++i) {
        const unsigned c = (unsigned char)d[i] - '0';
        bad |= c > 9;
        limb = limb * 10 + c;
      }
      if (bad) atomicOr(err, kErrBadDigit);
      if (begin == 0 && nd > 1 && d[0] == '0') atomicOr(err, kErrLeadingZero);
    }
    limbs[t] = limb;
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

int grid_for(unsigned long long n, int threads) {
  unsigned long long b = (n + threads - 1) / threads;
  const unsigned long long cap = 148ull * 16;
  return int(b < 1 ? 1 : (b > cap ? cap : b));
}

template <int LOGR>
void set_smem(const void* fn, int bytes) {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done = true;
  }
}

template <int LOGR>
void pass_fwd_t(const PassArgs& a, unsigned long long ncols, int np, cudaStream_t st) {
  const int sm = (1 << LOGR) * W * 8 + (1 << LOGR) / 2 * 16;
  set_smem<LOGR>((const void*)k_pass_fwd<LOGR>, sm);
  k_pass_fwd<LOGR><<<dim3(unsigned((ncols + W - 1) / W), np), NT, sm, st>>>(a);
}
template <int LOGR>
void pass_inv_t(const PassArgs& a, unsigned long long ncols, int np, cudaStream_t st) {
  const int sm = (1 << LOGR) * W * 8 + (1 << LOGR) / 2 * 16;
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute((const void*)k_pass_inv<LOGR>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    done = true;
  }
  k_pass_inv<LOGR><<<dim3(unsigned((ncols + W - 1) / W), np), NT, sm, st>>>(a);
}
template <int LOGR>
void pass_fused_t(const PassArgs& a, unsigned long long ncols, int np, cudaStream_t st) {
  const int sm = (1 << LOGR) * W * 8 + (1 << LOGR) * 16;
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute((const void*)k_pass_fused<LOGR>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    done = true;
  }
  k_pass_fused<LOGR><<<dim3(unsigned((ncols + W - 1) / W), np), NT, sm, st>>>(a);
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
    k_radix3_inv<<<dim3(g, np), 256, 0, st>>>(a);
  else
    k_radix3_fwd<<<dim3(g, np), 256, 0, st>>>(a);
}

void launch_gen_pass_table(TwPair* out, u64 root_mont, u64 scale_mont, int R, int /*logR*/, unsigned long long S,
                           u64 p, u64 recip, cudaStream_t st) {
  GenArgs g;
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
  g.M = (unsigned long long)R * S;
  k_gen_table<<<grid_for(g.M, 256), 256, 0, st>>>(g);
}

void launch_pack(const char* digits, unsigned long long nd, unsigned be, u64* limbs, unsigned long long total,
                 unsigned* err, cudaStream_t st) {
  k_pack<<<grid_for(total, 256), 256, 0, st>>>(digits, nd, be, limbs, total, err);
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

}  // namespace dmg
