// Kernel parameter blocks and launch helpers shared by kernels.cu and engine.cu.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "modarith.cuh"

namespace dmg {

constexpr int kTileLogW = 4;  // 16 columns per pass tile: one 128 B row segment per tile row
constexpr int kTileW = 1 << kTileLogW;
constexpr int kPassThreads = 256;
constexpr int kMaxPassLog = 9;  // radix of one pass <= 512 (64 KiB tile)

// ---- programmatic dependent launch (PDL) for the product's kernel chain ----
// Chain kernels are launched with programmatic stream serialization: the next grid is
// launched as this grid's CTAs exit (implicit trigger) and its CTAs wait at entry in
// griddepcontrol.wait until the predecessor's writes are visible.
// (An explicit launch_dependents at kernel entry let the whole chain launch at once
// and park in the wait: config 1 ran 2x slower.) Measured: config 1 -19%, config 3 -1%.
// griddepcontrol.wait is a no-op for kernels launched without the attribute;
// DECMUL_PDL=0 disables the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// DMG_PDL_MID=1 (A/B): chain kernels signal launch_dependents once their inputs are staged, so
// the next grid is scheduled (and parks in its wait) while this one still computes.
#ifndef DMG_PDL_MID
#define DMG_PDL_MID 0
#endif
__device__ __forceinline__ void pdl_trigger_mid() {
#if DMG_PDL_MID
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Per-launch profiling (decmul_gpu_profile_*): when the calling thread's engine has profiling
// on, records a CUDA event on st after the kernel just enqueued, tagged with its name and its
// algorithmic work (modular multiplications, HBM bytes); name == nullptr marks the start of
// a product. No-op otherwise.
void prof_mark(const char* name, cudaStream_t st, double modmuls = 0, double bytes = 0);

// Error bits raised by kernels (device flag, read by the host after a product).
enum : unsigned {
  kErrBadDigit = 1u,
  kErrLeadingZero = 2u,
  kErrCoeffBound = 4u,
  kErrCarryBound = 8u,
};

// One pass of a multi-pass transform over both primes.
struct PassArgs {
  const u64* src[2];       // input (may equal dst; pass 0 of an operand reads the shared packed limbs)
  u64* dst[2];             // output
  const u64* other[2];     // fused pass: the other operand's spectrum (nullptr = square)
  const TwPair* dft_fwd[2];  // omega_R^k, k < R/2
  const TwPair* dft_inv[2];  // omega_R^-k, k < R/2
  const TwPair* pass_tw[2];  // T[f][s] = omega_M^{+-f s} (* scale), R x S; nullptr when S == 1
                             // (tw_lbits > 0: the factorised lo[f][s mod 2^tw_lbits], R x 2^tw_lbits)
  const TwPair* pass_hi[2];  // factorised: hi[f][s >> tw_lbits] (* scale), R x S / 2^tw_lbits
  TwPair final_scale[2];   // fused single-pass transforms: (c, c') applied after the inverse
  u64 p[2], pp[2];
  unsigned long long S;    // column stride (elements)
  int logS;
  int has_final_scale;
  int np;                  // primes in this launch; blockIdx.x = tile * np + prime (primes of one tile adjacent)
  unsigned long long G;    // groups of R x S (row passes: tiles run group-fastest)
  // twiddle addressing: T[f << tw_logS + tw_off + s]. Unsharded: tw_logS = logS, tw_off = 0.
  // Column-sharded pass (this rank owns columns [tw_off, tw_off + S) of a global S' = 2^tw_logS).
  int tw_logS;
  unsigned long long tw_off;
  int tw_lbits;            // 0: full R x S twiddle table; else the factorised pair (see pass_tw)
  int lazy_out;            // inverse / fused passes: outputs may stay in [0, 2p) (the next pass is an
                           // inverse row pass, whose first step is a Shoup twiddle product)
  int two;                 // fused pass: other = the first operand before its last forward pass
  int nops;                // forward passes: 2 = a second operand in the same launch (blockIdx.y = 1)
  // Pass 1 after a twiddle-free radix-3 pass (N = 3 S): group g of the pass is radix-3 row f = g.
  // omega_N^{f s}, s = r S1 + c, splits into omega_{3 R}^{f r} (a pre-multiply of the column
  // input r: pre[g R + r], g > 0) and omega_N^{f c}, which commutes with the column DFT and
  // merges into the group's own twiddle table (tables per group: + g tw_gstride / hi_gstride).
  const TwPair* pre[2];
  unsigned long long tw_gstride, hi_gstride;
  const u64* src_b[2];     // the second operand's input / output (nops == 2)
  u64* dst_b[2];
};

// Tensor maps (CUtensorMap, opaque 128 bytes each) of the source arrays of a forward / inverse
// row pass, [operand * 2 + prime], and of its destination arrays, [4 + operand * 2 + prime]; the
// tiles are fetched (and optionally stored) by TMA (kernels.cu stage_rows_tma / store_rows_tma).
struct alignas(64) TileMaps {
  unsigned char m[10][128];  // [8 + prime]: the pass's inter-pass twiddle table (L2 prefetch of its rows)
};

// Radix-3 pass over N = 3 S. The twiddle omega_N^{+-f s} (times the convolution
// scale on the inverse) is factorised as lo[f][s mod L] * hi[f][s / L], L = 2^lbits,
// so the tables are 3 (L + S / L) pairs instead of 3 S (both stay L2-resident).
struct Radix3Args {
  const u64* src[2];
  u64* dst[2];
  const TwPair* lo[2];  // 3 x L
  const TwPair* hi[2];  // 3 x (S / L)
  u64 p[2];
  TwPair lam[2];        // omega_3 (forward) or omega_3^-1 (inverse)
  unsigned long long S;    // local columns
  int lbits;
  unsigned long long hrow;  // entries per f-row of hi (global S >> lbits)
  // local column l -> global column s = ((l >> cb) << sb) + off + (l & (2^cb - 1)).
  // Unsharded: cb = sb = 0, off = 0 (s = l).
  int cb, sb;
  unsigned long long off;
  // Merged twiddles (when the next power-of-two pass carries them, see PassArgs::pre):
  //  * forward: notw = 1, the length-3 DFT alone (omega_N^{f s} moves to pass 1);
  //  * inverse: pinv[f R1 + (s >> pre_shift)] = omega_{3 R1}^{-f r} replaces
  //    lo * hi: one Shoup product per element (r = pass 1's row of global column s).
  int notw;
  const TwPair* pinv[2];
  int pre_shift;
  int pre_rows;  // R1
};

// Launchers (kernels.cu).
void launch_pass_fwd(int logR, const PassArgs& a, unsigned long long ncols, int nprimes, cudaStream_t st);
void launch_pass_inv(int logR, const PassArgs& a, unsigned long long ncols, int nprimes, cudaStream_t st);
void launch_pass_fused(int logR, const PassArgs& a, unsigned long long ncols, int nprimes, cudaStream_t st);
void launch_radix3(bool inverse, const Radix3Args& a, int nprimes, cudaStream_t st);

// out[f][s] = root^(f s mod order) * scale (Shoup pairs), f < R, s < S; order 0 = R S.
// f_off: rows f_off .. f_off + R - 1 (out[f - f_off][s]). f_mul / f_add: the exponent of
// entry [f][s] is (f_mul f + f_add) s (mod order).
void launch_gen_pass_table(TwPair* out, u64 root_m, u64 scale, int R, int logR, unsigned long long S, u64 p,
                           u64 recip, cudaStream_t st, unsigned long long order = 0, int f_off = 0,
                           unsigned long long f_mul = 1, unsigned long long f_add = 0);
// Local limb i is global limb ((i >> row_bits) * row_stride) + off + (i & (2^row_bits - 1)):
// unsharded packs use row_bits = 63, off = 0 (limb i = i). Sharded packs need 2^row_bits >= 256.
// lead_check false (unsharded map only): no leading-zero check (a rank's compacted digit slices).
void launch_pack(const char* digits, unsigned long long nd, unsigned base_exp, u64* limbs,
                 unsigned long long nlimbs_total, unsigned* err, cudaStream_t st, int row_bits = 63,
                 unsigned long long row_stride = 0, unsigned long long off = 0, bool lead_check = true);
// Both operands of a product in one launch (blockIdx.y = operand; unsharded, leading-zero check).
void launch_pack2(const char* dx, unsigned long long nx, u64* limbs_x, const char* dy, unsigned long long ny,
                  u64* limbs_y, unsigned base_exp, unsigned long long nlimbs_total, unsigned* err, cudaStream_t st);
// Pack fused with the forward radix-3 pass (N = 3 S, unsharded): digits -> pass 0's output
// of both primes (a.dst), lo/hi/lam/p/lbits/hrow as for launch_radix3; a.src unused.
void launch_pack_radix3(const char* digits, unsigned long long nd, unsigned base_exp, const Radix3Args& a,
                        unsigned* err, cudaStream_t st);
// Block reorder between the all-to-all layout [peer][row][c] and segment rows [row][peer][c]
// (c < width, row < rows, peer < peers); to_segments selects the direction.
void launch_block_reorder(const u64* src, u64* dst, unsigned long long peers, unsigned long long rows,
                          unsigned long long width, bool to_segments, cudaStream_t st);
void launch_pointwise(u64* a, const u64* b, unsigned long long n, u64 p, u64 pp, cudaStream_t st);
void launch_mont_scale(u64* a, unsigned long long n, u64 factor, u64 p, u64 pp, cudaStream_t st);
void launch_gather(const u64* src, u64* dst, const unsigned long long* map, unsigned long long n, cudaStream_t st);
// DecimalNumber::parse checks on device digits (decimal.cpp:29-36): non-digit bytes and a
// leading zero raise kErrBadDigit / kErrLeadingZero in *err.
void launch_validate(const char* d, unsigned long long n, unsigned* err, cudaStream_t st);

// Carry pipeline (decimal recovery).
struct CarryArgs {
  const u64* z1;        // residues mod p1, natural order, N
  const u64* z2;        // residues mod p2
  unsigned long long n;  // N coefficients; limbs k in [0, n + 2)
  u64 p1, p2, p2_prime, r_tilde;  // CRT (reference decimal.cpp:136-152)
  DivB div;
  u64 coeff_cap_lo, coeff_cap_hi;  // (B-1)^2 * min_limbs
  unsigned base_exp;
  u64* s;               // n + 2 digit sums s_k < 3B
  unsigned* maps;       // per-chunk transfer maps / carry-ins
  unsigned* err;
  unsigned long long top_candidates[2];
  unsigned long long* meta;  // [0] top limb index, [1] top digit count, [2] output length
  char* out;
  // Sharded product (rank owns global coefficients [k_off, k_off + n)); unsharded: all zero / tail = 1.
  unsigned long long k_off;
  u64 halo1[2], halo2[2];  // residues of global coefficients k_off - 2, k_off - 1 (zeros on the first rank)
  int tail;                // this rank also emits the two trailing limbs N, N + 1 (last rank)
  unsigned* ticket;        // small products: CTA completion counter of the split (0 between uses)
  unsigned char* pm;       // optional, K bytes: per-limb in-chunk exclusive prefix maps (split -> emit)
};
constexpr int kCarryChunk = 2048;       // limbs per carry chunk (large products, shards)
constexpr int kCarryThreads = 256;
constexpr int kCarryChunkSmall = 512;   // small products: 4x the CTAs
// maps[] entries the carry of K limbs may use (sized for the small chunk)
inline std::size_t carry_map_words(std::size_t K) { return (K + kCarryChunkSmall - 1) / kCarryChunkSmall; }
// Returns the number of kernels launched.
int launch_carry(const CarryArgs& a, cudaStream_t st);
// Inverse radix-3 pass fused with the recovery (N = 3 S, unsharded, tail = 1): r holds the
// radix-3 inverse arguments (r.src = the last inverse power-of-two pass's output of both
// primes); a.z1/a.z2 are unused. Applies when carry_r3_fusable(S) (S a multiple of the carry
// chunk and a large product). Returns kernels launched.
int launch_carry_r3(const CarryArgs& a, const Radix3Args& r, cudaStream_t st);
bool carry_r3_fusable(unsigned long long S);
// General recovery for small forced bases (lambda < 14, where a coefficient can need more than
// three base-B digits): every coefficient's D base-B digits are added into the limb sums
// s[i + j] (s zeroed first), then `rounds` normalisation passes t_k = s_k mod B + s_{k-1} / B
// (ping-pong through tmp, result back in a.s) bring every sum to <= 3 (B - 1), so the {0,1,2}
// carry scan of launch_carry applies to the K = n + D + rounds limbs. Returns kernels launched.
int launch_carry_general(const CarryArgs& a, int D, int rounds, u64* tmp, unsigned long long K, cudaStream_t st);
// Sharded carry: split + per-chunk exclusive prefix maps; *rank_map_dev gets the rank's composed map.
void launch_carry_shard_begin(const CarryArgs& a, unsigned* rank_map_dev, cudaStream_t st);
// z at the global limbs `cand` owned by this rank (others UINT64_MAX), given the carry into the rank.
void launch_carry_shard_probe(const CarryArgs& a, unsigned rank_cin, u64* z_dev, cudaStream_t st);
// Convert prefix maps to carry-ins, then print this rank's limbs at their global positions.
void launch_carry_shard_emit(const CarryArgs& a, unsigned rank_cin, cudaStream_t st);

// One-CTA-per-product batch kernel (small transforms).
struct SmallArgs {
  const char* xs;               // count operands, x digits at xs + i * x_stride
  const char* ys;
  unsigned long long x_stride, y_stride, nx, ny;
  char* outs;                   // outputs at outs + i * out_stride
  unsigned long long out_stride;
  unsigned long long* out_lens; // per product
  unsigned count;
  unsigned base_exp;
  int logc;                     // power-of-two part: row length c = 2^logc
  int three;                    // N = 3 c if set, else N = c
  u64 p[2], pp[2];
  const TwPair* dft_fwd[2];     // omega_c^k, k < c/2
  const TwPair* dft_inv[2];
  const TwPair* r3_fwd[2];      // 3 x c: omega_N^{f s}
  const TwPair* r3_inv[2];      // 3 x c: omega_N^{-f s} * scale
  TwPair lam[2], lam_inv[2];
  TwPair scale[2];              // used when !three
  u64 p2_prime, r_tilde;
  DivB div;
  u64 coeff_cap_lo, coeff_cap_hi;
  unsigned* err;
  int squaring;
};
bool launch_small(const SmallArgs& a, cudaStream_t st);
int small_max_logc(int three);
// CTAs of the one-CTA kernel resident per SM (occupancy API)
int small_resident_ctas(int logc, int three, int squaring);

// Seeded digit generator (gen.cu): operand j = seed0 + j * seed_step, n digits at out + j * stride.
void launch_generate(u64 seed0, u64 seed_step, unsigned long long count, unsigned long long n,
                     unsigned long long stride, int mode, char* out, cudaStream_t st);
// Integer-pipe roofline denominator (diag.cu): modmul/s, variant 0 Shoup, 1 Montgomery.
double measure_modmul_rate(int variant, cudaStream_t st);

// In-place transposes (reference transpose.cpp) on device memory.
void launch_transpose_square_sub(u64* a, unsigned long long n, unsigned long long stride, cudaStream_t st);
// rho per row of 2n words (n rows), through scratch (>= 2 n^2 words); inverse = unpermute_rho.
// rho permutation of every 2n-word row, in place; scratch holds rho_scratch_words(n) words
// (0 when a row fits shared memory, else 2n per resident CTA)
std::size_t rho_scratch_words(unsigned long long n);
void launch_rho(u64* a, u64* scratch, unsigned long long n, bool inverse, cudaStream_t st);

}  // namespace dmg
