/* decmul_gpu.h — C ABI of the B200 decimal multiplier (libdecmul_gpu.so).
 *
 * The drop-in boundary for the hot path of the reference decimal multiplier
 * (arXiv 2011.11524, reference tree proj/). Plain pointers and sizes only; the
 * C++ header include/decmul/decimal.hpp re-exposes the reference's own C++ API
 * (DecimalNumber, MultiplyOptions, OperandTooLarge, multiply, ...) on top of it.
 * Every entry point cites the reference interface it replaces.
 *
 * Conventions
 *  - Every call returns an int status (DECMUL_OK or one DECMUL_E* code); the
 *    message of the last failure on a context is decmul_gpu_last_error(ctx).
 *    Codes map one-to-one onto the reference's exception types so a C++
 *    wrapper rethrows the same type with the same text.
 *  - Buffers are caller-owned. "d_" parameters are device pointers on the
 *    context's GPU; all others are host pointers.
 *  - A context is internally locked: one context may be shared by threads,
 *    or use one context per thread — matching the reference's reentrant
 *    multiply and its single plan-cache mutex
 *    (conv.cpp:311-322). Concurrent calls on one context do not simply
 *    serialise: small products are coalesced into batch launches, large
 *    products and batches from pinned buffers overlap their transfers (see
 *    "Concurrency" below).
 */
#ifndef DECMUL_GPU_H
#define DECMUL_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DECMUL_OK = 0,
  DECMUL_EINVAL = 1,    /* std::invalid_argument (decimal.cpp:30-34, :104; conv.cpp:221-238, :274-295) */
  DECMUL_ETOOLARGE = 2, /* decmul::OperandTooLarge (decimal.hpp:20-22; decimal.cpp:96, :99) */
  DECMUL_ECORRUPT = 3,  /* std::runtime_error: analytic bound violated (decimal.cpp:174-180) */
  DECMUL_ELOGIC = 4,    /* std::logic_error: internal self-check (primes.cpp:87,92; decimal.cpp:144) */
  DECMUL_ECUDA = 5,     /* CUDA runtime failure */
  DECMUL_ENOMEM = 6,    /* device or host allocation failure */
  DECMUL_ESPACE = 7     /* caller's output buffer too small */
};

typedef struct decmul_gpu_ctx decmul_gpu_ctx;

typedef struct {
  unsigned base_exp;  /* lambda: limb base 10^lambda */
  size_t length;      /* transform length N (2^k or 3 * 2^k) */
  uint64_t p1, p2;    /* prime pair used (the reference pair unless N > 3 * 2^24) */
  int large_pair;     /* 1 when the reference pair cannot hold N (reference: OperandTooLarge) */
  int one_cta;        /* 1 when the whole product runs inside one CTA */
} decmul_gpu_plan_info;

/* ---- context ---- */
int decmul_gpu_create(decmul_gpu_ctx** ctx, int device);
/* A context over n GPUs (multi-GPU fan-out hidden behind the context). Host-buffer
 * calls use every device: uniform and mixed batches split into contiguous ranges per device; one
 * product with a transform of >= 2^22 words is sharded (columns/rows of the six-step over the
 * devices, the transposition as peer copies over NVLink). Device-pointer calls and the parity
 * hooks run on devices[0]. devices may repeat (ranks sharing a GPU; tests). */
int decmul_gpu_create_multi(decmul_gpu_ctx** ctx, const int* devices, int n);
int decmul_gpu_context_devices(decmul_gpu_ctx* ctx, int* devices, int cap, int* n);
void decmul_gpu_destroy(decmul_gpu_ctx* ctx);
const char* decmul_gpu_last_error(const decmul_gpu_ctx* ctx); /* ctx may be NULL (create failures) */
int decmul_gpu_device_count(int* count);

/* ---- planning: decimal.cpp:54-100 (select_base_and_length, smallest_supported_length) ---- */
int decmul_gpu_select_base_and_length(size_t digits_x, size_t digits_y, uint64_t p1, uint64_t p2,
                                      unsigned forced_base_exp, unsigned* base_exp, size_t* length);
int decmul_gpu_smallest_supported_length(size_t need, uint64_t p1, uint64_t p2, size_t* length);
int decmul_gpu_plan(decmul_gpu_ctx* ctx, size_t digits_x, size_t digits_y, unsigned forced_base_exp,
                    decmul_gpu_plan_info* info);

/* ---- multiply: decmul::multiply, decimal.hpp:176-177 / decimal.cpp:191-216 ----
 * x, y: most-significant-first ASCII digits (the DecimalNumber text, decimal.hpp:26-38).
 * out receives the product digits (cap >= nx + ny); *out_len its length.
 * alias != 0 is the reference's &x == &y squaring path (decimal.cpp:198); equal texts
 * are detected as squaring too. forced_base_exp = MultiplyOptions::forced_base_exp.
 * Products past the largest transform the large pair holds (N > 3 * 2^30 limbs; the reference
 * raises OperandTooLarge past 3 * 2^24) run as a block convolution: block products of 6e9
 * digits fanned out over the context's devices and summed on the host (csrc/blocked.cu). */
int decmul_gpu_multiply(decmul_gpu_ctx* ctx, const char* x, size_t nx, const char* y, size_t ny, char* out,
                        size_t cap, size_t* out_len, unsigned forced_base_exp, int alias);

/* decmul_gpu_multiply with the options of the reference's multiply (MultiplyOptions,
 * decimal.hpp:170-173) plus the prime pair of its planner (select_base_and_length(dx, dy, pair,
 * forced), decimal.hpp:71-72, which the reference's multiply pins to production_primes(),
 * decimal.cpp:194): p1 = p2 = 0 picks the reference pair, or the large pair beyond its
 * 3 * 2^24 cap; otherwise two primes p1 < p2 < 2^63 (DECMUL_EINVAL if not; DECMUL_ETOOLARGE
 * when the pair cannot hold the product, as the reference's planner raises OperandTooLarge). */
typedef struct {
  unsigned forced_base_exp;
  uint64_t p1, p2;
  int alias; /* the reference's &x == &y squaring path */
} decmul_gpu_multiply_options;
int decmul_gpu_multiply_ex(decmul_gpu_ctx* ctx, const char* x, size_t nx, const char* y, size_t ny, char* out,
                           size_t cap, size_t* out_len, const decmul_gpu_multiply_options* opt);

/* decmul_gpu_multiply sharded over the context's devices whatever the size (a product too
 * small for the shard shape fails with DECMUL_EINVAL); what decmul_gpu_multiply does on its own
 * for large products. Exposed for parity tests of the sharded path at small sizes. */
int decmul_gpu_multiply_sharded(decmul_gpu_ctx* ctx, const char* x, size_t nx, const char* y, size_t ny, char* out,
                                size_t cap, size_t* out_len, int alias);

/* Concurrency: decmul_gpu_multiply calls from several threads on one context whose products run
 * as one CTA each (transform length <= 3 * 2^10 or 2^11, no forced base, no alias) are
 * coalesced: the first caller leads, waits for the context, and runs every product queued by
 * then as one batch launch; the others sleep until their result is in. Results and errors are
 * per call (a failing batch is rerun product by product). DECMUL_COALESCE=0 disables it.
 * decmul_gpu_coalesce_stats reports the batches and products run that way.
 * decmul_gpu_multiply[_ex] calls with >= 2^24 digits in all (pinned buffers always; pageable ones
 * while another such call is in flight) run upload, compute and download as separate stages over
 * two sets of digit buffers, the context lock held only around the compute, so one call's
 * download overlaps the next call's upload and compute; decmul_gpu_multiply_batch calls from
 * pinned buffers (two waves of one-CTA products or more) release the context once their chunks
 * are enqueued and alternate between two buffer sets. DECMUL_OVERLAP=0 disables both. */
int decmul_gpu_coalesce_stats(decmul_gpu_ctx* ctx, unsigned long long* batches, unsigned long long* products);

/* Device-resident variant: digits in and out stay in HBM. stream = cudaStream_t (NULL = the
 * context's stream). If out_len is NULL the call is asynchronous (no host sync; read the
 * length later with decmul_gpu_result_length after synchronising the stream). */
int decmul_gpu_multiply_device(decmul_gpu_ctx* ctx, const char* d_x, size_t nx, const char* d_y, size_t ny,
                               char* d_out, size_t cap, size_t* out_len, unsigned forced_base_exp, int squaring,
                               void* stream);
int decmul_gpu_result_length(decmul_gpu_ctx* ctx, size_t* out_len);

/* Batch of `count` independent products of uniform sizes (operand i at xs + i * x_stride,
 * product i at outs + i * out_stride, out_stride >= nx + ny). One CTA per product when the
 * transform fits shared memory. The reference runs products one multiply() at a time. */
int decmul_gpu_multiply_batch(decmul_gpu_ctx* ctx, size_t count, const char* xs, size_t x_stride, size_t nx,
                              const char* ys, size_t y_stride, size_t ny, char* outs, size_t out_stride,
                              size_t* out_lens);
/* Mixed-size batch from host memory (the pointer-array form of SURVEY §8(b)): product i is
 * xs[i] (nxs[i] digits) times ys[i] (nys[i] digits) into outs[i] (caps[i] >= nxs[i] + nys[i]),
 * length to out_lens[i]. Products of equal size pairs run as one batch each (the uniform path
 * above, one CTA per product where N <= 3 * 2^10); the rest one by one. Errors (bad digits,
 * too large) fail the call like the reference's multiply would for the first bad pair. */
int decmul_gpu_multiply_batch_ptrs(decmul_gpu_ctx* ctx, size_t count, const char* const* xs, const size_t* nxs,
                                   const char* const* ys, const size_t* nys, char* const* outs, const size_t* caps,
                                   size_t* out_lens);
/* Device-resident batch, asynchronous on `stream` (NULL = the context's stream). Input errors
 * (non-digit bytes, leading zeros) and bound violations of the asynchronous entry points
 * (this call and multiply_device without out_len) are collected in a stream-ordered error
 * word of their own: decmul_gpu_check_errors(ctx, stream) synchronises the stream, clears the
 * word and returns the matching code (DECMUL_EINVAL, DECMUL_ECORRUPT) for the calls since the
 * last check; decmul_gpu_result_length does the same. Synchronous calls never see them. */
int decmul_gpu_multiply_batch_device(decmul_gpu_ctx* ctx, size_t count, const char* d_xs, size_t x_stride,
                                     size_t nx, const char* d_ys, size_t y_stride, size_t ny, char* d_outs,
                                     size_t out_stride, unsigned long long* d_lens, void* stream);
int decmul_gpu_check_errors(decmul_gpu_ctx* ctx, void* stream);

/* ---- parity hooks on host arrays (conv.hpp:59-71) ----
 * p must be one of the supported primes (the reference pair or the large pair); n = 2^k or
 * 3 * 2^k dividing p - 1. forward_transform output follows the reference's documented storage
 * order for its default plan (conv.hpp:19-24); inverse_transform consumes that order. */
int decmul_gpu_convolve_mod_p(decmul_gpu_ctx* ctx, uint64_t p, size_t n, const uint64_t* x, size_t nx,
                              const uint64_t* y, size_t ny, uint64_t* out);
int decmul_gpu_forward_transform(decmul_gpu_ctx* ctx, uint64_t p, size_t n, uint64_t* a);
int decmul_gpu_inverse_transform(decmul_gpu_ctx* ctx, uint64_t p, size_t n, uint64_t* a);
int decmul_gpu_pointwise_product(decmul_gpu_ctx* ctx, uint64_t p, size_t n, uint64_t* a, const uint64_t* b);
/* The same hooks for a plan built with a non-default six-step threshold, build_conv_plan(ctx, n,
 * six_step_threshold) (conv.hpp:59-60, conv.cpp:243-269; 0 = kDefaultSixStepThreshold = 2^15):
 * the spectrum is stored in that plan's order (kDirect when n <= threshold, else kSixStep with
 * n1 = 2^floor(k/2); the three-row shape hands the threshold to its row plan), as the
 * reference's forced-shape checks need (test_conv.cpp:183-196, selftest.cpp:109-118).
 * conv_plan_info reports the plan's shape (0 direct, 1 six-step, 2 three-row), its plain
 * primitive root (primes.cpp:99-112) and the six-step factors; it needs no GPU. */
int decmul_gpu_forward_transform_ex(decmul_gpu_ctx* ctx, uint64_t p, size_t n, size_t six_step_threshold,
                                    uint64_t* a);
int decmul_gpu_inverse_transform_ex(decmul_gpu_ctx* ctx, uint64_t p, size_t n, size_t six_step_threshold,
                                    uint64_t* a);
int decmul_gpu_conv_plan_info(uint64_t p, size_t n, size_t six_step_threshold, int* shape, uint64_t* root,
                              size_t* n1, size_t* n2);

/* ---- stage hooks ----
 * pack: decimal.cpp:102-118. recover_decimal: crt2 over the two residue vectors
 * (decimal.cpp:148-152, :209-211), recover_digits (:154-189) and to_decimal (:120-134);
 * digits_sum = digit count of x plus digit count of y (bounds the product length). */
int decmul_gpu_pack(decmul_gpu_ctx* ctx, const char* digits, size_t nd, unsigned base_exp, uint64_t* limbs,
                    size_t cap, size_t* nlimbs);
int decmul_gpu_recover_decimal(decmul_gpu_ctx* ctx, const uint64_t* r1, const uint64_t* r2, size_t n, uint64_t p1,
                               uint64_t p2, unsigned base_exp, size_t min_limbs, size_t digits_sum, char* out,
                               size_t cap, size_t* out_len);

/* ---- in-place transposition: transpose.hpp:11-24 ---- */
int decmul_gpu_transpose_square_sub(decmul_gpu_ctx* ctx, uint64_t* a, size_t n, size_t stride);
int decmul_gpu_transpose_n_x_2n(decmul_gpu_ctx* ctx, uint64_t* a, size_t n);
int decmul_gpu_transpose_2n_x_n(decmul_gpu_ctx* ctx, uint64_t* a, size_t n);

/* ---- sharded large products (one product over `ranks` GPUs; not in the reference, which is
 * single-threaded and caps N at 3 * 2^24). The caller owns the exchange (NCCL all-to-all or any
 * transport) and runs, on every rank q, with device buffers of local_len words per prime:
 *   pack(x) -> transform(COL_FWD) -> [reorder-free all-to-all] -> reorder(to_segments=1) ->
 *   transform(ROW_FWD)  (same for y with ROW_FWD_CONV against x) -> reorder(to_segments=0) ->
 *   all-to-all -> transform(COL_INV) -> all-to-all -> reorder(to_segments=1) ->
 *   carry_begin (halo = p1, p1, p2, p2 residues of the two coefficients before this rank's block,
 *   gathered from rank q-1) -> all-gather rank maps -> carry_probe -> all-gather -> carry_emit.
 * All-to-all chunks are contiguous: local_len / ranks words per peer per prime.
 * paper_2011_11524_b200/sharded.py is the reference driver. ---- */
typedef struct {
  size_t length;          /* N */
  unsigned base_exp;      /* lambda */
  uint64_t p1, p2;
  int ranks;              /* G (power of two) */
  int col_passes;         /* K: passes run column-sharded */
  size_t rows;            /* Rtot: rows of the column phase (multiple of G) */
  size_t seg_len;         /* Sc = N / Rtot */
  size_t col_width;       /* Bc = Sc / G: this rank's columns */
  size_t local_len;       /* N / G */
  size_t s_words;         /* words of the carry scratch (d_s) */
  size_t map_words;       /* words of the chunk-map scratch (d_maps) */
  size_t digits_x, digits_y;
  unsigned long long top_candidates[2];
} decmul_gpu_shard_plan;

enum { DECMUL_SHARD_COL_FWD = 0, DECMUL_SHARD_ROW_FWD = 1, DECMUL_SHARD_ROW_FWD_CONV = 2, DECMUL_SHARD_COL_INV = 3 };

int decmul_gpu_shard_plan_create(decmul_gpu_ctx* ctx, size_t digits_x, size_t digits_y, int ranks,
                                 decmul_gpu_shard_plan* plan);
int decmul_gpu_shard_pack(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* plan, int rank, const char* d_digits,
                          size_t nd, uint64_t* d_out, void* stream);
int decmul_gpu_shard_transform(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* plan, int rank, int stage,
                               const uint64_t* d_src1, const uint64_t* d_src2, uint64_t* d_dst1, uint64_t* d_dst2,
                               const uint64_t* d_other1, const uint64_t* d_other2, void* stream);
int decmul_gpu_shard_reorder(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* plan, int to_segments,
                             const uint64_t* d_src, uint64_t* d_dst, void* stream);
int decmul_gpu_shard_carry_begin(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* plan, int rank,
                                 const uint64_t* d_z1, const uint64_t* d_z2, const uint64_t halo[4], uint64_t* d_s,
                                 unsigned* d_maps, unsigned* rank_map, void* stream);
int decmul_gpu_shard_carry_probe(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* plan, int rank,
                                 unsigned rank_carry_in, const uint64_t* d_z1, const uint64_t* d_z2,
                                 const uint64_t* d_s, unsigned* d_maps, uint64_t z_out[2], void* stream);
int decmul_gpu_shard_carry_emit(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* plan, int rank,
                                unsigned rank_carry_in, unsigned long long top, unsigned top_len,
                                const uint64_t* d_z1, const uint64_t* d_z2, const uint64_t* d_s, unsigned* d_maps,
                                char* d_out, void* stream);

/* ---- workload generation (not in the reference: its bench_mul draws digits on the host,
 * bench.cpp:107-116). Seeded counter-based splitmix64 digits written in place in HBM:
 * operand j (seed seed0 + j * seed_step) gets n digits at d_out + j * stride; mode 0 uniform
 * with a nonzero leading digit, mode 1 all nines. Bit-identical to the host generator. ---- */
int decmul_gpu_generate_digits(decmul_gpu_ctx* ctx, uint64_t seed0, uint64_t seed_step, size_t count, size_t n,
                               size_t stride, int mode, char* d_out, void* stream);

/* ---- introspection ---- */
/* Integer-pipe roofline denominator: measured modmul/s on this GPU, chained independent lanes on
 * all SMs (reference bench_modmul, bench.cpp:49-94): variant 0 Shoup (the transforms' form),
 * 1 Montgomery REDC, 2 the Solinas reduction for the Goldilocks prime 2^64 - 2^32 + 1. */
int decmul_gpu_measure_modmul_rate(decmul_gpu_ctx* ctx, int variant, double* modmul_per_s);
typedef struct {
  int last_launches;       /* kernels launched by the last product */
  size_t table_bytes;      /* device bytes held by cached twiddle tables */
} decmul_gpu_stats;
int decmul_gpu_get_stats(decmul_gpu_ctx* ctx, decmul_gpu_stats* out);
/* Per-launch timing (diagnostics, bench.py's roofline): while enabled, a CUDA event follows every
 * kernel the context enqueues. decmul_gpu_profile_report synchronises and writes one line per
 * launch since the last enable/report, "name<TAB>ms<TAB>modmuls<TAB>hbm_bytes\n" (ms since the
 * previous event on the product's stream; modmuls and bytes are the launch's algorithmic work),
 * NUL-terminated to report (truncated to cap; *len = full length), and clears the records
 * (report == NULL only returns *len and keeps them). */
int decmul_gpu_profile(decmul_gpu_ctx* ctx, int enable);
int decmul_gpu_profile_report(decmul_gpu_ctx* ctx, char* report, size_t cap, size_t* len);

/* GPU self-test, replaces run_selftest (selftest.cpp:79-219; CLI `selftest [--inject-fault]`,
 * main.cpp:162): field identities, transform round trips, convolution vs a direct O(n^2)
 * sum, CRT, base division, carry recovery and small products, all on the device path and
 * checked on the host. inject_fault corrupts one root-table entry of a plan (restored
 * afterwards) and adds a suite that must fail. The report ("suite=<name> checks=<n>
 * failures=<n>" lines, then "selftest_failures=<n>", the reference's format) is written
 * NUL-terminated to report (truncated to cap); *failures gets the total. Returns 0 when
 * the test ran, whatever its outcome. */
int decmul_gpu_selftest(decmul_gpu_ctx* ctx, int inject_fault, char* report, size_t cap, int* failures);

#ifdef __cplusplus
}
#endif
#endif /* DECMUL_GPU_H */
