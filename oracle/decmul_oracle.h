/* TEST INFRASTRUCTURE (oracle), not product code.
 *
 * Plain-C restatement of the reference decimal-multiplication hot path
 * (arXiv 2011.11524, /root/reference/proj). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it, and only as the checker.
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * reference's own known-answer tests (copied as numbers into
 * tests/golden/golden.json, "kat") and against the compiled reference
 * (oracle/_ref, and its outputs frozen in golden.json "ref").
 *
 * Return codes: 0 ok, 1 invalid argument, 2 operand too large,
 * 3 runtime error (bound violation), 4 logic error, 6 buffer too small.
 */
#ifndef DECMUL_ORACLE_H
#define DECMUL_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* or_last_error(void);

/* Montgomery field, R = 2^64 (montgomery.hpp:11-55). */
int or_make_ctx(uint64_t p, uint64_t* p_prime, uint64_t* r_mod_p, uint64_t* r2_mod_p);
uint64_t or_redc(uint64_t p, uint64_t x, uint64_t y);
uint64_t or_to_mont(uint64_t p, uint64_t x);
uint64_t or_from_mont(uint64_t p, uint64_t x);
uint64_t or_mont_pow(uint64_t p, uint64_t base_mont, uint64_t e);

/* Primes and roots (primes.cpp). */
int or_is_prime(uint64_t n);
void or_production_primes(uint64_t* p1, uint64_t* p2);
int or_find_primes(unsigned w, unsigned n_min, unsigned ell, uint64_t* out);
int or_primitive_root(uint64_t p, uint64_t n, uint64_t* root_plain);

/* Power-of-two kernels (ntt.cpp). */
int or_ntt_plan(uint64_t p, size_t n, uint64_t* fwd, uint64_t* inv, uint64_t* root, uint64_t* psi,
                uint64_t* psi_prime);
int or_dif_forward(uint64_t p, size_t n, uint64_t* a);
int or_dit_inverse(uint64_t p, size_t n, uint64_t* a);
void or_bit_rev_permute(uint64_t* a, size_t n);
int or_ntt_plan_root(uint64_t p, size_t n, uint64_t root, uint64_t* fwd, uint64_t* inv);
int or_dif_forward_root(uint64_t p, size_t n, uint64_t root, uint64_t* a);

/* Transposition (transpose.cpp). */
void or_transpose_square_sub(uint64_t* a, size_t n, size_t stride);
void or_transpose_n_x_2n(uint64_t* a, size_t n);
void or_transpose_2n_x_n(uint64_t* a, size_t n);

/* Convolution (conv.cpp). thr = six-step threshold (0 = default 2^15).
 * shape: 0 direct, 1 six-step, 2 three-row. */
int or_conv_plan_info(uint64_t p, size_t n, size_t thr, int* shape, uint64_t* root, uint64_t* psi,
                      uint64_t* psi_prime, size_t* n1, size_t* n2);
int or_forward_transform(uint64_t p, size_t n, size_t thr, uint64_t* a);
int or_inverse_transform(uint64_t p, size_t n, size_t thr, uint64_t* a);
int or_pointwise_product(uint64_t p, size_t n, uint64_t* a, const uint64_t* b);
int or_convolve_mod_p(uint64_t p, size_t n, size_t thr, const uint64_t* x, size_t nx, const uint64_t* y,
                      size_t ny, uint64_t* out);

/* Decimal layer (decimal.cpp). p1 == 0 selects the production pair. */
int or_smallest_supported_length(size_t need, uint64_t p1, uint64_t p2, size_t* out);
int or_select_base_and_length(size_t dx, size_t dy, uint64_t p1, uint64_t p2, unsigned forced,
                              unsigned* base_exp, size_t* length);
int or_pack(const char* digits, size_t nd, unsigned base_exp, uint64_t* limbs, size_t cap, size_t* nlimbs);
int or_to_decimal(const uint64_t* limbs, size_t nl, unsigned base_exp, char* out, size_t cap, size_t* len);
int or_crt2(uint64_t p1, uint64_t p2, uint64_t a1, uint64_t a2, uint64_t* lo, uint64_t* hi);
int or_recover_digits(const uint64_t* coeffs_lohi, size_t n, unsigned base_exp, size_t min_limbs,
                      uint64_t* out, size_t cap, size_t* nout);
int or_multiply(const char* x, size_t nx, const char* y, size_t ny, char* out, size_t cap, size_t* out_len,
                unsigned forced_base_exp, uint64_t p1, uint64_t p2);

/* Quadratic checkers (tests/oracle.cpp). */
int or_naive_dft(const uint64_t* x, size_t n, uint64_t root, uint64_t p, uint64_t* out);
int or_naive_convolve(const uint64_t* x, const uint64_t* y, size_t n, uint64_t p, uint64_t* out);
int or_schoolbook_multiply(const char* x, size_t nx, const char* y, size_t ny, char* out, size_t cap,
                           size_t* out_len);

/* Decimal value of s[0..n) mod q (fingerprint for products beyond the quadratic oracle). */
uint64_t or_residue_mod(const char* s, size_t n, uint64_t q);
int or_carry_u16(const unsigned short* acc, size_t n, char* out);
int or_add_shifted(unsigned char* acc, size_t acc_len, const char* p, size_t plen, size_t shift);
void or_residues_multi(const char* s, size_t n, const uint64_t* qs, int nq, uint64_t* out);

/* Shared seeded digit generator; mode 0 uniform, 1 all nines. */
void or_gen_digits(uint64_t seed, int mode, size_t n, char* out);
void or_gen_residues(uint64_t seed, size_t n, uint64_t p, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
