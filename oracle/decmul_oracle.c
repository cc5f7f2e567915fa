/* TEST INFRASTRUCTURE (oracle), not product code — see decmul_oracle.h.
 *
 * A plain-C restatement of the reference's decimal multiplication path.
 * Each function cites the reference file:line (under /root/reference/proj)
 * whose algorithm it restates. It deliberately follows the reference's
 * structure (Montgomery tables, six-step / three-row decomposition, reciprocal
 * bounds) so spectra, plans and products can be compared value for value;
 * where the reference uses a precomputed-reciprocal division the oracle uses
 * plain 128-bit division (the mathematically defining operation).
 */
#include "decmul_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef unsigned __int128 u128;

static __thread char g_err[256];
const char* or_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

static const u64 kP1 = 9223372036015915009ull; /* primes.hpp:30 */
static const u64 kP2 = 9223372036166909953ull; /* primes.hpp:31 */
#define DEFAULT_THR ((size_t)1 << 15)          /* conv.hpp:15 */

/* ---------------- Montgomery field (montgomery.hpp / montgomery.cpp) ---------------- */

typedef struct {
  u64 p, pp, r, r2;
} mctx;

/* make_ctx, montgomery.cpp:28-41 (p' by Newton iteration instead of extended Euclid). */
static int make_ctx(u64 p, mctx* c) {
  if (p <= 2 || !(p & 1) || p >= (1ull << 63)) return fail(1, "make_ctx: bad modulus");
  u64 inv = p; /* p * inv == 1 mod 2^64 */
  for (int i = 0; i < 6; ++i) inv *= 2 - p * inv;
  c->p = p;
  c->pp = (u64)0 - inv;
  c->r = ((u64)0 - p) % p;
  c->r2 = (u64)(((u128)c->r * c->r) % p);
  return 0;
}

/* mont_reduce, montgomery.hpp:26-34: a < p 2^64 -> a R^-1 mod p. */
static u64 mreduce(const mctx* c, u128 a) {
  u64 m = (u64)a * c->pp;
  u128 t = a + (u128)m * c->p; /* < 2^128 for legal inputs a < p 2^64; low word is 0 */
  u64 hi = (u64)(t >> 64);
  return hi >= c->p ? hi - c->p : hi;
}
static u64 redc(const mctx* c, u64 x, u64 y) { return mreduce(c, (u128)x * y); }   /* :36-39 */
static u64 to_mont(const mctx* c, u64 x) { return redc(c, x, c->r2); }              /* :51 */
static u64 from_mont(const mctx* c, u64 x) { return mreduce(c, (u128)x); }           /* :52 */
static u64 mont_pow(const mctx* c, u64 b, u64 e) {                                   /* montgomery.cpp:43-52 */
  u64 r = c->r;
  while (e) {
    if (e & 1) r = redc(c, r, b);
    b = redc(c, b, b);
    e >>= 1;
  }
  return r;
}
static u64 mod_add(u64 a, u64 b, u64 p) { u64 s = a + b; return s >= p ? s - p : s; } /* words.hpp:48-51 */
static u64 mod_sub(u64 a, u64 b, u64 p) { return a >= b ? a - b : a + p - b; }        /* words.hpp:54-57 */

int or_make_ctx(u64 p, u64* pp, u64* r, u64* r2) {
  mctx c;
  int rc = make_ctx(p, &c);
  if (rc) return rc;
  *pp = c.pp;
  *r = c.r;
  *r2 = c.r2;
  return 0;
}
u64 or_redc(u64 p, u64 x, u64 y) { mctx c; make_ctx(p, &c); return redc(&c, x, y); }
u64 or_to_mont(u64 p, u64 x) { mctx c; make_ctx(p, &c); return to_mont(&c, x); }
u64 or_from_mont(u64 p, u64 x) { mctx c; make_ctx(p, &c); return from_mont(&c, x); }
u64 or_mont_pow(u64 p, u64 b, u64 e) { mctx c; make_ctx(p, &c); return mont_pow(&c, b, e); }

/* ---------------- primes (primes.cpp) ---------------- */

static u64 mulmod(u64 a, u64 b, u64 n) { return (u64)((u128)a * b % n); }
static u64 powmod(u64 a, u64 e, u64 n) {
  u64 r = 1 % n;
  a %= n;
  while (e) {
    if (e & 1) r = mulmod(r, a, n);
    a = mulmod(a, a, n);
    e >>= 1;
  }
  return r;
}

/* is_prime, primes.cpp:24-49: Miller-Rabin over the first twelve prime bases. */
int or_is_prime(u64 n) {
  static const u64 bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i) {
    if (n == bases[i]) return 1;
    if (n % bases[i] == 0) return 0;
  }
  u64 d = n - 1;
  int s = __builtin_ctzll(d);
  d >>= s;
  for (int i = 0; i < 12; ++i) {
    u64 x = powmod(bases[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int comp = 1;
    for (int k = 1; k < s; ++k) {
      x = mulmod(x, x, n);
      if (x == n - 1) { comp = 0; break; }
    }
    if (comp) return 0;
  }
  return 1;
}

void or_production_primes(u64* p1, u64* p2) { *p1 = kP1; *p2 = kP2; } /* primes.cpp:83-97 */

/* find_primes_for_n / find_primes, primes.cpp:51-81. */
static int cmp_desc(const void* a, const void* b) {
  u64 x = *(const u64*)a, y = *(const u64*)b;
  return x < y ? 1 : (x > y ? -1 : 0);
}
int or_find_primes(unsigned w, unsigned n_min, unsigned ell, u64* out) {
  if (w != 64) return fail(1, "find_primes: only w = 64 is supported");
  const u64 p_max = (1ull << 63) - 1;
  size_t cap = (size_t)ell * 64, cnt = 0;
  u64* all = (u64*)malloc(cap * sizeof(u64));
  for (unsigned n = n_min; n <= w - 2; ++n) {
    if (n >= 63) continue;
    int64_t psi = (int64_t)((p_max - 1) >> n);
    if (psi % 2 == 0) psi -= 1;
    while (psi > 0 && psi % 3 != 0) psi -= 2;
    if (psi <= 0) continue;
    unsigned got = 0;
    while (psi > 0 && got < ell) {
      u64 p = ((u64)psi << n) + 1;
      if (or_is_prime(p)) {
        int dup = 0;
        for (size_t i = 0; i < cnt; ++i) dup |= all[i] == p;
        if (!dup) all[cnt++] = p;
        ++got;
      }
      psi -= 6;
    }
  }
  if (cnt < ell) { free(all); return fail(3, "find_primes: not enough primes of the required form"); }
  qsort(all, cnt, sizeof(u64), cmp_desc);
  memcpy(out, all, ell * sizeof(u64));
  free(all);
  return 0;
}

/* primitive_root_of_unity, primes.cpp:99-112: candidates 2, 3, 5, 7, ...; Montgomery result. */
static int prim_root(const mctx* c, u64 n, u64* out_mont) {
  const u64 p = c->p;
  if (n == 0 || (p - 1) % n) return fail(1, "primitive_root_of_unity: n must divide p-1");
  if (n == 1) { *out_mont = c->r; return 0; }
  for (u64 g = 2; g < p; g = (g == 2 ? 3 : g + 2)) {
    u64 xi = mont_pow(c, to_mont(c, g), (p - 1) / n);
    if (n % 2 == 0 && mont_pow(c, xi, n / 2) == c->r) continue;
    if (n % 3 == 0 && mont_pow(c, xi, n / 3) == c->r) continue;
    *out_mont = xi;
    return 0;
  }
  return fail(4, "primitive_root_of_unity: no generator found");
}
int or_primitive_root(u64 p, u64 n, u64* root_plain) {
  mctx c;
  int rc = make_ctx(p, &c);
  u64 m;
  if (rc || (rc = prim_root(&c, n, &m))) return rc;
  *root_plain = from_mont(&c, m);
  return 0;
}

/* ---------------- power-of-two kernels (ntt.hpp / ntt.cpp) ---------------- */

typedef struct {
  mctx c;
  size_t n;
  unsigned log2n;
  u64 root, psi, psi_prime;
  u64 *fwd, *inv; /* flat stage slices, ntt.hpp:10-19 */
} nttplan;

/* build_table, ntt.cpp:13-27. */
static void build_table(const mctx* c, size_t n, unsigned log2n, u64 root, u64* t) {
  if (n == 1) return;
  size_t half = n / 2;
  u64* top = t + (half - 1);
  u64 rh = to_mont(c, root);
  top[0] = c->r;
  for (size_t i = 1; i < half; ++i) top[i] = redc(c, top[i - 1], rh);
  for (unsigned s = log2n - 1; s >= 1; --s) {
    u64* sl = t + (((size_t)1 << (s - 1)) - 1);
    for (size_t i = 0; i < ((size_t)1 << (s - 1)); ++i) sl[i] = top[i << (log2n - s)];
  }
}

/* build_plan_with_root, ntt.cpp:88-112. */
static int ntt_plan_root(const mctx* c, size_t n, u64 root, nttplan* pl) {
  if (n == 0 || (n & (n - 1))) return fail(1, "build_plan: n must be a power of two");
  if (n > 1 && (c->p - 1) % n) return fail(1, "build_plan: n does not divide p-1");
  memset(pl, 0, sizeof *pl);
  pl->c = *c;
  pl->n = n;
  pl->log2n = (unsigned)__builtin_ctzll(n);
  pl->root = root % c->p;
  u64 rh = to_mont(c, pl->root);
  if (mont_pow(c, rh, n) != c->r) return fail(1, "build_plan: root^n != 1");
  if (n > 1 && mont_pow(c, rh, n / 2) == c->r) return fail(1, "build_plan: root is not primitive");
  u64 rinv = from_mont(c, mont_pow(c, rh, n - 1));
  pl->fwd = (u64*)calloc(n, sizeof(u64));
  pl->inv = (u64*)calloc(n, sizeof(u64));
  build_table(c, n, pl->log2n, pl->root, pl->fwd);
  build_table(c, n, pl->log2n, rinv, pl->inv);
  pl->psi = mont_pow(c, to_mont(c, (u64)n % c->p), c->p - 2);
  pl->psi_prime = redc(c, pl->psi, c->r2);
  return 0;
}
static int ntt_plan(const mctx* c, size_t n, nttplan* pl) { /* build_plan, ntt.cpp:83-86 */
  u64 root = 1;
  if (n > 1) {
    u64 m;
    int rc = prim_root(c, n, &m);
    if (rc) return rc;
    root = from_mont(c, m);
  }
  return ntt_plan_root(c, n, root, pl);
}
static void ntt_free(nttplan* pl) { free(pl->fwd); free(pl->inv); pl->fwd = pl->inv = NULL; }

/* dif_impl, ntt.cpp:29-50: Gentleman-Sande, natural in, bit-reversed out. */
static void dif(const nttplan* pl, u64* a) {
  const u64 p = pl->c.p;
  for (size_t m = pl->n; m >= 2; m >>= 1) {
    size_t h = m >> 1;
    const u64* tb = pl->fwd + (h - 1);
    for (size_t k = 0; k < pl->n; k += m) {
      u64 *x = a + k, *y = x + h;
      for (size_t j = 0; j < h; ++j) {
        u64 u = x[j], v = y[j];
        x[j] = mod_add(u, v, p);
        y[j] = j == 0 ? mod_sub(u, v, p) : mreduce(&pl->c, (u128)(u - v + p) * tb[j]);
      }
    }
  }
}
/* dit_impl, ntt.cpp:52-73: Cooley-Tukey, bit-reversed in, natural out, unscaled. */
static void dit(const nttplan* pl, u64* a) {
  const u64 p = pl->c.p;
  for (size_t m = 2; m <= pl->n; m <<= 1) {
    size_t h = m >> 1;
    const u64* tb = pl->inv + (h - 1);
    for (size_t k = 0; k < pl->n; k += m) {
      u64 *x = a + k, *y = x + h;
      for (size_t j = 0; j < h; ++j) {
        u64 u = x[j];
        u64 w = j == 0 ? y[j] : redc(&pl->c, tb[j], y[j]);
        x[j] = mod_add(u, w, p);
        y[j] = mod_sub(u, w, p);
      }
    }
  }
}
/* bit_rev_permute, ntt.cpp:114-126. */
void or_bit_rev_permute(u64* a, size_t n) {
  for (size_t i = 0, j = 0; i < n; ++i) {
    if (i < j) { u64 t = a[i]; a[i] = a[j]; a[j] = t; }
    size_t mask = n >> 1;
    while (j & mask) { j ^= mask; mask >>= 1; }
    j |= mask;
  }
}

int or_ntt_plan(u64 p, size_t n, u64* fwd, u64* inv, u64* root, u64* psi, u64* psi_prime) {
  mctx c;
  nttplan pl;
  int rc = make_ctx(p, &c);
  if (rc || (rc = ntt_plan(&c, n, &pl))) return rc;
  if (n > 1) {
    memcpy(fwd, pl.fwd, (n - 1) * sizeof(u64));
    memcpy(inv, pl.inv, (n - 1) * sizeof(u64));
  }
  *root = pl.root;
  *psi = pl.psi;
  *psi_prime = pl.psi_prime;
  ntt_free(&pl);
  return 0;
}
int or_dif_forward(u64 p, size_t n, u64* a) {
  mctx c;
  nttplan pl;
  int rc = make_ctx(p, &c);
  if (rc || (rc = ntt_plan(&c, n, &pl))) return rc;
  dif(&pl, a);
  ntt_free(&pl);
  return 0;
}
int or_dit_inverse(u64 p, size_t n, u64* a) {
  mctx c;
  nttplan pl;
  int rc = make_ctx(p, &c);
  if (rc || (rc = ntt_plan(&c, n, &pl))) return rc;
  dit(&pl, a);
  ntt_free(&pl);
  return 0;
}

/* ---------------- transposition (transpose.cpp) ---------------- */

/* transpose_square_sub, transpose.cpp:12-25 (untiled: the oracle needs only the result). */
void or_transpose_square_sub(u64* a, size_t n, size_t stride) {
  for (size_t i = 0; i < n; ++i)
    for (size_t j = i + 1; j < n; ++j) {
      u64 t = a[i * stride + j];
      a[i * stride + j] = a[j * stride + i];
      a[j * stride + i] = t;
    }
}
/* permute_rho / unpermute_rho, transpose.cpp:27-41. */
static void rho(u64* row, size_t n, u64* s, int inverse) {
  memcpy(s, row, 2 * n * sizeof(u64));
  for (size_t i = 0; i < n; ++i) {
    if (!inverse) { row[i] = s[2 * i]; row[i + n] = s[2 * i + 1]; }
    else { row[2 * i] = s[i]; row[2 * i + 1] = s[i + n]; }
  }
}
/* transpose_n_x_2n, transpose.cpp:43-47. */
void or_transpose_n_x_2n(u64* a, size_t n) {
  u64* s = (u64*)malloc(2 * n * sizeof(u64));
  for (size_t i = 0; i < n; ++i) rho(a + i * 2 * n, n, s, 0);
  or_transpose_square_sub(a, n, 2 * n);
  or_transpose_square_sub(a + n, n, 2 * n);
  free(s);
}
/* transpose_2n_x_n, transpose.cpp:49-53. */
void or_transpose_2n_x_n(u64* a, size_t n) {
  u64* s = (u64*)malloc(2 * n * sizeof(u64));
  or_transpose_square_sub(a, n, 2 * n);
  or_transpose_square_sub(a + n, n, 2 * n);
  for (size_t i = 0; i < n; ++i) rho(a + i * 2 * n, n, s, 1);
  free(s);
}

/* ---------------- convolution (conv.hpp / conv.cpp) ---------------- */

typedef struct convplan {
  mctx c;
  size_t n;
  int shape; /* 0 direct, 1 six-step, 2 three-row (conv.hpp:11) */
  u64 root, psi, psi_prime;
  nttplan direct;
  size_t n1, n2;
  nttplan col, row;
  u64 xi, xi_inv;
  struct convplan* rowplan;
  u64 gamma, gamma2, lam, lam2, gamma_inv, gamma2_inv, lam_inv, lam2_inv;
} convplan;

static u64 pow_plain(const mctx* c, u64 b, u64 e) { return from_mont(c, mont_pow(c, to_mont(c, b), e)); }

/* build_conv_plan_with_root, conv.cpp:217-271. */
static int conv_plan_root(const mctx* c, size_t n, u64 root, size_t thr, convplan* pl) {
  int pow2 = n > 0 && !(n & (n - 1));
  int three = n % 3 == 0 && n / 3 > 0 && !((n / 3) & (n / 3 - 1));
  if (!pow2 && !three) return fail(1, "build_conv_plan: length must be 2^k or 3*2^k");
  if (n > 1 && (c->p - 1) % n) return fail(1, "build_conv_plan: length does not divide p-1");
  memset(pl, 0, sizeof *pl);
  pl->c = *c;
  pl->n = n;
  pl->root = root % c->p;
  u64 rh = to_mont(c, pl->root);
  if (mont_pow(c, rh, n) != c->r) return fail(1, "build_conv_plan: root^n != 1");
  if (n % 2 == 0 && mont_pow(c, rh, n / 2) == c->r) return fail(1, "build_conv_plan: root is not primitive");
  if (n % 3 == 0 && mont_pow(c, rh, n / 3) == c->r) return fail(1, "build_conv_plan: root is not primitive");
  pl->psi = mont_pow(c, to_mont(c, (u64)n % c->p), c->p - 2);
  pl->psi_prime = redc(c, pl->psi, c->r2);
  int rc = 0;
  if (three) {
    size_t cc = n / 3;
    pl->shape = 2;
    pl->rowplan = (convplan*)calloc(1, sizeof(convplan));
    rc = conv_plan_root(c, cc, pow_plain(c, pl->root, 3), thr, pl->rowplan);
    pl->gamma = rh;
    pl->gamma2 = redc(c, rh, rh);
    pl->lam = mont_pow(c, rh, cc);
    pl->lam2 = redc(c, pl->lam, pl->lam);
    u64 rinv = mont_pow(c, rh, n - 1);
    pl->gamma_inv = rinv;
    pl->gamma2_inv = redc(c, rinv, rinv);
    pl->lam_inv = mont_pow(c, rinv, cc);
    pl->lam2_inv = redc(c, pl->lam_inv, pl->lam_inv);
  } else if (n <= thr) {
    pl->shape = 0;
    rc = ntt_plan_root(c, n, pl->root, &pl->direct);
  } else {
    unsigned k = (unsigned)__builtin_ctzll(n);
    pl->shape = 1;
    pl->n1 = (size_t)1 << (k / 2);
    pl->n2 = n / pl->n1;
    rc = ntt_plan_root(c, pl->n1, pow_plain(c, pl->root, pl->n2), &pl->col);
    if (!rc) rc = ntt_plan_root(c, pl->n2, pow_plain(c, pl->root, pl->n1), &pl->row);
    pl->xi = rh;
    pl->xi_inv = mont_pow(c, rh, n - 1);
  }
  return rc;
}
static int conv_plan(u64 p, size_t n, size_t thr, convplan* pl) { /* build_conv_plan, conv.cpp:212-215 */
  mctx c;
  int rc = make_ctx(p, &c);
  if (rc) return rc;
  u64 root = 1;
  if (n > 1) {
    u64 m;
    if ((rc = prim_root(&c, n, &m))) return rc;
    root = from_mont(&c, m);
  }
  return conv_plan_root(&c, n, root, thr ? thr : DEFAULT_THR, pl);
}
static void conv_free(convplan* pl) {
  ntt_free(&pl->direct);
  ntt_free(&pl->col);
  ntt_free(&pl->row);
  if (pl->rowplan) { conv_free(pl->rowplan); free(pl->rowplan); pl->rowplan = NULL; }
}

/* six_transpose, conv.cpp:30-38. */
static void six_transpose(const convplan* pl, u64* a, int to_wide) {
  if (pl->n1 == pl->n2) or_transpose_square_sub(a, pl->n1, pl->n1);
  else if (to_wide) or_transpose_n_x_2n(a, pl->n1);
  else or_transpose_2n_x_n(a, pl->n1);
}

static void fwd_in_place(const convplan* pl, u64* a);
static void inv_in_place(const convplan* pl, u64* a, u64 phi);

/* six_step_forward, conv.cpp:72-87 with six_twiddle_forward :41-54. */
static void six_fwd(const convplan* pl, u64* a) {
  const mctx* c = &pl->c;
  six_transpose(pl, a, 1);
  for (size_t r = 0; r < pl->n2; ++r) {
    dif(&pl->col, a + r * pl->n1);
    or_bit_rev_permute(a + r * pl->n1, pl->n1);
  }
  six_transpose(pl, a, 0);
  u64 seed = pl->xi;
  for (size_t i = 1; i < pl->n1; ++i) {
    u64* row = a + i * pl->n2;
    u64 f = seed;
    for (size_t j = 1; j < pl->n2; ++j) {
      row[j] = redc(c, row[j], f);
      f = redc(c, f, seed);
    }
    seed = redc(c, seed, pl->xi);
  }
  for (size_t r = 0; r < pl->n1; ++r) dif(&pl->row, a + r * pl->n2);
}

/* six_step_inverse, conv.cpp:89-104 with six_twiddle_inverse :57-70. */
static void six_inv(const convplan* pl, u64* a, u64 phi) {
  const mctx* c = &pl->c;
  for (size_t r = 0; r < pl->n1; ++r) dit(&pl->row, a + r * pl->n2);
  u64 seed = c->r;
  for (size_t i = 0; i < pl->n1; ++i) {
    u64* row = a + i * pl->n2;
    u64 f = phi;
    for (size_t j = 0; j < pl->n2; ++j) {
      row[j] = redc(c, row[j], f);
      f = redc(c, f, seed);
    }
    seed = redc(c, seed, pl->xi_inv);
  }
  six_transpose(pl, a, 1);
  for (size_t r = 0; r < pl->n2; ++r) {
    or_bit_rev_permute(a + r * pl->n1, pl->n1);
    dit(&pl->col, a + r * pl->n1);
  }
  six_transpose(pl, a, 0);
}

/* three_row_forward_columns + rows, conv.cpp:109-125, :149-156. */
static void three_fwd(const convplan* pl, u64* a) {
  const mctx* c = &pl->c;
  const u64 p = c->p;
  size_t cc = pl->n / 3;
  u64 *r0 = a, *r1 = a + cc, *r2 = a + 2 * cc;
  u64 g1 = c->r, g2 = c->r;
  for (size_t j = 0; j < cc; ++j) {
    u64 x = r0[j], y = r1[j], z = r2[j];
    u64 ya = redc(c, y, pl->lam), za = redc(c, z, pl->lam2);
    u64 yb = redc(c, y, pl->lam2), zb = redc(c, z, pl->lam);
    r0[j] = mod_add(mod_add(x, y, p), z, p);
    r1[j] = redc(c, mod_add(mod_add(x, ya, p), za, p), g1);
    r2[j] = redc(c, mod_add(mod_add(x, yb, p), zb, p), g2);
    g1 = redc(c, g1, pl->gamma);
    g2 = redc(c, g2, pl->gamma2);
  }
  for (int r = 0; r < 3; ++r) fwd_in_place(pl->rowplan, a + r * cc);
}

/* three_row_inverse + columns, conv.cpp:129-147, :158-166. */
static void three_inv(const convplan* pl, u64* a, u64 phi) {
  const mctx* c = &pl->c;
  const u64 p = c->p;
  size_t cc = pl->n / 3;
  for (int r = 0; r < 3; ++r) inv_in_place(pl->rowplan, a + r * cc, c->r);
  u64 *r0 = a, *r1 = a + cc, *r2 = a + 2 * cc;
  u64 f1 = phi, f2 = phi;
  for (size_t j = 0; j < cc; ++j) {
    u64 x = redc(c, r0[j], phi), y = redc(c, r1[j], f1), z = redc(c, r2[j], f2);
    u64 ya = redc(c, y, pl->lam_inv), za = redc(c, z, pl->lam2_inv);
    u64 yb = redc(c, y, pl->lam2_inv), zb = redc(c, z, pl->lam_inv);
    r0[j] = mod_add(mod_add(x, y, p), z, p);
    r1[j] = mod_add(mod_add(x, ya, p), za, p);
    r2[j] = mod_add(mod_add(x, yb, p), zb, p);
    f1 = redc(c, f1, pl->gamma_inv);
    f2 = redc(c, f2, pl->gamma2_inv);
  }
}

/* forward_in_place / inverse_in_place, conv.cpp:168-203. */
static void fwd_in_place(const convplan* pl, u64* a) {
  if (pl->shape == 0) dif(&pl->direct, a);
  else if (pl->shape == 1) six_fwd(pl, a);
  else three_fwd(pl, a);
}
static void inv_in_place(const convplan* pl, u64* a, u64 phi) {
  if (pl->shape == 0) {
    dit(&pl->direct, a);
    if (phi != pl->c.r)
      for (size_t i = 0; i < pl->n; ++i) a[i] = redc(&pl->c, a[i], phi);
  } else if (pl->shape == 1) {
    six_inv(pl, a, phi);
  } else {
    three_inv(pl, a, phi);
  }
}

int or_conv_plan_info(u64 p, size_t n, size_t thr, int* shape, u64* root, u64* psi, u64* psi_prime, size_t* n1,
                      size_t* n2) {
  convplan pl;
  int rc = conv_plan(p, n, thr, &pl);
  if (rc) return rc;
  *shape = pl.shape;
  *root = pl.root;
  *psi = pl.psi;
  *psi_prime = pl.psi_prime;
  *n1 = pl.n1;
  *n2 = pl.n2;
  conv_free(&pl);
  return 0;
}
int or_forward_transform(u64 p, size_t n, size_t thr, u64* a) { /* conv.cpp:273-276 */
  convplan pl;
  int rc = conv_plan(p, n, thr, &pl);
  if (rc) return rc;
  fwd_in_place(&pl, a);
  conv_free(&pl);
  return 0;
}
int or_inverse_transform(u64 p, size_t n, size_t thr, u64* a) { /* conv.cpp:278-281 */
  convplan pl;
  int rc = conv_plan(p, n, thr, &pl);
  if (rc) return rc;
  inv_in_place(&pl, a, pl.psi);
  conv_free(&pl);
  return 0;
}
int or_pointwise_product(u64 p, size_t n, u64* a, const u64* b) { /* conv.cpp:283-290, :205-208 */
  mctx c;
  int rc = make_ctx(p, &c);
  if (rc) return rc;
  for (size_t i = 0; i < n; ++i) a[i] = redc(&c, a[i], b[i]);
  return 0;
}
/* convolve_mod_p, conv.cpp:292-309. */
static int convolve(const convplan* pl, const u64* x, size_t nx, const u64* y, size_t ny, u64* out) {
  size_t n = pl->n;
  if (nx > n || ny > n) return fail(1, "convolve_mod_p: input longer than plan length");
  memset(out, 0, n * sizeof(u64));
  memcpy(out, x, nx * sizeof(u64));
  fwd_in_place(pl, out);
  if (x == y && nx == ny) {
    for (size_t i = 0; i < n; ++i) out[i] = redc(&pl->c, out[i], out[i]);
  } else {
    u64* fy = (u64*)calloc(n, sizeof(u64));
    memcpy(fy, y, ny * sizeof(u64));
    fwd_in_place(pl, fy);
    for (size_t i = 0; i < n; ++i) out[i] = redc(&pl->c, out[i], fy[i]);
    free(fy);
  }
  inv_in_place(pl, out, pl->psi_prime);
  return 0;
}
int or_convolve_mod_p(u64 p, size_t n, size_t thr, const u64* x, size_t nx, const u64* y, size_t ny, u64* out) {
  convplan pl;
  int rc = conv_plan(p, n, thr, &pl);
  if (rc) return rc;
  rc = convolve(&pl, x, nx, y, ny, out);
  conv_free(&pl);
  return rc;
}

/* ---------------- decimal layer (decimal.hpp / decimal.cpp) ---------------- */

static u64 pow10u(unsigned e) { u64 b = 1; while (e--) b *= 10; return b; } /* decimal.hpp:49-53 */

/* smallest_supported_length, decimal.cpp:54-76. */
int or_smallest_supported_length(size_t need, u64 p1, u64 p2, size_t* out) {
  if (!p1) { p1 = kP1; p2 = kP2; }
  unsigned v1 = (unsigned)__builtin_ctzll(p1 - 1), v2 = (unsigned)__builtin_ctzll(p2 - 1);
  int t1 = ((p1 - 1) >> v1) % 3 == 0, t2 = ((p2 - 1) >> v2) % 3 == 0;
  unsigned kmax = v1 < v2 ? v1 : v2;
  if (need < 2) need = 2;
  *out = 0;
  if (need > ((size_t)1 << 62)) return 0;
  size_t best = 0, two = 1;
  while (two < need) two <<= 1;
  if ((unsigned)__builtin_ctzll(two) <= kmax) best = two;
  if (t1 && t2) {
    size_t half = 1, q = (need + 2) / 3;
    while (half < q) half <<= 1;
    if ((unsigned)__builtin_ctzll(half) <= kmax && (best == 0 || 3 * half < best)) best = 3 * half;
  }
  *out = best;
  return 0;
}

/* select_base_and_length, decimal.cpp:78-100. */
int or_select_base_and_length(size_t dx, size_t dy, u64 p1, u64 p2, unsigned forced, unsigned* base_exp,
                              size_t* length) {
  if (!p1) { p1 = kP1; p2 = kP2; }
  if (dx < 1 || dy < 1) return fail(1, "select_base_and_length: digit counts must be >= 1");
  if (forced > 17) return fail(1, "select_base_and_length: unsupported forced base");
  u128 modulus = (u128)p1 * p2;
  unsigned lo = forced ? forced : 14, hi = forced ? forced : 17;
  for (unsigned be = hi; be >= lo; --be) {
    u64 top = pow10u(be) - 1;
    size_t lx = (dx + be - 1) / be, ly = (dy + be - 1) / be;
    size_t mn = lx < ly ? lx : ly;
    if ((u128)mn > (modulus - 1) / ((u128)top * top)) continue;
    size_t len;
    or_smallest_supported_length(lx + ly, p1, p2, &len);
    if (!len) return fail(2, "operands exceed the largest supported transform length");
    *base_exp = be;
    *length = len;
    return 0;
  }
  return fail(2, "operands violate the coefficient bound at every supported base");
}

/* pack, decimal.cpp:102-118: lambda digits per limb counted from the least-significant end. */
int or_pack(const char* s, size_t nd, unsigned be, u64* limbs, size_t cap, size_t* nl) {
  if (be < 1 || be > 17) return fail(1, "pack: unsupported base");
  size_t cnt = 0, end = nd;
  while (end > 0) {
    size_t begin = end > be ? end - be : 0;
    u64 limb = 0;
    for (size_t i = begin; i < end; ++i) limb = limb * 10 + (u64)(s[i] - '0');
    if (cnt >= cap) return fail(6, "pack: buffer too small");
    limbs[cnt++] = limb;
    end = begin;
  }
  *nl = cnt;
  return 0;
}

/* to_decimal, decimal.cpp:120-134. */
int or_to_decimal(const u64* limbs, size_t nl, unsigned be, char* out, size_t cap, size_t* len) {
  size_t top = nl;
  while (top > 1 && limbs[top - 1] == 0) --top;
  if (top == 0) {
    if (cap < 1) return fail(6, "to_decimal: buffer too small");
    out[0] = '0';
    *len = 1;
    return 0;
  }
  char buf[32];
  int l = snprintf(buf, sizeof buf, "%llu", (unsigned long long)limbs[top - 1]);
  size_t need = (size_t)l + (top - 1) * be;
  if (need > cap) return fail(6, "to_decimal: buffer too small");
  memcpy(out, buf, (size_t)l);
  size_t pos = (size_t)l;
  for (size_t i = top - 1; i-- > 0;) {
    u64 v = limbs[i];
    for (unsigned d = be; d-- > 0;) { out[pos + d] = (char)('0' + v % 10); v /= 10; }
    pos += be;
  }
  *len = pos;
  return 0;
}

/* make_crt_ctx / crt2, decimal.cpp:136-152. */
int or_crt2(u64 p1, u64 p2, u64 a1, u64 a2, u64* lo, u64* hi) {
  if (p1 >= p2) return fail(1, "make_crt_ctx: requires p1 < p2");
  mctx c2;
  int rc = make_ctx(p2, &c2);
  if (rc) return rc;
  u64 rt = mont_pow(&c2, to_mont(&c2, p1), p2 - 2);
  u64 diff = mod_sub(a2, a1, p2);
  u64 q = redc(&c2, rt, diff);
  u128 m = (u128)p1 * q + a1;
  *lo = (u64)m;
  *hi = (u64)(m >> 64);
  return 0;
}

/* recover_digits, decimal.cpp:154-189 (divmod_base restated as plain u128 division). */
int or_recover_digits(const u64* cf, size_t n, unsigned be, size_t min_limbs, u64* out, size_t cap,
                      size_t* nout) {
  if (be < 1 || be > 19) return fail(1, "recover_digits: base out of range");
  if (min_limbs < 1) return fail(1, "recover_digits: min_limbs must be >= 1");
  u128 B = pow10u(be), top = B - 1;
  u128 unit = top * top;
  u128 ccap = (u128)min_limbs <= ~(u128)0 / unit ? unit * min_limbs : ~(u128)0;
  u128 kcap = top * min_limbs;
  u128 carry = 0;
  size_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    u128 ci = ((u128)cf[2 * i + 1] << 64) | cf[2 * i];
    if (ci > ccap) return fail(3, "recover_digits: coefficient exceeds analytic bound (upstream corruption)");
    u128 v = carry + ci;
    if (k >= cap) return fail(6, "recover_digits: buffer too small");
    out[k++] = (u64)(v % B);
    carry = v / B;
    if (carry >= kcap) return fail(3, "recover_digits: carry exceeds analytic bound (upstream corruption)");
  }
  while (carry > 0) {
    if (k >= cap) return fail(6, "recover_digits: buffer too small");
    out[k++] = (u64)(carry % B);
    carry /= B;
  }
  if (k == 0) {
    if (cap < 1) return fail(6, "recover_digits: buffer too small");
    out[k++] = 0;
  }
  *nout = k;
  return 0;
}

static int valid_decimal(const char* s, size_t n) { /* DecimalNumber::parse, decimal.cpp:29-36 */
  if (n == 0) return fail(1, "decimal: empty string");
  for (size_t i = 0; i < n; ++i)
    if (s[i] < '0' || s[i] > '9') return fail(1, "decimal: non-digit character");
  if (n > 1 && s[0] == '0') return fail(1, "decimal: leading zero");
  return 0;
}

/* multiply, decimal.cpp:191-216. */
int or_multiply(const char* x, size_t nx, const char* y, size_t ny, char* out, size_t cap, size_t* out_len,
                unsigned forced, u64 p1, u64 p2) {
  int rc;
  if ((rc = valid_decimal(x, nx)) || (rc = valid_decimal(y, ny))) return rc;
  if (!p1) { p1 = kP1; p2 = kP2; }
  if ((nx == 1 && x[0] == '0') || (ny == 1 && y[0] == '0')) {
    if (cap < 1) return fail(6, "multiply: buffer too small");
    out[0] = '0';
    *out_len = 1;
    return 0;
  }
  unsigned be;
  size_t n;
  if ((rc = or_select_base_and_length(nx, ny, p1, p2, forced, &be, &n))) return rc;
  int squaring = x == y || (nx == ny && memcmp(x, y, nx) == 0);
  size_t lx = (nx + be - 1) / be, ly = (ny + be - 1) / be, got;
  u64* px = (u64*)malloc(lx * sizeof(u64));
  u64* py = (u64*)malloc(ly * sizeof(u64));
  or_pack(x, nx, be, px, lx, &got);
  or_pack(y, ny, be, py, ly, &got);
  u64* c1 = (u64*)malloc(n * sizeof(u64));
  u64* c2 = (u64*)malloc(n * sizeof(u64));
  u64* cf = (u64*)malloc(2 * n * sizeof(u64));
  u64* z = (u64*)malloc((n + 2) * sizeof(u64));
  const u64 ps[2] = {p1, p2};
  u64* cs[2] = {c1, c2};
  for (int k = 0; k < 2 && !rc; ++k) {
    convplan pl;
    if ((rc = conv_plan(ps[k], n, 0, &pl))) break;
    rc = convolve(&pl, px, lx, squaring ? px : py, squaring ? lx : ly, cs[k]);
    conv_free(&pl);
  }
  for (size_t i = 0; i < n && !rc; ++i) rc = or_crt2(p1, p2, c1[i], c2[i], &cf[2 * i], &cf[2 * i + 1]);
  size_t nz = 0;
  if (!rc) rc = or_recover_digits(cf, n, be, lx < ly ? lx : ly, z, n + 2, &nz);
  if (!rc) rc = or_to_decimal(z, nz, be, out, cap, out_len);
  free(px); free(py); free(c1); free(c2); free(cf); free(z);
  return rc;
}

/* ---------------- quadratic checkers (tests/oracle.cpp) ---------------- */

/* naive_dft, oracle.cpp:49-60. */
int or_naive_dft(const u64* x, size_t n, u64 root, u64 p, u64* out) {
  for (size_t k = 0; k < n; ++k) {
    u64 acc = 0, w = powmod(root, k, p), f = 1;
    for (size_t i = 0; i < n; ++i) {
      acc = (u64)(((u128)acc + (u128)x[i] * f) % p);
      f = mulmod(f, w, p);
    }
    out[k] = acc;
  }
  return 0;
}
/* naive_convolve, oracle.cpp:77-89. */
int or_naive_convolve(const u64* x, const u64* y, size_t n, u64 p, u64* out) {
  for (size_t k = 0; k < n; ++k) {
    u64 acc = 0;
    for (size_t i = 0; i < n; ++i) acc = (u64)(((u128)acc + (u128)x[i] * y[(k + n - i) % n]) % p);
    out[k] = acc;
  }
  return 0;
}
/* schoolbook_multiply, oracle.cpp:124-144 (base 10^9 limbs, 128-bit columns). */
int or_schoolbook_multiply(const char* x, size_t nx, const char* y, size_t ny, char* out, size_t cap,
                           size_t* out_len) {
  size_t la, lb, nz = 0;
  u64* a = (u64*)malloc(((nx + 8) / 9 + 1) * sizeof(u64));
  u64* b = (u64*)malloc(((ny + 8) / 9 + 1) * sizeof(u64));
  or_pack(x, nx, 9, a, nx, &la);
  or_pack(y, ny, 9, b, ny, &lb);
  u128* acc = (u128*)calloc(la + lb + 1, sizeof(u128));
  for (size_t i = 0; i < la; ++i)
    for (size_t j = 0; j < lb; ++j) acc[i + j] += (u128)a[i] * b[j];
  u64* z = (u64*)malloc((la + lb + 4) * sizeof(u64));
  u128 carry = 0;
  for (size_t k = 0; k < la + lb; ++k) {
    u128 cur = acc[k] + carry;
    z[nz++] = (u64)(cur % 1000000000u);
    carry = cur / 1000000000u;
  }
  while (carry) { z[nz++] = (u64)(carry % 1000000000u); carry /= 1000000000u; }
  int rc = or_to_decimal(z, nz, 9, out, cap, out_len);
  free(a); free(b); free(acc); free(z);
  return rc;
}

/* ---------------- size-independent fingerprints (SURVEY §8(c) fast checks) ---------------- */

/* The decimal value of s[0..n) modulo q (Horner over 18-digit chunks). Used to
 * check z == x y (mod q) for products too large for the quadratic oracle. */
u64 or_residue_mod(const char* s, size_t n, u64 q) {
  u64 acc = 0;
  size_t i = 0, head = n % 18;
  const u64 p18 = 1000000000000000000ull % q;
  if (head) {
    u64 v = 0;
    for (; i < head; ++i) v = v * 10 + (u64)(s[i] - '0');
    acc = v % q;
  }
  for (; i < n; i += 18) {
    u64 v = 0;
    for (size_t j = 0; j < 18; ++j) v = v * 10 + (u64)(s[i + j] - '0');
    acc = (u64)(((u128)acc * p18 + v % q) % q);
  }
  return acc;
}

/* Composed-reference oracle for products beyond the reference's cap:
 * acc (little-endian decimal digits 0..9, acc_len of them) += p * 10^shift, where p is
 * plen ASCII digits, most significant first. Exact, with carry propagation; returns 0, or
 * 1 if the sum does not fit acc. */
int or_add_shifted(unsigned char* acc, size_t acc_len, const char* p, size_t plen, size_t shift) {
  unsigned carry = 0;
  size_t i = 0;
  for (; i < plen; ++i) {
    const size_t k = shift + i;
    if (k >= acc_len) return 1;
    const unsigned v = acc[k] + (unsigned)(p[plen - 1 - i] - '0') + carry;
    acc[k] = (unsigned char)(v >= 10 ? v - 10 : v);
    carry = v >= 10;
  }
  for (size_t k = shift + i; carry; ++k) {
    if (k >= acc_len) return 1;
    const unsigned v = acc[k] + carry;
    acc[k] = (unsigned char)(v >= 10 ? v - 10 : v);
    carry = v >= 10;
  }
  return 0;
}

/* Carry pass of a carry-free digit accumulator: acc[k] (little-endian positions, sums of
 * digit columns, each < 2^16) -> the decimal string, most significant digit first,
 * written to out[0, n] (n + 1 bytes; the top byte absorbs the final carry; leading
 * zeros are left for the caller to strip). Returns 0, or 1 if the carry overflows. */
int or_carry_u16(const unsigned short* acc, size_t n, char* out) {
  unsigned long long carry = 0;
  for (size_t k = 0; k < n; ++k) {
    const unsigned long long v = acc[k] + carry;
    out[n - k] = (char)('0' + v % 10);
    carry = v / 10;
  }
  if (carry > 9) return 1;
  out[0] = (char)('0' + carry);
  return 0;
}

/* Residues of one digit string modulo nq primes q < 2^62 in a single pass (fingerprints
 * of 1e10-digit products); callers combine chunk residues as
 * r(ab) = r(a) 10^|b| + r(b). Reentrant (no shared state), so chunks run on threads. */
void or_residues_multi(const char* s, size_t n, const u64* qs, int nq, u64* out) {
  u64 p18[16];
  if (nq > 16) nq = 16;
  for (int k = 0; k < nq; ++k) {
    p18[k] = 1000000000000000000ull % qs[k];
    out[k] = 0;
  }
  size_t i = 0, head = n % 18;
  if (head) {
    u64 v = 0;
    for (; i < head; ++i) v = v * 10 + (u64)(s[i] - '0');
    for (int k = 0; k < nq; ++k) out[k] = v % qs[k];
  }
  for (; i < n; i += 18) {
    u64 v = 0;
    for (size_t j = 0; j < 18; ++j) v = v * 10 + (u64)(s[i + j] - '0');
    for (int k = 0; k < nq; ++k) out[k] = (u64)(((u128)out[k] * p18[k] + v) % qs[k]);
  }
}

/* ---------------- shared seeded generator ---------------- */

static u64 sm_mix(u64 z) { /* splitmix64 finalizer, reference bench.cpp:40-45 */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
#define GOLDEN 0x9e3779b97f4a7c15ull
void or_gen_digits(u64 seed, int mode, size_t n, char* out) {
  u64 key = sm_mix(seed + GOLDEN);
  for (size_t i = 0; i < n; ++i) {
    if (mode == 1) { out[i] = '9'; continue; }
    u64 v = sm_mix(key + (u64)(i + 1) * GOLDEN);
    out[i] = (char)('0' + (i == 0 ? 1 + v % 9 : v % 10));
  }
}
void or_gen_residues(u64 seed, size_t n, u64 p, u64* out) {
  u64 key = sm_mix(seed + GOLDEN);
  for (size_t i = 0; i < n; ++i) out[i] = sm_mix(key + (u64)(i + 1) * GOLDEN) % p;
}

/* build_plan_with_root (ntt.cpp:88-112) + dif_impl (ntt.cpp:29-50) for an explicit root:
 * the reference's hand examples use p = 17, n = 4, root = 4 (test_ntt.cpp:23-37, :81-88). */
int or_ntt_plan_root(u64 p, size_t n, u64 root, u64* fwd, u64* inv) {
  mctx c;
  nttplan pl;
  int rc = make_ctx(p, &c);
  if (rc || (rc = ntt_plan_root(&c, n, root, &pl))) return rc;
  if (n > 1) {
    memcpy(fwd, pl.fwd, (n - 1) * sizeof(u64));
    memcpy(inv, pl.inv, (n - 1) * sizeof(u64));
  }
  ntt_free(&pl);
  return 0;
}
int or_dif_forward_root(u64 p, size_t n, u64 root, u64* a) {
  mctx c;
  nttplan pl;
  int rc = make_ctx(p, &c);
  if (rc || (rc = ntt_plan_root(&c, n, root, &pl))) return rc;
  dif(&pl, a);
  ntt_free(&pl);
  return 0;
}
