// TEST INFRASTRUCTURE (oracle), not product code.
//
// extern "C" wrapper compiled together with the UNMODIFIED reference sources
// (/root/reference/proj/src/*.cpp, built by oracle/Makefile into
// oracle/_ref/libdecmul_ref.so). It exposes the reference's own hot-path API
// (decimal.hpp / conv.hpp / ntt.hpp / transpose.hpp / primes.hpp /
// montgomery.hpp) through plain pointers so Python tests, the golden-vector
// generator and bench.py's reference arm can call it with ctypes.
//
// Return codes: 0 ok, 1 std::invalid_argument, 2 decmul::OperandTooLarge,
// 3 std::runtime_error, 4 std::logic_error, 5 other, 6 output buffer too small.
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "decmul/conv.hpp"
#include "decmul/decimal.hpp"
#include "decmul/montgomery.hpp"
#include "decmul/ntt.hpp"
#include "decmul/primes.hpp"
#include "decmul/transpose.hpp"

using namespace decmul;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const OperandTooLarge& e) {
    g_err = e.what();
    return 2;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

AdjustStrategy strat(int s) {
  return s == 0 ? AdjustStrategy::kBitWizardry : AdjustStrategy::kConditionalSelect;
}

ConvPlan plan_for(Word p, std::size_t n, std::size_t thr) {
  return build_conv_plan(make_ctx(p), n, thr ? thr : kDefaultSixStepThreshold);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_production_primes(Word* p1, Word* p2) {
  const PrimePair& pr = production_primes();
  *p1 = pr.p1;
  *p2 = pr.p2;
}

int ref_is_prime(Word n) { return is_prime(n) ? 1 : 0; }

int ref_find_primes(unsigned w, unsigned n_min, unsigned ell, Word* out) {
  return guarded([&] {
    auto v = find_primes(w, n_min, ell);
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = v[i];
  });
}

int ref_make_ctx(Word p, Word* pp, Word* r, Word* r2) {
  return guarded([&] {
    MontCtx c = make_ctx(p);
    *pp = c.p_prime;
    *r = c.r_mod_p;
    *r2 = c.r2_mod_p;
  });
}

Word ref_redc(Word p, Word x, Word y) { return redc(make_ctx(p), x, y); }
Word ref_to_mont(Word p, Word x) { return to_mont(make_ctx(p), x); }
Word ref_from_mont(Word p, Word x) { return from_mont(make_ctx(p), x); }

int ref_primitive_root(Word p, Word n, Word* root_plain) {
  return guarded([&] {
    MontCtx c = make_ctx(p);
    *root_plain = from_mont(c, primitive_root_of_unity(c, n));
  });
}

int ref_smallest_supported_length(std::size_t need, std::size_t* out) {
  return guarded([&] { *out = smallest_supported_length(need, production_primes()); });
}

int ref_smallest_supported_length_pair(std::size_t need, Word p1, Word p2, std::size_t* out) {
  return guarded([&] { *out = smallest_supported_length(need, PrimePair{p1, p2}); });
}

int ref_select_base_and_length(std::size_t dx, std::size_t dy, unsigned forced, unsigned* base_exp,
                               std::size_t* length) {
  return guarded([&] {
    BasePlan bp = select_base_and_length(dx, dy, production_primes(), forced);
    *base_exp = bp.base_exp;
    *length = bp.length;
  });
}

int ref_select_base_and_length_pair(std::size_t dx, std::size_t dy, Word p1, Word p2, unsigned forced,
                                    unsigned* base_exp, std::size_t* length) {
  return guarded([&] {
    BasePlan bp = select_base_and_length(dx, dy, PrimePair{p1, p2}, forced);
    *base_exp = bp.base_exp;
    *length = bp.length;
  });
}

// shape: 0 direct, 1 six-step, 2 three-row. row_n: three-row row length.
int ref_conv_plan_info(Word p, std::size_t n, std::size_t thr, int* shape, Word* root, Word* psi,
                       Word* psi_prime, std::size_t* n1, std::size_t* n2, Word* col_root, Word* row_root) {
  return guarded([&] {
    ConvPlan pl = plan_for(p, n, thr);
    *shape = int(pl.shape);
    *root = pl.root;
    *psi = pl.psi;
    *psi_prime = pl.psi_prime;
    *n1 = pl.n1;
    *n2 = pl.n2;
    *col_root = 0;
    *row_root = 0;
    if (pl.shape == ConvShape::kSixStep) {
      *col_root = pl.col_kernel.root;
      *row_root = pl.row_kernel.root;
    } else if (pl.shape == ConvShape::kFourStepThreeRows) {
      *row_root = pl.row_plan->root;
    } else {
      *row_root = pl.direct.root;
    }
  });
}

int ref_forward_transform(Word p, std::size_t n, std::size_t thr, Word* a) {
  return guarded([&] {
    ConvPlan pl = plan_for(p, n, thr);
    forward_transform(pl, std::span<Word>(a, n));
  });
}

int ref_inverse_transform(Word p, std::size_t n, std::size_t thr, Word* a) {
  return guarded([&] {
    ConvPlan pl = plan_for(p, n, thr);
    inverse_transform(pl, std::span<Word>(a, n));
  });
}

int ref_pointwise_product(Word p, std::size_t n, Word* a, const Word* b) {
  return guarded([&] {
    ConvPlan pl = plan_for(p, n, 0);
    pointwise_product(pl, std::span<Word>(a, n), std::span<const Word>(b, n));
  });
}

int ref_convolve_mod_p(Word p, std::size_t n, std::size_t thr, const Word* x, std::size_t nx, const Word* y,
                       std::size_t ny, Word* out) {
  return guarded([&] {
    ConvPlan pl = plan_for(p, n, thr);
    std::vector<Word> r = convolve_mod_p(pl, std::span<const Word>(x, nx), std::span<const Word>(y, ny));
    std::memcpy(out, r.data(), n * sizeof(Word));
  });
}

int ref_ntt_plan(Word p, std::size_t n, Word* fwd, Word* inv, Word* root, Word* psi, Word* psi_prime) {
  return guarded([&] {
    NttPlan pl = build_plan(make_ctx(p), n);
    if (n > 1) {
      std::memcpy(fwd, pl.fwd.data(), (n - 1) * sizeof(Word));
      std::memcpy(inv, pl.inv.data(), (n - 1) * sizeof(Word));
    }
    *root = pl.root;
    *psi = pl.psi;
    *psi_prime = pl.psi_prime;
  });
}

int ref_dif_forward(Word p, std::size_t n, Word* a) {
  return guarded([&] { dif_forward_no_bitrev(build_plan(make_ctx(p), n), std::span<Word>(a, n)); });
}

int ref_dit_inverse(Word p, std::size_t n, Word* a) {
  return guarded([&] { dit_inverse_no_bitrev(build_plan(make_ctx(p), n), std::span<Word>(a, n)); });
}

void ref_bit_rev_permute(Word* a, std::size_t n) { bit_rev_permute(std::span<Word>(a, n)); }

void ref_transpose_square_sub(Word* a, std::size_t n, std::size_t stride) { transpose_square_sub(a, n, stride); }

void ref_transpose_n_x_2n(Word* a, std::size_t n) {
  std::vector<Word> s(2 * n);
  transpose_n_x_2n(a, n, s.data());
}

void ref_transpose_2n_x_n(Word* a, std::size_t n) {
  std::vector<Word> s(2 * n);
  transpose_2n_x_n(a, n, s.data());
}

int ref_pack(const char* digits, std::size_t nd, unsigned base_exp, Word* limbs, std::size_t cap,
             std::size_t* nlimbs) {
  return guarded([&] {
    PackedOperand po = pack(DecimalNumber::parse(std::string_view(digits, nd)), base_exp);
    *nlimbs = po.limbs.size();
    if (po.limbs.size() > cap) throw std::length_error("cap");
    std::memcpy(limbs, po.limbs.data(), po.limbs.size() * sizeof(Word));
  });
}

int ref_to_decimal(const Word* limbs, std::size_t nl, unsigned base_exp, char* out, std::size_t cap,
                   std::size_t* len) {
  return guarded([&] {
    PackedOperand po;
    po.base_exp = base_exp;
    po.limbs.assign(limbs, limbs + nl);
    std::string s = to_decimal(po);
    *len = s.size();
    if (s.size() > cap) throw std::length_error("cap");
    std::memcpy(out, s.data(), s.size());
  });
}

int ref_crt2(Word p1, Word p2, Word a1, Word a2, Word* lo, Word* hi) {
  return guarded([&] {
    CrtCtx c = make_crt_ctx(PrimePair{p1, p2}, AdjustStrategy::kConditionalSelect);
    WidePair w = crt2(c, a1, a2);
    *lo = w.lo;
    *hi = w.hi;
  });
}

int ref_divmod_base(Word base, Word lo, Word hi, Word* qlo, Word* qhi, Word* r) {
  return guarded([&] {
    DivByConstB d = make_div_by_const(base);
    DivModResult dm = divmod_base(d, WidePair{lo, hi});
    *qlo = dm.quotient.lo;
    *qhi = dm.quotient.hi;
    *r = dm.remainder;
  });
}

// coeffs: n pairs (lo, hi).
int ref_recover_digits(const Word* coeffs, std::size_t n, unsigned base_exp, std::size_t min_limbs, Word* out,
                       std::size_t cap, std::size_t* nout) {
  return guarded([&] {
    std::vector<WidePair> c(n);
    for (std::size_t i = 0; i < n; ++i) c[i] = WidePair{coeffs[2 * i], coeffs[2 * i + 1]};
    PackedOperand po = recover_digits(c, base_exp, min_limbs);
    *nout = po.limbs.size();
    if (po.limbs.size() > cap) throw std::length_error("cap");
    std::memcpy(out, po.limbs.data(), po.limbs.size() * sizeof(Word));
  });
}

// Full decmul::multiply from digit strings. alias != 0 passes the same object
// twice (the reference's &x == &y squaring path, decimal.cpp:198).
int ref_multiply(const char* x, std::size_t nx, const char* y, std::size_t ny, char* out, std::size_t cap,
                 std::size_t* out_len, unsigned forced_base_exp, int strategy, int alias) {
  return guarded([&] {
    DecimalNumber a = DecimalNumber::parse(std::string_view(x, nx));
    MultiplyOptions opt{strat(strategy), forced_base_exp};
    DecimalNumber z;
    if (alias) {
      z = multiply(a, a, opt);
    } else {
      DecimalNumber b = DecimalNumber::parse(std::string_view(y, ny));
      z = multiply(a, b, opt);
    }
    *out_len = z.digit_count();
    if (z.digit_count() > cap) throw std::length_error("cap");
    std::memcpy(out, z.text().data(), z.digit_count());
  });
}

// Batch of independent products on `threads` std::threads over disjoint
// pairs (multiply is reentrant, reference SPEC.md:588). Operands are packed
// back to back: x_off[i]..x_off[i]+nx[i] in xs; outputs at out_off[i] with
// out_cap[i] bytes; out_len[i] receives each product length.
int ref_multiply_batch(std::size_t count, const char* xs, const std::size_t* x_off, const std::size_t* nx,
                       const char* ys, const std::size_t* y_off, const std::size_t* ny, char* outs,
                       const std::size_t* out_off, const std::size_t* out_cap, std::size_t* out_len,
                       int threads) {
  if (threads < 1) threads = 1;
  std::vector<int> rc(threads, 0);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      for (std::size_t i = t; i < count; i += threads) {
        int r = ref_multiply(xs + x_off[i], nx[i], ys + y_off[i], ny[i], outs + out_off[i], out_cap[i],
                             &out_len[i], 0, 1, 0);
        if (r && !rc[t]) rc[t] = r;
      }
    });
  }
  for (auto& th : pool) th.join();
  for (int r : rc)
    if (r) return r;
  return 0;
}

// The reference bench_mul input stream (proj/src/bench.cpp:107-116):
// one std::mt19937_64(seed), x drawn then y, lead digit U{1..9}, rest U{0..9}.
void ref_bench_inputs(std::size_t digits, std::uint64_t seed, char* x, char* y) {
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> lead(1, 9), any(0, 9);
  for (char* s : {x, y}) {
    s[0] = char('0' + lead(rng));
    for (std::size_t i = 1; i < digits; ++i) s[i] = char('0' + any(rng));
  }
}

// oracle::random_residues (proj/tests/oracle.cpp:205-210) on a fresh mt19937_64(seed).
void ref_random_residues(std::uint64_t seed, std::size_t n, Word p, Word* out) {
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<Word> dist(0, p - 1);
  for (std::size_t i = 0; i < n; ++i) out[i] = dist(rng);
}

}  // extern "C"
