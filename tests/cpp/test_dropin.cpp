// Drop-in C++ API test: the reference's own test cases (proj/tests/test_decimal.cpp,
// test_conv.cpp, test_transpose.cpp) written against include/decmul/*.hpp, which
// routes every call to libdecmul_gpu.so. Checker: the oracle's C restatement
// (oracle/decmul_oracle.h). Run by tests/test_gpu_cpp.py on a GPU box.
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "../../include/decmul/conv.hpp"
#include "../../include/decmul/decimal.hpp"
#include "../../include/decmul/transpose.hpp"
#include "../../oracle/decmul_oracle.h"

using namespace decmul;

static int checks = 0, failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++checks;                                                              \
    if (!(cond)) {                                                         \
      ++failures;                                                          \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                           \
  do {                                                                     \
    bool thrown_ = false;                                                  \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const T&) {                                                   \
      thrown_ = true;                                                      \
    } catch (...) {                                                        \
    }                                                                      \
    CHECK(thrown_);                                                        \
  } while (0)

static std::string mul(const std::string& a, const std::string& b) {
  return multiply(DecimalNumber::parse(a), DecimalNumber::parse(b)).text();
}

static std::string school(const std::string& a, const std::string& b) {
  std::string out(a.size() + b.size() + 1, '\0');
  size_t n = 0;
  or_schoolbook_multiply(a.data(), a.size(), b.data(), b.size(), out.data(), out.size(), &n);
  out.resize(n);
  return out;
}

static std::string random_decimal(std::mt19937_64& rng, size_t digits) {  // reference oracle.cpp:196-203
  std::uniform_int_distribution<int> lead(1, 9), any(0, 9);
  std::string s(digits, '0');
  s[0] = char('0' + lead(rng));
  for (size_t i = 1; i < digits; ++i) s[i] = char('0' + any(rng));
  return s;
}

static std::string all_nines_square(size_t n) {
  return std::string(n - 1, '9') + "8" + std::string(n - 1, '0') + "1";
}

int main() {
  // test_decimal.cpp:272-291 (known answers)
  CHECK(mul("12", "34") == "408");
  CHECK(mul("21", "43") == "903");
  CHECK(mul("0", "999999") == "0");
  CHECK(mul("999999", "0") == "0");
  CHECK(mul("1", "1") == "1");
  CHECK(mul("1", "123456789") == "123456789");
  CHECK(mul("10", "10") == "100");
  CHECK(mul("123456789123456789", "987654321987654321") == "121932631356500531347203169112635269");
  for (size_t n : {1, 2, 17, 18, 100, 1000}) {
    const std::string nines(n, '9');
    CHECK(mul(nines, nines) == all_nines_square(n));
  }
  // parse errors (test_decimal.cpp:18-32)
  CHECK_THROWS_AS(DecimalNumber::parse(""), std::invalid_argument);
  CHECK_THROWS_AS(DecimalNumber::parse("01"), std::invalid_argument);
  CHECK_THROWS_AS(DecimalNumber::parse("1a"), std::invalid_argument);
  // base selection (test_decimal.cpp:91-127)
  const PrimePair& pair = production_primes();
  CHECK(select_base_and_length(1, 1, pair).base_exp == 17);
  CHECK(select_base_and_length(1, 1, pair).length == 2);
  CHECK(select_base_and_length(35, 35, pair).length == 6);
  CHECK(select_base_and_length(144619, 144619, pair).base_exp == 17);
  CHECK(select_base_and_length(144620, 144620, pair).base_exp == 16);
  CHECK(select_base_and_length(100000000, 17, pair).base_exp == 17);
  CHECK_THROWS_AS(select_base_and_length(1, 1, pair, 18), std::invalid_argument);
  CHECK_THROWS_AS(select_base_and_length(3000000, 3000000, pair, 17), OperandTooLarge);
  CHECK_THROWS_AS(select_base_and_length(400000000, 400000000, pair), OperandTooLarge);
  CHECK(smallest_supported_length((size_t(3) << 24) + 1, pair) == 0);
  // pack / to_decimal (test_decimal.cpp:129-154)
  CHECK(pack(DecimalNumber::parse("12345"), 14).limbs == std::vector<Word>{12345});
  CHECK((pack(DecimalNumber::parse("100000000000000"), 14).limbs == std::vector<Word>{0, 1}));
  const std::string nines35(35, '9');
  CHECK((pack(DecimalNumber::parse(nines35), 17).limbs ==
         std::vector<Word>{99999999999999999ull, 99999999999999999ull, 9}));
  CHECK(to_decimal(pack(DecimalNumber::parse(nines35), 17)) == nines35);
  // random products vs the quadratic oracle (test_decimal.cpp:293-314)
  std::mt19937_64 rng(127);
  for (int i = 0; i < 200; ++i) {
    const std::string a = random_decimal(rng, 1 + rng() % 300), b = random_decimal(rng, 1 + rng() % 300);
    CHECK(mul(a, b) == school(a, b));
  }
  for (size_t d : {997, 2000, 5000}) {
    const std::string a = random_decimal(rng, d), b = random_decimal(rng, d - 1);
    CHECK(mul(a, b) == school(a, b));
  }
  // squaring: aliased and equal text (test_decimal.cpp:316-326)
  for (size_t d : {1, 40, 1234}) {
    const std::string s = random_decimal(rng, d);
    const DecimalNumber x = DecimalNumber::parse(s), y = DecimalNumber::parse(s);
    CHECK(multiply(x, x).text() == school(s, s));
    CHECK(multiply(x, y).text() == school(s, s));
  }
  // every base (test_decimal.cpp:328-340)
  {
    const std::string a = random_decimal(rng, 4211), b = random_decimal(rng, 3999);
    const std::string expect = school(a, b);
    for (unsigned be : {0u, 14u, 15u, 16u, 17u})
      CHECK(multiply(DecimalNumber::parse(a), DecimalNumber::parse(b), {AdjustStrategy::kBitWizardry, be}).text() ==
            expect);
  }
  // convolution hooks (test_conv.cpp:131-148, 198-214)
  for (Word p : {kProductionP1, kProductionP2}) {
    for (size_t n : {1, 2, 3, 4, 6, 8, 12, 16, 24, 48, 64, 192}) {
      std::vector<Word> x(n), y(n), want(n);
      or_gen_residues(n, n, p, x.data());
      or_gen_residues(n + 1, n, p, y.data());
      or_naive_convolve(x.data(), y.data(), n, p, want.data());
      CHECK(convolve_mod_p(*conv_plan_for(p, n), x, y) == want);
      std::vector<Word> a = x, r = x;
      forward_transform(*conv_plan_for(p, n), a);
      or_forward_transform(p, n, 0, r.data());
      CHECK(a == r);
      inverse_transform(*conv_plan_for(p, n), a);
      CHECK(a == x);
    }
  }
  // non-default plans (test_conv.cpp:183-196 "all shapes agree", selftest.cpp:109-118 forced shapes)
  for (Word p : {kProductionP1, kProductionP2}) {
    const MontCtx c = make_ctx(p);
    for (size_t n : {size_t(64), size_t(96), size_t(192)}) {
      std::vector<Word> x(n), y(n);
      or_gen_residues(n + 7, n, p, x.data());
      or_gen_residues(n + 8, n, p, y.data());
      const ConvPlan direct = build_conv_plan(c, n);
      CHECK(direct.shape == (n % 3 == 0 ? ConvShape::kFourStepThreeRows : ConvShape::kDirect));
      const std::vector<Word> ref = convolve_mod_p(direct, x, y);
      for (size_t thr : {size_t(32), size_t(8), size_t(4), size_t(2)}) {
        const ConvPlan alt = build_conv_plan(c, n, thr);
        if (n % 3) CHECK(alt.shape == ConvShape::kSixStep && alt.n1 * alt.n2 == n);
        CHECK(alt.root == direct.root);
        CHECK(convolve_mod_p(alt, x, y) == ref);
        std::vector<Word> a = x, r = x;
        forward_transform(alt, a);
        or_forward_transform(p, n, thr, r.data());
        CHECK(a == r);
        inverse_transform(alt, a);
        CHECK(a == x);
      }
    }
    CHECK_THROWS_AS(build_conv_plan(c, 5), std::invalid_argument);
    CHECK_THROWS_AS(build_conv_plan(c, size_t(1) << 40), std::invalid_argument);
  }
  // transposes (test_transpose.cpp:93-129)
  {
    std::vector<Word> a{1, 2, 3, 4, 5, 6, 7, 8};
    transpose_n_x_2n(a.data(), 2, nullptr);
    CHECK((a == std::vector<Word>{1, 5, 2, 6, 3, 7, 4, 8}));
    std::vector<Word> b{1, 2, 3, 4, 5, 6, 7, 8};
    transpose_2n_x_n(b.data(), 2, nullptr);
    CHECK((b == std::vector<Word>{1, 3, 5, 7, 2, 4, 6, 8}));
    for (size_t n = 1; n <= 40; n += 13) {
      std::vector<Word> m(n * 2 * n), want;
      for (size_t i = 0; i < m.size(); ++i) m[i] = rng();
      want = m;
      or_transpose_n_x_2n(want.data(), n);
      std::vector<Word> got = m;
      transpose_n_x_2n(got.data(), n, nullptr);
      CHECK(got == want);
      transpose_2n_x_n(got.data(), n, nullptr);
      CHECK(got == m);
    }
  }
  std::printf("suite=dropin checks=%d failures=%d\n", checks, failures);
  return failures ? 1 : 0;
}
