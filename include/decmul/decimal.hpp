// decmul/decimal.hpp — drop-in replacement for the reference header
// proj/include/decmul/decimal.hpp, backed by the B200 library through the C ABI
// (include/decmul_gpu.h, libdecmul_gpu.so). Same names, signatures, argument
// meaning and exception types as the reference; header-only.
//
// Kept from the reference (decimal.hpp line numbers):
//   OperandTooLarge :20-22, DecimalNumber :26-38, PackedOperand :41-44,
//   kMinBaseExp/kMaxBaseExp :46-47, pow10 :49-53, BasePlan :61-64,
//   select_base_and_length :71-72, smallest_supported_length :76,
//   pack :79, to_decimal :82, MultiplyOptions :170-173, multiply :176-177.
// Not kept: max_digits_per_limb (paper table only, never called by multiply),
// the CPU division/CRT helpers (the device path does them inside the carry kernel).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../decmul_gpu.h"

namespace decmul {

using Word = std::uint64_t;

enum class AdjustStrategy { kBitWizardry, kConditionalSelect };  // reference words.hpp:29 (codegen knob only)

struct OperandTooLarge : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct PrimePair {  // reference primes.hpp:24-26
  Word p1, p2;
};
inline constexpr Word kProductionP1 = 9223372036015915009ull;
inline constexpr Word kProductionP2 = 9223372036166909953ull;
inline const PrimePair& production_primes() {
  static const PrimePair pair{kProductionP1, kProductionP2};
  return pair;
}

namespace detail {

[[noreturn]] inline void throw_for(int rc, const char* msg) {
  const std::string m = msg ? msg : "decmul_gpu error";
  switch (rc) {
    case DECMUL_EINVAL: throw std::invalid_argument(m);
    case DECMUL_ETOOLARGE: throw OperandTooLarge(m);
    case DECMUL_ELOGIC: throw std::logic_error(m);
    case DECMUL_ENOMEM: throw std::bad_alloc();
    case DECMUL_ESPACE: throw std::length_error(m);
    default: throw std::runtime_error(m);
  }
}

// Process-wide context over every visible GPU (decmul_gpu_create_multi: large products shard,
// batches fan out), or only the device named by DECMUL_DEVICE.
inline decmul_gpu_ctx* context() {
  static std::once_flag once;
  static decmul_gpu_ctx* ctx = nullptr;
  static int rc = 0;
  std::call_once(once, [] {
    if (const char* d = std::getenv("DECMUL_DEVICE")) {
      rc = decmul_gpu_create(&ctx, std::atoi(d));
      return;
    }
    int n = 0;
    rc = decmul_gpu_device_count(&n);
    if (rc) return;
    std::vector<int> devs;
    for (int i = 0; i < n; ++i) devs.push_back(i);
    if (devs.empty()) devs.push_back(0);  // no GPU: creation fails loudly (DECMUL_ECUDA)
    rc = decmul_gpu_create_multi(&ctx, devs.data(), int(devs.size()));
  });
  if (rc) throw_for(rc, decmul_gpu_last_error(nullptr));
  return ctx;
}

inline void check(int rc, decmul_gpu_ctx* ctx) {
  if (rc) throw_for(rc, decmul_gpu_last_error(ctx));
}

}  // namespace detail

// Non-negative integer as a canonical ASCII digit string (reference decimal.hpp:26-38).
class DecimalNumber {
 public:
  DecimalNumber() = default;
  static DecimalNumber parse(std::string_view text) {  // reference decimal.cpp:29-36
    if (text.empty()) throw std::invalid_argument("decimal: empty string");
    for (char ch : text)
      if (ch < '0' || ch > '9') throw std::invalid_argument("decimal: non-digit character");
    if (text.size() > 1 && text.front() == '0') throw std::invalid_argument("decimal: leading zero");
    return DecimalNumber(std::string(text));
  }
  const std::string& text() const { return text_; }
  std::size_t digit_count() const { return text_.size(); }
  bool is_zero() const { return text_ == "0"; }

 private:
  explicit DecimalNumber(std::string t) : text_(std::move(t)) {}
  std::string text_ = "0";
  friend DecimalNumber from_device_result(std::string t);
};

// Device-produced digits are canonical by construction: no re-validation
// (the reference re-parses its own output, decimal.cpp:215).
inline DecimalNumber from_device_result(std::string t) { return DecimalNumber(std::move(t)); }

struct PackedOperand {
  unsigned base_exp = 0;
  std::vector<Word> limbs;
};

inline constexpr unsigned kMinBaseExp = 14;
inline constexpr unsigned kMaxBaseExp = 17;

constexpr Word pow10(unsigned e) {
  Word b = 1;
  for (unsigned i = 0; i < e; ++i) b *= 10;
  return b;
}

struct BasePlan {
  unsigned base_exp = 0;
  std::size_t length = 0;
};

inline BasePlan select_base_and_length(std::size_t n_digits_x, std::size_t n_digits_y, const PrimePair& pair,
                                       unsigned forced_base_exp = 0) {
  BasePlan bp;
  const int rc = decmul_gpu_select_base_and_length(n_digits_x, n_digits_y, pair.p1, pair.p2, forced_base_exp,
                                                   &bp.base_exp, &bp.length);
  if (rc) detail::throw_for(rc, decmul_gpu_last_error(nullptr));
  return bp;
}

inline std::size_t smallest_supported_length(std::size_t need, const PrimePair& pair) {
  std::size_t n = 0;
  const int rc = decmul_gpu_smallest_supported_length(need, pair.p1, pair.p2, &n);
  if (rc) detail::throw_for(rc, decmul_gpu_last_error(nullptr));
  return n;
}

inline PackedOperand pack(const DecimalNumber& x, unsigned base_exp) {
  if (base_exp < 1 || base_exp > kMaxBaseExp) throw std::invalid_argument("pack: unsupported base");
  PackedOperand out;
  out.base_exp = base_exp;
  out.limbs.resize((x.digit_count() + base_exp - 1) / base_exp);
  std::size_t n = 0;
  decmul_gpu_ctx* ctx = detail::context();
  detail::check(decmul_gpu_pack(ctx, x.text().data(), x.digit_count(), base_exp, out.limbs.data(), out.limbs.size(),
                                &n),
                ctx);
  out.limbs.resize(n);
  return out;
}

inline std::string to_decimal(const PackedOperand& x) {  // reference decimal.cpp:120-134 (host formatting)
  std::size_t top = x.limbs.size();
  while (top > 1 && x.limbs[top - 1] == 0) --top;
  if (top == 0) return "0";
  std::string out = std::to_string(x.limbs[top - 1]);
  for (std::size_t i = top - 1; i-- > 0;) {
    std::string part = std::to_string(x.limbs[i]);
    out.append(x.base_exp - part.size(), '0');
    out += part;
  }
  return out;
}

struct MultiplyOptions {
  AdjustStrategy strategy = AdjustStrategy::kConditionalSelect;  // accepted; products identical under both
  unsigned forced_base_exp = 0;
  // Extension (last, so the reference's initialisers still compile): the prime pair of the
  // planner, which the reference's multiply pins to production_primes() (decimal.cpp:194).
  // {0, 0}: the reference pair, or the large pair beyond its 3 * 2^24 cap.
  PrimePair primes{0, 0};
};

// Exact decimal product on the GPU; x and y may alias (squaring saves one transform).
inline DecimalNumber multiply(const DecimalNumber& x, const DecimalNumber& y, const MultiplyOptions& opt = {}) {
  if (x.is_zero() || y.is_zero()) return DecimalNumber();
  decmul_gpu_ctx* ctx = detail::context();
  std::string out(x.digit_count() + y.digit_count(), '\0');
  std::size_t n = 0;
  const decmul_gpu_multiply_options o{opt.forced_base_exp, opt.primes.p1, opt.primes.p2, &x == &y ? 1 : 0};
  detail::check(decmul_gpu_multiply_ex(ctx, x.text().data(), x.digit_count(), y.text().data(), y.digit_count(),
                                       out.data(), out.size(), &n, &o),
                ctx);
  out.resize(n);
  return from_device_result(std::move(out));
}

}  // namespace decmul
