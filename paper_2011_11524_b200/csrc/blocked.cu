// Block convolution: decmul::multiply for operands past the largest single transform
// (SURVEY §7 D1 fallback; the reference throws OperandTooLarge, decimal.cpp:94-96).
//
// x = sum_i X_i 10^(K i), y = sum_j Y_j 10^(K j) with decimal blocks of K digits counted from the
// least significant end; z = sum X_i Y_j 10^(K (i + j)). Every block product X_i Y_j is one
// ordinary device product (any engine of the context: the pairs fan out over the devices, one
// host thread each), and is added at digit offset K (i + j) into a little-endian host
// accumulator of nx + ny + 1 digits by a multithreaded ripple-carry add (chunk carries fixed up
// afterwards). Blocks are stripped of leading zeros (legal inside an operand) and all-zero
// blocks are skipped. The whole operands are validated first, with the reference's messages.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "multi.hpp"

namespace dmg {

namespace {

// Block [begin, end) of an operand text (block i from the least significant end).
void block_span(std::size_t n, std::size_t K, std::size_t i, std::size_t& begin, std::size_t& end) {
  end = n - std::min(n, i * K);
  begin = end > K ? end - K : 0;
}

// acc[off + t] += p[len - 1 - t] for t < len, carries propagated into acc (which has room):
// T threads add contiguous digit ranges, then the range carries ripple forward.
void add_shifted(unsigned char* acc, std::size_t acc_len, const char* p, std::size_t len, std::size_t off) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const std::size_t T = std::min<std::size_t>(std::min<std::size_t>(hw, 32), std::max<std::size_t>(1, len >> 22));
  std::vector<unsigned char> carry(T, 0);
  auto work = [&](std::size_t q) {
    const std::size_t b = len * q / T, e = len * (q + 1) / T;
    unsigned c = 0;
    for (std::size_t t = b; t < e; ++t) {
      unsigned v = acc[off + t] + unsigned(p[len - 1 - t] - '0') + c;
      c = v >= 10;
      acc[off + t] = (unsigned char)(c ? v - 10 : v);
    }
    carry[q] = (unsigned char)c;
  };
  if (T == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (std::size_t q = 0; q < T; ++q) th.emplace_back(work, q);
    for (auto& t : th) t.join();
  }
  for (std::size_t q = 0; q < T; ++q) {  // carry out of range q enters at the start of range q + 1
    std::size_t pos = off + len * (q + 1) / T;
    for (unsigned c = carry[q]; c && pos < acc_len; ++pos) {
      const unsigned v = acc[pos] + c;
      c = v >= 10;
      acc[pos] = (unsigned char)(c ? v - 10 : v);
    }
  }
}

}  // namespace

// Block size for decmul::multiply on host strings: 0 = one ordinary product. DECMUL_BLOCK_DIGITS
// (test knob) forces blocks of that many digits whenever an operand is longer.
std::size_t MultiEngine::block_digits(std::size_t nx, std::size_t ny, unsigned forced) const {
  if (const char* e = std::getenv("DECMUL_BLOCK_DIGITS")) {
    const std::size_t k = std::strtoull(e, nullptr, 10);
    if (k && std::max(nx, ny) > k) return k;
  }
  try {
    choose_pair(nx, ny, forced, true);
    return 0;
  } catch (const OperandTooLarge&) {
    return kBlockDigits;
  }
}

std::size_t MultiEngine::blocked_multiply(const char* x, std::size_t nx, const char* y, std::size_t ny, char* out,
                                          std::size_t cap, unsigned forced, std::size_t K) {
  // DecimalNumber::parse of both operands (decimal.cpp:29-36), with the reference's messages
  for (const auto& [d, n] : {std::pair<const char*, std::size_t>{x, nx}, {y, ny}}) {
    for (std::size_t i = 0; i < n; ++i)
      if (d[i] < '0' || d[i] > '9') throw std::invalid_argument("decimal: non-digit character");
    if (n > 1 && d[0] == '0') throw std::invalid_argument("decimal: leading zero");
  }
  if ((nx == 1 && x[0] == '0') || (ny == 1 && y[0] == '0')) {  // zero short-circuit (decimal.cpp:193)
    if (cap < 1) throw std::length_error("multiply: output buffer too small");
    out[0] = '0';
    return 1;
  }
  if (cap < nx + ny) throw std::length_error("multiply: output buffer too small");
  const std::size_t bx = (nx + K - 1) / K, by = (ny + K - 1) / K;
  std::vector<std::pair<std::size_t, std::size_t>> pairs;
  for (std::size_t i = 0; i < bx; ++i)
    for (std::size_t j = 0; j < by; ++j) pairs.push_back({i, j});
  const std::size_t acc_len = nx + ny + 1;
  std::vector<unsigned char> acc(acc_len, 0);
  std::mutex mu;  // one add into the accumulator at a time
  fan_out(pairs.size(), [&](Engine& e, std::size_t b, std::size_t end) {
    std::vector<char> prod(2 * K);
    for (std::size_t t = b; t < end; ++t) {
      const auto [i, j] = pairs[t];
      std::size_t xb, xe, yb, ye;
      block_span(nx, K, i, xb, xe);
      block_span(ny, K, j, yb, ye);
      while (xb + 1 < xe && x[xb] == '0') ++xb;  // leading zeros inside the operand
      while (yb + 1 < ye && y[yb] == '0') ++yb;
      if ((xe - xb == 1 && x[xb] == '0') || (ye - yb == 1 && y[yb] == '0')) continue;  // a zero block
      const std::size_t len = e.multiply_host(x + xb, xe - xb, y + yb, ye - yb, prod.data(), prod.size(), forced,
                                              false);
      std::lock_guard<std::mutex> lk(mu);
      add_shifted(acc.data(), acc_len, prod.data(), len, K * (i + j));
    }
  });
  std::size_t n = acc_len;
  while (n > 1 && acc[n - 1] == 0) --n;
  for (std::size_t t = 0; t < n; ++t) out[t] = char('0' + acc[n - 1 - t]);
  return n;
}

}  // namespace dmg
