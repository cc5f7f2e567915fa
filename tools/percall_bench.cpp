// Per-call throughput of decmul::multiply from T host threads sharing the process-wide
// context (the reference's multiply is reentrant; its arm in bench.py runs 16
// calls at once): each thread multiplies its own pair of std::string operands K times through
// the drop-in header. Small products are coalesced by the library into batch launches
// (DECMUL_COALESCE=0 turns that off).
//   tools/percall_bench [--threads T] [--digits D] [--iters K]
// Output: key=value like the reference CLI's bench surfaces.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "decmul/decimal.hpp"

static std::string random_decimal(unsigned seed, size_t digits) {
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> lead(1, 9), any(0, 9);
  std::string s(digits, '0');
  s[0] = char('0' + lead(rng));
  for (size_t i = 1; i < digits; ++i) s[i] = char('0' + any(rng));
  return s;
}

int main(int argc, char** argv) {
  int threads = 16, iters = 2000;
  size_t digits = 10000;
  for (int i = 1; i + 1 < argc; i += 2) {
    if (!std::strcmp(argv[i], "--threads")) threads = std::atoi(argv[i + 1]);
    else if (!std::strcmp(argv[i], "--digits")) digits = std::strtoull(argv[i + 1], nullptr, 10);
    else if (!std::strcmp(argv[i], "--iters")) iters = std::atoi(argv[i + 1]);
  }
  using decmul::DecimalNumber;
  std::vector<DecimalNumber> xs, ys;
  for (int t = 0; t < threads; ++t) {
    xs.push_back(DecimalNumber::parse(random_decimal(2 * t, digits)));
    ys.push_back(DecimalNumber::parse(random_decimal(2 * t + 1, digits)));
  }
  std::vector<size_t> sum(threads, 0);
  auto run = [&](int k) {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        for (int i = 0; i < k; ++i) sum[t] += decmul::multiply(xs[t], ys[t]).digit_count();
      });
    for (auto& th : pool) th.join();
  };
  run(std::max(1, iters / 20));  // warm-up: context, plans, buffers
  const auto t0 = std::chrono::steady_clock::now();
  run(iters);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const double products = double(threads) * iters;
  std::printf("bench=percall threads=%d digits=%zu iters=%d seconds=%.4f products_per_s=%.1f digits_per_s=%.4e "
              "us_per_call=%.2f\n",
              threads, digits, iters, s, products / s, products * 2.0 * double(digits) / s, s / iters * 1e6);
  return sum[0] ? 0 : 1;
}
