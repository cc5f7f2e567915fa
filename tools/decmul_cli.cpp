// `decmul` command line on the GPU path: the reference CLI's subcommands and output
// format (reference tools/main.cpp) backed by libdecmul_gpu.so.
//
//   decmul [--device N] [--adjust-strategy bitwise|cselect] mul A B
//   decmul mul --file PATH_A PATH_B
//   decmul bench mul --digits D [--digits D ...] [--iters K]
//   decmul bench modmul [--variant shoup|montgomery|solinas]
//   decmul selftest [--inject-fault]
//
// Errors print "error: <message>" and exit 1 (reference main.cpp:150-153).
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "decmul/decimal.hpp"
#include "decmul_gpu.h"

namespace {

[[noreturn]] void usage(const char* why) {
  throw std::invalid_argument(std::string(why) +
                              "\nusage: decmul [--device N] [--adjust-strategy bitwise|cselect] "
                              "{mul [--file] A B | bench mul --digits D... [--iters K] | "
                              "bench modmul [--variant shoup|montgomery|solinas] | selftest [--inject-fault]}");
}

// reference main.cpp:19-29
std::string read_operand_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  std::string s = ss.str();
  if (!s.empty() && s.back() == '\n') s.pop_back();
  if (!s.empty() && s.back() == '\r') s.pop_back();
  return s;
}

decmul_gpu_ctx* context() { return decmul::detail::context(); }

void check(int rc) {
  if (rc) decmul::detail::throw_for(rc, decmul_gpu_last_error(context()));
}

int cmd_mul(const std::string& a0, const std::string& b0, bool from_files) {
  const std::string a = from_files ? read_operand_file(a0) : a0;
  const std::string b = from_files ? read_operand_file(b0) : b0;
  const decmul::DecimalNumber z = decmul::multiply(decmul::DecimalNumber::parse(a), decmul::DecimalNumber::parse(b));
  std::fwrite(z.text().data(), 1, z.text().size(), stdout);
  std::fputc('\n', stdout);
  return 0;
}

// Operands drawn like the reference's bench_mul (bench.cpp:107-116): one mt19937_64(seed),
// x then y, leading digit uniform 1-9, the rest 0-9.
std::string bench_operand(std::mt19937_64& rng, std::size_t n) {
  std::uniform_int_distribution<int> lead(1, 9), any(0, 9);
  std::string s(n, '0');
  s[0] = char('0' + lead(rng));
  for (std::size_t i = 1; i < n; ++i) s[i] = char('0' + any(rng));
  return s;
}

int cmd_bench_mul(const std::vector<std::uint64_t>& sizes, std::uint64_t iters) {
  for (std::uint64_t digits : sizes) {
    if (digits == 0) usage("bench mul: --digits must be positive");
    const std::uint64_t k = iters ? iters : std::max<std::uint64_t>(1, 80000000ull / digits);  // auto_mul_iterations
    std::mt19937_64 rng(42);
    const std::string x = bench_operand(rng, digits), y = bench_operand(rng, digits);
    decmul_gpu_plan_info plan{};
    check(decmul_gpu_plan(context(), digits, digits, 0, &plan));
    std::string z(2 * digits, '\0');
    std::size_t len = 0;
    check(decmul_gpu_multiply(context(), x.data(), digits, y.data(), digits, &z[0], z.size(), &len, 0, 0));  // warm
    const auto t0 = std::chrono::steady_clock::now();
    for (std::uint64_t i = 0; i < k; ++i)
      check(decmul_gpu_multiply(context(), x.data(), digits, y.data(), digits, &z[0], z.size(), &len, 0, 0));
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("bench=mul digits=%" PRIu64 " iters=%" PRIu64 " base_exp=%u length=%zu seconds=%.6f"
                " seconds_per_mul=%.9f product_digits=%zu device=gpu\n",
                digits, k, plan.base_exp, plan.length, sec, sec / double(k), len);
  }
  return 0;
}

int cmd_bench_modmul(const std::string& variant) {
  int v;
  if (variant == "shoup")
    v = 0;
  else if (variant == "montgomery")
    v = 1;
  else if (variant == "solinas")
    v = 2;
  else
    throw std::invalid_argument("unknown variant: " + variant);
  double rate = 0;
  check(decmul_gpu_measure_modmul_rate(context(), v, &rate));
  std::printf("bench=modmul variant=%s device=gpu modmuls_per_second=%.6g ns_per_modmul=%.6f\n", variant.c_str(),
              rate, rate > 0 ? 1e9 / rate : 0.0);
  return 0;
}

int cmd_selftest(bool inject) {
  std::vector<char> report(1 << 14);
  int failures = 0;
  check(decmul_gpu_selftest(context(), inject ? 1 : 0, report.data(), report.size(), &failures));
  std::fputs(report.data(), stdout);
  return failures == 0 ? 0 : 1;
}

int run(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  std::size_t i = 0;
  while (i < args.size() && args[i].rfind("--", 0) == 0) {  // global options
    if (args[i] == "--device" && i + 1 < args.size()) {
      setenv("DECMUL_DEVICE", args[i + 1].c_str(), 1);
      i += 2;
    } else if (args[i] == "--adjust-strategy" && i + 1 < args.size()) {
      if (args[i + 1] != "bitwise" && args[i + 1] != "cselect") usage("--adjust-strategy: bitwise | cselect");
      i += 2;  // CPU codegen knob of the reference; products are identical (README.md:50-52)
    } else {
      usage(("unknown option " + args[i]).c_str());
    }
  }
  if (i >= args.size()) usage("a subcommand is required");
  const std::string cmd = args[i++];
  if (cmd == "mul") {
    bool files = false;
    std::vector<std::string> ops;
    for (; i < args.size(); ++i) {
      if (args[i] == "--file")
        files = true;
      else
        ops.push_back(args[i]);
    }
    if (ops.size() != 2) usage("mul: expected two operands");
    return cmd_mul(ops[0], ops[1], files);
  }
  if (cmd == "bench") {
    if (i >= args.size()) usage("bench: a subcommand is required");
    const std::string sub = args[i++];
    if (sub == "mul") {
      std::vector<std::uint64_t> sizes;
      std::uint64_t iters = 0;
      for (; i < args.size(); ++i) {
        if (args[i] == "--digits" && i + 1 < args.size())
          sizes.push_back(std::strtoull(args[++i].c_str(), nullptr, 10));
        else if (args[i] == "--iters" && i + 1 < args.size())
          iters = std::strtoull(args[++i].c_str(), nullptr, 10);
        else
          usage(("bench mul: unexpected " + args[i]).c_str());
      }
      if (sizes.empty()) usage("bench mul: --digits is required");
      return cmd_bench_mul(sizes, iters);
    }
    if (sub == "modmul") {
      std::string variant = "shoup";
      for (; i < args.size(); ++i) {
        if (args[i] == "--variant" && i + 1 < args.size())
          variant = args[++i];
        else
          usage(("bench modmul: unexpected " + args[i]).c_str());
      }
      return cmd_bench_modmul(variant);
    }
    usage(("bench: unknown subcommand " + sub).c_str());
  }
  if (cmd == "selftest") {
    bool inject = false;
    for (; i < args.size(); ++i) {
      if (args[i] == "--inject-fault")
        inject = true;
      else
        usage(("selftest: unexpected " + args[i]).c_str());
    }
    return cmd_selftest(inject);
  }
  usage(("unknown subcommand " + cmd).c_str());
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(argc, argv);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
