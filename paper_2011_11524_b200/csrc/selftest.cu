// GPU self-test: the reference's run_selftest (selftest.cpp:79-219) restated for the
// device path. Every suite runs the sm_100a code the products use — the field kernels
// below call the same modarith.cuh / carry.cuh routines as the transforms and the
// carry, and the transform, convolution, recovery and product suites go through the
// Engine's own entry points — and checks the results on the host with 128-bit
// arithmetic, a direct O(n^2) convolution and a schoolbook product.
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "carry.cuh"
#include "engine.hpp"

namespace dmg {

namespace {

// out[5 i + 0..4] = Shoup(x w), REDC(x y), x + y, x - y (mod p), and the Goldilocks
// Solinas product x y mod (2^64 - 2^32 + 1) of the benchmark variant
__global__ void k_st_field(const u64* x, const u64* y, const TwPair* w, u64* out, unsigned n, u64 p, u64 pp) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[5 * i + 0] = shoup_mul(x[i], w[i], p);
  out[5 * i + 1] = mont_mul(x[i], y[i], p, pp);
  out[5 * i + 2] = mod_add(x[i], y[i], p);
  out[5 * i + 3] = mod_sub(x[i], y[i], p);
  out[5 * i + 4] = solinas_mul(x[i] | (y[i] << 62), ~y[i]);  // full 64-bit operands
}

// (a1, a2) -> the 128-bit CRT value (reference crt2, decimal.cpp:147-152)
__global__ void k_st_crt(const u64* a1, const u64* a2, u64* out, unsigned n, u64 p1, u64 p2, u64 p2p, u64 rt) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  crt2(a1[i], a2[i], p1, p2, p2p, rt, out[2 * i], out[2 * i + 1]);
}

// c (< 2^126) -> base-B digits (d0, d1, d2) by the carry's split3, and the reference's
// divmod_base quotient/remainder (decimal.hpp:123-146)
__global__ void k_st_div(const u64* lo, const u64* hi, u64* out, unsigned n, DivB d) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  u64 d0, d1, d2, qlo, qhi;
  split3(d, lo[i], hi[i], d0, d1, d2);
  const u64 r = divmod_base(d, lo[i], hi[i], qlo, qhi);
  out[6 * i + 0] = d0;
  out[6 * i + 1] = d1;
  out[6 * i + 2] = d2;
  out[6 * i + 3] = r;
  out[6 * i + 4] = qlo;
  out[6 * i + 5] = qhi;
}

struct Suite {
  const char* name;
  int checks = 0, failures = 0;
  void expect(bool ok) {
    ++checks;
    if (!ok) ++failures;
  }
  int report(std::string& out) const {
    char line[160];
    std::snprintf(line, sizeof line, "suite=%s checks=%d failures=%d\n", name, checks, failures);
    out += line;
    return failures;
  }
};

template <class T>
T* to_device(const std::vector<T>& v) {
  T* d = nullptr;
  cuda_check(cudaMalloc(&d, std::max<std::size_t>(v.size(), 1) * sizeof(T)), "selftest alloc");
  cuda_check(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "selftest h2d");
  return d;
}
template <class T>
std::vector<T> to_host(const T* d, std::size_t n) {
  std::vector<T> v(n);
  cuda_check(cudaMemcpy(v.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost), "selftest d2h");
  return v;
}

std::vector<u64> random_residues(std::mt19937_64& rng, std::size_t n, u64 p) {
  std::uniform_int_distribution<u64> dist(0, p - 1);
  std::vector<u64> v(n);
  for (u64& w : v) w = dist(rng);
  return v;
}

// Direct double-loop cyclic convolution (reference selftest.cpp:38-47).
std::vector<u64> direct_cyclic(const std::vector<u64>& x, const std::vector<u64>& y, u64 p) {
  const std::size_t n = x.size();
  std::vector<u64> out(n, 0);
  for (std::size_t k = 0; k < n; ++k) {
    u128 sum = 0;
    for (std::size_t i = 0; i < n; ++i) sum += u128(x[i]) * y[(k + n - i) % n] % p;
    out[k] = u64(sum % p);
  }
  return out;
}

// Digit-string schoolbook product (reference selftest.cpp:50-68).
std::string schoolbook(const std::string& a, const std::string& b) {
  if (a == "0" || b == "0") return "0";
  std::vector<unsigned> acc(a.size() + b.size(), 0);
  for (std::size_t i = 0; i < a.size(); ++i)
    for (std::size_t j = 0; j < b.size(); ++j) acc[i + j + 1] += unsigned(a[i] - '0') * unsigned(b[j] - '0');
  for (std::size_t k = acc.size(); k-- > 1;) {
    acc[k - 1] += acc[k] / 10;
    acc[k] %= 10;
  }
  std::string s;
  std::size_t i = 0;
  while (i + 1 < acc.size() && acc[i] == 0) ++i;
  for (; i < acc.size(); ++i) s += char('0' + acc[i]);
  return s;
}

std::string random_decimal(std::mt19937_64& rng, std::size_t len) {
  std::uniform_int_distribution<int> lead(1, 9), any(0, 9);
  std::string s(len, '0');
  s[0] = char('0' + lead(rng));
  for (std::size_t i = 1; i < len; ++i) s[i] = char('0' + any(rng));
  return s;
}

u64 residue(const std::string& s, u64 q) {
  u128 r = 0;
  for (char c : s) r = (r * 10 + unsigned(c - '0')) % q;
  return u64(r);
}

}  // namespace

int Engine::selftest(bool inject_fault, std::string& out) {
  int total = 0;
  std::mt19937_64 rng(0xdecu);
  const u64 primes[4] = {kP1, kP2, kQ1, kQ2};

  {
    Suite s{"field_identities"};
    const unsigned n = 200;
    for (u64 p : primes) {
      HostField F(p);
      std::vector<u64> x = random_residues(rng, n, p), y = random_residues(rng, n, p);
      std::vector<TwPair> w(n);
      for (auto& t : w) {
        const u64 v = random_residues(rng, 1, p)[0];
        t = TwPair{v, F.shoup(v)};
      }
      x[0] = 0;
      x[1] = p - 1;
      y[1] = p - 1;
      u64 *dx = to_device(x), *dy = to_device(y), *dout = nullptr;
      TwPair* dw = to_device(w);
      cuda_check(cudaMalloc(&dout, 5 * n * sizeof(u64)), "selftest alloc");
      k_st_field<<<(n + 127) / 128, 128>>>(dx, dy, dw, dout, n, p, F.pp);
      cuda_check(cudaGetLastError(), "selftest field");
      const std::vector<u64> r = to_host(dout, 5 * std::size_t(n));
      const u64 rinv = F.inv(F.r);
      for (unsigned i = 0; i < n; ++i) {
        s.expect(r[5 * i + 0] == F.mul(x[i], w[i].w));
        s.expect(r[5 * i + 1] == F.mul(F.mul(x[i], y[i]), rinv));
        s.expect(r[5 * i + 2] == F.add(x[i], y[i]));
        s.expect(r[5 * i + 3] == F.sub(x[i], y[i]));
        const u64 sa = x[i] | (y[i] << 62), sb = ~y[i];
        s.expect(r[5 * i + 4] == u64(u128(sa) * sb % kSolinasPrime));
      }
      s.expect(F.pow(5, p - 1) == 1);  // Fermat (the host planner's field)
      cudaFree(dx);
      cudaFree(dy);
      cudaFree(dw);
      cudaFree(dout);
    }
    total += s.report(out);
  }

  {
    Suite s{"transform_roundtrip"};
    for (u64 p : {kP1, kP2}) {
      // the reference's sizes, plus multi-pass, narrow-tile and radix-3 pass lengths
      for (std::size_t n : {2u, 4u, 16u, 64u, 256u, 3u, 6u, 48u, 192u, 768u, 4096u, 12288u, 131072u, 98304u}) {
        const std::vector<u64> x = random_residues(rng, n, p);
        std::vector<u64> v = x;
        forward_transform(p, n, v.data());
        inverse_transform(p, n, v.data());
        s.expect(v == x);
      }
    }
    total += s.report(out);
  }

  {
    Suite s{"convolution_vs_direct"};
    for (u64 p : {kP1, kP2, kQ1}) {
      for (std::size_t n : {4u, 8u, 12u, 16u, 24u, 96u, 384u, 4096u}) {
        const std::vector<u64> x = random_residues(rng, n, p), y = random_residues(rng, n, p);
        std::vector<u64> z(n);
        convolve_mod_p(p, n, x.data(), n, y.data(), n, z.data());
        s.expect(z == direct_cyclic(x, y, p));
      }
    }
    total += s.report(out);
  }

  {
    Suite s{"crt_recompose"};
    const u64 pairs[2][2] = {{kP1, kP2}, {kQ1, kQ2}};
    for (const auto& pr : pairs) {
      const u128 M = u128(pr[0]) * pr[1];
      const unsigned n = 1000;
      std::uniform_int_distribution<u64> lo(0, ~u64(0)), hi(0, u64((M - 1) >> 64));
      std::vector<u128> xs(n);
      std::vector<u64> a1(n), a2(n);
      for (unsigned i = 0; i < n; ++i) {
        u128 x = (u128(hi(rng)) << 64) | lo(rng);
        if (x >= M) x -= M;
        if (i == 0) x = 0;
        if (i == 1) x = M - 1;
        xs[i] = x;
        a1[i] = u64(x % pr[0]);
        a2[i] = u64(x % pr[1]);
      }
      const CrtConsts cc = crt_consts(pr[0], pr[1]);
      u64 *d1 = to_device(a1), *d2 = to_device(a2), *dout = nullptr;
      cuda_check(cudaMalloc(&dout, 2 * n * sizeof(u64)), "selftest alloc");
      k_st_crt<<<(n + 127) / 128, 128>>>(d1, d2, dout, n, pr[0], pr[1], cc.p2_prime, cc.r_tilde);
      cuda_check(cudaGetLastError(), "selftest crt");
      const std::vector<u64> r = to_host(dout, 2 * std::size_t(n));
      for (unsigned i = 0; i < n; ++i) s.expect(((u128(r[2 * i + 1]) << 64) | r[2 * i]) == xs[i]);
      cudaFree(d1);
      cudaFree(d2);
      cudaFree(dout);
    }
    total += s.report(out);
  }

  {
    Suite s{"base_division"};
    for (unsigned e = 14; e <= 17; ++e) {
      const u64 B = pow10u(e);
      const unsigned n = 1000;
      std::uniform_int_distribution<u64> lo(0, ~u64(0)), hi(0, (u64(1) << 62) - 1);
      std::vector<u64> xl(n), xh(n);
      for (unsigned i = 0; i < n; ++i) {
        xl[i] = lo(rng);
        xh[i] = hi(rng);  // x < 2^126
      }
      xl[0] = xh[0] = 0;
      xl[1] = ~u64(0);
      xh[1] = (u64(1) << 62) - 1;
      u64 *dl = to_device(xl), *dh = to_device(xh), *dout = nullptr;
      cuda_check(cudaMalloc(&dout, 6 * n * sizeof(u64)), "selftest alloc");
      k_st_div<<<(n + 127) / 128, 128>>>(dl, dh, dout, n, div_for(B));
      cuda_check(cudaGetLastError(), "selftest div");
      const std::vector<u64> r = to_host(dout, 6 * std::size_t(n));
      for (unsigned i = 0; i < n; ++i) {
        const u128 x = (u128(xh[i]) << 64) | xl[i];
        const u64 *d = &r[6 * i];
        s.expect(d[0] < B && d[1] < B && d[2] < B);
        s.expect(u128(d[0]) + u128(d[1]) * B + u128(d[2]) * B * B == x);
        s.expect(d[3] < B && ((u128(d[5]) << 64) | d[4]) * B + d[3] == x);
      }
      cudaFree(dl);
      cudaFree(dh);
      cudaFree(dout);
    }
    total += s.report(out);
  }

  {
    // reference selftest.cpp:180-190 at lambda = 14: coefficients (3, B, 8, 0) carry
    // into limbs (3, 0, 9, 0), i.e. 9 * 10^28 + 3; all-zero coefficients give "0"
    Suite s{"carry_recovery"};
    const u64 B = pow10u(14);
    const u64 c[4] = {3, B, 8, 0};
    char buf[64] = {0};
    std::size_t len = recover_decimal(c, c, 4, kP1, kP2, 14, 1, 30, buf, sizeof buf);
    s.expect(std::string(buf, len) == "9" + std::string(27, '0') + "3");
    const u64 zero[6] = {0, 0, 0, 0, 0, 0};
    len = recover_decimal(zero, zero, 6, kP1, kP2, 14, 1, 2, buf, sizeof buf);
    s.expect(std::string(buf, len) == "0");
    total += s.report(out);
  }

  {
    Suite s{"small_products"};
    auto mul = [&](const std::string& a, const std::string& b) {
      std::string z(a.size() + b.size(), '\0');
      const std::size_t n = multiply_host(a.data(), a.size(), b.data(), b.size(), &z[0], z.size(), 0, false);
      z.resize(n);
      return z;
    };
    s.expect(mul("12", "34") == "408");
    s.expect(mul("21", "43") == "903");
    s.expect(mul("0", "999") == "0");
    s.expect(mul("1", "1") == "1");
    for (int i = 0; i < 100; ++i) {
      std::uniform_int_distribution<std::size_t> len(1, 60);
      const std::string a = random_decimal(rng, len(rng)), b = random_decimal(rng, len(rng));
      s.expect(mul(a, b) == schoolbook(a, b));
    }
    const std::string sq = random_decimal(rng, 40);
    s.expect(mul(sq, sq) == schoolbook(sq, sq));
    // one-CTA sizes against the schoolbook product, multi-pass sizes by fingerprints
    for (std::size_t n : {700u, 2500u}) {
      const std::string a = random_decimal(rng, n), b = random_decimal(rng, n + 13);
      s.expect(mul(a, b) == schoolbook(a, b));
    }
    const u64 q = 2305843009213693951ull;  // 2^61 - 1
    for (std::size_t n : {30000u, 150000u, 400000u}) {
      const std::string a = random_decimal(rng, n), b = random_decimal(rng, n / 2 + 7);
      const std::string z = mul(a, b);
      s.expect(z.size() + 1 >= a.size() + b.size() && z[0] != '0');
      s.expect(residue(z, q) == u64(u128(residue(a, q)) * residue(b, q) % q));
    }
    total += s.report(out);
  }

  if (inject_fault) {
    // Flip one root-table entry of a locally used plan; the round trip and the
    // convolution identity must now fail (reference selftest.cpp:205-216). The entry is
    // restored afterwards, so the context stays usable.
    Suite s{"fault_injection"};
    const std::size_t n = 64;
    const PrimePlan& P = prime_plan(kP1, n);
    TwPair* entry = P.passes.front()->dft_fwd.ptr + 5;
    TwPair saved{}, bad{};
    cuda_check(cudaMemcpy(&saved, entry, sizeof saved, cudaMemcpyDeviceToHost), "fault read");
    bad = saved;
    bad.w ^= 1;
    cuda_check(cudaMemcpy(entry, &bad, sizeof bad, cudaMemcpyHostToDevice), "fault write");
    const std::vector<u64> x = random_residues(rng, n, kP1), y = random_residues(rng, n, kP1);
    std::vector<u64> v = x, z(n);
    forward_transform(kP1, n, v.data());
    inverse_transform(kP1, n, v.data());
    s.expect(v == x);
    convolve_mod_p(kP1, n, x.data(), n, y.data(), n, z.data());
    s.expect(z == direct_cyclic(x, y, kP1));
    cuda_check(cudaMemcpy(entry, &saved, sizeof saved, cudaMemcpyHostToDevice), "fault restore");
    total += s.report(out);
  }

  char line[64];
  std::snprintf(line, sizeof line, "selftest_failures=%d\n", total);
  out += line;
  return total;
}

}  // namespace dmg
