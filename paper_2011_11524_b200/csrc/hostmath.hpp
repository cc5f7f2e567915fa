// Host-side number theory for planning: Montgomery context, powers, primality,
// deterministic roots of unity, base/length selection.
//
// These decide WHICH field elements the device computes with, so they follow
// the reference's choices exactly (same primes, same root search order, same
// lambda/length selection):
//   make_ctx            montgomery.cpp:28-41
//   is_prime            primes.cpp:24-49
//   primitive root      primes.cpp:99-112
//   smallest length     decimal.cpp:54-76
//   base selection      decimal.cpp:78-100
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

namespace dmg {

typedef unsigned long long u64;
typedef unsigned __int128 u128;

// Embedded production pair (reference primes.hpp:30-31).
constexpr u64 kP1 = 9223372036015915009ull;  // 91625968973 * 3 * 2^25 + 1
constexpr u64 kP2 = 9223372036166909953ull;  // 183251937949 * 3 * 2^24 + 1
// Large-length pair: the two largest results of the reference's own search
// find_primes(64, 30, 2) (primes.cpp:70-81). Used only when the
// production pair cannot hold the transform (N > 3 * 2^24).
constexpr u64 kQ1 = 9223371938070528001ull;  // 715827875 * 3 * 2^32 + 1
constexpr u64 kQ2 = 9223371941291753473ull;  // 2863311501 * 3 * 2^30 + 1

struct OperandTooLarge : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct HostField {
  u64 p = 0, pp = 0, r = 0, r2 = 0;  // p' with p p' = -1 mod 2^64; R mod p; R^2 mod p

  explicit HostField(u64 prime) : p(prime) {
    if (p <= 2 || !(p & 1) || p >= (1ull << 63)) throw std::invalid_argument("make_ctx: bad modulus");
    u64 inv = p;
    for (int i = 0; i < 6; ++i) inv *= 2 - p * inv;  // Newton: p inv == 1 mod 2^64
    pp = 0 - inv;
    r = (0 - p) % p;
    r2 = u64((u128)r * r % p);
  }
  u64 mul(u64 a, u64 b) const { return u64((u128)a * b % p); }
  u64 add(u64 a, u64 b) const { u64 s = a + b; return s >= p ? s - p : s; }
  u64 sub(u64 a, u64 b) const { return a >= b ? a - b : a + p - b; }
  u64 pow(u64 a, u64 e) const {
    u64 acc = 1 % p;
    a %= p;
    while (e) {
      if (e & 1) acc = mul(acc, a);
      a = mul(a, a);
      e >>= 1;
    }
    return acc;
  }
  u64 inv(u64 a) const { return pow(a, p - 2); }
  u64 to_mont(u64 a) const { return u64(((u128)(a % p) << 64) % p); }
  u64 shoup(u64 w) const { return u64(((u128)w << 64) / p); }  // w' = floor(w 2^64 / p)

  // primitive_root_of_unity (reference primes.cpp:99-112), returned PLAIN.
  u64 root_of_unity(u64 n) const {
    if (n == 0 || (p - 1) % n) throw std::invalid_argument("primitive_root_of_unity: n must divide p-1");
    if (n == 1) return 1;
    for (u64 g = 2; g < p; g = (g == 2 ? 3 : g + 2)) {
      u64 xi = pow(g, (p - 1) / n);
      if (n % 2 == 0 && pow(xi, n / 2) == 1) continue;
      if (n % 3 == 0 && pow(xi, n / 3) == 1) continue;
      return xi;
    }
    throw std::logic_error("primitive_root_of_unity: no generator found");
  }
};

inline bool is_prime(u64 n) {
  static const u64 bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (u64 b : bases) {
    if (n == b) return true;
    if (n % b == 0) return false;
  }
  u64 d = n - 1;
  int s = __builtin_ctzll(d);
  d >>= s;
  auto mulm = [n](u64 a, u64 b) { return u64((u128)a * b % n); };
  for (u64 b : bases) {
    u64 x = 1, a = b, e = d;
    while (e) {
      if (e & 1) x = mulm(x, a);
      a = mulm(a, a);
      e >>= 1;
    }
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 1; i < s; ++i) {
      x = mulm(x, x);
      if (x == n - 1) {
        comp = false;
        break;
      }
    }
    if (comp) return false;
  }
  return true;
}

inline u64 pow10u(unsigned e) {
  u64 b = 1;
  while (e--) b *= 10;
  return b;
}

// smallest_supported_length (decimal.cpp:54-76): smallest 2^k or 3*2^k >= need dividing both p-1; 0 if none.
inline std::size_t smallest_supported_length(std::size_t need, u64 p1, u64 p2) {
  unsigned v1 = __builtin_ctzll(p1 - 1), v2 = __builtin_ctzll(p2 - 1);
  bool t1 = ((p1 - 1) >> v1) % 3 == 0, t2 = ((p2 - 1) >> v2) % 3 == 0;
  unsigned kmax = v1 < v2 ? v1 : v2;
  if (need < 2) need = 2;
  if (need > (std::size_t(1) << 62)) return 0;
  std::size_t best = 0, two = 1;
  while (two < need) two <<= 1;
  if (unsigned(__builtin_ctzll(two)) <= kmax) best = two;
  if (t1 && t2) {
    std::size_t half = 1, q = (need + 2) / 3;
    while (half < q) half <<= 1;
    if (unsigned(__builtin_ctzll(half)) <= kmax && (best == 0 || 3 * half < best)) best = 3 * half;
  }
  return best;
}

struct BasePlan {
  unsigned base_exp = 0;
  std::size_t length = 0;
};

// select_base_and_length (decimal.cpp:78-100) for one prime pair.
inline BasePlan select_base_and_length(std::size_t dx, std::size_t dy, u64 p1, u64 p2, unsigned forced) {
  if (dx < 1 || dy < 1) throw std::invalid_argument("select_base_and_length: digit counts must be >= 1");
  if (forced > 17) throw std::invalid_argument("select_base_and_length: unsupported forced base");
  const u128 modulus = (u128)p1 * p2;
  const unsigned lo = forced ? forced : 14, hi = forced ? forced : 17;
  for (unsigned be = hi; be >= lo; --be) {
    const u64 top = pow10u(be) - 1;
    const std::size_t lx = (dx + be - 1) / be, ly = (dy + be - 1) / be;
    if ((u128)(lx < ly ? lx : ly) > (modulus - 1) / ((u128)top * top)) continue;
    const std::size_t len = smallest_supported_length(lx + ly, p1, p2);
    if (len == 0) throw OperandTooLarge("operands exceed the largest supported transform length");
    return {be, len};
  }
  throw OperandTooLarge("operands violate the coefficient bound at every supported base");
}

// Pass radices of a length-N transform (N = 2^k or 3 * 2^k): a radix-3 pass first when
// 3 | N, then the power of two split into ceil(k / maxlog) balanced radix-2^e passes,
// larger ones first (each tile of 2^e x 16 columns must fit shared memory).
inline std::vector<int> pass_radices(std::size_t N, int maxlog) {
  std::vector<int> r;
  std::size_t c = N;
  if (N % 3 == 0) {
    r.push_back(3);
    c = N / 3;
  }
  const int k = c > 1 ? __builtin_ctzll(c) : 0;
  if (k > 0) {
    const int m = (k + maxlog - 1) / maxlog;
    for (int i = 0; i < m; ++i) r.push_back(1 << (k / m + (i < k % m ? 1 : 0)));
  }
  return r;
}

// Column/row split of the passes for G ranks; see engine.hpp ShardGeom.
struct ShardShape {
  int K = 0;
  std::size_t Rtot = 1, Sc = 0, Bc = 0;
};
inline ShardShape shard_shape(std::size_t N, const std::vector<int>& radices, int G, std::size_t min_width) {
  if (G < 1 || (G & (G - 1))) throw std::invalid_argument("shard: the rank count must be a power of two");
  if (radices.size() < 2 || radices.back() == 3) throw std::invalid_argument("shard: product too small to shard");
  ShardShape s;
  for (std::size_t i = 0; i + 1 < radices.size(); ++i) {
    s.Rtot *= std::size_t(radices[i]);
    s.K = int(i) + 1;
    s.Sc = N / s.Rtot;
    if (s.Rtot % std::size_t(G) == 0 && s.Sc % std::size_t(G) == 0 && s.Sc / std::size_t(G) >= min_width) {
      s.Bc = s.Sc / std::size_t(G);
      for (int j = 0; j + 1 < s.K; ++j)
        if (radices[j] != 3) throw std::logic_error("shard: unsupported column-phase pass layout");
      return s;
    }
  }
  throw std::invalid_argument("shard: product too small for this many ranks");
}

struct PairChoice {
  u64 p1 = 0, p2 = 0;
  BasePlan bp;
  bool large_pair = false;  // true when the q-pair had to be used (beyond the reference's 3*2^24 cap)
};

// The reference pair wherever it can hold the product (bit-comparable spectra);
// otherwise the larger-2-adic pair from the reference's own prime search.
// DECMUL_FORCE_LARGE_PAIR=1 (test knob) selects the large pair at any size so its
// code path is parity-tested on small operands.
inline PairChoice choose_pair(std::size_t dx, std::size_t dy, unsigned forced, bool allow_large) {
  const char* force = std::getenv("DECMUL_FORCE_LARGE_PAIR");
  if (allow_large && force && force[0] == '1')
    return {kQ1, kQ2, select_base_and_length(dx, dy, kQ1, kQ2, forced), true};
  try {
    return {kP1, kP2, select_base_and_length(dx, dy, kP1, kP2, forced), false};
  } catch (const OperandTooLarge&) {
    if (!allow_large) throw;
    return {kQ1, kQ2, select_base_and_length(dx, dy, kQ1, kQ2, forced), true};
  }
}

}  // namespace dmg
