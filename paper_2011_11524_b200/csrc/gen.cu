// Seeded synthetic digit generator: a counter-based splitmix64
// stream shared bit-for-bit with the host (oracle or_gen_digits and
// paper_2011_11524_b200.inputs), so 10^10-digit operands can be produced in
// place in HBM. Digit 0 (most significant) is 1 + v mod 9, others v mod 10;
// mode 1 gives all nines (config 3's worst case).
#include "kernels.cuh"

namespace dmg {

namespace {

__device__ __forceinline__ u64 sm_mix(u64 z) {  // splitmix64 finalizer (reference bench.cpp:40-45)
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
constexpr u64 kGolden = 0x9e3779b97f4a7c15ull;

__global__ void k_gen(u64 seed0, u64 seed_step, unsigned long long count, unsigned long long n,
                      unsigned long long stride, int mode, char* out) {
  const unsigned long long total = count * n;
  for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < total;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long j = t / n, i = t % n;
    char c = '9';
    if (mode == 0) {
      const u64 key = sm_mix(seed0 + j * seed_step + kGolden);
      const u64 v = sm_mix(key + (u64)(i + 1) * kGolden);
      c = char('0' + (i == 0 ? 1 + v % 9 : v % 10));
    }
    out[j * stride + i] = c;
  }
}

}  // namespace

void launch_generate(u64 seed0, u64 seed_step, unsigned long long count, unsigned long long n,
                     unsigned long long stride, int mode, char* out, cudaStream_t st) {
  const unsigned long long total = count * n;
  unsigned long long blocks = (total + 255) / 256;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  if (blocks < 1) blocks = 1;
  k_gen<<<unsigned(blocks), 256, 0, st>>>(seed0, seed_step, count, n, stride, mode, out);
}

}  // namespace dmg
