// Integer-pipe roofline denominator R_mm: throughput of
// independent-lane 63-bit modular multiplications on all SMs, measured live so
// bench.py can report the transform kernels as a fraction of it. Variant 0 is
// the Shoup form the transforms use for every root-of-unity factor; variant 1 is
// the reference's Montgomery REDC (montgomery.hpp:26-39); variant 2 the reference's
// Solinas reduction for the Goldilocks prime (montgomery.hpp:60-77, bench.cpp:82-88).
#include "kernels.cuh"

namespace dmg {

namespace {

template <int V>
__global__ void k_modmul_rate(u64* out, u64 p, u64 pp, int iters, const TwPair* ks) {
  constexpr int C = 8;
  u64 acc[C];
  TwPair k[C];
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    acc[c] = (u64(t) * 0x9e3779b97f4a7c15ull + c) % p;
    k[c] = ks[c];
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      acc[c] = V == 0 ? shoup_mul(acc[c], k[c], p) : V == 1 ? mont_mul(acc[c], k[c].w, p, pp) : solinas_mul(acc[c], k[c].w);
  }
  u64 s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s ^= acc[c];
  out[t] = s;
}

}  // namespace

double measure_modmul_rate(int variant, cudaStream_t st) {
  const u64 p = 9223372036015915009ull;
  u64 inv = p;
  for (int i = 0; i < 6; ++i) inv *= 2 - p * inv;
  const u64 pp = 0 - inv;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  TwPair hk[8];
  for (int c = 0; c < 8; ++c) {
    const u64 w = (0x243f6a8885a308d3ull * u64(c + 1)) % p;
    hk[c] = TwPair{w, u64(((unsigned __int128)w << 64) / p)};
  }
  const int threads = 256, blocks = sms * 8, iters = 4096;
  TwPair* dk = nullptr;
  u64* dout = nullptr;
  if (cudaMalloc(&dk, sizeof hk) != cudaSuccess) return 0;
  if (cudaMalloc(&dout, sizeof(u64) * threads * blocks) != cudaSuccess) return 0;
  cudaMemcpyAsync(dk, hk, sizeof hk, cudaMemcpyHostToDevice, st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, st);
    if (variant == 0)
      k_modmul_rate<0><<<blocks, threads, 0, st>>>(dout, p, pp, iters, dk);
    else if (variant == 1)
      k_modmul_rate<1><<<blocks, threads, 0, st>>>(dout, p, pp, iters, dk);
    else
      k_modmul_rate<2><<<blocks, threads, 0, st>>>(dout, p, pp, iters, dk);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(dk);
  cudaFree(dout);
  return double(blocks) * threads * iters * 8 / (best * 1e-3);
}

}  // namespace dmg
