// Throughput micro-benchmark for 63-bit modular multiplication on sm_100a.
// Fixes R_mm, the integer-pipe denominator of the NTT roofline.
// Variants: Montgomery REDC (reference montgomery.hpp:26-39 restated),
// Shoup (precomputed w' = floor(w 2^64 / p)), pseudo-Mersenne (p = 2^63 - eps),
// and the bare 64x64->128 product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__device__ __forceinline__ u64 mont(u64 a, u64 b, u64 p, u64 pp) {
  u64 lo = a * b, hi = __umul64hi(a, b);
  u64 m = lo * pp;
  u64 r = hi + __umul64hi(m, p) + (lo != 0);
  return r >= p ? r - p : r;
}
__device__ __forceinline__ u64 shoup(u64 x, u64 w, u64 wp, u64 p) {
  u64 q = __umul64hi(x, wp);
  u64 r = x * w - q * p;
  return r >= p ? r - p : r;
}
// p = 2^63 - eps, eps < 2^32
__device__ __forceinline__ u64 pmers(u64 a, u64 b, u64 p, u64 eps) {
  u64 lo = a * b, hi = __umul64hi(a, b);
  u64 H = (hi << 1) | (lo >> 63);
  u64 L = lo & 0x7fffffffffffffffull;
  u64 l2 = H * eps, h2 = __umul64hi(H, eps);
  u64 y = l2 + L;
  h2 += (y < L);
  u64 H2 = (h2 << 1) | (y >> 63);
  u64 z = (y & 0x7fffffffffffffffull) + H2 * eps;
  return z >= p ? z - p : z;
}

template <int V>
__global__ void bench(u64* out, u64 p, u64 pp, u64 eps, int iters, const u64* ks) {
  const int C = 8;
  u64 acc[C], k[C], kp[C];
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int c = 0; c < C; ++c) {
    acc[c] = (u64(t) * 0x9e3779b97f4a7c15ull + c) % p;
    k[c] = ks[2 * c];
    kp[c] = ks[2 * c + 1];
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (V == 0) acc[c] = mont(acc[c], k[c], p, pp);
      else if (V == 1) acc[c] = shoup(acc[c], k[c], kp[c], p);
      else if (V == 2) acc[c] = pmers(acc[c], k[c], p, eps);
      else { u64 lo = acc[c] * k[c], hi = __umul64hi(acc[c], k[c]); acc[c] = lo ^ hi; }
    }
  }
  u64 s = 0;
  for (int c = 0; c < C; ++c) s ^= acc[c];
  out[t] = s;
}

__global__ void copyk(const u64* __restrict__ a, u64* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

int main() {
  const u64 p = 9223372036015915009ull, pp = 8519684594239275007ull;
  const u64 eps = (1ull << 63) - p;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int sms = prop.multiProcessorCount;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\":\"%s\",\"sms\":%d,\"clock_khz\":%d}\n", prop.name, sms, clk);
  u64 hks[16];
  for (int c = 0; c < 8; ++c) {
    u64 w = (0x243f6a8885a308d3ull * (c + 1)) % p;
    hks[2 * c] = w;
    hks[2 * c + 1] = (u64)(((unsigned __int128)w << 64) / p);
  }
  u64 *ks, *out;
  cudaMalloc(&ks, sizeof hks);
  cudaMemcpy(ks, hks, sizeof hks, cudaMemcpyHostToDevice);
  int threads = 256, blocks = sms * 8;
  cudaMalloc(&out, sizeof(u64) * threads * blocks);
  int iters = 4096;
  const char* names[] = {"montgomery", "shoup", "pseudo_mersenne", "mul128"};
  for (int v = 0; v < 4; ++v) {
    for (int occ : {2, 4, 8}) {
      blocks = sms * occ;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        if (v == 0) bench<0><<<blocks, threads>>>(out, p, pp, eps, iters, ks);
        if (v == 1) bench<1><<<blocks, threads>>>(out, p, pp, eps, iters, ks);
        if (v == 2) bench<2><<<blocks, threads>>>(out, p, pp, eps, iters, ks);
        if (v == 3) bench<3><<<blocks, threads>>>(out, p, pp, eps, iters, ks);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
      double ops = double(blocks) * threads * iters * 8;
      printf("{\"variant\":\"%s\",\"blocks_per_sm\":%d,\"ms\":%.4f,\"gmodmul_per_s\":%.1f}\n", names[v], occ,
             best, ops / best / 1e6);
    }
  }
  // HBM copy
  size_t n = (size_t)1 << 28;
  u64 *a, *b;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 1, n * 8);
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    copyk<<<sms * 16, 512>>>(a, b, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  printf("{\"variant\":\"copy_u64\",\"GBps\":%.1f}\n", 2.0 * n * 8 / best / 1e6);
  cudaError_t err = cudaDeviceSynchronize();
  printf("{\"status\":\"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
