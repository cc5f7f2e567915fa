// In-place transposition kernels (reference transpose.cpp). On the fused
// transform path the transposes are folded into strided pass addressing; these
// standalone kernels back the parity hooks and the memory-tight in-place mode.
//
//  transpose_square_sub (transpose.cpp:12-25): the n x n submatrix at a with row
//  stride `stride`, swapped as 32 x 32 tile pairs staged through shared memory:
//  one CTA owns one (i <= j) tile pair, so the swap is race-free in place.
//  permute_rho / unpermute_rho (transpose.cpp:27-41) per row of 2n words.
#include "kernels.cuh"

namespace dmg {

namespace {

constexpr int T = 32;

__global__ void k_transpose_square(u64* a, unsigned long long n, unsigned long long stride, unsigned ntiles) {
  __shared__ u64 ta[T][T + 1], tb[T][T + 1];
  // blockIdx.x enumerates pairs (bi, bj), bi <= bj, row-major over the upper triangle.
  unsigned long long idx = blockIdx.x;
  unsigned bi = 0;
  while (idx >= ntiles - bi) {
    idx -= ntiles - bi;
    ++bi;
  }
  const unsigned bj = bi + unsigned(idx);
  const unsigned long long r0 = (unsigned long long)bi * T, c0 = (unsigned long long)bj * T;
  for (int y = threadIdx.y; y < T; y += blockDim.y) {
    const int x = threadIdx.x;
    const unsigned long long ra = r0 + y, ca = c0 + x;  // tile A = rows bi, cols bj
    const unsigned long long rb = c0 + y, cb = r0 + x;  // tile B = rows bj, cols bi
    if (ra < n && ca < n) ta[y][x] = a[ra * stride + ca];
    if (rb < n && cb < n) tb[y][x] = a[rb * stride + cb];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < T; y += blockDim.y) {
    const int x = threadIdx.x;
    const unsigned long long ra = r0 + y, ca = c0 + x;
    const unsigned long long rb = c0 + y, cb = r0 + x;
    if (ra < n && ca < n) a[ra * stride + ca] = tb[x][y];  // A <- B^T
    if (rb < n && cb < n) a[rb * stride + cb] = ta[x][y];  // B <- A^T
  }
}

__global__ void k_rho(const u64* a, u64* s, unsigned long long n, int inverse) {
  const unsigned long long total = 2 * n * n;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long row = i / (2 * n), j = i % (2 * n);
    // destination index j of the permuted row
    unsigned long long from;
    if (!inverse)
      from = j < n ? 2 * j : 2 * (j - n) + 1;  // row[j] = old[2j], row[n+j] = old[2j+1]
    else
      from = (j & 1) ? n + j / 2 : j / 2;      // row[2i] = old[i], row[2i+1] = old[n+i]
    s[i] = a[row * 2 * n + from];
  }
}

}  // namespace

void launch_transpose_square_sub(u64* a, unsigned long long n, unsigned long long stride, cudaStream_t st) {
  if (n == 0) return;
  const unsigned nt = unsigned((n + T - 1) / T);
  const unsigned long long pairs = (unsigned long long)nt * (nt + 1) / 2;
  k_transpose_square<<<unsigned(pairs), dim3(T, 8), 0, st>>>(a, n, stride, nt);
}

void launch_rho(u64* a, u64* scratch, unsigned long long n, bool inverse, cudaStream_t st) {
  if (n == 0) return;
  const unsigned long long total = 2 * n * n;
  unsigned long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_rho<<<unsigned(blocks), 256, 0, st>>>(a, scratch, n, inverse ? 1 : 0);
  cudaMemcpyAsync(a, scratch, total * sizeof(u64), cudaMemcpyDeviceToDevice, st);
}

}  // namespace dmg
