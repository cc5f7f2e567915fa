// In-place transposition kernels (reference transpose.cpp). On the fused
// transform path the transposes are folded into strided pass addressing; these
// standalone kernels back the parity hooks and the memory-tight in-place mode.
//
//  transpose_square_sub (transpose.cpp:12-25): the n x n submatrix at a with row
//  stride `stride`, swapped as 32 x 32 tile pairs staged through shared memory:
//  one CTA owns one (i <= j) tile pair, so the swap is race-free in place.
//  permute_rho / unpermute_rho (transpose.cpp:27-41) per row of 2n words.
#include <cstdlib>

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

// permute_rho / unpermute_rho in place, one row of 2n words at a time per CTA: the row is
// staged in shared memory (2n <= kRhoSmemWords) or in this CTA's own 2n-word slice of a small
// global scratch, like the reference's 2n words of scratch per row (transpose.cpp:27-47).
constexpr unsigned long long kRhoSmemWords = 16384;  // 128 KiB

template <bool SMEM>
__global__ void k_rho_rows(u64* a, u64* scratch, unsigned long long n, int inverse) {
  extern __shared__ u64 rho_stage[];
  const unsigned long long w = 2 * n;
  u64* s = SMEM ? rho_stage : scratch + blockIdx.x * w;
  for (unsigned long long row = blockIdx.x; row < n; row += gridDim.x) {
    u64* r = a + row * w;
    for (unsigned long long j = threadIdx.x; j < w; j += blockDim.x) s[j] = r[j];
    __syncthreads();
    for (unsigned long long j = threadIdx.x; j < w; j += blockDim.x) {
      unsigned long long from;
      if (!inverse)
        from = j < n ? 2 * j : 2 * (j - n) + 1;  // row[j] = old[2j], row[n+j] = old[2j+1]
      else
        from = (j & 1) ? n + j / 2 : j / 2;      // row[2i] = old[i], row[2i+1] = old[n+i]
      r[j] = s[from];
    }
    __syncthreads();
  }
}

}  // namespace

void launch_transpose_square_sub(u64* a, unsigned long long n, unsigned long long stride, cudaStream_t st) {
  if (n == 0) return;
  const unsigned nt = unsigned((n + T - 1) / T);
  const unsigned long long pairs = (unsigned long long)nt * (nt + 1) / 2;
  k_transpose_square<<<unsigned(pairs), dim3(T, 8), 0, st>>>(a, n, stride, nt);
}

unsigned rho_ctas(unsigned long long n) { return unsigned(n < 148 * 2 ? n : 148 * 2); }

// DECMUL_RHO_GLOBAL=1 forces the global-scratch variant at small n (tests)
bool rho_in_smem(unsigned long long n) {
  const char* e = std::getenv("DECMUL_RHO_GLOBAL");
  return 2 * n <= kRhoSmemWords && !(e && e[0] == '1');
}

std::size_t rho_scratch_words(unsigned long long n) {
  return rho_in_smem(n) ? 0 : std::size_t(rho_ctas(n)) * 2 * n;
}

void launch_rho(u64* a, u64* scratch, unsigned long long n, bool inverse, cudaStream_t st) {
  if (n == 0) return;
  const unsigned ctas = rho_ctas(n);
  if (rho_in_smem(n)) {
    const std::size_t smem = 2 * n * sizeof(u64);
    cudaFuncSetAttribute(k_rho_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k_rho_rows<true><<<ctas, 256, smem, st>>>(a, nullptr, n, inverse ? 1 : 0);
  } else {
    k_rho_rows<false><<<ctas, 256, 0, st>>>(a, scratch, n, inverse ? 1 : 0);
  }
}

}  // namespace dmg
