// PCIe transfer probe: DMA copies (whole / chunked, one direction / both) versus SM-driven
// zero-copy (kernels loading from and storing to mapped pinned host memory).
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/pcie_probe.cu -o tools/pcie_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));        \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)

__global__ void k_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

// one kernel: half the CTAs read host->device, half write device->host
__global__ void k_duplex(const uint4* __restrict__ hsrc, uint4* __restrict__ ddst, const uint4* __restrict__ dsrc,
                         uint4* __restrict__ hdst, size_t n) {
  const unsigned half = gridDim.x / 2;
  const bool up = blockIdx.x < half;
  const unsigned b = up ? blockIdx.x : blockIdx.x - half;
  for (size_t i = b * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(half) * blockDim.x) {
    if (up) ddst[i] = hsrc[i];
    else hdst[i] = dsrc[i];
  }
}

int main() {
  const size_t n = 82u << 20;
  char *h1, *h2, *d1, *d2;
  CK(cudaHostAlloc(&h1, n, cudaHostAllocMapped));
  CK(cudaHostAlloc(&h2, n, cudaHostAllocMapped));
  CK(cudaMalloc(&d1, n));
  CK(cudaMalloc(&d2, n));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, j1, j2;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&j1));
  CK(cudaEventCreate(&j2));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  auto timed = [&](const char* name, auto fn, double bytes_per_dir) {
    fn();
    CK(cudaDeviceSynchronize());
    const int reps = 10;
    CK(cudaEventRecord(e0, s1));
    CK(cudaStreamWaitEvent(s2, e0, 0));
    for (int r = 0; r < reps; ++r) fn();
    CK(cudaEventRecord(j2, s2));
    CK(cudaStreamWaitEvent(s1, j2, 0));
    CK(cudaEventRecord(e1, s1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    std::printf("%-28s %7.3f ms  %6.1f GB/s per direction\n", name, ms, bytes_per_dir / ms / 1e6);
  };
  timed("dma h2d", [&] { CK(cudaMemcpyAsync(d1, h1, n, cudaMemcpyHostToDevice, s1)); }, n);
  timed("dma d2h", [&] { CK(cudaMemcpyAsync(h2, d2, n, cudaMemcpyDeviceToHost, s2)); }, n);
  timed("dma both", [&] {
    CK(cudaMemcpyAsync(d1, h1, n, cudaMemcpyHostToDevice, s1));
    CK(cudaMemcpyAsync(h2, d2, n, cudaMemcpyDeviceToHost, s2));
  }, n);
  for (int chunks : {4, 10, 20}) {
    char name[64];
    std::snprintf(name, sizeof name, "dma both, %d chunks", chunks);
    timed(name, [&] {
      const size_t c = n / chunks;
      for (int i = 0; i < chunks; ++i) {
        CK(cudaMemcpyAsync(d1 + i * c, h1 + i * c, c, cudaMemcpyHostToDevice, s1));
        CK(cudaMemcpyAsync(h2 + i * c, d2 + i * c, c, cudaMemcpyDeviceToHost, s2));
      }
    }, n);
  }
  for (int per_sm : {2, 4, 8}) {
    char name[64];
    std::snprintf(name, sizeof name, "zero-copy h2d (%d CTA/SM)", per_sm);
    timed(name, [&] { k_copy<<<sms * per_sm, 512, 0, s1>>>((const uint4*)h1, (uint4*)d1, n / 16); }, n);
    std::snprintf(name, sizeof name, "zero-copy d2h (%d CTA/SM)", per_sm);
    timed(name, [&] { k_copy<<<sms * per_sm, 512, 0, s1>>>((const uint4*)d2, (uint4*)h2, n / 16); }, n);
    std::snprintf(name, sizeof name, "zero-copy both (%d CTA/SM)", per_sm);
    timed(name, [&] {
      k_duplex<<<sms * per_sm, 512, 0, s1>>>((const uint4*)h1, (uint4*)d1, (const uint4*)d2, (uint4*)h2, n / 16);
    }, n);
  }
  timed("dma h2d + zero-copy d2h", [&] {
    CK(cudaMemcpyAsync(d1, h1, n, cudaMemcpyHostToDevice, s1));
    k_copy<<<sms * 4, 512, 0, s2>>>((const uint4*)d2, (uint4*)h2, n / 16);
  }, n);
  return 0;
}
