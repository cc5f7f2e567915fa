// Host-side transfer probe: pageable cudaMemcpy (driver-staged) vs pinned DMA, and host
// memcpy bandwidth with 1..8 threads (the staging cost of a pageable-buffer pipeline).
// Build: g++ -O2 -std=c++17 tools/host_probe.cpp -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
  const size_t n = 200u << 20;
  std::vector<char> page_a(n, 1), page_b(n, 2);
  char *pin, *dev;
  cudaMallocHost(&pin, n);
  cudaMalloc(&dev, n);
  memset(pin, 3, n);
  for (int rep = 0; rep < 2; ++rep) {
    double t = now();
    cudaMemcpy(dev, page_a.data(), n, cudaMemcpyHostToDevice);
    double h2d_page = now() - t;
    t = now();
    cudaMemcpy(page_b.data(), dev, n, cudaMemcpyDeviceToHost);
    double d2h_page = now() - t;
    t = now();
    cudaMemcpy(dev, pin, n, cudaMemcpyHostToDevice);
    double h2d_pin = now() - t;
    t = now();
    cudaMemcpy(pin, dev, n, cudaMemcpyDeviceToHost);
    double d2h_pin = now() - t;
    std::printf("pageable h2d %.1f GB/s d2h %.1f GB/s | pinned h2d %.1f d2h %.1f\n", n / h2d_page / 1e9,
                n / d2h_page / 1e9, n / h2d_pin / 1e9, n / d2h_pin / 1e9);
  }
  for (int th : {1, 2, 4, 8}) {
    for (int rep = 0; rep < 2; ++rep) {
      double t = now();
      std::vector<std::thread> ts;
      for (int i = 0; i < th; ++i)
        ts.emplace_back([&, i] { memcpy(pin + n / th * i, page_a.data() + n / th * i, n / th); });
      for (auto& x : ts) x.join();
      double dt = now() - t;
      if (rep) std::printf("memcpy pageable->pinned %d threads: %.1f GB/s\n", th, n / dt / 1e9);
    }
  }
  return 0;
}
