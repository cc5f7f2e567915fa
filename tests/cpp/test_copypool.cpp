// CopyPool (csrc/hostio.cu): the pageable <-> pinned staging copy split over host threads must
// cover every byte for any length, including lengths whose per-part share is an exact
// multiple of 4 KiB plus a few bytes (the partition rounds the CEILING quotient up to 4 KiB).
// CPU-only: CopyPool is plain host code inside libdecmul_gpu.so.
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../paper_2011_11524_b200/csrc/engine.hpp"

int main() {
  int failures = 0, checks = 0;
  for (int threads = 1; threads <= 4; ++threads) {
    dmg::CopyPool pool(threads);
    const std::size_t parts = std::size_t(threads) + 1;
    for (std::size_t k : {64, 128, 257}) {
      for (std::size_t r = 0; r <= 4; ++r) {
        const std::size_t n = parts * 4096 * k + r;
        std::vector<char> src(n), dst(n, 0);
        for (std::size_t i = 0; i < n; ++i) src[i] = char(1 + (i * 131 + 7) % 251);
        pool.copy(dst.data(), src.data(), n);
        ++checks;
        if (std::memcmp(dst.data(), src.data(), n) != 0) {
          ++failures;
          std::printf("mismatch: threads=%d n=%zu\n", threads, n);
        }
      }
    }
  }
  std::printf("suite=copypool checks=%d failures=%d\n", checks, failures);
  return failures ? 1 : 0;
}
