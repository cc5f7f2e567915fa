// Multi-device context (see multi.cu): one Engine per device of the context; batches fan out
// over the devices, one large product is sharded over them.
#pragma once
#include <exception>
#include <memory>
#include <thread>
#include <vector>

#include "engine.hpp"

namespace dmg {

class MultiEngine {
 public:
  // devices may repeat (ranks sharing a GPU: the exchange becomes local copies; tests)
  MultiEngine(const int* devices, int n);
  ~MultiEngine();

  int size() const { return int(eng_.size()); }
  Engine& rank(int q) { return *eng_[q]; }
  Engine& primary() { return *eng_[0]; }
  std::vector<int> devices() const;

  // decmul::multiply on host strings: sharded over every device when the product is large
  // enough (shards()), else on the first device
  std::size_t multiply_host(const char* x, std::size_t nx, const char* y, std::size_t ny, char* out,
                            std::size_t cap, unsigned forced_base_exp, bool alias, u64 p1 = 0, u64 p2 = 0);
  // The engine that would run this product alone on one device with overlappable transfers
  // (Engine::overlap_ok: large, pinned buffers; not sharded, not block-convolved), else nullptr.
  // Its multiply_host_overlapped is called WITHOUT the context lock held.
  Engine* overlap_engine(const char* x, std::size_t nx, const char* y, std::size_t ny, const char* out,
                         unsigned forced_base_exp, bool concurrent, u64 p1 = 0, u64 p2 = 0);
  // batches: contiguous ranges of products per device, one host thread per device
  void multiply_batch_host(std::size_t count, const char* xs, std::size_t x_stride, std::size_t nx,
                           const char* ys, std::size_t y_stride, std::size_t ny, char* outs,
                           std::size_t out_stride, std::size_t* lens,
                           std::unique_lock<std::mutex>* ctx_lock = nullptr);
  void multiply_batch_ptrs(std::size_t count, const char* const* xs, const std::size_t* nxs, const char* const* ys,
                           const std::size_t* nys, char* const* outs, const std::size_t* caps, std::size_t* lens);
  // whether multiply_host shards this product (G > 1, N >= 2^22, a valid shard shape)
  bool shards(std::size_t nx, std::size_t ny, unsigned forced) const;
  // the sharded product itself (any size the shard shape admits)
  std::size_t sharded_multiply(const char* x, std::size_t nx, const char* y, std::size_t ny, char* out,
                               std::size_t cap, bool squaring);
  // block convolution (blocked.cu): products past the largest transform as sums of block
  // products of K digits each, fanned out over the devices; block_digits: the K multiply_host
  // uses (0 = one ordinary product)
  static constexpr std::size_t kBlockDigits = 6000000000ull;
  std::size_t block_digits(std::size_t nx, std::size_t ny, unsigned forced) const;
  std::size_t blocked_multiply(const char* x, std::size_t nx, const char* y, std::size_t ny, char* out,
                               std::size_t cap, unsigned forced, std::size_t K);

 private:
  template <class F>
  void fan_out(std::size_t count, F&& f);
  std::size_t upload_slice(Engine& e, const ShardPlan& sp, int q, const char* d, std::size_t nd, char* dst,
                           cudaStream_t st);
  void all_to_all(const std::vector<u64*>& send, const std::vector<u64*>& recv, std::size_t L);
  void sync_all();

  std::vector<std::unique_ptr<Engine>> eng_;
  std::vector<cudaEvent_t> ready_, done_;
  static constexpr std::size_t kPinnedWords = 7 * 64;  // halo, rank maps, probes of up to 64 ranks
  u64* pinned_ = nullptr;
};

// Runs f(rank, begin, end) for the G contiguous ranges of [0, count) on G host threads (each
// engine on its own device); rethrows the first failure.
template <class F>
inline void MultiEngine::fan_out(std::size_t count, F&& f) {
  const std::size_t G = eng_.size();
  std::vector<std::exception_ptr> errs(G);
  std::vector<std::thread> th;
  for (std::size_t q = 0; q < G; ++q) {
    const std::size_t b = count * q / G, e = count * (q + 1) / G;
    if (b == e) continue;
    th.emplace_back([&, q, b, e] {
      try {
        cuda_check(cudaSetDevice(eng_[q]->device()), "cudaSetDevice");
        f(*eng_[q], b, e);
      } catch (...) {
        errs[q] = std::current_exception();
      }
    });
  }
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

}  // namespace dmg
