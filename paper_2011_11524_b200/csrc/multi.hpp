// Multi-device context (see multi.cu): one Engine per device of the context; batches fan out
// over the devices, one large product is sharded over them.
#pragma once
#include <memory>
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
  // batches: contiguous ranges of products per device, one host thread per device
  void multiply_batch_host(std::size_t count, const char* xs, std::size_t x_stride, std::size_t nx,
                           const char* ys, std::size_t y_stride, std::size_t ny, char* outs,
                           std::size_t out_stride, std::size_t* lens);
  void multiply_batch_ptrs(std::size_t count, const char* const* xs, const std::size_t* nxs, const char* const* ys,
                           const std::size_t* nys, char* const* outs, const std::size_t* caps, std::size_t* lens);
  // whether multiply_host shards this product (G > 1, N >= 2^22, a valid shard shape)
  bool shards(std::size_t nx, std::size_t ny, unsigned forced) const;
  // the sharded product itself (any size the shard shape admits)
  std::size_t sharded_multiply(const char* x, std::size_t nx, const char* y, std::size_t ny, char* out,
                               std::size_t cap, bool squaring);

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

}  // namespace dmg
