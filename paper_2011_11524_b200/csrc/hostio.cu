// Host <-> device transfers for the host-buffer API (the drop-in decmul::multiply with
// std::string operands): pinned buffers go straight to the DMA engines;
// large pageable ones are pipelined through a ring of pinned slots, the host threads of
// a CopyPool filling (or draining) slot c while the DMA engine moves slot c - 1.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "engine.hpp"

namespace dmg {

CopyPool::CopyPool(int threads) {
  for (int i = 0; i < threads; ++i) th_.emplace_back([this, i] { worker(i); });
}

CopyPool::~CopyPool() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  go_.notify_all();
  for (auto& t : th_) t.join();
}

void CopyPool::copy(char* dst, const char* src, std::size_t n) {
  const std::size_t parts = th_.size() + 1;
  if (th_.empty() || n < (std::size_t(1) << 20)) {
    std::memcpy(dst, src, n);
    return;
  }
  // ceiling quotient, rounded up to 4 KiB: parts * per >= n, so the parts cover every byte
  const std::size_t per = ((n + parts - 1) / parts + 4095) & ~std::size_t(4095);
  {
    std::lock_guard<std::mutex> lk(mu_);
    dst_ = dst;
    src_ = src;
    n_ = n;
    per_ = per;
    pending_ = int(th_.size());
    ++gen_;
  }
  go_.notify_all();
  std::memcpy(dst, src, std::min(per, n));  // part 0 on the calling thread
  std::unique_lock<std::mutex> lk(mu_);
  done_.wait(lk, [this] { return pending_ == 0; });
}

void CopyPool::worker(int i) {
  unsigned long long seen = 0;
  for (;;) {
    char* dst;
    const char* src;
    std::size_t n, per;
    {
      std::unique_lock<std::mutex> lk(mu_);
      go_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      dst = dst_;
      src = src_;
      n = n_;
      per = per_;
    }
    const std::size_t off = per * std::size_t(i + 1);
    if (off < n) std::memcpy(dst + off, src + off, std::min(per, n - off));
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
}

namespace {

bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

constexpr std::size_t kStageMin = std::size_t(4) << 20;  // below this the driver's own path is as fast

}  // namespace

void Engine::ensure_staging() {
  if (stage_[0]) return;
  for (int s = 0; s < kStageSlots; ++s) {
    cuda_check(cudaMallocHost(&stage_[s], kStageSlot), "cudaMallocHost");
    cuda_check(cudaEventCreateWithFlags(&stage_ev_[s], cudaEventDisableTiming), "cudaEventCreate");
  }
  int threads = 4;
  if (const char* e = std::getenv("DECMUL_COPY_THREADS")) threads = std::max(0, std::atoi(e));
  threads = std::min<int>(threads, std::max(1u, std::thread::hardware_concurrency()) - 1);
  copy_pool_ = std::make_unique<CopyPool>(std::max(0, threads));
}

void Engine::stage_h2d(void* dst, const void* src, std::size_t n, cudaStream_t st) {
  if (n < kStageMin || is_pinned(src)) {
    cuda_check(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st), "h2d");
    return;
  }
  ensure_staging();
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  for (std::size_t off = 0, c = 0; off < n; off += kStageSlot, ++c) {
    const int k = int(c % kStageSlots);
    const std::size_t len = std::min(kStageSlot, n - off);
    cuda_check(cudaEventSynchronize(stage_ev_[k]), "stage wait");  // the slot's previous DMA is done
    copy_pool_->copy(stage_[k], s + off, len);
    cuda_check(cudaMemcpyAsync(d + off, stage_[k], len, cudaMemcpyHostToDevice, st), "h2d");
    cuda_check(cudaEventRecord(stage_ev_[k], st), "event");
  }
}

void Engine::stage_d2h(void* dst, const void* src, std::size_t n, cudaStream_t st) {
  if (n < kStageMin || is_pinned(dst)) {
    cuda_check(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st), "d2h");
    cuda_check(cudaStreamSynchronize(st), "sync");
    return;
  }
  ensure_staging();
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  const std::size_t nch = (n + kStageSlot - 1) / kStageSlot;
  auto len = [&](std::size_t c) { return std::min(kStageSlot, n - c * kStageSlot); };
  auto issue = [&](std::size_t c) {
    const int k = int(c % kStageSlots);
    cuda_check(cudaMemcpyAsync(stage_[k], s + c * kStageSlot, len(c), cudaMemcpyDeviceToHost, st), "d2h");
    cuda_check(cudaEventRecord(stage_ev_[k], st), "event");
  };
  std::size_t issued = 0;
  for (; issued < std::min<std::size_t>(kStageSlots, nch); ++issued) issue(issued);
  for (std::size_t c = 0; c < nch; ++c) {
    const int k = int(c % kStageSlots);
    cuda_check(cudaEventSynchronize(stage_ev_[k]), "stage wait");
    copy_pool_->copy(d + c * kStageSlot, stage_[k], len(c));
    if (issued < nch) issue(issued++);  // refills slot k, whose data has just been copied out
  }
}

}  // namespace dmg
