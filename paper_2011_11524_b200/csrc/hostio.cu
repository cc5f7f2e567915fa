// Host <-> device transfers for the host-buffer API (the drop-in decmul::multiply with
// std::string operands): pinned buffers go straight to the DMA engines;
// large pageable ones are pipelined through a ring of pinned slots, the host threads of
// a CopyPool filling (or draining) slot c while the DMA engine moves slot c - 1.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>

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

// ---- overlapped host products (concurrent callers, pinned buffers) ----
// Below kOverlapMin digits the transfers are too short to matter; above kOverlapMax the four
// extra digit buffers (2 slots x (inputs + output)) would not fit beside a config-5-size plan.
constexpr std::size_t kOverlapMin = std::size_t(1) << 24;
constexpr std::size_t kOverlapMax = std::size_t(4) << 30;

bool Engine::overlap_ok(const char* x, std::size_t nx, const char* y, std::size_t ny, const char* out,
                        bool concurrent) const {
  if (const char* e = std::getenv("DECMUL_OVERLAP"))
    if (e[0] == '0') return false;
  if (nx == 0 || ny == 0 || !x || !y || !out) return false;
  const std::size_t n = nx + ny;
  if (n < kOverlapMin || n > kOverlapMax) return false;
  // pinned buffers go straight to DMA. Pageable ones move through the stages' own staging rings
  // (192 MB of pinned memory, ~45 ms to set up), so they take this path only while another
  // large call is in flight on the context; a lone caller keeps the locked path and its one ring.
  return concurrent || (is_pinned(x) && is_pinned(y) && is_pinned(out));
}

std::size_t Engine::multiply_host_overlapped(std::mutex& ctx_mu, const char* x, std::size_t nx, const char* y,
                                             std::size_t ny, char* out, std::size_t cap, unsigned forced,
                                             bool alias, u64 p1, u64 p2) {
  const bool squaring = alias || (nx == ny && (x == y || std::memcmp(x, y, nx) == 0));
  const ProductPlan pp = plan_product(nx, ny, forced, p1, p2);
  if (cap < nx + ny) throw std::length_error("multiply: output buffer too small");
  // DECMUL_OVERLAP_TRACE=1: one stderr line of stage timestamps (ms since the call began)
  static const bool trace = [] {
    const char* e = std::getenv("DECMUL_OVERLAP_TRACE");
    return e && e[0] == '1';
  }();
  const auto t_begin = std::chrono::steady_clock::now();
  auto ms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_begin).count(); };
  double t_up = 0, t_dl = 0, t_comp = 0, t_enq = 0, t_ydone = 0, t_cdone = 0;
  // stage 1, uploads (in call order): x starts at once, also while the previous product computes
  std::unique_lock<std::mutex> up(ov_up_mu_);
  t_up = ms();
  if (!ov_up_stream_) {
    cuda_check(cudaStreamCreateWithFlags(&ov_up_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    for (OvSlot& s : ov_) {
      cuda_check(cudaStreamCreateWithFlags(&s.dl_stream, cudaStreamNonBlocking), "cudaStreamCreate");
      cuda_check(cudaEventCreateWithFlags(&s.ev_x, cudaEventDisableTiming), "cudaEventCreate");
      cuda_check(cudaEventCreateWithFlags(&s.ev_y, cudaEventDisableTiming), "cudaEventCreate");
      cuda_check(cudaMallocHost(&s.h_len, sizeof *s.h_len), "cudaMallocHost");
    }
  }
  OvSlot& s = ov_[ov_slot_ ^= 1];
  // the slot's inputs are free: its previous product finished computing before the product
  // after it could take the context lock, and that one released ov_up_mu_ only later
  s.dx.ensure(nx);
  if (!squaring) s.dy.ensure(ny);
  // from here on a DMA may be reading the caller's buffers: no error leaves this function
  // before the upload stream has drained
  struct DrainOnError {
    cudaStream_t st;
    int live = std::uncaught_exceptions();
    ~DrainOnError() {
      if (std::uncaught_exceptions() > live) cudaStreamSynchronize(st);
    }
  } drain{ov_up_stream_};
  ov_up_ring_.h2d(s.dx.ptr, x, nx, ov_up_stream_);
  cuda_check(cudaEventRecord(s.ev_x, ov_up_stream_), "event");
  // the slot's output buffer: wait out the download of the product that used it last
  std::unique_lock<std::mutex> dl(s.dl_mu);
  t_dl = ms();
  s.dout.ensure(nx + ny);
  // stage 2, compute, under the context lock (workspace, plans, error word)
  std::unique_lock<std::mutex> comp(ctx_mu);
  t_comp = ms();
  cudaStream_t st = stream_;
  cuda_check(cudaStreamWaitEvent(st, s.ev_x, 0), "wait");
  run_product(pp, s.dx.ptr, squaring ? s.dx.ptr : s.dy.ptr, squaring, s.dout.ptr, st, err_.ptr, [&] {
    if (squaring) return;
    ov_up_ring_.h2d(s.dy.ptr, y, ny, ov_up_stream_);
    cuda_check(cudaEventRecord(s.ev_y, ov_up_stream_), "event");
    cuda_check(cudaStreamWaitEvent(st, s.ev_y, 0), "wait");
  });
  // (into pinned memory: a copy to pageable memory would block this thread, and with it the
  // upload lock, until the whole product has been computed)
  cuda_check(cudaMemcpyAsync(s.h_len, meta_.ptr + 2, sizeof *s.h_len, cudaMemcpyDeviceToHost, st), "len");
  t_enq = ms();
  cuda_check(cudaEventSynchronize(squaring ? s.ev_x : s.ev_y), "upload wait");
  up.unlock();  // this product's digits are in HBM: the next call may upload
  t_ydone = ms();
  check_err(st);
  t_cdone = ms();
  const unsigned long long len = *s.h_len;
  if (len > cap) throw std::length_error("multiply: output buffer too small");
  comp.unlock();
  // stage 3, download, outside the context lock
  s.dl_ring.d2h(out, s.dout.ptr, std::size_t(len), s.dl_stream);
  if (trace)
    std::fprintf(stderr,
                 "overlap slot %d: up lock %.1f, out slot %.1f, ctx lock %.1f, enqueued %.1f, uploads done %.1f, "
                 "computed %.1f, downloaded %.1f ms\n",
                 int(&s - ov_), t_up, t_dl, t_comp, t_enq, t_ydone, t_cdone, ms());
  return std::size_t(len);
}

void PinnedBuf::ensure(size_t count) {
  if (count <= n) return;
  if (ptr) cudaFreeHost(ptr);
  ptr = nullptr;
  n = 0;
  const size_t want = std::max<size_t>(count + count / 2, size_t(1) << 20);
  cuda_check(cudaMallocHost(&ptr, want), "cudaMallocHost");
  n = want;
}

StageRing::~StageRing() {
  pool.reset();
  for (int k = 0; k < kSlots; ++k) {
    if (slot[k]) cudaFreeHost(slot[k]);
    if (ev[k]) cudaEventDestroy(ev[k]);
  }
}

void StageRing::ensure() {
  if (slot[0]) return;
  for (int k = 0; k < kSlots; ++k) {
    cuda_check(cudaMallocHost(&slot[k], kSlot), "cudaMallocHost");
    cuda_check(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming), "cudaEventCreate");
  }
  int threads = 4;
  if (const char* e = std::getenv("DECMUL_COPY_THREADS")) threads = std::max(0, std::atoi(e));
  threads = std::min<int>(threads, std::max(1u, std::thread::hardware_concurrency()) - 1);
  pool = std::make_unique<CopyPool>(std::max(0, threads));
}

void StageRing::h2d(void* dst, const void* src, std::size_t n, cudaStream_t st) {
  if (n < kStageMin || is_pinned(src)) {
    cuda_check(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st), "h2d");
    return;
  }
  ensure();
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  for (std::size_t off = 0, c = 0; off < n; off += kSlot, ++c) {
    const int k = int(c % kSlots);
    const std::size_t len = std::min(kSlot, n - off);
    cuda_check(cudaEventSynchronize(ev[k]), "stage wait");  // the slot's previous DMA is done
    pool->copy(slot[k], s + off, len);
    cuda_check(cudaMemcpyAsync(d + off, slot[k], len, cudaMemcpyHostToDevice, st), "h2d");
    cuda_check(cudaEventRecord(ev[k], st), "event");
  }
}

void StageRing::d2h(void* dst, const void* src, std::size_t n, cudaStream_t st) {
  if (n < kStageMin || is_pinned(dst)) {
    cuda_check(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st), "d2h");
    cuda_check(cudaStreamSynchronize(st), "sync");
    return;
  }
  ensure();
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  const std::size_t nch = (n + kSlot - 1) / kSlot;
  auto len = [&](std::size_t c) { return std::min(kSlot, n - c * kSlot); };
  auto issue = [&](std::size_t c) {
    const int k = int(c % kSlots);
    cuda_check(cudaMemcpyAsync(slot[k], s + c * kSlot, len(c), cudaMemcpyDeviceToHost, st), "d2h");
    cuda_check(cudaEventRecord(ev[k], st), "event");
  };
  std::size_t issued = 0;
  for (; issued < std::min<std::size_t>(kSlots, nch); ++issued) issue(issued);
  for (std::size_t c = 0; c < nch; ++c) {
    const int k = int(c % kSlots);
    cuda_check(cudaEventSynchronize(ev[k]), "stage wait");
    pool->copy(d + c * kSlot, slot[k], len(c));
    if (issued < nch) issue(issued++);  // refills slot k, whose data has just been copied out
  }
}

bool Engine::host_pinned(const void* p) { return is_pinned(p); }
bool Engine::stage_direct(const void* host, std::size_t n) const { return n < kStageMin || is_pinned(host); }
void Engine::stage_h2d(void* dst, const void* src, std::size_t n, cudaStream_t st) { ring_.h2d(dst, src, n, st); }
void Engine::stage_d2h(void* dst, const void* src, std::size_t n, cudaStream_t st) { ring_.d2h(dst, src, n, st); }

}  // namespace dmg
