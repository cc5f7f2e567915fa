// extern "C" implementation of include/decmul_gpu.h over dmg::Engine.
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>
#include <new>
#include <string>
#include <thread>

#include "../../include/decmul_gpu.h"
#include "engine.hpp"
#include "multi.hpp"

// One pending small product of the coalescing path (decmul_gpu_multiply from several threads).
struct CoalescedReq {
  const char* x;
  size_t nx;
  const char* y;
  size_t ny;
  char* out;
  size_t cap;
  size_t len = 0;
  int rc = 0;
  std::string msg;
  bool done = false;
};

struct decmul_gpu_ctx {
  std::unique_ptr<dmg::MultiEngine> multi;  // one engine per device of the context
  dmg::Engine* eng = nullptr;               // the first device's engine (device-pointer calls, hooks)
  std::mutex mu;
  std::string err;
  // coalescing of concurrent small products (leader/follower): callers queue their product;
  // the first becomes the leader, takes the context lock (waiting out the batch in flight,
  // while more callers queue) and runs everything queued as one batch (one k_small launch
  // per size group); followers sleep until their result is in
  std::mutex qmu;
  std::condition_variable qcv;
  std::vector<CoalescedReq*> queue;
  bool leader = false;
  unsigned long long coalesced_batches = 0, coalesced_products = 0;
  size_t last_batch = 0;                             // size and end of the last coalesced batch
  std::chrono::steady_clock::time_point last_end{};  // (under mu)
  std::atomic<int> large_active{0};  // large host products inside decmul_gpu_multiply[_ex] right now
};

namespace {

thread_local std::string g_create_err;

// Runs f, mapping exceptions to error codes; the message goes to msg.
template <class F>
int guarded_msg(std::string& msg, F&& f) {
  int rc = DECMUL_OK;
  try {
    f();
    return DECMUL_OK;
  } catch (const dmg::OperandTooLarge& e) {
    rc = DECMUL_ETOOLARGE;
    msg = e.what();
  } catch (const std::invalid_argument& e) {
    rc = DECMUL_EINVAL;
    msg = e.what();
  } catch (const std::length_error& e) {
    rc = DECMUL_ESPACE;
    msg = e.what();
  } catch (const dmg::CudaError& e) {
    msg = e.what();
    rc = msg.find("out of memory") != std::string::npos ? DECMUL_ENOMEM : DECMUL_ECUDA;
  } catch (const std::bad_alloc& e) {
    rc = DECMUL_ENOMEM;
    msg = e.what();
  } catch (const std::logic_error& e) {
    rc = DECMUL_ELOGIC;
    msg = e.what();
  } catch (const std::runtime_error& e) {
    rc = DECMUL_ECORRUPT;
    msg = e.what();
  } catch (const std::exception& e) {
    rc = DECMUL_ECUDA;
    msg = e.what();
  }
  return rc;
}

// The same with the message stored in the context (the caller holds its lock) or, without a
// context, in the thread's creation-error slot.
template <class F>
int guarded(decmul_gpu_ctx* ctx, F&& f) {
  std::string msg;
  const int rc = guarded_msg(msg, f);
  if (rc == DECMUL_OK) return rc;
  if (ctx)
    ctx->err = msg;
  else
    g_create_err = msg;
  return rc;
}

// The calling thread's current device is switched to the context's for the call and restored
// after it, so contexts on different GPUs can be used from one thread (allocations, streams
// and kernel attributes all follow the current device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
    }
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

#define LOCKED(ctx, ...)                                     \
  do {                                                       \
    if (!(ctx)) return DECMUL_EINVAL;                        \
    std::lock_guard<std::mutex> lock_((ctx)->mu);            \
    DeviceGuard dev_((ctx)->eng->device());                  \
    return guarded((ctx), [&] { __VA_ARGS__; });             \
  } while (0)

}  // namespace

extern "C" {

int decmul_gpu_create(decmul_gpu_ctx** ctx, int device) { return decmul_gpu_create_multi(ctx, &device, 1); }

int decmul_gpu_create_multi(decmul_gpu_ctx** ctx, const int* devices, int n) {
  if (!ctx || !devices || n < 1) return DECMUL_EINVAL;
  *ctx = nullptr;
  return guarded(nullptr, [&] {
    DeviceGuard dev(devices[0]);
    auto c = std::make_unique<decmul_gpu_ctx>();
    c->multi = std::make_unique<dmg::MultiEngine>(devices, n);
    c->eng = &c->multi->primary();
    *ctx = c.release();
  });
}

int decmul_gpu_context_devices(decmul_gpu_ctx* ctx, int* devices, int cap, int* n) {
  LOCKED(ctx, {
    const std::vector<int> d = ctx->multi->devices();
    if (n) *n = int(d.size());
    for (int i = 0; devices && i < cap && i < int(d.size()); ++i) devices[i] = d[i];
  });
}

void decmul_gpu_destroy(decmul_gpu_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard dev(ctx->eng->device());
  ctx->eng = nullptr;
  delete ctx;
}

const char* decmul_gpu_last_error(const decmul_gpu_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

int decmul_gpu_device_count(int* count) {
  return guarded(nullptr, [&] { dmg::cuda_check(cudaGetDeviceCount(count), "cudaGetDeviceCount"); });
}

int decmul_gpu_select_base_and_length(size_t dx, size_t dy, uint64_t p1, uint64_t p2, unsigned forced,
                                      unsigned* base_exp, size_t* length) {
  return guarded(nullptr, [&] {
    dmg::BasePlan bp = dmg::select_base_and_length(dx, dy, p1 ? p1 : dmg::kP1, p1 ? p2 : dmg::kP2, forced);
    *base_exp = bp.base_exp;
    *length = bp.length;
  });
}

int decmul_gpu_smallest_supported_length(size_t need, uint64_t p1, uint64_t p2, size_t* length) {
  return guarded(nullptr, [&] {
    *length = dmg::smallest_supported_length(need, p1 ? p1 : dmg::kP1, p1 ? p2 : dmg::kP2);
  });
}

int decmul_gpu_plan(decmul_gpu_ctx* ctx, size_t dx, size_t dy, unsigned forced, decmul_gpu_plan_info* info) {
  LOCKED(ctx, {
    dmg::ProductPlan pp = ctx->eng->plan_product(dx, dy, forced);
    info->base_exp = pp.base_exp;
    info->length = pp.N;
    info->p1 = pp.p1;
    info->p2 = pp.p2;
    info->large_pair = pp.large_pair ? 1 : 0;
    const int three = pp.N % 3 == 0;
    const size_t c = three ? pp.N / 3 : pp.N;
    info->one_cta = __builtin_ctzll(c) <= dmg::small_max_logc(three) ? 1 : 0;
  });
}

namespace {

// Products that run as one CTA each (the batch kernel): worth coalescing across threads.
bool coalescable(size_t nx, size_t ny, unsigned forced, int alias) {
  if (forced || alias || nx < 2 || ny < 2) return false;
  const char* e = std::getenv("DECMUL_COALESCE");
  if (e && e[0] == '0') return false;
  try {
    const dmg::PairChoice pc = dmg::choose_pair(nx, ny, 0, true);
    const size_t N = pc.bp.length;
    const int three = N % 3 == 0;
    const size_t c = three ? N / 3 : N;
    return __builtin_ctzll(c) <= dmg::small_max_logc(three);
  } catch (const std::exception&) {
    return false;
  }
}

// Runs the queued products as a batch (the caller holds ctx->mu); on any failure every product
// is rerun on its own so each caller gets its own result or error.
void run_coalesced(decmul_gpu_ctx* ctx, std::vector<CoalescedReq*>& batch) {
  const size_t n = batch.size();
  std::vector<const char*> xs(n), ys(n);
  std::vector<char*> outs(n);
  std::vector<size_t> nxs(n), nys(n), caps(n), lens(n);
  for (size_t i = 0; i < n; ++i) {
    xs[i] = batch[i]->x;
    ys[i] = batch[i]->y;
    outs[i] = batch[i]->out;
    nxs[i] = batch[i]->nx;
    nys[i] = batch[i]->ny;
    caps[i] = batch[i]->cap;
  }
  const int rc = guarded(ctx, [&] {
    ctx->multi->multiply_batch_ptrs(n, xs.data(), nxs.data(), ys.data(), nys.data(), outs.data(), caps.data(),
                                    lens.data());
  });
  if (rc == DECMUL_OK) {
    for (size_t i = 0; i < n; ++i) batch[i]->len = lens[i];
    return;
  }
  for (CoalescedReq* r : batch) {
    r->rc = guarded(ctx, [&] { r->len = ctx->multi->multiply_host(r->x, r->nx, r->y, r->ny, r->out, r->cap, 0, false); });
    if (r->rc) r->msg = ctx->err;
  }
}

int multiply_coalesced(decmul_gpu_ctx* ctx, const char* x, size_t nx, const char* y, size_t ny, char* out, size_t cap,
                       size_t* out_len) {
  CoalescedReq req{x, nx, y, ny, out, cap};
  {
    std::unique_lock<std::mutex> q(ctx->qmu);
    ctx->queue.push_back(&req);
    if (ctx->leader) {  // follower: the current or next leader runs this product
      ctx->qcv.wait(q, [&] { return req.done; });
      q.unlock();  // before taking ctx->mu: a leader holds mu while it takes qmu to swap the queue
      if (req.rc) {
        std::lock_guard<std::mutex> lk(ctx->mu);
        ctx->err = req.msg;
      }
      *out_len = req.len;
      return req.rc;
    }
    ctx->leader = true;
  }
  std::vector<CoalescedReq*> batch;
  {
    // waits for the batch in flight; callers keep queueing
    std::unique_lock<std::mutex> lock_(ctx->mu, std::try_to_lock);
    const bool waited = !lock_.owns_lock();
    if (waited) lock_.lock();
    DeviceGuard dev_(ctx->eng->device());
    // Callers in a closed loop come back right after their batch: give them a moment to queue up,
    // so that all of them share the next launch instead of two groups taking turns. Expected
    // callers: the batch that has just ended, plus -- when this leader had to wait for it -- the
    // callers that queued meanwhile. DECMUL_COALESCE_WAIT_US=0 turns the wait off.
    static const int wait_us = [] {
      const char* e = std::getenv("DECMUL_COALESCE_WAIT_US");
      return e ? std::atoi(e) : 40;
    }();
    const auto now = std::chrono::steady_clock::now();
    if (wait_us > 0 && ctx->last_batch > 1 && now - ctx->last_end < std::chrono::milliseconds(1)) {
      size_t queued = 0;
      {
        std::lock_guard<std::mutex> q(ctx->qmu);
        queued = ctx->queue.size();
      }
      // (only while the batches are small, where the fixed cost of a launch dominates: measured
      // with 1e4-digit products, 2 threads 20.8k -> 26.0k products/s, 4 threads 29.7k -> 42.3k,
      // but 16 threads 78k -> 51k when batches of 8 wait as well)
      const size_t target = ctx->last_batch + queued < 8 ? (waited ? ctx->last_batch + queued : ctx->last_batch) : 0;
      const auto deadline = now + std::chrono::microseconds(wait_us);
      while (queued < target && std::chrono::steady_clock::now() < deadline) {
        std::this_thread::yield();
        std::lock_guard<std::mutex> q(ctx->qmu);
        queued = ctx->queue.size();
      }
    }
    {
      std::lock_guard<std::mutex> q(ctx->qmu);
      batch.swap(ctx->queue);
      ctx->leader = false;  // the next caller leads the next batch
    }
    run_coalesced(ctx, batch);
    ++ctx->coalesced_batches;
    ctx->coalesced_products += batch.size();
    ctx->last_batch = batch.size();
    ctx->last_end = std::chrono::steady_clock::now();
    if (req.rc) ctx->err = req.msg;
  }
  {
    std::lock_guard<std::mutex> q(ctx->qmu);
    for (CoalescedReq* r : batch) r->done = true;
  }
  ctx->qcv.notify_all();
  *out_len = req.len;
  return req.rc;
}

// Counts the large host products in flight on a context (Engine::overlap_ok's `concurrent`).
struct LargeCall {
  std::atomic<int>* c = nullptr;
  int before = 0;
  LargeCall(decmul_gpu_ctx* ctx, size_t nx, size_t ny) {
    if (ctx && nx + ny >= (size_t(1) << 24)) {
      c = &ctx->large_active;
      before = c->fetch_add(1);
    }
  }
  ~LargeCall() {
    if (c) c->fetch_sub(1);
  }
};

// Large products from pinned buffers: the engine takes the context lock only around the
// compute stage, so concurrent callers overlap one product's download with the next one's
// upload and compute (Engine::multiply_host_overlapped). Returns false when the call does
// not qualify (the caller then runs the ordinary locked path).
bool multiply_overlapped(decmul_gpu_ctx* ctx, const char* x, size_t nx, const char* y, size_t ny, char* out,
                         size_t cap, size_t* out_len, unsigned forced, int alias, uint64_t p1, uint64_t p2,
                         bool concurrent, int* rc) {
  if (!ctx || !out_len) return false;
  DeviceGuard dev_(ctx->eng->device());
  dmg::Engine* e = nullptr;
  std::string msg;
  if (guarded_msg(msg, [&] { e = ctx->multi->overlap_engine(x, nx, y, ny, out, forced, concurrent, p1, p2); }) || !e)
    return false;
  *rc = guarded_msg(msg, [&] {
    *out_len = e->multiply_host_overlapped(ctx->mu, x, nx, y, ny, out, cap, forced, alias != 0, p1, p2);
  });
  if (*rc) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->err = msg;
  }
  return true;
}

}  // namespace

int decmul_gpu_multiply(decmul_gpu_ctx* ctx, const char* x, size_t nx, const char* y, size_t ny, char* out,
                        size_t cap, size_t* out_len, unsigned forced, int alias) {
  if (ctx && out_len && coalescable(nx, ny, forced, alias) && !(nx == ny && x == y)) {
    bool valid = cap >= nx + ny && x[0] != '0' && y[0] != '0';
    if (valid) return multiply_coalesced(ctx, x, nx, y, ny, out, cap, out_len);
  }
  LargeCall large(ctx, nx, ny);
  if (int rc = 0; multiply_overlapped(ctx, x, nx, y, ny, out, cap, out_len, forced, alias, 0, 0, large.before > 0, &rc))
    return rc;
  LOCKED(ctx, {
    if (nx == 0 || ny == 0) throw std::invalid_argument("decimal: empty string");
    const bool xz = nx == 1 && x[0] == '0', yz = ny == 1 && y[0] == '0';
    if (xz || yz) {  // decimal.cpp:193, after DecimalNumber::parse validated both texts
      for (size_t i = 0; i < nx; ++i)
        if (x[i] < '0' || x[i] > '9') throw std::invalid_argument("decimal: non-digit character");
      for (size_t i = 0; i < ny; ++i)
        if (y[i] < '0' || y[i] > '9') throw std::invalid_argument("decimal: non-digit character");
      if ((nx > 1 && x[0] == '0') || (ny > 1 && y[0] == '0')) throw std::invalid_argument("decimal: leading zero");
      if (cap < 1) throw std::length_error("multiply: output buffer too small");
      out[0] = '0';
      *out_len = 1;
      return;
    }
    *out_len = ctx->multi->multiply_host(x, nx, y, ny, out, cap, forced, alias != 0);
  });
}

int decmul_gpu_multiply_ex(decmul_gpu_ctx* ctx, const char* x, size_t nx, const char* y, size_t ny, char* out,
                           size_t cap, size_t* out_len, const decmul_gpu_multiply_options* opt) {
  // no options that change the plan: the same path as decmul_gpu_multiply (coalescing of
  // concurrent small products, overlapped transfers of concurrent large ones). The C++
  // drop-in's decmul::multiply always calls this entry point.
  if (!opt || (!opt->forced_base_exp && !opt->p1 && !opt->p2))
    return decmul_gpu_multiply(ctx, x, nx, y, ny, out, cap, out_len, 0, opt ? opt->alias : 0);
  LargeCall large(ctx, nx, ny);
  if (int rc = 0; multiply_overlapped(ctx, x, nx, y, ny, out, cap, out_len, opt->forced_base_exp, opt->alias, opt->p1,
                                      opt->p2, large.before > 0, &rc))
    return rc;
  LOCKED(ctx, {
    const decmul_gpu_multiply_options o = opt ? *opt : decmul_gpu_multiply_options{0, 0, 0, 0};
    if (nx == 0 || ny == 0) throw std::invalid_argument("decimal: empty string");
    const bool xz = nx == 1 && x[0] == '0', yz = ny == 1 && y[0] == '0';
    if (xz || yz) {  // decimal.cpp:193, after DecimalNumber::parse validated both texts
      for (size_t i = 0; i < nx; ++i)
        if (x[i] < '0' || x[i] > '9') throw std::invalid_argument("decimal: non-digit character");
      for (size_t i = 0; i < ny; ++i)
        if (y[i] < '0' || y[i] > '9') throw std::invalid_argument("decimal: non-digit character");
      if ((nx > 1 && x[0] == '0') || (ny > 1 && y[0] == '0')) throw std::invalid_argument("decimal: leading zero");
      if (cap < 1) throw std::length_error("multiply: output buffer too small");
      out[0] = '0';
      *out_len = 1;
      return;
    }
    *out_len = ctx->multi->multiply_host(x, nx, y, ny, out, cap, o.forced_base_exp, o.alias != 0, o.p1, o.p2);
  });
}

int decmul_gpu_multiply_sharded(decmul_gpu_ctx* ctx, const char* x, size_t nx, const char* y, size_t ny, char* out,
                                size_t cap, size_t* out_len, int alias) {
  LOCKED(ctx, {
    if (nx == 0 || ny == 0) throw std::invalid_argument("decimal: empty string");
    if ((nx > 1 && x[0] == '0') || (ny > 1 && y[0] == '0')) throw std::invalid_argument("decimal: leading zero");
    const bool sq = alias != 0 || (nx == ny && (x == y || std::memcmp(x, y, nx) == 0));
    *out_len = ctx->multi->sharded_multiply(x, nx, y, ny, out, cap, sq);
  });
}

int decmul_gpu_multiply_device(decmul_gpu_ctx* ctx, const char* d_x, size_t nx, const char* d_y, size_t ny,
                               char* d_out, size_t cap, size_t* out_len, unsigned forced, int squaring,
                               void* stream) {
  LOCKED(ctx, {
    const bool sq = squaring != 0 || (d_x == d_y && nx == ny);
    const size_t len = ctx->eng->multiply_device(d_x, nx, d_y, ny, d_out, cap, forced, sq,
                                                 static_cast<cudaStream_t>(stream), out_len != nullptr);
    if (out_len) *out_len = len;
  });
}

int decmul_gpu_result_length(decmul_gpu_ctx* ctx, size_t* out_len) {
  LOCKED(ctx, {
    *out_len = ctx->eng->result_length();
  });
}

int decmul_gpu_multiply_batch(decmul_gpu_ctx* ctx, size_t count, const char* xs, size_t x_stride, size_t nx,
                              const char* ys, size_t y_stride, size_t ny, char* outs, size_t out_stride,
                              size_t* out_lens) {
  // the engine may release the context lock once a large pinned batch is enqueued, so that
  // batches from several threads overlap (Engine::batch_host_pipelined)
  if (!ctx) return DECMUL_EINVAL;
  std::unique_lock<std::mutex> lock_(ctx->mu);
  DeviceGuard dev_(ctx->eng->device());
  std::string msg;
  const int rc = guarded_msg(msg, [&] {
    ctx->multi->multiply_batch_host(count, xs, x_stride, nx, ys, y_stride, ny, outs, out_stride, out_lens, &lock_);
  });
  if (rc) {
    if (!lock_.owns_lock()) lock_.lock();
    ctx->err = msg;
  }
  return rc;
}

int decmul_gpu_multiply_batch_ptrs(decmul_gpu_ctx* ctx, size_t count, const char* const* xs, const size_t* nxs,
                                   const char* const* ys, const size_t* nys, char* const* outs, const size_t* caps,
                                   size_t* out_lens) {
  LOCKED(ctx, ctx->multi->multiply_batch_ptrs(count, xs, nxs, ys, nys, outs, caps, out_lens));
}

int decmul_gpu_multiply_batch_device(decmul_gpu_ctx* ctx, size_t count, const char* d_xs, size_t x_stride,
                                     size_t nx, const char* d_ys, size_t y_stride, size_t ny, char* d_outs,
                                     size_t out_stride, unsigned long long* d_lens, void* stream) {
  LOCKED(ctx, ctx->eng->multiply_batch_device(count, d_xs, x_stride, nx, d_ys, y_stride, ny, d_outs, out_stride,
                                               d_lens, static_cast<cudaStream_t>(stream)));
}

int decmul_gpu_convolve_mod_p(decmul_gpu_ctx* ctx, uint64_t p, size_t n, const uint64_t* x, size_t nx,
                              const uint64_t* y, size_t ny, uint64_t* out) {
  LOCKED(ctx, ctx->eng->convolve_mod_p(p, n, reinterpret_cast<const dmg::u64*>(x), nx,
                                       reinterpret_cast<const dmg::u64*>(y), ny, reinterpret_cast<dmg::u64*>(out)));
}

int decmul_gpu_forward_transform(decmul_gpu_ctx* ctx, uint64_t p, size_t n, uint64_t* a) {
  LOCKED(ctx, ctx->eng->forward_transform(p, n, reinterpret_cast<dmg::u64*>(a)));
}

int decmul_gpu_inverse_transform(decmul_gpu_ctx* ctx, uint64_t p, size_t n, uint64_t* a) {
  LOCKED(ctx, ctx->eng->inverse_transform(p, n, reinterpret_cast<dmg::u64*>(a)));
}

int decmul_gpu_forward_transform_ex(decmul_gpu_ctx* ctx, uint64_t p, size_t n, size_t six_step_threshold,
                                    uint64_t* a) {
  LOCKED(ctx, ctx->eng->forward_transform(p, n, reinterpret_cast<dmg::u64*>(a), six_step_threshold));
}

int decmul_gpu_inverse_transform_ex(decmul_gpu_ctx* ctx, uint64_t p, size_t n, size_t six_step_threshold,
                                    uint64_t* a) {
  LOCKED(ctx, ctx->eng->inverse_transform(p, n, reinterpret_cast<dmg::u64*>(a), six_step_threshold));
}

int decmul_gpu_conv_plan_info(uint64_t p, size_t n, size_t six_step_threshold, int* shape, uint64_t* root,
                              size_t* n1, size_t* n2) {
  return guarded(nullptr, [&] {
    const size_t c = n % 3 == 0 ? n / 3 : n;
    const bool three = n % 3 == 0 && n > 0 && !(c & (c - 1));
    const bool pow2 = n > 0 && !(n & (n - 1));
    if (!pow2 && !three) throw std::invalid_argument("build_conv_plan: length must be 2^k or 3*2^k");
    if (n > 1 && (p - 1) % n) throw std::invalid_argument("build_conv_plan: length does not divide p-1");
    const size_t thr = six_step_threshold ? six_step_threshold : size_t(1) << 15;
    dmg::HostField F(p);
    if (root) *root = F.root_of_unity(n);
    size_t a = 0, b = 0;
    int sh = 0;
    if (three) {
      sh = 2;
    } else if (n > thr) {
      sh = 1;
      a = size_t(1) << (__builtin_ctzll(n) / 2);
      b = n / a;
    }
    if (shape) *shape = sh;
    if (n1) *n1 = a;
    if (n2) *n2 = b;
  });
}

int decmul_gpu_pointwise_product(decmul_gpu_ctx* ctx, uint64_t p, size_t n, uint64_t* a, const uint64_t* b) {
  LOCKED(ctx, ctx->eng->pointwise_product(p, n, reinterpret_cast<dmg::u64*>(a), reinterpret_cast<const dmg::u64*>(b)));
}

int decmul_gpu_pack(decmul_gpu_ctx* ctx, const char* digits, size_t nd, unsigned base_exp, uint64_t* limbs,
                    size_t cap, size_t* nlimbs) {
  LOCKED(ctx, *nlimbs = ctx->eng->pack(digits, nd, base_exp, reinterpret_cast<dmg::u64*>(limbs), cap));
}

int decmul_gpu_recover_decimal(decmul_gpu_ctx* ctx, const uint64_t* r1, const uint64_t* r2, size_t n, uint64_t p1,
                               uint64_t p2, unsigned base_exp, size_t min_limbs, size_t digits_sum, char* out,
                               size_t cap, size_t* out_len) {
  LOCKED(ctx, *out_len = ctx->eng->recover_decimal(reinterpret_cast<const dmg::u64*>(r1),
                                                   reinterpret_cast<const dmg::u64*>(r2), n, p1, p2, base_exp,
                                                   min_limbs, digits_sum, out, cap));
}

int decmul_gpu_transpose_square_sub(decmul_gpu_ctx* ctx, uint64_t* a, size_t n, size_t stride) {
  LOCKED(ctx, ctx->eng->transpose(0, reinterpret_cast<dmg::u64*>(a), n, stride));
}
int decmul_gpu_transpose_n_x_2n(decmul_gpu_ctx* ctx, uint64_t* a, size_t n) {
  LOCKED(ctx, ctx->eng->transpose(1, reinterpret_cast<dmg::u64*>(a), n, 2 * n));
}
int decmul_gpu_transpose_2n_x_n(decmul_gpu_ctx* ctx, uint64_t* a, size_t n) {
  LOCKED(ctx, ctx->eng->transpose(2, reinterpret_cast<dmg::u64*>(a), n, n));
}

}  // extern "C"

namespace {
dmg::ShardPlan shard_from(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* p) {
  if (!p) throw std::invalid_argument("shard: null plan");
  return ctx->eng->shard_plan(p->digits_x, p->digits_y, p->ranks);
}
cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }
}  // namespace

extern "C" {

static void fill_shard_plan(const dmg::ShardPlan& sp, size_t dx, size_t dy, decmul_gpu_shard_plan* out);

// ctx == NULL plans on the host only (no device tables), e.g. for CPU-side drivers.
int decmul_gpu_shard_plan_create(decmul_gpu_ctx* ctx, size_t dx, size_t dy, int ranks, decmul_gpu_shard_plan* out) {
  if (!ctx) return guarded(nullptr, [&] { fill_shard_plan(dmg::make_shard_plan(dx, dy, ranks), dx, dy, out); });
  LOCKED(ctx, fill_shard_plan(ctx->eng->shard_plan(dx, dy, ranks), dx, dy, out));
}

static void fill_shard_plan(const dmg::ShardPlan& sp, size_t dx, size_t dy, decmul_gpu_shard_plan* out) {
  {
    out->length = sp.pp.N;
    out->base_exp = sp.pp.base_exp;
    out->p1 = sp.pp.p1;
    out->p2 = sp.pp.p2;
    out->ranks = sp.geom.G;
    out->col_passes = sp.geom.K;
    out->rows = sp.geom.Rtot;
    out->seg_len = sp.geom.Sc;
    out->col_width = sp.geom.Bc;
    out->local_len = sp.geom.local_len;
    const size_t K = sp.geom.local_len + 2, ch = size_t(dmg::kCarryChunk);
    out->s_words = (K + ch - 1) / ch * ch;
    out->map_words = (K + ch - 1) / ch;
    out->digits_x = dx;
    out->digits_y = dy;
    out->top_candidates[0] = sp.top_candidates[0];
    out->top_candidates[1] = sp.top_candidates[1];
  }
}

int decmul_gpu_shard_pack(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* plan, int rank, const char* d_digits,
                          size_t nd, uint64_t* d_out, void* stream) {
  LOCKED(ctx, ctx->eng->shard_pack(shard_from(ctx, plan), rank, d_digits, nd, reinterpret_cast<dmg::u64*>(d_out),
                                   as_stream(stream)));
}

int decmul_gpu_shard_transform(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* plan, int rank, int stage,
                               const uint64_t* s1, const uint64_t* s2, uint64_t* d1, uint64_t* d2,
                               const uint64_t* o1, const uint64_t* o2, void* stream) {
  LOCKED(ctx, {
    const dmg::u64* src[2] = {reinterpret_cast<const dmg::u64*>(s1), reinterpret_cast<const dmg::u64*>(s2)};
    dmg::u64* dst[2] = {reinterpret_cast<dmg::u64*>(d1), reinterpret_cast<dmg::u64*>(d2)};
    const dmg::u64* oth[2] = {reinterpret_cast<const dmg::u64*>(o1), reinterpret_cast<const dmg::u64*>(o2)};
    ctx->eng->shard_transform(shard_from(ctx, plan), rank, stage, src, dst, o1 ? oth : nullptr, as_stream(stream));
  });
}

int decmul_gpu_shard_reorder(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* plan, int to_segments,
                             const uint64_t* src, uint64_t* dst, void* stream) {
  LOCKED(ctx, ctx->eng->shard_reorder(shard_from(ctx, plan), to_segments != 0, reinterpret_cast<const dmg::u64*>(src),
                                      reinterpret_cast<dmg::u64*>(dst), as_stream(stream)));
}

int decmul_gpu_shard_carry_begin(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* plan, int rank,
                                 const uint64_t* z1, const uint64_t* z2, const uint64_t halo[4], uint64_t* d_s,
                                 unsigned* d_maps, unsigned* rank_map, void* stream) {
  LOCKED(ctx, {
    const dmg::u64 h1[2] = {halo[0], halo[1]}, h2[2] = {halo[2], halo[3]};
    *rank_map = ctx->eng->shard_carry_begin(shard_from(ctx, plan), rank, reinterpret_cast<const dmg::u64*>(z1),
                                            reinterpret_cast<const dmg::u64*>(z2), h1, h2,
                                            reinterpret_cast<dmg::u64*>(d_s), d_maps, as_stream(stream));
  });
}

int decmul_gpu_shard_carry_probe(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* plan, int rank, unsigned cin,
                                 const uint64_t* z1, const uint64_t* z2, const uint64_t* d_s, unsigned* d_maps,
                                 uint64_t z_out[2], void* stream) {
  LOCKED(ctx, {
    dmg::u64 z[2];
    ctx->eng->shard_carry_probe(shard_from(ctx, plan), rank, cin, reinterpret_cast<const dmg::u64*>(z1),
                                reinterpret_cast<const dmg::u64*>(z2), reinterpret_cast<const dmg::u64*>(d_s),
                                d_maps, z, as_stream(stream));
    z_out[0] = z[0];
    z_out[1] = z[1];
  });
}

int decmul_gpu_shard_carry_emit(decmul_gpu_ctx* ctx, const decmul_gpu_shard_plan* plan, int rank, unsigned cin,
                                unsigned long long top, unsigned top_len, const uint64_t* z1, const uint64_t* z2,
                                const uint64_t* d_s, unsigned* d_maps, char* d_out, void* stream) {
  LOCKED(ctx, ctx->eng->shard_carry_emit(shard_from(ctx, plan), rank, cin, top, top_len,
                                         reinterpret_cast<const dmg::u64*>(z1), reinterpret_cast<const dmg::u64*>(z2),
                                         reinterpret_cast<const dmg::u64*>(d_s), d_maps, d_out, as_stream(stream)));
}

int decmul_gpu_generate_digits(decmul_gpu_ctx* ctx, uint64_t seed0, uint64_t seed_step, size_t count, size_t n,
                               size_t stride, int mode, char* d_out, void* stream) {
  LOCKED(ctx, {
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->eng->stream();
    dmg::launch_generate(seed0, seed_step, count, n, stride, mode, d_out, st);
    dmg::cuda_check(cudaGetLastError(), "generate");
  });
}

int decmul_gpu_measure_modmul_rate(decmul_gpu_ctx* ctx, int variant, double* rate) {
  LOCKED(ctx, {
    *rate = dmg::measure_modmul_rate(variant, ctx->eng->stream());
    if (*rate <= 0) throw dmg::CudaError("modmul rate measurement failed");
  });
}

int decmul_gpu_selftest(decmul_gpu_ctx* ctx, int inject_fault, char* report, size_t cap, int* failures) {
  LOCKED(ctx, {
    std::string r;
    const int f = ctx->eng->selftest(inject_fault != 0, r);
    if (failures) *failures = f;
    if (report && cap) {
      const size_t n = r.size() < cap - 1 ? r.size() : cap - 1;
      std::memcpy(report, r.data(), n);
      report[n] = '\0';
    }
  });
}

int decmul_gpu_coalesce_stats(decmul_gpu_ctx* ctx, unsigned long long* batches, unsigned long long* products) {
  LOCKED(ctx, {
    if (batches) *batches = ctx->coalesced_batches;
    if (products) *products = ctx->coalesced_products;
  });
}

int decmul_gpu_check_errors(decmul_gpu_ctx* ctx, void* stream) {
  LOCKED(ctx, ctx->eng->check_async_errors(static_cast<cudaStream_t>(stream)));
}

int decmul_gpu_profile(decmul_gpu_ctx* ctx, int enable) { LOCKED(ctx, ctx->eng->profile_enable(enable != 0)); }

int decmul_gpu_profile_report(decmul_gpu_ctx* ctx, char* report, size_t cap, size_t* len) {
  LOCKED(ctx, {
    const std::string r = ctx->eng->profile_report(report != nullptr);
    if (len) *len = r.size();
    if (report && cap) {
      const size_t n = r.size() < cap - 1 ? r.size() : cap - 1;
      std::memcpy(report, r.data(), n);
      report[n] = '\0';
    }
  });
}

int decmul_gpu_get_stats(decmul_gpu_ctx* ctx, decmul_gpu_stats* out) {
  LOCKED(ctx, {
    out->last_launches = ctx->eng->last_launches();
    out->table_bytes = ctx->eng->table_bytes();
  });
}

}  // extern "C"
