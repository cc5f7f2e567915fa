// Multi-device context: one Engine per GPU of the context (SURVEY §8(b) "multi-GPU fan-out is
// hidden behind the context"; §8(e) partitioning), driven from one host thread.
//
//  * Batches of independent products split into contiguous ranges, one per device, each run
//    by that device's engine on its own host thread (no data-path exchange).
//  * One large product is sharded (§8(e) configs 4, 5): the first K passes run column-sharded
//    (rank q owns columns [q Bc, (q + 1) Bc) of the Rtot x Sc pass matrix), the rest on whole
//    segments; the layout changes are all-to-alls done as peer copies (cudaMemcpyPeerAsync over
//    NVLink between GPUs; plain device copies when ranks share a GPU), ordered by events; the
//    carries are resolved with per-rank {0,1,2}-carry maps. The sequence mirrors the reference's
//    six-step (conv.cpp:72-104) with its transposition as the exchange.
//
// Memory per rank ~ 1/G of the product: rank q receives only its digit slices (one 2-D copy per
// operand: the rows of its column block, compacted so that its local limb i is limb i of the
// slice string), holds N/G words per array, factorised twiddle tables (no R x S table), and only
// its own contiguous range of the product's digits.
#include <algorithm>
#include <cstring>
#include <thread>

#include "multi.hpp"

namespace dmg {

namespace {

// [lo, hi) of the product text printed by rank q (limbs [q L, (q + 1) L), top limb unpadded)
void rank_digit_range(std::size_t L, unsigned be, int q, std::size_t n, std::size_t& lo, std::size_t& hi) {
  const std::size_t top = (n - 1) / be, top_len = n - top * be;
  const std::size_t k_lo = std::size_t(q) * L, k_hi = std::min((std::size_t(q) + 1) * L - 1, top);
  if (k_lo > top) {
    lo = hi = n;
    return;
  }
  auto pos = [&](std::size_t k) { return k == top ? 0 : top_len + (top - 1 - k) * be; };
  lo = pos(k_hi);
  hi = pos(k_lo) + (k_lo == top ? top_len : be);
}

unsigned map_apply_h(unsigned m, unsigned c) { return (m >> (2 * c)) & 3u; }
unsigned map_compose_h(unsigned later, unsigned earlier) {
  unsigned r = 0;
  for (unsigned c = 0; c < 3; ++c) r |= map_apply_h(later, map_apply_h(earlier, c)) << (2 * c);
  return r;
}

unsigned decimal_len_h(u64 v) {
  unsigned n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}

}  // namespace

MultiEngine::MultiEngine(const int* devices, int n) {
  if (n < 1) throw std::invalid_argument("decmul_gpu_create_multi: at least one device");
  for (int i = 0; i < n; ++i) {
    cuda_check(cudaSetDevice(devices[i]), "cudaSetDevice");
    eng_.push_back(std::make_unique<Engine>(devices[i]));
    if (n > 1) eng_.back()->set_factor_all(true);
  }
  // peer access between distinct GPUs (NVLink); ranks on one GPU copy locally
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      if (devices[i] == devices[j]) continue;
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, devices[i], devices[j]);
      if (ok) {
        cudaSetDevice(devices[i]);
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "peer access");
        cudaGetLastError();
      }
    }
  cuda_check(cudaSetDevice(devices[0]), "cudaSetDevice");
  cuda_check(cudaMallocHost(&pinned_, kPinnedWords * sizeof(u64)), "cudaMallocHost");
  for (int i = 0; i < n; ++i) {
    cudaSetDevice(devices[i]);
    cudaEvent_t a, b;
    cuda_check(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "event");
    ready_.push_back(a);
    done_.push_back(b);
  }
  cudaSetDevice(devices[0]);
}

MultiEngine::~MultiEngine() {
  for (std::size_t i = 0; i < eng_.size(); ++i) {
    cudaSetDevice(eng_[i]->device());
    cudaStreamSynchronize(eng_[i]->stream());
    cudaEventDestroy(ready_[i]);
    cudaEventDestroy(done_[i]);
  }
  if (pinned_) cudaFreeHost(pinned_);
  eng_.clear();
}

std::vector<int> MultiEngine::devices() const {
  std::vector<int> d;
  for (const auto& e : eng_) d.push_back(e->device());
  return d;
}

bool MultiEngine::shards(std::size_t nx, std::size_t ny, unsigned forced) const {
  if (eng_.size() < 2 || forced) return false;
  try {
    const ShardPlan sp = make_shard_plan(nx, ny, int(eng_.size()));
    // ~2^22 words and up: below that one GPU finishes in well under a millisecond
    return sp.pp.N >= (std::size_t(1) << 22);
  } catch (const std::exception&) {
    return false;  // not shardable over this many ranks (too small, or G not a power of two)
  }
}

std::size_t MultiEngine::multiply_host(const char* x, std::size_t nx, const char* y, std::size_t ny, char* out,
                                       std::size_t cap, unsigned forced, bool alias, u64 p1, u64 p2) {
  if (nx == 0 || ny == 0) throw std::invalid_argument("decimal: empty string");
  const bool zero = (nx == 1 && x[0] == '0') || (ny == 1 && y[0] == '0');
  if (!zero && !p1 && !p2) {  // past the largest transform: block convolution (blocked.cu)
    const std::size_t K = block_digits(nx, ny, forced);
    if (K) return blocked_multiply(x, nx, y, ny, out, cap, forced, K);
  }
  if (!zero && !p1 && !p2 && shards(nx, ny, forced)) {
    const bool squaring = alias || (nx == ny && (x == y || std::memcmp(x, y, nx) == 0));
    if ((nx > 1 && x[0] == '0') || (ny > 1 && y[0] == '0')) throw std::invalid_argument("decimal: leading zero");
    return sharded_multiply(x, nx, y, ny, out, cap, squaring);
  }
  cudaSetDevice(eng_[0]->device());
  return eng_[0]->multiply_host(x, nx, y, ny, out, cap, forced, alias, p1, p2);
}

Engine* MultiEngine::overlap_engine(const char* x, std::size_t nx, const char* y, std::size_t ny, const char* out,
                                    unsigned forced, bool concurrent, u64 p1, u64 p2) {
  Engine& e = *eng_[0];
  if (!e.overlap_ok(x, nx, y, ny, out, concurrent)) return nullptr;
  if ((nx == 1 && x[0] == '0') || (ny == 1 && y[0] == '0')) return nullptr;
  if (!p1 && !p2 && (block_digits(nx, ny, forced) || shards(nx, ny, forced))) return nullptr;
  return &e;
}

void MultiEngine::multiply_batch_host(std::size_t count, const char* xs, std::size_t x_stride, std::size_t nx,
                                      const char* ys, std::size_t y_stride, std::size_t ny, char* outs,
                                      std::size_t out_stride, std::size_t* lens,
                                      std::unique_lock<std::mutex>* ctx_lock) {
  if (eng_.size() == 1 || count < 2 * eng_.size()) {
    cudaSetDevice(eng_[0]->device());
    eng_[0]->multiply_batch_host(count, xs, x_stride, nx, ys, y_stride, ny, outs, out_stride, lens, ctx_lock);
    return;
  }
  fan_out(count, [&](Engine& e, std::size_t b, std::size_t end) {
    e.multiply_batch_host(end - b, xs + b * x_stride, x_stride, nx, ys + b * y_stride, y_stride, ny,
                          outs + b * out_stride, out_stride, lens + b);
  });
}

void MultiEngine::multiply_batch_ptrs(std::size_t count, const char* const* xs, const std::size_t* nxs,
                                      const char* const* ys, const std::size_t* nys, char* const* outs,
                                      const std::size_t* caps, std::size_t* lens) {
  if (eng_.size() == 1 || count < 2 * eng_.size()) {
    cudaSetDevice(eng_[0]->device());
    eng_[0]->multiply_batch_ptrs(count, xs, nxs, ys, nys, outs, caps, lens);
    return;
  }
  fan_out(count, [&](Engine& e, std::size_t b, std::size_t end) {
    e.multiply_batch_ptrs(end - b, xs + b, nxs + b, ys + b, nys + b, outs + b, caps + b, lens + b);
  });
}

// ---------------- the sharded product ----------------

// Rank q's digit slice of one operand (nd digits, most significant first): the rows of its
// column block, limbs [r Sc + q Bc, r Sc + (q + 1) Bc) for r = top row .. 0, concatenated in
// string order (a partial top row first). Returns the slice length.
std::size_t MultiEngine::upload_slice(Engine& e, const ShardPlan& sp, int q, const char* d, std::size_t nd,
                                      char* dst, cudaStream_t st) {
  const std::size_t be = sp.pp.base_exp, Sc = sp.geom.Sc, Bc = sp.geom.Bc, off = std::size_t(q) * Bc;
  const std::size_t rows = sp.geom.Rtot;
  const std::size_t wbytes = Bc * be, pitch = Sc * be;
  // row r covers string positions [nd - (r Sc + off + Bc) be, nd - (r Sc + off) be)
  std::size_t full = 0;  // rows 0 .. full - 1 lie entirely inside the string
  while (full < rows && (full * Sc + off + Bc) * be <= nd) ++full;
  std::size_t part = 0;  // digits of the partial row `full` (clipped at the string's start)
  if (full < rows && (full * Sc + off) * be < nd) part = nd - (full * Sc + off) * be;
  (void)e;
  if (part) cuda_check(cudaMemcpyAsync(dst, d, part, cudaMemcpyHostToDevice, st), "slice h2d");
  if (full) {
    const char* src = d + nd - ((full - 1) * Sc + off + Bc) * be;  // row full - 1, the first in string order
    cuda_check(cudaMemcpy2DAsync(dst + part, wbytes, src, pitch, wbytes, full, cudaMemcpyHostToDevice, st),
               "slice h2d");
  }
  return part + full * wbytes;
}

// All-to-all of one prime's array: rank s sends words [d n, (d + 1) n) of send[s] to words
// [s n, (s + 1) n) of recv[d] (n = L / G). Every receiver waits for every sender's producing
// work; every sender then waits until all copies that read its buffer are done.
void MultiEngine::all_to_all(const std::vector<u64*>& send, const std::vector<u64*>& recv, std::size_t L) {
  const int G = int(eng_.size());
  const std::size_t n = L / std::size_t(G), bytes = n * sizeof(u64);
  for (int q = 0; q < G; ++q) {
    cudaSetDevice(eng_[q]->device());
    cuda_check(cudaEventRecord(ready_[q], eng_[q]->stream()), "event");
  }
  for (int d = 0; d < G; ++d) {
    cudaSetDevice(eng_[d]->device());
    cudaStream_t st = eng_[d]->stream();
    for (int s = 0; s < G; ++s) cuda_check(cudaStreamWaitEvent(st, ready_[s], 0), "wait");
    for (int s = 0; s < G; ++s) {
      u64* dst = recv[d] + std::size_t(s) * n;
      const u64* src = send[s] + std::size_t(d) * n;
      if (eng_[d]->device() == eng_[s]->device())
        cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st), "exchange");
      else
        cuda_check(cudaMemcpyPeerAsync(dst, eng_[d]->device(), src, eng_[s]->device(), bytes, st), "exchange");
    }
    cuda_check(cudaEventRecord(done_[d], st), "event");
  }
  for (int q = 0; q < G; ++q) {
    cudaSetDevice(eng_[q]->device());
    for (int d = 0; d < G; ++d) cuda_check(cudaStreamWaitEvent(eng_[q]->stream(), done_[d], 0), "wait");
  }
}

std::size_t MultiEngine::sharded_multiply(const char* x, std::size_t nx, const char* y, std::size_t ny, char* out,
                                          std::size_t cap, bool squaring) {
  const int G = int(eng_.size());
  if (cap < nx + ny) throw std::length_error("multiply: output buffer too small");
  std::vector<ShardPlan> sp(G);
  for (int q = 0; q < G; ++q) {
    cudaSetDevice(eng_[q]->device());
    sp[q] = eng_[q]->shard_plan(nx, ny, G);  // device tables of both primes on every rank
  }
  const ShardPlan& P = sp[0];
  const std::size_t L = P.geom.local_len;
  const std::size_t s_words = (L + 2 + kCarryChunk - 1) / kCarryChunk * kCarryChunk;
  const std::size_t map_words = (L + 2 + kCarryChunk - 1) / kCarryChunk;
  auto B = [&](int q) -> ShardBufs& { return eng_[q]->shard_bufs(); };
  auto dev = [&](int q) { cuda_check(cudaSetDevice(eng_[q]->device()), "cudaSetDevice"); };
  auto st = [&](int q) { return eng_[q]->stream(); };
  const std::size_t wmax = P.geom.Rtot * P.geom.Bc * P.pp.base_exp;  // slice bytes (upper bound)
  for (int q = 0; q < G; ++q) {
    dev(q);
    ShardBufs& b = B(q);
    for (int pr = 0; pr < 2; ++pr) {
      b.X[pr].ensure(L);
      if (!squaring) b.Y[pr].ensure(L);
    }
    b.P.ensure(L);
    b.R.ensure(L);
    b.S.ensure(s_words);
    b.M.ensure(map_words);
    b.dx.ensure(std::min(wmax, nx));
    if (!squaring) b.dy.ensure(std::min(wmax, ny));
  }
  // (1) digit slices and the column phase of x (and y)
  auto load = [&](const char* d, std::size_t nd, bool is_y) {
    for (int q = 0; q < G; ++q) {
      dev(q);
      ShardBufs& b = B(q);
      char* slice = is_y ? b.dy.ptr : b.dx.ptr;
      const std::size_t ns = upload_slice(*eng_[q], sp[q], q, d, nd, slice, st(q));
      eng_[q]->shard_pack_compact(sp[q], slice, ns, b.P.ptr, st(q));
      const u64* src[2] = {b.P.ptr, b.P.ptr};
      u64* dst[2] = {is_y ? b.Y[0].ptr : b.X[0].ptr, is_y ? b.Y[1].ptr : b.X[1].ptr};
      eng_[q]->shard_transform(sp[q], q, kShardColFwd, src, dst, nullptr, st(q));
    }
  };
  // column layout -> all-to-all -> block reorder into whole segments (and back)
  auto to_segments = [&](bool is_y) {
    for (int pr = 0; pr < 2; ++pr) {
      std::vector<u64*> send(G), recv(G);
      for (int q = 0; q < G; ++q) {
        send[q] = is_y ? B(q).Y[pr].ptr : B(q).X[pr].ptr;
        recv[q] = B(q).R.ptr;
      }
      all_to_all(send, recv, L);
      for (int q = 0; q < G; ++q) {
        dev(q);
        eng_[q]->shard_reorder(sp[q], true, B(q).R.ptr, send[q], st(q));
      }
    }
  };
  auto to_columns = [&](bool is_y) {
    for (int pr = 0; pr < 2; ++pr) {
      std::vector<u64*> send(G), recv(G);
      for (int q = 0; q < G; ++q) {
        dev(q);
        u64* a = is_y ? B(q).Y[pr].ptr : B(q).X[pr].ptr;
        eng_[q]->shard_reorder(sp[q], false, a, B(q).R.ptr, st(q));
        send[q] = B(q).R.ptr;
        recv[q] = a;
      }
      all_to_all(send, recv, L);
    }
  };
  load(x, nx, false);
  to_segments(false);
  const bool key_y = !squaring;
  if (squaring) {
    for (int q = 0; q < G; ++q) {
      dev(q);
      u64* d[2] = {B(q).X[0].ptr, B(q).X[1].ptr};
      const u64* s[2] = {d[0], d[1]};
      eng_[q]->shard_transform(sp[q], q, kShardRowFwdConv, s, d, nullptr, st(q));
    }
  } else {
    for (int q = 0; q < G; ++q) {
      dev(q);
      u64* d[2] = {B(q).X[0].ptr, B(q).X[1].ptr};
      const u64* s[2] = {d[0], d[1]};
      eng_[q]->shard_transform(sp[q], q, kShardRowFwd, s, d, nullptr, st(q));
    }
    load(y, ny, true);
    to_segments(true);
    for (int q = 0; q < G; ++q) {
      dev(q);
      u64* d[2] = {B(q).Y[0].ptr, B(q).Y[1].ptr};
      const u64* s[2] = {d[0], d[1]};
      const u64* o[2] = {B(q).X[0].ptr, B(q).X[1].ptr};
      eng_[q]->shard_transform(sp[q], q, kShardRowFwdConv, s, d, o, st(q));
    }
  }
  to_columns(key_y);
  for (int q = 0; q < G; ++q) {
    dev(q);
    u64* d[2] = {key_y ? B(q).Y[0].ptr : B(q).X[0].ptr, key_y ? B(q).Y[1].ptr : B(q).X[1].ptr};
    const u64* s[2] = {d[0], d[1]};
    eng_[q]->shard_transform(sp[q], q, kShardColInv, s, d, nullptr, st(q));
  }
  to_segments(key_y);  // rank q now holds coefficients [q L, (q + 1) L) in natural order
  auto Z = [&](int q, int pr) { return key_y ? B(q).Y[pr].ptr : B(q).X[pr].ptr; };

  // (2) distributed carry. pinned_: [4 G] halo words, [G] rank maps, [2 G] probes
  u64* halo = pinned_;
  unsigned* rmaps = reinterpret_cast<unsigned*>(pinned_ + 4 * G);
  u64* probes = pinned_ + 5 * G;
  for (int q = 0; q + 1 < G; ++q) {  // the last two residues of each prime go to rank q + 1
    dev(q);
    for (int pr = 0; pr < 2; ++pr)
      cuda_check(cudaMemcpyAsync(halo + 4 * (q + 1) + 2 * pr, Z(q, pr) + L - 2, 2 * sizeof(u64),
                                 cudaMemcpyDeviceToHost, st(q)),
                 "halo");
  }
  for (int k = 0; k < 4; ++k) halo[k] = 0;
  sync_all();
  for (int q = 0; q < G; ++q) {
    dev(q);
    const u64 h1[2] = {halo[4 * q], halo[4 * q + 1]}, h2[2] = {halo[4 * q + 2], halo[4 * q + 3]};
    eng_[q]->shard_carry_begin_async(sp[q], q, Z(q, 0), Z(q, 1), h1, h2, B(q).S.ptr, B(q).M.ptr, rmaps + q, st(q));
  }
  sync_all();
  std::vector<unsigned> cin(G);
  unsigned acc = 0x24u;  // identity map
  for (int q = 0; q < G; ++q) {
    cin[q] = map_apply_h(acc, 0);
    acc = map_compose_h(rmaps[q], acc);
  }
  for (int q = 0; q < G; ++q) {
    dev(q);
    eng_[q]->shard_carry_probe_async(sp[q], q, cin[q], Z(q, 0), Z(q, 1), B(q).S.ptr, B(q).M.ptr, probes + 2 * q,
                                     st(q));
  }
  sync_all();
  u64 zc[2] = {0, 0};
  for (int t = 0; t < 2; ++t)
    for (int q = 0; q < G; ++q)
      if (probes[2 * q + t] != ~0ull) {
        zc[t] = probes[2 * q + t];
        break;
      }
  unsigned long long top;
  u64 z;
  if (zc[1] != 0) {
    top = P.top_candidates[1];
    z = zc[1];
  } else if (zc[0] != 0) {
    top = P.top_candidates[0];
    z = zc[0];
  } else {
    top = 0;
    z = 0;
  }
  const unsigned top_len = decimal_len_h(z);
  const std::size_t n = top_len + std::size_t(top) * P.pp.base_exp;
  // (3) every rank prints its own digit range straight into its slice of the output
  std::vector<std::size_t> lo(G), hi(G);
  for (int q = 0; q < G; ++q) {
    rank_digit_range(L, P.pp.base_exp, q, n, lo[q], hi[q]);
    if (lo[q] >= hi[q]) continue;
    dev(q);
    ShardBufs& b = B(q);
    b.dout.ensure(hi[q] - lo[q]);
    eng_[q]->shard_carry_emit_async(sp[q], q, cin[q], top, top_len, Z(q, 0), Z(q, 1), b.S.ptr, b.M.ptr,
                                    b.dout.ptr - lo[q], st(q));
    cuda_check(cudaMemcpyAsync(out + lo[q], b.dout.ptr, hi[q] - lo[q], cudaMemcpyDeviceToHost, st(q)), "d2h");
  }
  // bad digits, bound violations: every rank's error word is read and cleared (syncs its
  // stream), then the first error is raised
  std::exception_ptr first;
  for (int q = 0; q < G; ++q) {
    dev(q);
    try {
      eng_[q]->check_errors_sync(st(q));
    } catch (...) {
      if (!first) first = std::current_exception();
    }
  }
  dev(0);
  if (first) std::rethrow_exception(first);
  return n;
}

void MultiEngine::sync_all() {
  for (auto& e : eng_) {
    cuda_check(cudaSetDevice(e->device()), "cudaSetDevice");
    cuda_check(cudaStreamSynchronize(e->stream()), "sync");
  }
}

}  // namespace dmg
