// Host orchestration of the device pipeline: per-(prime, length) transform
// plans with device-resident twiddle tables, workspace management, and the
// multiply / batch / parity-hook entry points used by the C ABI (capi.cu).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "hostmath.hpp"
#include "kernels.cuh"

namespace dmg {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CorruptionError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);

// Pinned host scratch that only grows.
struct PinnedBuf {
  char* ptr = nullptr;
  size_t n = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() {
    if (ptr) cudaFreeHost(ptr);
  }
  void ensure(size_t count);
};

template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (ptr) cudaFree(ptr);
  }
  void ensure(size_t count) {
    if (count <= n) return;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    n = 0;
    cuda_check(cudaMalloc(&ptr, count * sizeof(T) + 16), "cudaMalloc");
    n = count;
  }
};

struct PassPlan {
  bool radix3 = false;
  int logR = 0, R = 0;
  unsigned long long S = 0;
  int logS = 0;
  DevBuf<TwPair> tw_fwd, tw_inv;    // R x S inter-pass twiddles (power-of-two passes, S > 1), or the
                                    // factorised lo tables R x 2^tw_lbits when tw_lbits > 0
  DevBuf<TwPair> hi_fwd, hi_inv;    // factorised: R x S / 2^tw_lbits (the inverse carries the scale)
  int tw_lbits = 0;
  DevBuf<TwPair> dft_fwd, dft_inv;  // omega_R^{+-k}, k < R/2
  // radix-3 passes: omega_N^{+-f s} = lo[f][s mod 2^lbits] * hi[f][s >> lbits]
  DevBuf<TwPair> r3_lo_fwd, r3_hi_fwd, r3_lo_inv, r3_hi_inv;
  int r3_lbits = 0;
  // per-group twiddle tables (pass 1 after a merged radix-3 pass): group g at + g * stride
  unsigned long long tw_gstride = 0, hi_gstride = 0;
};

// Transform plan for one prime and one length N = 2^k or 3*2^k (root chosen
// exactly as the reference does: primitive_root_of_unity(N), primes.cpp:99-112).
struct PrimePlan {
  u64 p = 0, pp = 0;
  std::size_t N = 0;
  int three = 0, k = 0;
  u64 xi = 0;          // plain primitive N-th root
  u64 conv_scale = 0;  // R N^-1 mod p: undoes N (unscaled inverse) and R^-1 (pointwise REDC)
  TwPair final_scale{};  // Shoup pair of conv_scale (used when no pass table carries it)
  TwPair lam{}, lam_inv{};
  std::vector<std::unique_ptr<PassPlan>> passes;  // pass 0 first
  bool last_pow2 = false;  // last pass is a power-of-two pass with S == 1 (fusable)
  // radix-3 twiddles merged into pass 1 (build_passes): pre = omega_{3 R1}^{f r} (forward, pass 1's
  // column inputs), pinv = omega_{3 R1}^{-f r} scale (inverse radix-3), 3 x R1 Shoup pairs each
  bool r3_merged = false;
  DevBuf<TwPair> r3_pre, r3_pinv;
  // one-CTA kernel tables (N small): row length c = N / 3^three
  DevBuf<TwPair> small_fwd, small_inv, r3_fwd, r3_inv;
  bool small_ok = false;

  // position of spectrum index f in this plan's forward output, and inverse.
  std::size_t position_of(std::size_t spec) const;
};

struct ProductPlan {
  std::size_t dx = 0, dy = 0;
  unsigned base_exp = 0;
  std::size_t N = 0;
  u64 p1 = 0, p2 = 0;
  bool large_pair = false;
};

// Distribution of one large product over G ranks. The first K passes
// (their rows multiply to Rtot, a multiple of G) run column-sharded: rank q owns
// columns [q Bc, (q + 1) Bc) of the Rtot x Sc matrix. An all-to-all then gives each
// rank Rtot / G whole segments of length Sc for the remaining passes, the pointwise
// product and the first inverse passes; the inverse undoes this, and a last exchange
// leaves rank q with the natural-order coefficients [q N / G, (q + 1) N / G) for the
// distributed carry.
struct ShardGeom {
  int G = 1, q = 0, K = 0;
  std::size_t Rtot = 1, Sc = 0, Bc = 0, local_len = 0;
};

struct ShardPlan {
  ProductPlan pp;
  ShardGeom geom;  // q unset
  std::size_t lx = 0, ly = 0, min_limbs = 0;
  unsigned long long top_candidates[2] = {0, 0};
};

// Reciprocal-division constants for B = 10^lambda (reference make_div_by_const, decimal.hpp:93-104).
DivB div_for(u64 base);
// CRT constants of a pair (reference make_crt_ctx, decimal.cpp:136-146).
struct CrtConsts {
  u64 p2_prime, r_tilde;
};
CrtConsts crt_consts(u64 p1, u64 p2);

// Host-only shard planning (no device): decmul_gpu_shard_plan_create with a NULL context.
ShardPlan make_shard_plan(std::size_t dx, std::size_t dy, int G);

// Local geometry of one pass on a (possibly sharded) array.
struct PassLocal {
  unsigned long long S = 0, groups = 0, ncols = 0, tw_off = 0, off = 0;
  int logS = 0, tw_logS = 0, cb = 0, sb = 0;
};

enum ShardStage {
  kShardColFwd = 0,        // passes [0, K): src (packed limbs) -> dst, column layout
  kShardRowFwd = 1,        // passes [K, m): segment layout, in place
  kShardRowFwdConv = 2,    // passes [K, m-1), last pass fused with the pointwise product
                           // against `other` (null = square) and its inverse, then inverse [K, m-1)
  kShardColInv = 3,        // inverse passes [0, K): column layout, in place
};

// Persistent host threads splitting one large memcpy (pageable <-> pinned staging):
// measured on the GPU box, 4 threads copy pageable -> pinned at ~42 GB/s vs ~13 GB/s
// for one; the driver's own pageable DMA path reaches 9.7 GB/s H2D, 15 GB/s D2H.
class CopyPool {
 public:
  explicit CopyPool(int threads);
  ~CopyPool();
  void copy(char* dst, const char* src, std::size_t n);

 private:
  void worker(int i);
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable go_, done_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  std::size_t n_ = 0, per_ = 0;
  unsigned long long gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

// A ring of pinned staging slots with its own copy threads: large pageable host buffers are
// moved slot by slot, the host threads filling (or draining) one slot while the DMA engine
// moves another (hostio.cu). Pinned buffers and small ones go straight to cudaMemcpyAsync.
struct StageRing {
  static constexpr int kSlots = 4;
  static constexpr std::size_t kSlot = std::size_t(16) << 20;
  char* slot[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  std::unique_ptr<CopyPool> pool;
  ~StageRing();
  void ensure();
  void h2d(void* dst, const void* src, std::size_t n, cudaStream_t st);  // asynchronous for pinned src
  void d2h(void* dst, const void* src, std::size_t n, cudaStream_t st);  // returns with dst complete
};

// One rank's device buffers of a sharded product driven inside the library (multi.cu).
struct ShardBufs {
  DevBuf<u64> X[2], Y[2], P, R, S;
  DevBuf<unsigned> M;
  DevBuf<char> dx, dy, dout;
  DevBuf<unsigned long long> tmp;  // halo words, rank maps, probes
};

class Engine {
 public:
  explicit Engine(int device);
  ~Engine();

  int device() const { return device_; }
  cudaStream_t stream() const { return stream_; }

  // p1 = p2 = 0: the reference pair, or the large pair beyond its 3 * 2^24 cap; else that pair
  ProductPlan plan_product(std::size_t dx, std::size_t dy, unsigned forced_base_exp, u64 p1 = 0, u64 p2 = 0) const;

  // Host strings -> host string (reference decmul::multiply semantics).
  std::size_t multiply_host(const char* x, std::size_t nx, const char* y, std::size_t ny, char* out,
                            std::size_t cap, unsigned forced_base_exp, bool alias, u64 p1 = 0, u64 p2 = 0);
  // The same product for concurrent callers with large pinned buffers: the caller does NOT hold
  // the context lock; uploads, compute (under ctx_mu) and the download are separate stages over
  // two buffer slots, so one call's download overlaps the next call's upload and compute and the
  // next upload starts while this product still computes (PCIe is full duplex; hostio.cu).
  // concurrent: another large host product is in flight on the context
  bool overlap_ok(const char* x, std::size_t nx, const char* y, std::size_t ny, const char* out,
                  bool concurrent) const;
  std::size_t multiply_host_overlapped(std::mutex& ctx_mu, const char* x, std::size_t nx, const char* y,
                                       std::size_t ny, char* out, std::size_t cap, unsigned forced_base_exp,
                                       bool alias, u64 p1 = 0, u64 p2 = 0);
  // Device digits -> device digits; stream-ordered; *out_len written (host) after sync.
  std::size_t multiply_device(const char* dx, std::size_t nx, const char* dy, std::size_t ny, char* dout,
                              std::size_t cap, unsigned forced_base_exp, bool squaring, cudaStream_t st,
                              bool sync);
  // Uniform-size batch (config 2 shape), device buffers.
  void multiply_batch_device(std::size_t count, const char* dxs, std::size_t x_stride, std::size_t nx,
                             const char* dys, std::size_t y_stride, std::size_t ny, char* douts,
                             std::size_t out_stride, unsigned long long* dlens, cudaStream_t st);
  // Mixed sizes from host pointers: equal (nx, ny) groups through multiply_batch_host.
  void multiply_batch_ptrs(std::size_t count, const char* const* xs, const std::size_t* nxs, const char* const* ys,
                           const std::size_t* nys, char* const* outs, const std::size_t* caps, std::size_t* lens);
  // ctx_lock: the caller's (held) context lock; a large batch from pinned buffers releases it
  // once its chunks are enqueued, so batches from several threads overlap (batch_host_pipelined)
  void multiply_batch_host(std::size_t count, const char* xs, std::size_t x_stride, std::size_t nx,
                           const char* ys, std::size_t y_stride, std::size_t ny, char* outs,
                           std::size_t out_stride, std::size_t* lens,
                           std::unique_lock<std::mutex>* ctx_lock = nullptr);

  // Parity hooks (reference conv.hpp:59-71), host arrays, one prime.
  void convolve_mod_p(u64 p, std::size_t n, const u64* x, std::size_t nx, const u64* y, std::size_t ny,
                      u64* out);
  // reference storage order (conv.hpp:19-24) of a plan built with six-step threshold thr
  // (0 = the default 2^15)
  void forward_transform(u64 p, std::size_t n, u64* a, std::size_t thr = 0);
  void inverse_transform(u64 p, std::size_t n, u64* a, std::size_t thr = 0);
  void pointwise_product(u64 p, std::size_t n, u64* a, const u64* b);
  // Stage hooks on the device path (decimal.cpp pack / crt2 + recover_digits + to_decimal).
  std::size_t pack(const char* digits, std::size_t nd, unsigned base_exp, u64* limbs, std::size_t cap);
  std::size_t recover_decimal(const u64* r1, const u64* r2, std::size_t n, u64 p1, u64 p2, unsigned base_exp,
                              std::size_t min_limbs, std::size_t dsum, char* out, std::size_t cap);
  // In-place transposes (reference transpose.cpp) of a host matrix through the device.
  void transpose(int kind, u64* a, std::size_t n, std::size_t stride);

  // ---- sharded large products: device steps on caller-owned buffers (both primes) ----
  ShardPlan shard_plan(std::size_t dx, std::size_t dy, int G);
  // digits of one operand (full string, device) -> this rank's column-layout limbs
  void shard_pack(const ShardPlan& sp, int q, const char* d_digits, std::size_t nd, u64* d_out, cudaStream_t st);
  void shard_transform(const ShardPlan& sp, int q, int stage, const u64* const src[2], u64* const dst[2],
                       const u64* const other[2], cudaStream_t st);
  void shard_reorder(const ShardPlan& sp, bool to_segments, const u64* src, u64* dst, cudaStream_t st);
  // carry over this rank's natural block; halo = residues (p1: h1[0..1], p2: h2[0..1]) of the
  // two coefficients before the block. Returns the rank's composed carry map (syncs).
  unsigned shard_carry_begin(const ShardPlan& sp, int q, const u64* z1, const u64* z2, const u64 h1[2],
                             const u64 h2[2], u64* s_buf, unsigned* maps_buf, cudaStream_t st);
  void shard_carry_probe(const ShardPlan& sp, int q, unsigned rank_cin, const u64* z1, const u64* z2,
                         const u64* s_buf, unsigned* maps_buf, u64 z_out[2], cudaStream_t st);
  void shard_carry_emit(const ShardPlan& sp, int q, unsigned rank_cin, unsigned long long top, unsigned top_len,
                        const u64* z1, const u64* z2, const u64* s_buf, unsigned* maps_buf, char* d_out,
                        cudaStream_t st);

  // async forms for the in-library multi-device driver (multi.cu): no host sync; results land
  // in the caller's pinned host memory once st completes
  void shard_pack_compact(const ShardPlan& sp, const char* d_compact, std::size_t nd_compact, u64* d_out,
                          cudaStream_t st);
  void shard_carry_begin_async(const ShardPlan& sp, int q, const u64* z1, const u64* z2, const u64 h1[2],
                               const u64 h2[2], u64* s_buf, unsigned* maps_buf, unsigned* h_rank_map,
                               cudaStream_t st);
  void shard_carry_probe_async(const ShardPlan& sp, int q, unsigned rank_cin, const u64* z1, const u64* z2,
                               const u64* s_buf, unsigned* maps_buf, u64* h_z, cudaStream_t st);
  void shard_carry_emit_async(const ShardPlan& sp, int q, unsigned rank_cin, unsigned long long top,
                              unsigned top_len, const u64* z1, const u64* z2, const u64* s_buf, unsigned* maps_buf,
                              char* d_out, cudaStream_t st);
  ShardBufs& shard_bufs() { return shard_; }
  // every pass with S > 1 gets factorised twiddle tables (ranks of a sharded context: table
  // memory independent of N)
  void set_factor_all(bool on) { factor_all_ = on; }
  void check_errors_sync(cudaStream_t st) { check_err(st); }

  const PrimePlan& prime_plan(u64 p, std::size_t N);
  // Length of the last product (after its stream was synchronised); raises its errors.
  std::size_t result_length();

  // GPU self-test mirroring the reference's run_selftest (selftest.cpp:79-219): suites of
  // field identities, transform round trips, convolution vs direct, CRT, base division,
  // carry recovery and small products on the device path; inject_fault corrupts one
  // root-table entry of a plan (restored afterwards) to prove the checks detect it.
  // Appends "suite=... checks=... failures=..." lines to report; returns the failures.
  int selftest(bool inject_fault, std::string& report);

  // bytes of device tables currently held by plans
  std::size_t table_bytes() const;

  // Launch count of the last product (for the bench's gpu_launches claim).
  int last_launches() const { return launches_; }

  // Per-launch profiling (decmul_gpu_profile_*): while on, every kernel this engine enqueues
  // is followed by a CUDA event; report() syncs and returns "name<TAB>ms<TAB>modmuls<TAB>bytes"
  // lines (one per launch, ms since the previous mark); clear drops the records.
  void profile_enable(bool on);
  std::string profile_report(bool clear);
  void prof_record(const char* name, cudaStream_t st, double modmuls, double bytes);
  // Stream-ordered error word of the asynchronous entry points (multiply_device without sync,
  // multiply_batch_device): read and cleared by check_async_errors / result_length.
  void check_async_errors(cudaStream_t st);

 private:
  void build_passes(PrimePlan& pl);
  void build_small_tables(PrimePlan& pl);
  // before_y (optional) runs on the host after x's pack and forward transform are
  // enqueued and before anything reads dy: the host path uploads y there, so the
  // upload overlaps x's transform.
  void run_product(const ProductPlan& pp, const char* dx, const char* dy, bool squaring, char* dout,
                   cudaStream_t st, unsigned* err, const std::function<void()>& before_y = nullptr);
  // multiply_batch_device with an explicit error word (err_ for the synchronous host paths)
  void batch_device(std::size_t count, const char* dxs, std::size_t x_stride, std::size_t nx, const char* dys,
                    std::size_t y_stride, std::size_t ny, char* douts, std::size_t out_stride,
                    unsigned long long* dlens, cudaStream_t st, unsigned* err);
  // Host <-> device copies for the host-buffer API: pinned or small buffers go straight
  // to DMA; large pageable ones are pipelined through a pinned ring (CopyPool threads
  // fill/drain slot c while the DMA engine moves slot c - 1). stage_h2d returns once the
  // source may be reused (copies stream-ordered on st); stage_d2h returns when dst holds
  // the data.
  void stage_h2d(void* dst, const void* src, std::size_t n, cudaStream_t st);
  bool stage_direct(const void* host, std::size_t n) const;  // no staging ring: pinned or small
  void stage_d2h(void* dst, const void* src, std::size_t n, cudaStream_t st);
  void transform_forward(const PrimePlan* pl[2], int np, const u64* const src[2], u64* const dst[2],
                         bool include_last, cudaStream_t st);
  void transform_forward_packed(const PrimePlan* pl[2], u64* const data[2], bool include_last, cudaStream_t st);
  void transform_fused_last(const PrimePlan* pl[2], int np, u64* const data[2], const u64* const other[2],
                            cudaStream_t st);
  void transform_inverse(const PrimePlan* pl[2], int np, u64* const data[2], bool skip_last, cudaStream_t st);
  PassLocal local_pass(const PrimePlan& pl, std::size_t i, const ShardGeom* sg) const;
  // src_b / dst_b: a second operand in the same launches (power-of-two passes only)
  void passes_fwd(const PrimePlan* pl[2], int np, const u64* const src[2], u64* const dst[2], std::size_t begin,
                  std::size_t end, const ShardGeom* sg, cudaStream_t st, const u64* const src_b[2] = nullptr,
                  u64* const dst_b[2] = nullptr);
  // two: other[] holds the first operand before its last forward pass (run inside the kernel)
  void pass_fused(const PrimePlan* pl[2], int np, u64* const data[2], const u64* const other[2],
                  const ShardGeom* sg, cudaStream_t st, bool two = false);
  void passes_inv(const PrimePlan* pl[2], int np, u64* const data[2], std::size_t begin, std::size_t end,
                  const ShardGeom* sg, cudaStream_t st);
  // digits -> the first (radix-3) pass's output of both primes, one fused kernel
  void pack_radix3(const PrimePlan* pl[2], const char* digits, std::size_t nd, unsigned be, u64* const dst[2],
                   unsigned* err, cudaStream_t st);
  CarryArgs carry_args(const ProductPlan& pp, const u64* z1, const u64* z2, std::size_t n, char* out) const;
  void check_err(cudaStream_t st);
  void check_word(unsigned* word, cudaStream_t st);
  // decimal recovery of a product's coefficients: the 3-digit {0,1,2}-carry pipeline when every
  // coefficient is < B^3, else the general small-base path (forced lambda < 14)
  int recover(CarryArgs c, unsigned be, std::size_t min_limbs, bool allow_s_in_x, cudaStream_t st);

  // H2D / compute / D2H pipeline of multiply_batch_host (one-CTA products)
  void batch_host_pipelined(std::size_t count, const char* xs, std::size_t x_stride, std::size_t nx, const char* ys,
                            std::size_t y_stride, std::size_t ny, char* outs, std::size_t out_stride,
                            std::size_t* lens, std::unique_lock<std::mutex>* ctx_lock);
  static bool host_pinned(const void* p);
  static void throw_err_bits(unsigned e);

  int device_ = 0;
  cudaStream_t stream_ = nullptr;
  static constexpr int kPipe = 3;        // upload, compute, download
  static constexpr int kMaxChunks = 64;
  cudaStream_t pipe_[kPipe] = {};
  cudaEvent_t pipe_ev_ = nullptr;
  cudaEvent_t up_ev_[kMaxChunks] = {}, done_ev_[kMaxChunks] = {};
  unsigned long long* host_lens_ = nullptr;  // pinned
  std::size_t host_lens_n_ = 0;
  static constexpr std::size_t kGatherMax = std::size_t(64) << 20;
  PinnedBuf gather_;                // multiply_batch_ptrs: operands / products of a small group
  StageRing ring_;                  // the locked host path (under the context lock)
  StageRing ov_up_ring_;            // the overlapped path's upload stage (under ov_up_mu_)
  std::mutex mu_;
  std::map<std::pair<u64, std::size_t>, std::unique_ptr<PrimePlan>> plans_;
  DevBuf<u64> X_[2], Y_[2], Px_, Py_, S_, S2_;
  DevBuf<unsigned> maps_, err_, async_err_, ticket_;  // ticket_: the small carry's last-CTA counter
  DevBuf<unsigned char> pm_;                         // per-limb prefix maps of the carry (split -> emit)
  DevBuf<unsigned long long> meta_, lens_;
  DevBuf<char> din_x_, din_y_, dout_;
  // multiply_host_overlapped: two slots of digit buffers; ov_up_mu_ orders the uploads, the
  // context lock the compute, a slot's dl_mu its output buffer (held from before the compute
  // that fills it to the end of its download)
  struct OvSlot {
    DevBuf<char> dx, dy, dout;
    std::mutex dl_mu;
    cudaStream_t dl_stream = nullptr;
    cudaEvent_t ev_x = nullptr, ev_y = nullptr;
    unsigned long long* h_len = nullptr;  // pinned: the product length, read back without blocking
    StageRing dl_ring;  // pageable outputs: the two slots' downloads may run at the same time
  };
  // batch_host_pipelined in overlap mode: two sets of batch buffers
  struct BatchSet {
    DevBuf<char> dx, dy, dout;
    DevBuf<unsigned long long> lens;
    DevBuf<unsigned> err;
    PinnedBuf h_lens;
    unsigned* h_err = nullptr;
    cudaEvent_t done = nullptr;
    std::mutex mu;
  };
  BatchSet bsets_[2];
  int bset_ = 0;
  std::atomic<int> batch_active_{0};  // batch_host_pipelined calls in flight
  OvSlot ov_[2];
  std::mutex ov_up_mu_;
  cudaStream_t ov_up_stream_ = nullptr;
  int ov_slot_ = 0;
  int launches_ = 0;
  struct ProfRec {
    std::string name;
    double modmuls, bytes;
    cudaEvent_t ev;
  };
  bool prof_on_ = false;
  std::vector<ProfRec> prof_;
  ShardBufs shard_;
  bool factor_all_ = false;
};

// The engine whose launches the calling thread is currently enqueueing (prof_mark target).
struct ProfScope {
  explicit ProfScope(Engine* e);
  ~ProfScope();
  Engine* prev;
};

}  // namespace dmg
