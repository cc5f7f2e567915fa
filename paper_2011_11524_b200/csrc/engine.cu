// Host orchestration for the device multiplier. See engine.hpp.
#include "engine.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <stdexcept>

namespace dmg {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

TwPair shoup_pair(const HostField& F, u64 w) { return TwPair{w, F.shoup(w)}; }

// Factorised inter-pass twiddle tables for a pass whose full R x S table would take more than
// 4 GB per direction... per prime (config 5's first power-of-two pass: 8 GB; config 4 keeps its
// 1 GB tables: the second Shoup product per element costs more than the table read saves).
// DECMUL_FACTOR_TABLES=1 factorises every pass with S > 1 (tests), =0 none.
bool factor_tables(std::size_t entries) {
  if (const char* e = std::getenv("DECMUL_FACTOR_TABLES")) return e[0] == '1';
  return entries * sizeof(TwPair) > (std::size_t(4) << 30);
}


// Radix-3 twiddles merged into pass 1 (PassArgs::pre): the radix-3 passes run twiddle-free
// forward and with a 3 x R1 table inverse; pass 1 gets one twiddle table per radix-3 row.
// DECMUL_R3_MERGE=0 keeps the factorised lo * hi twiddles in the radix-3 passes (tests, A/B).
bool r3_merge_enabled() {
  const char* e = std::getenv("DECMUL_R3_MERGE");
  return !(e && e[0] == '0');
}

u64 recip_of(u64 d) {  // reference make_div_by_const (decimal.hpp:93-104), for a normalized divisor
  return u64(~(u128)0 / d - ((u128)1 << 64));
}

DivB div_for_impl(u64 base) {
  DivB d;
  d.base = base;
  d.shift = __builtin_clzll(base);
  d.d_norm = base << d.shift;
  d.recip = recip_of(d.d_norm);
  const u128 b2 = (u128)base * base;
  d.b2lo = u64(b2);
  d.b2hi = u64(b2 >> 64);
  d.inv_b2 = 1.0 / (double(base) * double(base));
  return d;
}

int bitrev_h(std::size_t x, int bits) {
  std::size_t r = 0;
  for (int i = 0; i < bits; ++i) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return int(r);
}

// The reference's storage -> spectrum map (conv.hpp:19-24) for a plan built with six-step
// threshold thr (build_conv_plan, conv.cpp:243-269; default 2^15; checked by
// test_conv.cpp:18-32). The three-row shape hands thr on to its row plan.
std::size_t ref_order_of(std::size_t n, std::size_t k, std::size_t thr) {
  if (n <= 1) return 0;
  if (n % 3 == 0) {
    const std::size_t c = n / 3;
    return k / c + 3 * ref_order_of(c, k % c, thr);
  }
  const int lg = __builtin_ctzll(n);
  if (n <= thr) return std::size_t(bitrev_h(k, lg));
  const std::size_t n1 = std::size_t(1) << (lg / 2), n2 = n / n1;
  const std::size_t i = k / n2, j = k % n2;
  return i + n1 * std::size_t(bitrev_h(j, __builtin_ctzll(n2)));
}

std::vector<int> split_log(int k, int maxlog) {
  std::vector<int> parts;
  if (k <= 0) return parts;
  const int m = (k + maxlog - 1) / maxlog;
  for (int i = 0; i < m; ++i) parts.push_back(k / m + (i < k % m ? 1 : 0));
  return parts;
}

template <class T>
void upload(DevBuf<T>& b, const std::vector<T>& v, cudaStream_t st) {
  b.ensure(std::max<std::size_t>(v.size(), 1));
  if (!v.empty())
    cuda_check(cudaMemcpyAsync(b.ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st), "upload");
}

__host__ u64 padded_len(const PrimePlan& pl) {
  std::size_t n = std::max<std::size_t>(pl.N, 1);
  if (pl.last_pow2) {
    const std::size_t blk = std::size_t(pl.passes.back()->R) * kTileW;
    n = (n + blk - 1) / blk * blk;
  }
  return n;
}

}  // namespace

std::size_t PrimePlan::position_of(std::size_t spec) const {
  std::size_t pos = 0, rem = spec;
  for (const auto& ps : passes) {
    const std::size_t f = rem % ps->R;
    rem /= ps->R;
    const std::size_t r = ps->radix3 ? f : std::size_t(bitrev_h(f, ps->logR));
    pos += r * ps->S;
  }
  return pos;
}

Engine::Engine(int device) : device_(device) {
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  for (auto& s : pipe_) cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  cuda_check(cudaEventCreateWithFlags(&pipe_ev_, cudaEventDisableTiming), "cudaEventCreate");
  for (int i = 0; i < kMaxChunks; ++i) {
    cuda_check(cudaEventCreateWithFlags(&up_ev_[i], cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&done_ev_[i], cudaEventDisableTiming), "cudaEventCreate");
  }
  err_.ensure(1);
  async_err_.ensure(1);
  ticket_.ensure(1);
  meta_.ensure(4);
  cuda_check(cudaMemsetAsync(ticket_.ptr, 0, sizeof(unsigned), stream_), "memset");
  cuda_check(cudaMemsetAsync(err_.ptr, 0, sizeof(unsigned), stream_), "memset");
  cuda_check(cudaMemsetAsync(async_err_.ptr, 0, sizeof(unsigned), stream_), "memset");
  cuda_check(cudaStreamSynchronize(stream_), "init");
}

Engine::~Engine() {
  cudaSetDevice(device_);
  cudaStreamSynchronize(stream_);
  for (auto& r : prof_) cudaEventDestroy(r.ev);
  for (auto s : pipe_) cudaStreamSynchronize(s);
  plans_.clear();
  for (auto s : pipe_) cudaStreamDestroy(s);
  cudaEventDestroy(pipe_ev_);
  for (int i = 0; i < kMaxChunks; ++i) {
    cudaEventDestroy(up_ev_[i]);
    cudaEventDestroy(done_ev_[i]);
  }
  if (host_lens_) cudaFreeHost(host_lens_);
  for (BatchSet& b : bsets_) {
    if (b.done) cudaEventDestroy(b.done);
    if (b.h_err) cudaFreeHost(b.h_err);
  }
  if (ov_up_stream_) cudaStreamDestroy(ov_up_stream_);
  for (OvSlot& s : ov_) {
    if (s.dl_stream) cudaStreamDestroy(s.dl_stream);
    if (s.ev_x) cudaEventDestroy(s.ev_x);
    if (s.ev_y) cudaEventDestroy(s.ev_y);
    if (s.h_len) cudaFreeHost(s.h_len);
  }
  cudaStreamDestroy(stream_);
}

const PrimePlan& Engine::prime_plan(u64 p, std::size_t N) {
  std::lock_guard<std::mutex> lock(mu_);
  auto key = std::make_pair(p, N);
  auto it = plans_.find(key);
  if (it != plans_.end()) return *it->second;
  auto pl = std::make_unique<PrimePlan>();
  HostField F(p);
  pl->p = p;
  pl->pp = F.pp;
  pl->N = N;
  pl->three = (N % 3 == 0) ? 1 : 0;
  const std::size_t c = pl->three ? N / 3 : N;
  if (N == 0 || (c & (c - 1))) throw std::invalid_argument("build_conv_plan: length must be 2^k or 3*2^k");
  if (N > 1 && (p - 1) % N) throw std::invalid_argument("build_conv_plan: length does not divide p-1");
  pl->k = __builtin_ctzll(c);
  pl->xi = N > 1 ? F.root_of_unity(N) : 1;
  pl->conv_scale = F.mul(F.r, F.inv(N % p));
  pl->final_scale = shoup_pair(F, pl->conv_scale);
  if (pl->three) {
    pl->lam = shoup_pair(F, F.pow(pl->xi, N / 3));
    pl->lam_inv = shoup_pair(F, F.pow(pl->xi, 2 * (N / 3)));
  }
  build_passes(*pl);
  build_small_tables(*pl);
  cuda_check(cudaStreamSynchronize(stream_), "plan build");
  auto* raw = pl.get();
  plans_.emplace(key, std::move(pl));
  return *raw;
}

void Engine::build_passes(PrimePlan& pl) {
  HostField F(pl.p);
  const u64 recip = recip_of(pl.p << __builtin_clzll(pl.p));
  std::vector<std::pair<bool, int>> spec;  // (radix3, logR)
  for (int r : pass_radices(pl.N, kMaxPassLog)) spec.push_back({r == 3, r == 3 ? 0 : __builtin_ctz(unsigned(r))});
  std::size_t done = 1;
  int last_table = -1;
  for (std::size_t i = 0; i < spec.size(); ++i) {
    auto ps = std::make_unique<PassPlan>();
    ps->radix3 = spec[i].first;
    ps->logR = spec[i].second;
    ps->R = ps->radix3 ? 3 : (1 << ps->logR);
    done *= std::size_t(ps->R);
    ps->S = pl.N / done;
    ps->logS = ps->S ? __builtin_ctzll(ps->S) : 0;
    if (ps->radix3 || ps->S > 1) last_table = int(i);
    pl.passes.push_back(std::move(ps));
  }
  // merged radix-3 twiddles need pass 1 to be a staged row pass (S1 > 1, 16 <= R1)
  pl.r3_merged = pl.passes.size() >= 2 && pl.passes[0]->radix3 && pl.passes[1]->S > 1 && pl.passes[1]->logR >= 4 &&
                 r3_merge_enabled();
  if (pl.r3_merged) {
    // pre[f R1 + r] = omega_{3 R1}^{f r}; pinv[f R1 + r] = omega_{3 R1}^{-f r} (the convolution
    // scale rides on the highest pass with a table, never pass 0 here: pass 1 has S > 1)
    const int R1 = pl.passes[1]->R;
    const u64 w = F.pow(pl.xi, pl.N / (3 * std::size_t(R1))), wi = F.inv(w);
    std::vector<TwPair> pre(3 * R1), pinv(3 * R1);
    for (int f = 0; f < 3; ++f) {
      const u64 sf = F.pow(w, f), sfi = F.pow(wi, f);
      u64 a = 1, b = last_table == 0 ? pl.conv_scale : 1;
      for (int r = 0; r < R1; ++r) {
        pre[f * R1 + r] = shoup_pair(F, a);
        pinv[f * R1 + r] = shoup_pair(F, b);
        a = F.mul(a, sf);
        b = F.mul(b, sfi);
      }
    }
    upload(pl.r3_pre, pre, stream_);
    upload(pl.r3_pinv, pinv, stream_);
    cuda_check(cudaStreamSynchronize(stream_), "radix-3 merged tables");
  }
  for (std::size_t i = 0; i < pl.passes.size(); ++i) {
    PassPlan& ps = *pl.passes[i];
    const std::size_t M = std::size_t(ps.R) * ps.S;
    const u64 wM = F.pow(pl.xi, pl.N / M);
    if (ps.radix3) {
      // factorised twiddles: omega^{f s} = omega^{f (s mod L)} * omega^{f L (s / L)}
      const std::size_t L = std::min<std::size_t>(ps.S, 8192), H = ps.S / L;
      ps.r3_lbits = __builtin_ctzll(L);
      const u64 scale = int(i) == last_table ? pl.conv_scale : 1;
      std::vector<TwPair> lf(3 * L), li(3 * L), hf(3 * H), hi(3 * H);
      const u64 wMi = F.inv(wM), wL = F.pow(wM, L), wLi = F.inv(wL);
      for (int f = 0; f < 3; ++f) {
        const u64 sf = F.pow(wM, f), sfi = F.pow(wMi, f), hf_step = F.pow(wL, f), hi_step = F.pow(wLi, f);
        u64 a = 1, b = 1;
        for (std::size_t s = 0; s < L; ++s) {
          lf[f * L + s] = shoup_pair(F, a);
          li[f * L + s] = shoup_pair(F, b);
          a = F.mul(a, sf);
          b = F.mul(b, sfi);
        }
        a = 1;
        b = scale;
        for (std::size_t s = 0; s < H; ++s) {
          hf[f * H + s] = shoup_pair(F, a);
          hi[f * H + s] = shoup_pair(F, b);
          a = F.mul(a, hf_step);
          b = F.mul(b, hi_step);
        }
      }
      upload(ps.r3_lo_fwd, lf, stream_);
      upload(ps.r3_hi_fwd, hf, stream_);
      upload(ps.r3_lo_inv, li, stream_);
      upload(ps.r3_hi_inv, hi, stream_);
      cuda_check(cudaStreamSynchronize(stream_), "radix-3 tables");
    } else if (i == 1 && pl.r3_merged) {
      // pass 1 after a twiddle-free radix-3 pass: group g (radix-3 row g) uses
      // omega_N^{(3 f1 + g) c} = omega_S^{f1 c} (its own twiddle) * omega_N^{g c} (the radix-3
      // twiddle's part that commutes with the column DFT); one table (or lo / hi pair) per group
      const std::size_t N = pl.N;
      const u64 xi = pl.xi, xii = F.inv(pl.xi);
      const std::size_t cnt = std::size_t(ps.R) * ps.S;
      const u64 scale = int(i) == last_table ? pl.conv_scale : 1;
      if (factor_all_ || factor_tables(3 * cnt)) {
        const int lb = std::max(kTileLogW, (ps.logS + 1) / 2);
        const std::size_t L = std::size_t(1) << lb, H = ps.S / L;
        ps.tw_lbits = lb;
        ps.tw_gstride = std::size_t(ps.R) * L;
        ps.hi_gstride = std::size_t(ps.R) * H;
        ps.tw_fwd.ensure(3 * ps.tw_gstride);
        ps.tw_inv.ensure(3 * ps.tw_gstride);
        ps.hi_fwd.ensure(3 * ps.hi_gstride);
        ps.hi_inv.ensure(3 * ps.hi_gstride);
        for (int g = 0; g < 3; ++g) {
          launch_gen_pass_table(ps.tw_fwd.ptr + g * ps.tw_gstride, F.to_mont(xi), F.to_mont(1), ps.R, ps.logR, L, pl.p,
                                recip, stream_, N, 0, 3, g);
          launch_gen_pass_table(ps.tw_inv.ptr + g * ps.tw_gstride, F.to_mont(xii), F.to_mont(1), ps.R, ps.logR, L,
                                pl.p, recip, stream_, N, 0, 3, g);
          launch_gen_pass_table(ps.hi_fwd.ptr + g * ps.hi_gstride, F.to_mont(F.pow(xi, L)), F.to_mont(1), ps.R,
                                ps.logR, H, pl.p, recip, stream_, N / L, 0, 3, g);
          launch_gen_pass_table(ps.hi_inv.ptr + g * ps.hi_gstride, F.to_mont(F.pow(xii, L)), F.to_mont(scale), ps.R,
                                ps.logR, H, pl.p, recip, stream_, N / L, 0, 3, g);
        }
      } else {
        ps.tw_gstride = cnt;
        ps.tw_fwd.ensure(3 * cnt);
        ps.tw_inv.ensure(3 * cnt);
        for (int g = 0; g < 3; ++g) {
          launch_gen_pass_table(ps.tw_fwd.ptr + g * cnt, F.to_mont(xi), F.to_mont(1), ps.R, ps.logR, ps.S, pl.p, recip,
                                stream_, N, 0, 3, g);
          launch_gen_pass_table(ps.tw_inv.ptr + g * cnt, F.to_mont(xii), F.to_mont(scale), ps.R, ps.logR, ps.S, pl.p,
                                recip, stream_, N, 0, 3, g);
        }
      }
      cuda_check(cudaGetLastError(), "gen table");
    } else if (ps.S > 1) {
      const std::size_t cnt = std::size_t(ps.R) * ps.S;
      const u64 scale = int(i) == last_table ? pl.conv_scale : 1;
      if (factor_all_ || factor_tables(cnt)) {
        // omega_M^{f s} = omega_M^{f (s mod L)} * (omega_M^L)^{f (s / L)}: R (L + S / L) pairs instead
        // of R S, for one more Shoup product per element of the pass (memory-bound plans only)
        const int lb = std::max(kTileLogW, (ps.logS + 1) / 2);
        const std::size_t L = std::size_t(1) << lb, H = ps.S / L;
        ps.tw_lbits = lb;
        ps.tw_fwd.ensure(std::size_t(ps.R) * L);
        ps.tw_inv.ensure(std::size_t(ps.R) * L);
        ps.hi_fwd.ensure(std::size_t(ps.R) * H);
        ps.hi_inv.ensure(std::size_t(ps.R) * H);
        const u64 wMi = F.inv(wM);
        // lo: exponents f sl mod M over R x L; hi: (omega^L)^{f sh} mod M / L over R x H
        launch_gen_pass_table(ps.tw_fwd.ptr, F.to_mont(wM), F.to_mont(1), ps.R, ps.logR, L, pl.p, recip, stream_,
                              std::size_t(ps.R) * ps.S);
        launch_gen_pass_table(ps.tw_inv.ptr, F.to_mont(wMi), F.to_mont(1), ps.R, ps.logR, L, pl.p, recip, stream_,
                              std::size_t(ps.R) * ps.S);
        launch_gen_pass_table(ps.hi_fwd.ptr, F.to_mont(F.pow(wM, L)), F.to_mont(1), ps.R, ps.logR, H, pl.p, recip,
                              stream_, std::size_t(ps.R) * ps.S / L);
        launch_gen_pass_table(ps.hi_inv.ptr, F.to_mont(F.pow(wMi, L)), F.to_mont(scale), ps.R, ps.logR, H, pl.p,
                              recip, stream_, std::size_t(ps.R) * ps.S / L);
      } else {
        ps.tw_fwd.ensure(cnt);
        ps.tw_inv.ensure(cnt);
        launch_gen_pass_table(ps.tw_fwd.ptr, F.to_mont(wM), F.to_mont(1), ps.R, ps.logR, ps.S, pl.p, recip, stream_);
        launch_gen_pass_table(ps.tw_inv.ptr, F.to_mont(F.inv(wM)), F.to_mont(scale), ps.R, ps.logR, ps.S, pl.p,
                              recip, stream_);
      }
      cuda_check(cudaGetLastError(), "gen table");
    }
    if (!ps.radix3) {
      const u64 wR = F.pow(pl.xi, pl.N / std::size_t(ps.R)), wRi = F.inv(wR);
      std::vector<TwPair> tf(std::max(ps.R / 2, 1)), ti(std::max(ps.R / 2, 1));
      u64 a = 1, b = 1;
      for (int j = 0; j < ps.R / 2; ++j) {
        tf[j] = shoup_pair(F, a);
        ti[j] = shoup_pair(F, b);
        a = F.mul(a, wR);
        b = F.mul(b, wRi);
      }
      upload(ps.dft_fwd, tf, stream_);
      upload(ps.dft_inv, ti, stream_);
      cuda_check(cudaStreamSynchronize(stream_), "table upload");
    }
  }
  pl.last_pow2 = !pl.passes.empty() && !pl.passes.back()->radix3;
  if (last_table < 0) {
    // no table carries the convolution scale: the last inverse kernel applies final_scale
  }
}

void Engine::build_small_tables(PrimePlan& pl) {
  const int maxlog = small_max_logc(pl.three);
  if (pl.k > maxlog) return;
  HostField F(pl.p);
  const std::size_t c = std::size_t(1) << pl.k;
  const u64 wc = F.pow(pl.xi, pl.N / c), wci = F.inv(wc);
  std::vector<TwPair> tf(std::max<std::size_t>(c / 2, 1)), ti(std::max<std::size_t>(c / 2, 1));
  u64 a = 1, b = 1;
  for (std::size_t j = 0; j < c / 2; ++j) {
    tf[j] = shoup_pair(F, a);
    ti[j] = shoup_pair(F, b);
    a = F.mul(a, wc);
    b = F.mul(b, wci);
  }
  upload(pl.small_fwd, tf, stream_);
  upload(pl.small_inv, ti, stream_);
  if (pl.three) {
    std::vector<TwPair> r3f(3 * c), r3i(3 * c);
    const u64 xin = F.inv(pl.xi);
    for (int f = 0; f < 3; ++f) {
      const u64 sf = F.pow(pl.xi, f), sfi = F.pow(xin, f);
      u64 w = 1, wi = pl.conv_scale;
      for (std::size_t s = 0; s < c; ++s) {
        r3f[f * c + s] = shoup_pair(F, w);
        r3i[f * c + s] = shoup_pair(F, wi);
        w = F.mul(w, sf);
        wi = F.mul(wi, sfi);
      }
    }
    upload(pl.r3_fwd, r3f, stream_);
    upload(pl.r3_inv, r3i, stream_);
  }
  cuda_check(cudaStreamSynchronize(stream_), "small tables");
  pl.small_ok = true;
}

std::size_t Engine::table_bytes() const {
  std::size_t b = 0;
  for (const auto& kv : plans_)
    for (const auto& ps : kv.second->passes)
      b += (ps->tw_fwd.n + ps->tw_inv.n + ps->hi_fwd.n + ps->hi_inv.n + ps->dft_fwd.n + ps->dft_inv.n +
            ps->r3_lo_fwd.n + ps->r3_hi_fwd.n + ps->r3_lo_inv.n + ps->r3_hi_inv.n) *
           sizeof(TwPair);
  return b;
}

ProductPlan Engine::plan_product(std::size_t dx, std::size_t dy, unsigned forced, u64 p1, u64 p2) const {
  PairChoice pc;
  if (p1 || p2) {  // caller-chosen pair (the reference's select_base_and_length(dx, dy, pair, forced))
    if (!(p1 < p2) || p2 >= (u64(1) << 63) || !is_prime(p1) || !is_prime(p2))
      throw std::invalid_argument("multiply: prime pair must be two primes p1 < p2 < 2^63");
    pc = PairChoice{p1, p2, select_base_and_length(dx, dy, p1, p2, forced), false};
  } else {
    pc = choose_pair(dx, dy, forced, /*allow_large=*/true);
  }
  ProductPlan pp;
  pp.dx = dx;
  pp.dy = dy;
  pp.base_exp = pc.bp.base_exp;
  pp.N = pc.bp.length;
  pp.p1 = pc.p1;
  pp.p2 = pc.p2;
  pp.large_pair = pc.large_pair;
  return pp;
}

// Local geometry of pass i. Unsharded: the whole array. Column phase (i < K): this
// rank owns columns [q Bc, (q + 1) Bc) of every row of the first K passes' matrix,
// so pass i keeps its groups, its stride shrinks to S_i / G, and its twiddle column
// is the global one. Row phase (i >= K): this rank owns whole segments of length Sc,
// so pass i keeps its stride and owns 1/G of the groups.
PassLocal Engine::local_pass(const PrimePlan& pl, std::size_t i, const ShardGeom* sg) const {
  const PassPlan& P = *pl.passes[i];
  PassLocal L;
  L.S = P.S;
  L.logS = P.logS;
  L.groups = pl.N / (std::size_t(P.R) * P.S);
  L.ncols = pl.N / std::size_t(P.R);
  L.tw_logS = P.logS;
  L.tw_off = 0;
  L.cb = L.sb = 0;
  L.off = 0;
  if (!sg) return L;
  const std::size_t G = std::size_t(sg->G);
  L.ncols = sg->local_len / std::size_t(P.R);
  if (int(i) < sg->K) {
    L.S = P.S / G;
    L.logS = __builtin_ctzll(L.S);
    L.tw_off = std::size_t(sg->q) * sg->Bc;  // valid for the last column pass (S_i = Sc)
    L.cb = __builtin_ctzll(sg->Bc);
    L.sb = __builtin_ctzll(sg->Sc);
    L.off = std::size_t(sg->q) * sg->Bc;
  } else {
    L.groups /= G;
  }
  return L;
}

// Whether inverse pass i may leave its outputs in [0, 2p): yes unless it is the last inverse
// pass (pass 0), whose outputs the carry and the parity hooks read as residues in [0, p).
static bool inverse_lazy_ok(const PrimePlan& pl, std::size_t i) {
  // every inverse pass below the last starts by multiplying each input (a power-of-two row
  // pass by its twiddle, the radix-3 pass / fused carry by its twiddle or the scale)
  (void)pl;
  return i > 0;
}

void Engine::passes_fwd(const PrimePlan* pl[2], int np, const u64* const src[2], u64* const dst[2], std::size_t begin,
                        std::size_t end, const ShardGeom* sg, cudaStream_t st, const u64* const src_b[2],
                        u64* const dst_b[2]) {
  for (std::size_t i = begin; i < end; ++i) {
    const bool first = i == begin;
    const PassLocal L = local_pass(*pl[0], i, sg);
    if (pl[0]->passes[i]->radix3) {
      if (src_b) throw std::logic_error("two-operand passes: power-of-two passes only");
      Radix3Args a{};
      for (int q = 0; q < np; ++q) {
        a.src[q] = first ? src[q] : dst[q];
        a.dst[q] = dst[q];
        a.lo[q] = pl[q]->passes[i]->r3_lo_fwd.ptr;
        a.hi[q] = pl[q]->passes[i]->r3_hi_fwd.ptr;
        a.p[q] = pl[q]->p;
        a.lam[q] = pl[q]->lam;
      }
      a.notw = pl[0]->r3_merged ? 1 : 0;
      a.S = L.S;
      a.lbits = pl[0]->passes[i]->r3_lbits;
      a.hrow = pl[0]->passes[i]->S >> a.lbits;
      a.cb = L.cb;
      a.sb = L.sb;
      a.off = L.off;
      launch_radix3(false, a, np, st);
      prof_mark("k_radix3_fwd", st, double(np) * 3.0 * double(L.S), double(np) * 48.0 * double(L.S));
    } else {
      PassArgs a{};
      const PassPlan& P = *pl[0]->passes[i];
      for (int q = 0; q < np; ++q) {
        const PassPlan& Pq = *pl[q]->passes[i];
        a.src[q] = first ? src[q] : dst[q];
        a.dst[q] = dst[q];
        a.dft_fwd[q] = Pq.dft_fwd.ptr;
        a.dft_inv[q] = Pq.dft_inv.ptr;
        a.pass_tw[q] = Pq.S > 1 ? Pq.tw_fwd.ptr : nullptr;
        a.pass_hi[q] = Pq.hi_fwd.ptr;
        a.p[q] = pl[q]->p;
        a.pp[q] = pl[q]->pp;
        if (src_b) {
          a.src_b[q] = first ? src_b[q] : dst_b[q];
          a.dst_b[q] = dst_b[q];
        }
        a.pre[q] = (i == 1 && pl[q]->r3_merged) ? pl[q]->r3_pre.ptr : nullptr;
      }
      a.tw_gstride = P.tw_gstride;
      a.hi_gstride = P.hi_gstride;
      a.nops = src_b ? 2 : 1;
      a.tw_lbits = P.tw_lbits;
      a.S = L.S;
      a.logS = L.logS;
      a.G = L.groups;
      a.tw_logS = L.tw_logS;
      a.tw_off = L.tw_off;
      launch_pass_fwd(P.logR, a, L.ncols, np, st);
      if (prof_on_) {
        char nm[64];
        std::snprintf(nm, sizeof nm, "k_pass_fwd<%d,%s>", P.logR, L.S > 1 ? "rows" : "cols");
        const double n = double(L.ncols) * P.R;
        // algorithmic HBM bytes: the data once in, once out, plus the inter-pass twiddle table
        // (one 16-byte pair per element; shared by the pass's groups unless pass 1 carries a
        // table per radix-3 row; factorised tables are small)
        const double tb = (L.S > 1 && !P.tw_lbits) ? np * 16.0 * n / (P.tw_gstride ? 1.0 : double(L.groups)) : 0.0;
        prof_mark(nm, st, a.nops * np * (n / 2 * P.logR + (L.S > 1 ? n : 0)), a.nops * np * 16 * n + tb);
      }
    }
    ++launches_;
  }
}

void Engine::pass_fused(const PrimePlan* pl[2], int np, u64* const data[2], const u64* const other[2],
                        const ShardGeom* sg, cudaStream_t st, bool two) {
  const std::size_t m = pl[0]->passes.size();
  const PassPlan& P = *pl[0]->passes[m - 1];
  const PassLocal L = local_pass(*pl[0], m - 1, sg);
  bool any_table = false;
  for (const auto& ps : pl[0]->passes) any_table |= ps->radix3 || ps->S > 1;
  PassArgs a{};
  for (int q = 0; q < np; ++q) {
    const PassPlan& Pq = *pl[q]->passes[m - 1];
    a.src[q] = data[q];
    a.dst[q] = data[q];
    a.other[q] = other ? other[q] : nullptr;
    a.dft_fwd[q] = Pq.dft_fwd.ptr;
    a.dft_inv[q] = Pq.dft_inv.ptr;
    a.pass_tw[q] = nullptr;
    a.final_scale[q] = pl[q]->final_scale;
    a.p[q] = pl[q]->p;
    a.pp[q] = pl[q]->pp;
  }
  a.S = 1;
  a.logS = 0;
  a.G = L.groups;
  a.tw_logS = 0;
  a.has_final_scale = any_table ? 0 : 1;
  a.lazy_out = inverse_lazy_ok(*pl[0], m - 1) ? 1 : 0;
  a.two = two ? 1 : 0;
  launch_pass_fused(P.logR, a, L.ncols, np, st);
  if (prof_on_) {
    char nm[64];
    std::snprintf(nm, sizeof nm, two ? "k_pass_fused2<%d>" : "k_pass_fused<%d>", P.logR);
    const double n = double(L.ncols) * P.R;
    prof_mark(nm, st, np * (n * P.logR * (two ? 1.5 : 1.0) + n + (a.has_final_scale ? n : 0)),
              np * (other ? 24 : 16) * n);
  }
  ++launches_;
}

void Engine::passes_inv(const PrimePlan* pl[2], int np, u64* const data[2], std::size_t begin, std::size_t end,
                        const ShardGeom* sg, cudaStream_t st) {
  bool any_table = false;
  for (const auto& ps : pl[0]->passes) any_table |= ps->radix3 || ps->S > 1;
  for (std::size_t ii = end; ii-- > begin;) {
    const PassLocal L = local_pass(*pl[0], ii, sg);
    if (pl[0]->passes[ii]->radix3) {
      Radix3Args a{};
      for (int q = 0; q < np; ++q) {
        a.src[q] = data[q];
        a.dst[q] = data[q];
        a.lo[q] = pl[q]->passes[ii]->r3_lo_inv.ptr;
        a.hi[q] = pl[q]->passes[ii]->r3_hi_inv.ptr;
        a.p[q] = pl[q]->p;
        a.lam[q] = pl[q]->lam_inv;
        a.pinv[q] = pl[q]->r3_merged ? pl[q]->r3_pinv.ptr : nullptr;
      }
      if (pl[0]->r3_merged) {
        a.pre_shift = pl[0]->passes[1]->logS;
        a.pre_rows = pl[0]->passes[1]->R;
      }
      a.S = L.S;
      a.lbits = pl[0]->passes[ii]->r3_lbits;
      a.hrow = pl[0]->passes[ii]->S >> a.lbits;
      a.cb = L.cb;
      a.sb = L.sb;
      a.off = L.off;
      launch_radix3(true, a, np, st);
      prof_mark("k_radix3_inv", st, double(np) * 4.0 * double(L.S), double(np) * 48.0 * double(L.S));
    } else {
      PassArgs a{};
      const PassPlan& P = *pl[0]->passes[ii];
      for (int q = 0; q < np; ++q) {
        const PassPlan& Pq = *pl[q]->passes[ii];
        a.src[q] = data[q];
        a.dst[q] = data[q];
        a.dft_fwd[q] = Pq.dft_fwd.ptr;
        a.dft_inv[q] = Pq.dft_inv.ptr;
        a.pass_tw[q] = Pq.S > 1 ? Pq.tw_inv.ptr : nullptr;
        a.pass_hi[q] = Pq.hi_inv.ptr;
        a.final_scale[q] = pl[q]->final_scale;
        a.p[q] = pl[q]->p;
        a.pp[q] = pl[q]->pp;
      }
      a.S = L.S;
      a.logS = L.logS;
      a.G = L.groups;
      a.tw_logS = L.tw_logS;
      a.tw_off = L.tw_off;
      a.has_final_scale = (!any_table && ii == 0) ? 1 : 0;
      a.lazy_out = inverse_lazy_ok(*pl[0], ii) ? 1 : 0;
      a.tw_lbits = P.tw_lbits;
      a.tw_gstride = P.tw_gstride;
      a.hi_gstride = P.hi_gstride;
      launch_pass_inv(P.logR, a, L.ncols, np, st);
      if (prof_on_) {
        char nm[64];
        std::snprintf(nm, sizeof nm, "k_pass_inv<%d,%s>", P.logR, L.S > 1 ? "rows" : "cols");
        const double n = double(L.ncols) * P.R;
        const double tb = (L.S > 1 && !P.tw_lbits) ? np * 16.0 * n / (P.tw_gstride ? 1.0 : double(L.groups)) : 0.0;
        prof_mark(nm, st, np * (n / 2 * P.logR + (L.S > 1 ? n : 0) + (a.has_final_scale ? n : 0)), np * 16 * n + tb);
      }
    }
    ++launches_;
  }
}

void Engine::transform_forward(const PrimePlan* pl[2], int np, const u64* const src[2], u64* const dst[2],
                               bool include_last, cudaStream_t st) {
  const std::size_t m = pl[0]->passes.size();
  passes_fwd(pl, np, src, dst, 0, include_last ? m : (m ? m - 1 : 0), nullptr, st);
}

// Forward transform of limbs packed into data[1] (both primes' outputs in data[0..1]).
void Engine::transform_forward_packed(const PrimePlan* pl[2], u64* const data[2], bool include_last,
                                      cudaStream_t st) {
  const std::size_t m = pl[0]->passes.size();
  const std::size_t end = include_last ? m : (m ? m - 1 : 0);
  if (end == 0) {  // no forward pass at all (N == 1, or one fused pass): just duplicate
    cuda_check(cudaMemcpyAsync(data[0], data[1], padded_len(*pl[0]) * sizeof(u64), cudaMemcpyDeviceToDevice, st),
               "copy");
    return;
  }
  const u64* packed[2] = {data[1], data[1]};
  const PrimePlan* p0[2] = {pl[0], pl[0]};
  const PrimePlan* p1[2] = {pl[1], pl[1]};
  u64* d0[2] = {data[0], data[0]};
  u64* d1[2] = {data[1], data[1]};
  passes_fwd(p0, 1, packed, d0, 0, 1, nullptr, st);  // prime 0 reads the packed limbs ...
  passes_fwd(p1, 1, packed, d1, 0, 1, nullptr, st);  // ... before prime 1 overwrites them in place
  passes_fwd(pl, 2, data, data, 1, end, nullptr, st);
}

void Engine::transform_fused_last(const PrimePlan* pl[2], int np, u64* const data[2], const u64* const other[2],
                                  cudaStream_t st) {
  pass_fused(pl, np, data, other, nullptr, st);
}

void Engine::transform_inverse(const PrimePlan* pl[2], int np, u64* const data[2], bool skip_last,
                               cudaStream_t st) {
  const std::size_t m = pl[0]->passes.size();
  passes_inv(pl, np, data, 0, skip_last ? (m ? m - 1 : 0) : m, nullptr, st);
}

void Engine::check_err(cudaStream_t st) { check_word(err_.ptr, st); }
void Engine::check_async_errors(cudaStream_t st) { check_word(async_err_.ptr, st ? st : stream_); }

void Engine::check_word(unsigned* word, cudaStream_t st) {
  unsigned e = 0;
  cuda_check(cudaMemcpyAsync(&e, word, sizeof e, cudaMemcpyDeviceToHost, st), "err readback");
  cuda_check(cudaStreamSynchronize(st), "sync");
  if (e) {
    cuda_check(cudaMemsetAsync(word, 0, sizeof(unsigned), st), "memset");
    cuda_check(cudaStreamSynchronize(st), "sync");
  }
  throw_err_bits(e);
}

void Engine::throw_err_bits(unsigned e) {
  if (e & kErrBadDigit) throw std::invalid_argument("decimal: non-digit character");
  if (e & kErrLeadingZero) throw std::invalid_argument("decimal: leading zero");
  if (e & kErrCoeffBound)
    throw CorruptionError("recover_digits: coefficient exceeds analytic bound (upstream corruption)");
  if (e & kErrCarryBound) throw CorruptionError("recover_digits: carry exceeds analytic bound (upstream corruption)");
}

namespace {

CrtConsts crt_consts_impl(u64 p1, u64 p2) {  // make_crt_ctx, decimal.cpp:136-146
  if (p1 >= p2) throw std::invalid_argument("make_crt_ctx: requires p1 < p2");
  HostField F2(p2);
  return {F2.pp, F2.to_mont(F2.inv(p1 % p2))};
}

void coeff_cap(unsigned be, std::size_t min_limbs, u64& lo, u64& hi) {
  const u128 top = pow10u(be) - 1, unit = top * top;
  const u128 cap = (u128)min_limbs <= ~(u128)0 / unit ? unit * min_limbs : ~(u128)0;
  lo = u64(cap);
  hi = u64(cap >> 64);
}

}  // namespace

const unsigned long long kOneLen = 1;  // product length of the zero short-circuit

// Algorithmic modular multiplications of one product: T(2^k) = (N/2) k (+ N for
// a six-step twiddle when N > 2^15), T(3c) = 8c + 3 T(c); M = 2 (3 T(N) + N) + N, squaring
// 2 (2 T(N) + N) + N.
static double alg_modmuls(std::size_t N, bool squaring) {
  std::function<double(std::size_t)> T = [&](std::size_t m) -> double {
    if (m % 3 == 0) return 8.0 * double(m / 3) + 3.0 * T(m / 3);
    const int k = m > 1 ? __builtin_ctzll(m) : 0;
    return double(m / 2) * k + (m > (std::size_t(1) << 15) ? double(m) : 0.0);
  };
  return 2.0 * ((squaring ? 2.0 : 3.0) * T(N) + double(N)) + double(N);
}

// Whether every coefficient c <= (B - 1)^2 min_limbs is < B^3, so three base-B digits and
// {0,1,2} carries suffice (always for lambda >= 13: c < p1 p2 < 2^127 < 10^39).
static bool carry3_exact(unsigned be, std::size_t min_limbs) {
  if (be >= 13) return true;
  const u128 B = pow10u(be), top = B - 1;
  return top * top * (u128)min_limbs < B * B * B;
}

int Engine::recover(CarryArgs c, unsigned be, std::size_t min_limbs, bool allow_s_in_x, cudaStream_t st) {
  (void)allow_s_in_x;
  c.ticket = ticket_.ptr;
  if (carry3_exact(be, min_limbs)) {
    pm_.ensure((c.n + 2 + 2 * kCarryChunk) / kCarryChunk * kCarryChunk);
    c.pm = pm_.ptr;
    return launch_carry(c, st);
  }
  // D = base-B digits of the coefficient cap; normalisation rounds until every sum <= 3 (B - 1)
  const u128 B = pow10u(be), cap = ((u128)c.coeff_cap_hi << 64) | c.coeff_cap_lo;
  int D = 1;
  for (u128 pw = B; pw <= cap; ++D) {
    if (pw > ~(u128)0 / B) {
      ++D;
      break;
    }
    pw *= B;
  }
  int rounds = 0;
  for (u128 bound = (u128)D * (B - 1); bound > 3 * (B - 1); ++rounds) bound = (B - 1) + bound / B;
  const std::size_t K = c.n + std::size_t(D) + std::size_t(rounds);
  const std::size_t s_words = (K + kCarryChunk - 1) / kCarryChunk * kCarryChunk;
  S_.ensure(s_words);
  S2_.ensure(s_words);
  maps_.ensure(carry_map_words(K));
  c.s = S_.ptr;
  c.maps = maps_.ptr;
  pm_.ensure((K + 2 * kCarryChunk) / kCarryChunk * kCarryChunk);
  c.pm = pm_.ptr;
  return launch_carry_general(c, D, rounds, S2_.ptr, K, st);
}

void Engine::pack_radix3(const PrimePlan* pl[2], const char* digits, std::size_t nd, unsigned be, u64* const dst[2],
                         unsigned* err, cudaStream_t st) {
  const PassPlan& P = *pl[0]->passes[0];
  Radix3Args a{};
  for (int q = 0; q < 2; ++q) {
    a.src[q] = nullptr;
    a.dst[q] = dst[q];
    a.lo[q] = pl[q]->passes[0]->r3_lo_fwd.ptr;
    a.hi[q] = pl[q]->passes[0]->r3_hi_fwd.ptr;
    a.p[q] = pl[q]->p;
    a.lam[q] = pl[q]->lam;
  }
  a.notw = pl[0]->r3_merged ? 1 : 0;
  a.S = P.S;
  a.lbits = P.r3_lbits;
  a.hrow = P.S >> a.lbits;
  launch_pack_radix3(digits, nd, be, a, err, st);
  ++launches_;
  prof_mark("k_pack_radix3", st, 2.0 * double(P.S) * 5.0, double(nd) + 48.0 * double(P.S));
}

void Engine::run_product(const ProductPlan& pp, const char* dx, const char* dy, bool squaring, char* dout,
                         cudaStream_t st, unsigned* err, const std::function<void()>& before_y) {
  const PrimePlan& P1 = prime_plan(pp.p1, pp.N);
  const PrimePlan& P2 = prime_plan(pp.p2, pp.N);
  const unsigned be = pp.base_exp;
  const std::size_t lx = (pp.dx + be - 1) / be, ly = (pp.dy + be - 1) / be;
  const CrtConsts cc = crt_consts(pp.p1, pp.p2);
  const DivB div = div_for(pow10u(be));
  u64 cap_lo, cap_hi;
  coeff_cap(be, std::min(lx, ly), cap_lo, cap_hi);
  const bool carry3 = carry3_exact(be, std::min(lx, ly));
  launches_ = 0;
  ProfScope prof_scope(this);
  prof_mark(nullptr, st);

  if (P1.small_ok && P2.small_ok && carry3) {
    if (before_y) before_y();
    SmallArgs a{};
    a.xs = dx;
    a.ys = squaring ? dx : dy;
    a.x_stride = a.y_stride = 0;
    a.nx = pp.dx;
    a.ny = pp.dy;
    a.outs = dout;
    a.out_stride = 0;
    lens_.ensure(1);
    a.out_lens = lens_.ptr;
    a.count = 1;
    a.base_exp = be;
    a.logc = P1.k;
    a.three = P1.three;
    const PrimePlan* pls[2] = {&P1, &P2};
    for (int q = 0; q < 2; ++q) {
      a.p[q] = pls[q]->p;
      a.pp[q] = pls[q]->pp;
      a.dft_fwd[q] = pls[q]->small_fwd.ptr;
      a.dft_inv[q] = pls[q]->small_inv.ptr;
      a.r3_fwd[q] = pls[q]->r3_fwd.ptr;
      a.r3_inv[q] = pls[q]->r3_inv.ptr;
      a.lam[q] = pls[q]->lam;
      a.lam_inv[q] = pls[q]->lam_inv;
      a.scale[q] = pls[q]->final_scale;
    }
    a.p2_prime = cc.p2_prime;
    a.r_tilde = cc.r_tilde;
    a.div = div;
    a.coeff_cap_lo = cap_lo;
    a.coeff_cap_hi = cap_hi;
    a.err = err;
    a.squaring = squaring ? 1 : 0;
    if (!launch_small(a, st)) throw CudaError("small kernel launch failed");
    cuda_check(cudaGetLastError(), "small kernel");
    prof_mark("k_small", st, alg_modmuls(pp.N, squaring), double(2 * (pp.dx + pp.dy)));
    cuda_check(cudaMemcpyAsync(meta_.ptr + 2, lens_.ptr, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st),
               "meta");
    launches_ = 1;
    return;
  }

  // HBM plan. Large transforms (>= 2 GB per residue array; config 5 is 12.9 GB) pack
  // the limbs straight into the second prime's array, and the first pass reads them from
  // there (prime 0 out of place, then prime 1 in place), so no packed-limb buffers; the
  // carry's limb sums reuse the x spectrum, dead after the pointwise product. Smaller
  // ones keep separate packed buffers so the first pass runs both primes in one launch.
  const std::size_t npad = padded_len(P1);
  const std::size_t K = pp.N + 2;
  const std::size_t nchunks = (K + kCarryChunk - 1) / kCarryChunk;
  const std::size_t s_words = nchunks * kCarryChunk;
  const char* force_lean = std::getenv("DECMUL_FORCE_LEAN");  // test knob: lean plan at any size
  const bool lean = npad * sizeof(u64) >= (std::size_t(2) << 30) || (force_lean && force_lean[0] == '1');
  const bool s_in_x = lean && !squaring && carry3;
  X_[0].ensure(s_in_x ? std::max(npad, s_words) : npad);
  X_[1].ensure(npad);
  if (!squaring) {
    Y_[0].ensure(npad);
    Y_[1].ensure(npad);
  }
  // N = 3 S: the pack runs inside the first (radix-3) pass, no packed-limb buffer at all
  const bool fuse_r3 = !P1.passes.empty() && P1.passes[0]->radix3;
  if (!s_in_x) S_.ensure(s_words);
  if (!lean && !fuse_r3) {
    Px_.ensure(npad);
    if (!squaring) Py_.ensure(npad);
  }
  maps_.ensure(carry_map_words(K));
  u64* s_buf = s_in_x ? X_[0].ptr : S_.ptr;
  u64* px = lean ? X_[1].ptr : Px_.ptr;
  u64* py = lean ? Y_[1].ptr : Py_.ptr;

  const PrimePlan* pl[2] = {&P1, &P2};
  const std::size_t m = P1.passes.size();
  // the inverse radix-3 pass runs inside the carry split (no natural-order coefficients in HBM)
  const bool fuse_r3_carry = fuse_r3 && carry3 && carry_r3_fusable(P1.passes[0]->S);
  auto inverse = [&](u64* const z[2]) {
    passes_inv(pl, 2, z, fuse_r3_carry ? 1 : 0, P1.last_pow2 ? m - 1 : m, nullptr, st);
  };
  // digits -> forward transform (all passes, or all but the last when it is fused with the
  // pointwise product)
  auto load = [&](const char* dd, std::size_t nd, u64* packed, u64* const dst[2], bool include_last) {
    if (fuse_r3) {
      pack_radix3(pl, dd, nd, be, dst, err, st);
      const u64* src[2] = {dst[0], dst[1]};
      passes_fwd(pl, 2, src, dst, 1, include_last ? m : m - 1, nullptr, st);
      return;
    }
    launch_pack(dd, nd, be, packed, npad, err, st);
    prof_mark("k_pack", st, 0, double(nd) + 8.0 * npad);
    ++launches_;
    if (lean) {
      transform_forward_packed(pl, dst, include_last, st);
    } else {
      const u64* src[2] = {packed, packed};
      transform_forward(pl, 2, src, dst, include_last, st);
    }
  };
  u64* Z[2];
  if (squaring) {
    u64* X[2] = {X_[0].ptr, X_[1].ptr};
    load(dx, pp.dx, px, X, !P1.last_pow2);
    if (P1.last_pow2) {
      transform_fused_last(pl, 2, X, nullptr, st);
    } else {
      for (int q = 0; q < 2; ++q) launch_pointwise(X[q], X[q], pp.N, pl[q]->p, pl[q]->pp, st);
      prof_mark("k_pointwise", st, 2.0 * pp.N, 32.0 * pp.N);
      launches_ += 2;
    }
    inverse(X);
    Z[0] = X[0];
    Z[1] = X[1];
  } else {
    u64* X[2] = {X_[0].ptr, X_[1].ptr};
    u64* Y[2] = {Y_[0].ptr, Y_[1].ptr};
    // two-operand fused last pass (x's last forward pass inside the pointwise kernel) when the
    // transform has at least two passes (DECMUL_FUSE2=0: x's last pass as its own launch)
    const char* f2 = std::getenv("DECMUL_FUSE2");
    // (R = 512: two 64 KB tiles would leave one CTA per SM)
    const bool two = P1.last_pow2 && m >= 2 && P1.passes[m - 1]->logR <= 8 && !(f2 && f2[0] == '0');
    // small transforms are launch-latency bound: both operands share the pack launch and each
    // forward pass launch (blockIdx.y = operand); larger ones keep y's upload overlapping x's work
    const bool paired = two && !lean && !fuse_r3 && pp.N <= (std::size_t(1) << 21);
    if (paired) {
      if (before_y) before_y();
      launch_pack2(dx, pp.dx, px, dy, pp.dy, py, be, npad, err, st);
      prof_mark("k_pack2", st, 0, double(pp.dx + pp.dy) + 16.0 * npad);
      ++launches_;
      const u64* sx[2] = {px, px};
      const u64* sy[2] = {py, py};
      passes_fwd(pl, 2, sx, X, 0, m - 1, nullptr, st, sy, Y);
    } else {
      load(dx, pp.dx, px, X, !two);
      if (before_y) before_y();
      load(dy, pp.dy, py, Y, !P1.last_pow2);
    }
    if (P1.last_pow2) {
      const u64* oth[2] = {X[0], X[1]};
      pass_fused(pl, 2, Y, oth, nullptr, st, two);
    } else {
      for (int q = 0; q < 2; ++q) launch_pointwise(Y[q], X[q], pp.N, pl[q]->p, pl[q]->pp, st);
      prof_mark("k_pointwise", st, 2.0 * pp.N, 48.0 * pp.N);
      launches_ += 2;
    }
    inverse(Y);
    Z[0] = Y[0];
    Z[1] = Y[1];
  }
  if (P1.passes.empty()) {  // N == 1: no kernel carried the convolution scale
    for (int q = 0; q < 2; ++q) {
      HostField F(pl[q]->p);
      launch_mont_scale(Z[q], 1, F.to_mont(pl[q]->conv_scale), pl[q]->p, pl[q]->pp, st);
    }
  }
  CarryArgs c{};
  c.z1 = Z[0];
  c.z2 = Z[1];
  c.n = pp.N;
  c.p1 = pp.p1;
  c.p2 = pp.p2;
  c.p2_prime = cc.p2_prime;
  c.r_tilde = cc.r_tilde;
  c.div = div;
  c.coeff_cap_lo = cap_lo;
  c.coeff_cap_hi = cap_hi;
  c.base_exp = be;
  c.s = s_buf;
  c.maps = maps_.ptr;
  c.err = err;
  const unsigned long long dsum = pp.dx + pp.dy;
  c.top_candidates[0] = dsum >= 2 ? (dsum - 2) / be : 0;
  c.top_candidates[1] = (dsum - 1) / be;
  c.meta = meta_.ptr;
  c.out = dout;
  c.tail = 1;
  if (fuse_r3_carry) {
    const PassPlan& P0 = *P1.passes[0];
    Radix3Args r{};
    for (int q = 0; q < 2; ++q) {
      r.src[q] = Z[q];
      r.dst[q] = nullptr;
      r.lo[q] = pl[q]->passes[0]->r3_lo_inv.ptr;
      r.hi[q] = pl[q]->passes[0]->r3_hi_inv.ptr;
      r.p[q] = pl[q]->p;
      r.lam[q] = pl[q]->lam_inv;
      r.pinv[q] = pl[q]->r3_merged ? pl[q]->r3_pinv.ptr : nullptr;
    }
    if (P1.r3_merged) {
      r.pre_shift = P1.passes[1]->logS;
      r.pre_rows = P1.passes[1]->R;
    }
    r.S = P0.S;
    r.lbits = P0.r3_lbits;
    r.hrow = P0.S >> r.lbits;
    pm_.ensure((pp.N + 2 + 2 * kCarryChunk) / kCarryChunk * kCarryChunk);
    c.pm = pm_.ptr;
    launches_ += launch_carry_r3(c, r, st);
  } else {
    launches_ += recover(c, be, std::min(lx, ly), s_in_x, st);
  }
  cuda_check(cudaGetLastError(), "product kernels");
}

std::size_t Engine::multiply_device(const char* dx, std::size_t nx, const char* dy, std::size_t ny, char* dout,
                                    std::size_t cap, unsigned forced, bool squaring, cudaStream_t st, bool sync) {
  if (nx == 0 || ny == 0) throw std::invalid_argument("decimal: empty string");
  if (!st) st = stream_;
  if (nx == 1 || ny == 1) {  // zero short-circuit (decimal.cpp:193), before any size checks
    // both texts are validated first, as DecimalNumber::parse does for the reference's operands
    launch_validate(dx, nx, err_.ptr, st);
    if (!squaring) launch_validate(dy, ny, err_.ptr, st);
    char a = 0, b = 0;
    if (nx == 1) cuda_check(cudaMemcpyAsync(&a, dx, 1, cudaMemcpyDeviceToHost, st), "zero check");
    if (ny == 1) cuda_check(cudaMemcpyAsync(&b, dy, 1, cudaMemcpyDeviceToHost, st), "zero check");
    check_err(st);  // synchronises st: a and b are valid after this
    if (a == '0' || b == '0') {
      if (cap < 1) throw std::length_error("multiply: output buffer too small");
      cuda_check(cudaMemcpyAsync(dout, "0", 1, cudaMemcpyHostToDevice, st), "zero");
      cuda_check(cudaMemcpyAsync(meta_.ptr + 2, &kOneLen, sizeof kOneLen, cudaMemcpyHostToDevice, st), "meta");
      cuda_check(cudaStreamSynchronize(st), "sync");
      return 1;
    }
  }
  const ProductPlan pp = plan_product(nx, ny, forced);
  if (cap < nx + ny) throw std::length_error("multiply: output buffer too small");
  run_product(pp, dx, squaring ? dx : dy, squaring, dout, st, sync ? err_.ptr : async_err_.ptr);
  if (!sync) return 0;
  unsigned long long len = 0;
  cuda_check(cudaMemcpyAsync(&len, meta_.ptr + 2, sizeof len, cudaMemcpyDeviceToHost, st), "len");
  check_err(st);
  return std::size_t(len);
}

std::size_t Engine::result_length() {
  unsigned long long len = 0;
  cuda_check(cudaMemcpyAsync(&len, meta_.ptr + 2, sizeof len, cudaMemcpyDeviceToHost, stream_), "len");
  check_word(async_err_.ptr, stream_);
  return std::size_t(len);
}

std::size_t Engine::multiply_host(const char* x, std::size_t nx, const char* y, std::size_t ny, char* out,
                                  std::size_t cap, unsigned forced, bool alias, u64 p1, u64 p2) {
  if (nx == 0 || ny == 0) throw std::invalid_argument("decimal: empty string");
  if ((nx == 1 && x[0] == '0') || (ny == 1 && y[0] == '0')) {  // zero short-circuit (decimal.cpp:193)
    if (cap < 1) throw std::length_error("multiply: output buffer too small");
    out[0] = '0';
    return 1;
  }
  const bool squaring = alias || (nx == ny && (x == y || std::memcmp(x, y, nx) == 0));
  const ProductPlan pp = plan_product(nx, ny, forced, p1, p2);
  if (cap < nx + ny) throw std::length_error("multiply: output buffer too small");
  din_x_.ensure(nx);
  if (!squaring) din_y_.ensure(ny);
  dout_.ensure(nx + ny);
  // x uploads on the copy stream; the product runs on the context stream once x is in
  // HBM, and y uploads while x is packed and transformed (run_product's before_y)
  cudaStream_t cs = pipe_[0], st = stream_;
  cuda_check(cudaEventRecord(pipe_ev_, st), "event");
  cuda_check(cudaStreamWaitEvent(cs, pipe_ev_, 0), "wait");
  stage_h2d(din_x_.ptr, x, nx, cs);
  cuda_check(cudaEventRecord(up_ev_[0], cs), "event");
  cuda_check(cudaStreamWaitEvent(st, up_ev_[0], 0), "wait");
  run_product(pp, din_x_.ptr, squaring ? din_x_.ptr : din_y_.ptr, squaring, dout_.ptr, st, err_.ptr, [&] {
    if (squaring) return;
    stage_h2d(din_y_.ptr, y, ny, cs);
    cuda_check(cudaEventRecord(up_ev_[1], cs), "event");
    cuda_check(cudaStreamWaitEvent(st, up_ev_[1], 0), "wait");
  });
  // The length comes back through pinned memory and, when the output goes straight to DMA
  // (pinned or small), the product's nx + ny bytes are copied behind it before the error word
  // is read: one synchronisation instead of three (a product is nx + ny or nx + ny - 1 digits
  // long; cap >= nx + ny was checked above).
  if (host_lens_n_ < 1) {
    cuda_check(cudaMallocHost(&host_lens_, 1024 * sizeof(unsigned long long)), "cudaMallocHost");
    host_lens_n_ = 1024;
  }
  cuda_check(cudaMemcpyAsync(host_lens_, meta_.ptr + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st), "len");
  const bool direct = stage_direct(out, nx + ny);
  if (direct) cuda_check(cudaMemcpyAsync(out, dout_.ptr, nx + ny, cudaMemcpyDeviceToHost, st), "d2h");
  check_err(st);
  const unsigned long long len = host_lens_[0];
  if (len > cap) throw std::length_error("multiply: output buffer too small");
  if (!direct) stage_d2h(out, dout_.ptr, std::size_t(len), st);
  return std::size_t(len);
}

void Engine::multiply_batch_device(std::size_t count, const char* dxs, std::size_t x_stride, std::size_t nx,
                                   const char* dys, std::size_t y_stride, std::size_t ny, char* douts,
                                   std::size_t out_stride, unsigned long long* dlens, cudaStream_t st) {
  batch_device(count, dxs, x_stride, nx, dys, y_stride, ny, douts, out_stride, dlens, st ? st : stream_,
               async_err_.ptr);
}

void Engine::batch_device(std::size_t count, const char* dxs, std::size_t x_stride, std::size_t nx, const char* dys,
                          std::size_t y_stride, std::size_t ny, char* douts, std::size_t out_stride,
                          unsigned long long* dlens, cudaStream_t st, unsigned* err) {
  if (count == 0) return;
  if (nx == 0 || ny == 0) throw std::invalid_argument("decimal: empty string");
  if (out_stride < nx + ny) throw std::length_error("multiply_batch: output stride too small");
  const ProductPlan pp = plan_product(nx, ny, 0);
  const PrimePlan& P1 = prime_plan(pp.p1, pp.N);
  const PrimePlan& P2 = prime_plan(pp.p2, pp.N);
  if (!(P1.small_ok && P2.small_ok)) {
    // large products: one after another through the pass engine
    for (std::size_t i = 0; i < count; ++i) {
      run_product(pp, dxs + i * x_stride, dys + i * y_stride, false, douts + i * out_stride, st, err);
      cuda_check(cudaMemcpyAsync(dlens + i, meta_.ptr + 2, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st),
                 "len");
    }
    return;
  }
  const unsigned be = pp.base_exp;
  const std::size_t lx = (nx + be - 1) / be, ly = (ny + be - 1) / be;
  const CrtConsts cc = crt_consts(pp.p1, pp.p2);
  SmallArgs a{};
  a.xs = dxs;
  a.ys = dys;
  a.x_stride = x_stride;
  a.y_stride = y_stride;
  a.nx = nx;
  a.ny = ny;
  a.outs = douts;
  a.out_stride = out_stride;
  a.out_lens = dlens;
  a.base_exp = be;
  a.logc = P1.k;
  a.three = P1.three;
  const PrimePlan* pls[2] = {&P1, &P2};
  for (int q = 0; q < 2; ++q) {
    a.p[q] = pls[q]->p;
    a.pp[q] = pls[q]->pp;
    a.dft_fwd[q] = pls[q]->small_fwd.ptr;
    a.dft_inv[q] = pls[q]->small_inv.ptr;
    a.r3_fwd[q] = pls[q]->r3_fwd.ptr;
    a.r3_inv[q] = pls[q]->r3_inv.ptr;
    a.lam[q] = pls[q]->lam;
    a.lam_inv[q] = pls[q]->lam_inv;
    a.scale[q] = pls[q]->final_scale;
  }
  a.p2_prime = cc.p2_prime;
  a.r_tilde = cc.r_tilde;
  a.div = div_for(pow10u(be));
  coeff_cap(be, std::min(lx, ly), a.coeff_cap_lo, a.coeff_cap_hi);
  a.err = err;
  a.squaring = 0;
  ProfScope prof_scope(this);
  prof_mark(nullptr, st);
  const std::size_t maxgrid = 1u << 30;
  for (std::size_t off = 0; off < count; off += maxgrid) {
    SmallArgs b = a;
    b.count = unsigned(std::min(maxgrid, count - off));
    b.xs = dxs + off * x_stride;
    b.ys = dys + off * y_stride;
    b.outs = douts + off * out_stride;
    b.out_lens = dlens + off;
    if (!launch_small(b, st)) throw CudaError("small kernel launch failed");
  }
  launches_ = 1;
  cuda_check(cudaGetLastError(), "batch kernel");
  prof_mark("k_small", st, double(count) * alg_modmuls(pp.N, false), double(count) * 2.0 * double(nx + ny));
}

void Engine::multiply_batch_host(std::size_t count, const char* xs, std::size_t x_stride, std::size_t nx,
                                 const char* ys, std::size_t y_stride, std::size_t ny, char* outs,
                                 std::size_t out_stride, std::size_t* lens, std::unique_lock<std::mutex>* ctx_lock) {
  if (count == 0) return;
  if (nx == 0 || ny == 0) throw std::invalid_argument("decimal: empty string");
  const ProductPlan pp = plan_product(nx, ny, 0);
  // the chunked upload / compute / download pipeline pays from two waves of one-CTA products
  // up; a smaller batch (e.g. a handful of coalesced concurrent calls) is one partial wave:
  // one copy in, one launch, one copy out
  const PrimePlan& Pb = prime_plan(pp.p1, pp.N);
  if (Pb.small_ok && prime_plan(pp.p2, pp.N).small_ok) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_);
    const std::size_t wave = std::size_t(sms) * std::max(1, small_resident_ctas(Pb.k, Pb.three, 0));
    if (count >= 2 * wave) {
      batch_host_pipelined(count, xs, x_stride, nx, ys, y_stride, ny, outs, out_stride, lens, ctx_lock);
      return;
    }
  }
  const std::size_t xb = (count - 1) * x_stride + nx, yb = (count - 1) * y_stride + ny;
  const std::size_t ob = count * out_stride;
  din_x_.ensure(xb);
  din_y_.ensure(yb);
  dout_.ensure(ob);
  lens_.ensure(count);
  cuda_check(cudaMemcpyAsync(din_x_.ptr, xs, xb, cudaMemcpyHostToDevice, stream_), "h2d");
  cuda_check(cudaMemcpyAsync(din_y_.ptr, ys, yb, cudaMemcpyHostToDevice, stream_), "h2d");
  batch_device(count, din_x_.ptr, x_stride, nx, din_y_.ptr, y_stride, ny, dout_.ptr, out_stride, lens_.ptr,
               stream_, err_.ptr);
  // lengths into pinned memory: a pageable destination would block here until the kernel is done,
  // and the product copy behind it
  if (host_lens_n_ < count) {
    if (host_lens_) cudaFreeHost(host_lens_);
    host_lens_ = nullptr;
    host_lens_n_ = 0;
    const std::size_t want = std::max<std::size_t>(count, 1024);
    cuda_check(cudaMallocHost(&host_lens_, want * sizeof(unsigned long long)), "cudaMallocHost");
    host_lens_n_ = want;
  }
  cuda_check(cudaMemcpyAsync(host_lens_, lens_.ptr, count * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             stream_), "d2h");
  cuda_check(cudaMemcpyAsync(outs, dout_.ptr, ob, cudaMemcpyDeviceToHost, stream_), "d2h");
  check_err(stream_);
  for (std::size_t i = 0; i < count; ++i) lens[i] = std::size_t(host_lens_[i]);
}

// Chunks of products flow through three streams — upload, compute, download — linked by
// per-chunk events, so chunk c's H2D overlaps chunk c-1's kernel and chunk c-2's D2H (one
// copy engine per direction; PCIe is full duplex). One-CTA products share no device
// workspace, so the chunks are independent.
void Engine::batch_host_pipelined(std::size_t count, const char* xs, std::size_t x_stride, std::size_t nx,
                                  const char* ys, std::size_t y_stride, std::size_t ny, char* outs,
                                  std::size_t out_stride, std::size_t* lens, std::unique_lock<std::mutex>* ctx_lock) {
  // whole waves of the one-CTA kernel per chunk (a partial wave costs a full one)
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_);
  const ProductPlan pp = plan_product(nx, ny, 0);
  const PrimePlan& P1 = prime_plan(pp.p1, pp.N);
  const std::size_t wave = std::size_t(sms) * std::max(1, small_resident_ctas(P1.k, P1.three, 0));
  // ~5 equal chunks of whole waves: fewer chunks lengthen pipeline fill and drain, more
  // lose duplex copy throughput (measured on B200: both directions together sustain
  // ~41-49 GB/s each for 9-20 MB copies, ~36 GB/s for 4 MB ones).
  // DECMUL_PIPE_CHUNKS=k forces k equal chunks (tuning).
  // With another batch call in flight (calls from several threads overlap, below) fill and
  // drain hide behind the neighbours and larger copies win: 3 chunks (config 2 from three
  // threads: 2.08 ms per batch against 2.24 with 5; one caller alone: 2.52 against 2.47).
  struct InFlight {
    std::atomic<int>& c;
    int before;
    explicit InFlight(std::atomic<int>& c_) : c(c_), before(c_.fetch_add(1)) {}
    ~InFlight() { c.fetch_sub(1); }
  } in_flight(batch_active_);
  std::size_t k = in_flight.before > 0 ? 3 : 5;
  if (const char* e = std::getenv("DECMUL_PIPE_CHUNKS")) k = std::max<std::size_t>(1, std::strtoull(e, 0, 10));
  k = std::min<std::size_t>(std::min<std::size_t>(k, count), kMaxChunks);
  std::size_t per = (count + k - 1) / k;
  // whole waves per chunk for a lone call (rounding can add a short last chunk); equal chunks
  // when calls overlap
  if (!std::getenv("DECMUL_PIPE_CHUNKS") && in_flight.before == 0 && per > wave) per = (per + wave / 2) / wave * wave;
  while ((count + per - 1) / per > std::size_t(kMaxChunks)) per += wave;
  std::vector<std::size_t> bounds{0};
  for (std::size_t c = per; c < count; c += per) bounds.push_back(c);
  bounds.push_back(count);
  // Calls from several threads overlap (pinned buffers, the caller's context lock handed in):
  // the lock is held only while the chunks are enqueued; each call works in one of two buffer
  // sets (digits, lengths, error word), so the next call's uploads follow this call's on the
  // upload stream while this one still computes and downloads -- a call's pipeline fill and
  // drain disappear behind its neighbours'. The set's own lock is held until the lengths have
  // been copied out.
  const bool overlap = ctx_lock && ctx_lock->owns_lock() && host_pinned(xs) && host_pinned(ys) && host_pinned(outs) &&
                       !(std::getenv("DECMUL_OVERLAP") && std::getenv("DECMUL_OVERLAP")[0] == '0');
  BatchSet* B = nullptr;
  std::unique_lock<std::mutex> set_lock;
  if (overlap) {
    B = &bsets_[bset_ ^= 1];
    set_lock = std::unique_lock<std::mutex>(B->mu);  // waits for the call that used this set last
    if (!B->done) {
      cuda_check(cudaEventCreateWithFlags(&B->done, cudaEventDisableTiming), "cudaEventCreate");
      cuda_check(cudaMallocHost(&B->h_err, sizeof(unsigned)), "cudaMallocHost");
      B->err.ensure(1);
      cuda_check(cudaMemsetAsync(B->err.ptr, 0, sizeof(unsigned), stream_), "memset");
    }
    B->dx.ensure((count - 1) * x_stride + nx);
    B->dy.ensure((count - 1) * y_stride + ny);
    B->lens.ensure(count);
    B->dout.ensure(count * out_stride);
    B->h_lens.ensure(count * sizeof(unsigned long long));
  } else {
    din_x_.ensure((count - 1) * x_stride + nx);
    din_y_.ensure((count - 1) * y_stride + ny);
    lens_.ensure(count);
    dout_.ensure(count * out_stride);
    if (host_lens_n_ < count) {
      if (host_lens_) cudaFreeHost(host_lens_);
      host_lens_ = nullptr;
      host_lens_n_ = 0;
      cuda_check(cudaMallocHost(&host_lens_, count * sizeof(unsigned long long)), "cudaMallocHost");
      host_lens_n_ = count;
    }
  }
  char* const d_x = overlap ? B->dx.ptr : din_x_.ptr;
  char* const d_y = overlap ? B->dy.ptr : din_y_.ptr;
  char* const d_o = overlap ? B->dout.ptr : dout_.ptr;
  unsigned long long* const d_l = overlap ? B->lens.ptr : lens_.ptr;
  unsigned long long* const h_l = overlap ? reinterpret_cast<unsigned long long*>(B->h_lens.ptr) : host_lens_;
  unsigned* const d_err = overlap ? B->err.ptr : err_.ptr;
  cuda_check(cudaEventRecord(pipe_ev_, stream_), "event");  // after any earlier work of this context
  for (auto s : pipe_) cuda_check(cudaStreamWaitEvent(s, pipe_ev_, 0), "wait");
  // DECMUL_PIPE_TRACE=1: per-chunk stage timestamps on stderr (debugging the overlap)
  const bool trace = std::getenv("DECMUL_PIPE_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto mark = [&](cudaStream_t s) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    tev.push_back(e);
  };
  mark(stream_);
  int launched = 0;
  for (std::size_t c = 0; c + 1 < bounds.size(); ++c) {
    const std::size_t c0 = bounds[c], n = bounds[c + 1] - c0;
    if (n == 0) continue;
    cudaStream_t up = pipe_[0], comp = pipe_[1], down = pipe_[2];
    cuda_check(cudaMemcpyAsync(d_x + c0 * x_stride, xs + c0 * x_stride, (n - 1) * x_stride + nx,
                               cudaMemcpyHostToDevice, up), "h2d");
    cuda_check(cudaMemcpyAsync(d_y + c0 * y_stride, ys + c0 * y_stride, (n - 1) * y_stride + ny,
                               cudaMemcpyHostToDevice, up), "h2d");
    mark(up);
    cuda_check(cudaEventRecord(up_ev_[c], up), "event");
    cuda_check(cudaStreamWaitEvent(comp, up_ev_[c], 0), "wait");
    batch_device(n, d_x + c0 * x_stride, x_stride, nx, d_y + c0 * y_stride, y_stride, ny, d_o + c0 * out_stride,
                 out_stride, d_l + c0, comp, d_err);
    launched += launches_;
    mark(comp);
    cuda_check(cudaEventRecord(done_ev_[c], comp), "event");
    cuda_check(cudaStreamWaitEvent(down, done_ev_[c], 0), "wait");
    cuda_check(cudaMemcpyAsync(outs + c0 * out_stride, d_o + c0 * out_stride, n * out_stride, cudaMemcpyDeviceToHost,
                               down), "d2h");
    cuda_check(cudaMemcpyAsync(h_l + c0, d_l + c0, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, down),
               "d2h");
    mark(down);
  }
  if (overlap) {
    // the download stream is ordered after every chunk's kernel: the set's error word and the
    // completion event go there, the context lock is released, and only this caller waits
    cudaStream_t down = pipe_[2];
    cuda_check(cudaMemcpyAsync(B->h_err, B->err.ptr, sizeof(unsigned), cudaMemcpyDeviceToHost, down), "err");
    cuda_check(cudaEventRecord(B->done, down), "event");
    launches_ = launched;
    ctx_lock->unlock();
    cuda_check(cudaEventSynchronize(B->done), "batch wait");
    if (const unsigned e = *B->h_err) {
      cuda_check(cudaMemsetAsync(B->err.ptr, 0, sizeof(unsigned), down), "memset");
      cuda_check(cudaStreamSynchronize(down), "sync");
      throw_err_bits(e);
    }
    for (std::size_t i = 0; i < count; ++i) lens[i] = std::size_t(h_l[i]);
    return;
  }
  for (auto s : pipe_) {
    cuda_check(cudaEventRecord(pipe_ev_, s), "event");
    cuda_check(cudaStreamWaitEvent(stream_, pipe_ev_, 0), "wait");
  }
  check_err(stream_);
  if (trace) {
    for (std::size_t i = 1; i < tev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, tev[0], tev[i]);
      std::fprintf(stderr, "%s%.3f", i % 3 == 1 ? "\n  up/comp/down " : " ", ms);
    }
    std::fprintf(stderr, "\n");
    for (auto e : tev) cudaEventDestroy(e);
  }
  launches_ = launched;
  for (std::size_t i = 0; i < count; ++i) lens[i] = std::size_t(host_lens_[i]);
}

void Engine::multiply_batch_ptrs(std::size_t count, const char* const* xs, const std::size_t* nxs,
                                 const char* const* ys, const std::size_t* nys, char* const* outs,
                                 const std::size_t* caps, std::size_t* lens) {
  for (std::size_t i = 0; i < count; ++i)
    if (caps[i] < nxs[i] + nys[i]) throw std::length_error("multiply: output buffer too small");
  std::map<std::pair<std::size_t, std::size_t>, std::vector<std::size_t>> groups;
  for (std::size_t i = 0; i < count; ++i) groups[{nxs[i], nys[i]}].push_back(i);
  std::vector<char> vx, vy, vo;
  std::vector<std::size_t> bl;
  for (const auto& [shape, idx] : groups) {
    const auto [nx, ny] = shape;
    // singletons go one by one unless they are one-CTA products (then the gathered pinned
    // path below is the cheaper one: three DMA copies and one launch); so do empty and zero
    // operands (the error path and the zero short-circuit)
    bool single = nx == 0 || ny == 0;
    if (!single && idx.size() < 2) {
      single = true;
      if (!(nx == 1 && xs[idx[0]][0] == '0') && !(ny == 1 && ys[idx[0]][0] == '0')) {
        try {
          const ProductPlan pp = plan_product(nx, ny, 0);
          single = !(prime_plan(pp.p1, pp.N).small_ok && prime_plan(pp.p2, pp.N).small_ok);
        } catch (const std::exception&) {
        }
      }
    }
    if (single) {
      for (std::size_t i : idx) lens[i] = multiply_host(xs[i], nx, ys[i], ny, outs[i], caps[i], 0, false);
      continue;
    }
    const std::size_t m = idx.size(), ostride = nx + ny;
    // the group's operands gathered into one buffer each -- pinned while the group is small
    // (coalesced concurrent calls: a few products), so the batch moves by DMA in three copies
    // instead of the driver's staged pageable path
    char *bx, *by, *bo;
    if (2 * m * ostride <= kGatherMax) {
      gather_.ensure(2 * m * ostride);
      bx = gather_.ptr;
      by = bx + m * nx;
      bo = bx + m * ostride;
    } else {
      vx.resize(m * nx);
      vy.resize(m * ny);
      vo.resize(m * ostride);
      bx = vx.data();
      by = vy.data();
      bo = vo.data();
    }
    bl.resize(m);
    for (std::size_t j = 0; j < m; ++j) {
      std::memcpy(bx + j * nx, xs[idx[j]], nx);
      std::memcpy(by + j * ny, ys[idx[j]], ny);
    }
    multiply_batch_host(m, bx, nx, nx, by, ny, ny, bo, ostride, bl.data());
    for (std::size_t j = 0; j < m; ++j) {
      std::memcpy(outs[idx[j]], bo + j * ostride, bl[j]);
      lens[idx[j]] = bl[j];
    }
  }
}

// ---------------- parity hooks ----------------

void Engine::convolve_mod_p(u64 p, std::size_t n, const u64* x, std::size_t nx, const u64* y, std::size_t ny,
                            u64* out) {
  if (nx > n || ny > n) throw std::invalid_argument("convolve_mod_p: input longer than plan length");
  const PrimePlan& P = prime_plan(p, n);
  const bool squaring = x == y && nx == ny;
  const std::size_t npad = padded_len(P);
  X_[0].ensure(npad);
  Y_[0].ensure(npad);
  cudaStream_t st = stream_;
  cuda_check(cudaMemsetAsync(X_[0].ptr, 0, npad * 8, st), "memset");
  cuda_check(cudaMemcpyAsync(X_[0].ptr, x, nx * 8, cudaMemcpyHostToDevice, st), "h2d");
  if (!squaring) {
    cuda_check(cudaMemsetAsync(Y_[0].ptr, 0, npad * 8, st), "memset");
    cuda_check(cudaMemcpyAsync(Y_[0].ptr, y, ny * 8, cudaMemcpyHostToDevice, st), "h2d");
  }
  const PrimePlan* pl[2] = {&P, &P};
  u64* X[2] = {X_[0].ptr, nullptr};
  u64* Y[2] = {Y_[0].ptr, nullptr};
  const u64* sx[2] = {X_[0].ptr, nullptr};
  const u64* sy[2] = {Y_[0].ptr, nullptr};
  u64* Z = nullptr;
  if (squaring) {
    transform_forward(pl, 1, sx, X, !P.last_pow2, st);
    if (P.last_pow2)
      transform_fused_last(pl, 1, X, nullptr, st);
    else
      launch_pointwise(X[0], X[0], n, p, P.pp, st);
    transform_inverse(pl, 1, X, P.last_pow2, st);
    Z = X[0];
  } else {
    transform_forward(pl, 1, sx, X, true, st);
    transform_forward(pl, 1, sy, Y, !P.last_pow2, st);
    if (P.last_pow2) {
      const u64* oth[2] = {X[0], nullptr};
      transform_fused_last(pl, 1, Y, oth, st);
    } else {
      launch_pointwise(Y[0], X[0], n, p, P.pp, st);
    }
    transform_inverse(pl, 1, Y, P.last_pow2, st);
    Z = Y[0];
  }
  if (P.passes.empty()) {
    HostField F(p);
    launch_mont_scale(Z, 1, F.to_mont(P.conv_scale), p, P.pp, st);
  }
  cuda_check(cudaGetLastError(), "convolve");
  cuda_check(cudaMemcpyAsync(out, Z, n * 8, cudaMemcpyDeviceToHost, st), "d2h");
  cuda_check(cudaStreamSynchronize(st), "sync");
}

void Engine::forward_transform(u64 p, std::size_t n, u64* a, std::size_t thr) {
  if (thr == 0) thr = std::size_t(1) << 15;
  const PrimePlan& P = prime_plan(p, n);
  const std::size_t npad = padded_len(P);
  X_[0].ensure(npad);
  Y_[0].ensure(npad);
  cudaStream_t st = stream_;
  cuda_check(cudaMemcpyAsync(X_[0].ptr, a, n * 8, cudaMemcpyHostToDevice, st), "h2d");
  const PrimePlan* pl[2] = {&P, &P};
  u64* X[2] = {X_[0].ptr, nullptr};
  const u64* sx[2] = {X_[0].ptr, nullptr};
  transform_forward(pl, 1, sx, X, true, st);
  std::vector<unsigned long long> map(n);
  for (std::size_t k = 0; k < n; ++k) map[k] = P.position_of(ref_order_of(n, k, thr));
  DevBuf<unsigned long long> dmap;
  upload(dmap, map, st);
  launch_gather(X_[0].ptr, Y_[0].ptr, dmap.ptr, n, st);
  cuda_check(cudaGetLastError(), "forward");
  cuda_check(cudaMemcpyAsync(a, Y_[0].ptr, n * 8, cudaMemcpyDeviceToHost, st), "d2h");
  cuda_check(cudaStreamSynchronize(st), "sync");
}

void Engine::inverse_transform(u64 p, std::size_t n, u64* a, std::size_t thr) {
  if (thr == 0) thr = std::size_t(1) << 15;
  const PrimePlan& P = prime_plan(p, n);
  const std::size_t npad = padded_len(P);
  X_[0].ensure(npad);
  Y_[0].ensure(npad);
  cudaStream_t st = stream_;
  cuda_check(cudaMemcpyAsync(Y_[0].ptr, a, n * 8, cudaMemcpyHostToDevice, st), "h2d");
  // inverse of the forward gather: position_of(ref_order_of(k)) <- a[k]
  std::vector<unsigned long long> map(n);
  for (std::size_t k = 0; k < n; ++k) map[P.position_of(ref_order_of(n, k, thr))] = k;
  DevBuf<unsigned long long> dmap;
  upload(dmap, map, st);
  launch_gather(Y_[0].ptr, X_[0].ptr, dmap.ptr, n, st);
  const PrimePlan* pl[2] = {&P, &P};
  u64* X[2] = {X_[0].ptr, nullptr};
  transform_inverse(pl, 1, X, false, st);
  HostField F(p);
  // the inverse carries R N^-1 (the convolution fold); one REDC against 1 leaves N^-1
  if (P.passes.empty()) launch_mont_scale(X_[0].ptr, 1, F.to_mont(P.conv_scale), p, P.pp, st);
  launch_mont_scale(X_[0].ptr, n, 1, p, P.pp, st);
  cuda_check(cudaGetLastError(), "inverse");
  cuda_check(cudaMemcpyAsync(a, X_[0].ptr, n * 8, cudaMemcpyDeviceToHost, st), "d2h");
  cuda_check(cudaStreamSynchronize(st), "sync");
}

void Engine::pointwise_product(u64 p, std::size_t n, u64* a, const u64* b) {
  HostField F(p);
  X_[0].ensure(std::max<std::size_t>(n, 1));
  Y_[0].ensure(std::max<std::size_t>(n, 1));
  cudaStream_t st = stream_;
  cuda_check(cudaMemcpyAsync(X_[0].ptr, a, n * 8, cudaMemcpyHostToDevice, st), "h2d");
  cuda_check(cudaMemcpyAsync(Y_[0].ptr, b, n * 8, cudaMemcpyHostToDevice, st), "h2d");
  launch_pointwise(X_[0].ptr, Y_[0].ptr, n, p, F.pp, st);
  cuda_check(cudaGetLastError(), "pointwise");
  cuda_check(cudaMemcpyAsync(a, X_[0].ptr, n * 8, cudaMemcpyDeviceToHost, st), "d2h");
  cuda_check(cudaStreamSynchronize(st), "sync");
}

std::size_t Engine::pack(const char* digits, std::size_t nd, unsigned be, u64* limbs, std::size_t cap) {
  if (be < 1 || be > 17) throw std::invalid_argument("pack: unsupported base");
  if (nd == 0) throw std::invalid_argument("decimal: empty string");
  const std::size_t nl = (nd + be - 1) / be;
  if (nl > cap) throw std::length_error("pack: output buffer too small");
  din_x_.ensure(nd);
  Px_.ensure(nl);
  cuda_check(cudaMemcpyAsync(din_x_.ptr, digits, nd, cudaMemcpyHostToDevice, stream_), "h2d");
  launch_pack(din_x_.ptr, nd, be, Px_.ptr, nl, err_.ptr, stream_);
  cuda_check(cudaMemcpyAsync(limbs, Px_.ptr, nl * 8, cudaMemcpyDeviceToHost, stream_), "d2h");
  check_err(stream_);
  return nl;
}

std::size_t Engine::recover_decimal(const u64* r1, const u64* r2, std::size_t n, u64 p1, u64 p2, unsigned be,
                                    std::size_t min_limbs, std::size_t dsum, char* out, std::size_t cap) {
  if (be < 1 || be > 17) throw std::invalid_argument("recover_digits: base out of range");
  if (min_limbs < 1) throw std::invalid_argument("recover_digits: min_limbs must be >= 1");
  const CrtConsts cc = crt_consts(p1, p2);
  X_[0].ensure(n);
  X_[1].ensure(n);
  const std::size_t K = n + 2, nchunks = (K + kCarryChunk - 1) / kCarryChunk;
  S_.ensure(nchunks * kCarryChunk);
  maps_.ensure(carry_map_words(K));
  dout_.ensure(std::max<std::size_t>(dsum, 1) + 64);
  cudaStream_t st = stream_;
  cuda_check(cudaMemcpyAsync(X_[0].ptr, r1, n * 8, cudaMemcpyHostToDevice, st), "h2d");
  cuda_check(cudaMemcpyAsync(X_[1].ptr, r2, n * 8, cudaMemcpyHostToDevice, st), "h2d");
  CarryArgs c{};
  c.z1 = X_[0].ptr;
  c.z2 = X_[1].ptr;
  c.n = n;
  c.p1 = p1;
  c.p2 = p2;
  c.p2_prime = cc.p2_prime;
  c.r_tilde = cc.r_tilde;
  c.div = div_for(pow10u(be));
  coeff_cap(be, min_limbs, c.coeff_cap_lo, c.coeff_cap_hi);
  c.base_exp = be;
  c.s = S_.ptr;
  c.maps = maps_.ptr;
  c.err = err_.ptr;
  c.top_candidates[0] = dsum >= 2 ? (dsum - 2) / be : 0;
  c.top_candidates[1] = (dsum - 1) / be;
  c.meta = meta_.ptr;
  c.out = dout_.ptr;
  c.tail = 1;
  recover(c, be, min_limbs, false, st);
  cuda_check(cudaGetLastError(), "carry");
  unsigned long long len = 0;
  cuda_check(cudaMemcpyAsync(&len, meta_.ptr + 2, sizeof len, cudaMemcpyDeviceToHost, st), "len");
  check_err(st);
  if (len > cap) throw std::length_error("recover: output buffer too small");
  cuda_check(cudaMemcpy(out, dout_.ptr, len, cudaMemcpyDeviceToHost), "d2h");
  return std::size_t(len);
}

void Engine::transpose(int kind, u64* a, std::size_t n, std::size_t stride) {
  std::size_t total;
  if (kind == 0)
    total = n ? (n - 1) * stride + n : 0;
  else
    total = 2 * n * n;
  if (total == 0) return;
  X_[0].ensure(total);
  if (kind != 0) X_[1].ensure(std::max<std::size_t>(rho_scratch_words(n), 1));
  cudaStream_t st = stream_;
  cuda_check(cudaMemcpyAsync(X_[0].ptr, a, total * 8, cudaMemcpyHostToDevice, st), "h2d");
  if (kind == 0) {
    launch_transpose_square_sub(X_[0].ptr, n, stride, st);
  } else if (kind == 1) {  // n x 2n -> 2n x n: rho per row, then both square halves (transpose.cpp:43-47)
    launch_rho(X_[0].ptr, X_[1].ptr, n, false, st);
    launch_transpose_square_sub(X_[0].ptr, n, 2 * n, st);
    launch_transpose_square_sub(X_[0].ptr + n, n, 2 * n, st);
  } else {  // 2n x n -> n x 2n (transpose.cpp:49-53)
    launch_transpose_square_sub(X_[0].ptr, n, 2 * n, st);
    launch_transpose_square_sub(X_[0].ptr + n, n, 2 * n, st);
    launch_rho(X_[0].ptr, X_[1].ptr, n, true, st);
  }
  cuda_check(cudaGetLastError(), "transpose");
  cuda_check(cudaMemcpyAsync(a, X_[0].ptr, total * 8, cudaMemcpyDeviceToHost, st), "d2h");
  cuda_check(cudaStreamSynchronize(st), "sync");
}

// ---------------- per-launch profiling ----------------

namespace {
thread_local Engine* g_prof_engine = nullptr;
}

ProfScope::ProfScope(Engine* e) : prev(g_prof_engine) { g_prof_engine = e; }
ProfScope::~ProfScope() { g_prof_engine = prev; }

void prof_mark(const char* name, cudaStream_t st, double modmuls, double bytes) {
  if (g_prof_engine) g_prof_engine->prof_record(name, st, modmuls, bytes);
}

void Engine::prof_record(const char* name, cudaStream_t st, double modmuls, double bytes) {
  if (!prof_on_) return;
  cudaEvent_t e;
  cuda_check(cudaEventCreate(&e), "cudaEventCreate");
  cuda_check(cudaEventRecord(e, st), "cudaEventRecord");
  prof_.push_back({name ? std::string(name) : std::string(), modmuls, bytes, e});
}

void Engine::profile_enable(bool on) {
  cuda_check(cudaDeviceSynchronize(), "sync");
  for (auto& r : prof_) cudaEventDestroy(r.ev);
  prof_.clear();
  prof_on_ = on;
}

std::string Engine::profile_report(bool clear) {
  cuda_check(cudaDeviceSynchronize(), "sync");
  std::string out;
  char line[256];
  for (std::size_t i = 0; i < prof_.size(); ++i) {
    if (prof_[i].name.empty() || i == 0) continue;  // product-start marks
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, prof_[i - 1].ev, prof_[i].ev), "cudaEventElapsedTime");
    std::snprintf(line, sizeof line, "%s\t%.6f\t%.6g\t%.6g\n", prof_[i].name.c_str(), double(ms), prof_[i].modmuls,
                  prof_[i].bytes);
    out += line;
  }
  if (clear) {
    for (auto& r : prof_) cudaEventDestroy(r.ev);
    prof_.clear();
  }
  return out;
}

}  // namespace dmg

// ---------------- sharded large products ----------------

namespace dmg {

CarryArgs Engine::carry_args(const ProductPlan& pp, const u64* z1, const u64* z2, std::size_t n, char* out) const {
  const unsigned be = pp.base_exp;
  const std::size_t lx = (pp.dx + be - 1) / be, ly = (pp.dy + be - 1) / be;
  const CrtConsts cc = crt_consts(pp.p1, pp.p2);
  CarryArgs c{};
  c.z1 = z1;
  c.z2 = z2;
  c.n = n;
  c.p1 = pp.p1;
  c.p2 = pp.p2;
  c.p2_prime = cc.p2_prime;
  c.r_tilde = cc.r_tilde;
  c.div = div_for(pow10u(be));
  coeff_cap(be, std::min(lx, ly), c.coeff_cap_lo, c.coeff_cap_hi);
  c.base_exp = be;
  c.err = err_.ptr;
  const unsigned long long dsum = pp.dx + pp.dy;
  c.top_candidates[0] = dsum >= 2 ? (dsum - 2) / be : 0;
  c.top_candidates[1] = (dsum - 1) / be;
  c.meta = meta_.ptr;
  c.out = out;
  c.tail = 1;
  return c;
}

// Host-only planning (no device): usable without a GPU context.
ShardPlan make_shard_plan(std::size_t dx, std::size_t dy, int G) {
  ShardPlan sp;
  const PairChoice pc = choose_pair(dx, dy, 0, /*allow_large=*/true);
  sp.pp.dx = dx;
  sp.pp.dy = dy;
  sp.pp.base_exp = pc.bp.base_exp;
  sp.pp.N = pc.bp.length;
  sp.pp.p1 = pc.p1;
  sp.pp.p2 = pc.p2;
  sp.pp.large_pair = pc.large_pair;
  const ShardShape sh = shard_shape(sp.pp.N, pass_radices(sp.pp.N, kMaxPassLog), G, std::size_t(kTileW));
  ShardGeom& g = sp.geom;
  g.G = G;
  g.K = sh.K;
  g.Rtot = sh.Rtot;
  g.Sc = sh.Sc;
  g.Bc = sh.Bc;
  g.local_len = sp.pp.N / std::size_t(G);
  const unsigned be = sp.pp.base_exp;
  sp.lx = (dx + be - 1) / be;
  sp.ly = (dy + be - 1) / be;
  sp.min_limbs = std::min(sp.lx, sp.ly);
  const unsigned long long dsum = dx + dy;
  sp.top_candidates[0] = dsum >= 2 ? (dsum - 2) / be : 0;
  sp.top_candidates[1] = (dsum - 1) / be;
  return sp;
}

ShardPlan Engine::shard_plan(std::size_t dx, std::size_t dy, int G) {
  ShardPlan sp = make_shard_plan(dx, dy, G);
  prime_plan(sp.pp.p1, sp.pp.N);  // device tables
  prime_plan(sp.pp.p2, sp.pp.N);
  return sp;
}

void Engine::shard_pack(const ShardPlan& sp, int q, const char* d_digits, std::size_t nd, u64* d_out, cudaStream_t st) {
  if (!st) st = stream_;
  const ShardGeom& g = sp.geom;
  launch_pack(d_digits, nd, sp.pp.base_exp, d_out, g.local_len, err_.ptr, st, __builtin_ctzll(g.Bc), g.Sc,
              std::size_t(q) * g.Bc);
  ++launches_;  // shard steps accumulate launches_ (callers read differences via get_stats)
  cuda_check(cudaGetLastError(), "shard pack");
}

void Engine::shard_transform(const ShardPlan& sp, int q, int stage, const u64* const src[2], u64* const dst[2],
                             const u64* const other[2], cudaStream_t st) {
  if (!st) st = stream_;
  const PrimePlan* pl[2] = {&prime_plan(sp.pp.p1, sp.pp.N), &prime_plan(sp.pp.p2, sp.pp.N)};
  ShardGeom g = sp.geom;
  g.q = q;
  const std::size_t m = pl[0]->passes.size(), K = std::size_t(g.K);
  const u64* in_place[2] = {dst[0], dst[1]};
  switch (stage) {
    case kShardColFwd:
      passes_fwd(pl, 2, src, dst, 0, K, &g, st);
      break;
    case kShardRowFwd:
      passes_fwd(pl, 2, in_place, dst, K, m, &g, st);
      break;
    case kShardRowFwdConv:
      passes_fwd(pl, 2, in_place, dst, K, m - 1, &g, st);
      pass_fused(pl, 2, dst, other, &g, st);
      passes_inv(pl, 2, dst, K, m - 1, &g, st);
      break;
    case kShardColInv:
      passes_inv(pl, 2, dst, 0, K, &g, st);
      break;
    default:
      throw std::invalid_argument("shard: unknown stage");
  }
  cuda_check(cudaGetLastError(), "shard transform");
}

void Engine::shard_reorder(const ShardPlan& sp, bool to_segments, const u64* src, u64* dst, cudaStream_t st) {
  if (!st) st = stream_;
  const ShardGeom& g = sp.geom;
  launch_block_reorder(src, dst, std::size_t(g.G), g.Rtot / std::size_t(g.G), g.Bc, to_segments, st);
  ++launches_;
  cuda_check(cudaGetLastError(), "shard reorder");
}

unsigned Engine::shard_carry_begin(const ShardPlan& sp, int q, const u64* z1, const u64* z2, const u64 h1[2],
                                   const u64 h2[2], u64* s_buf, unsigned* maps_buf, cudaStream_t st) {
  if (!st) st = stream_;
  CarryArgs c = carry_args(sp.pp, z1, z2, sp.geom.local_len, nullptr);
  c.k_off = std::size_t(q) * sp.geom.local_len;
  c.halo1[0] = h1[0];
  c.halo1[1] = h1[1];
  c.halo2[0] = h2[0];
  c.halo2[1] = h2[1];
  c.tail = q == sp.geom.G - 1;
  c.s = s_buf;
  c.maps = maps_buf;
  lens_.ensure(1);
  unsigned* rmap = reinterpret_cast<unsigned*>(lens_.ptr);
  launch_carry_shard_begin(c, rmap, st);
  launches_ += 2;
  cuda_check(cudaGetLastError(), "shard carry");
  unsigned m = 0;
  cuda_check(cudaMemcpyAsync(&m, rmap, sizeof m, cudaMemcpyDeviceToHost, st), "rank map");
  check_err(st);
  return m;
}

void Engine::shard_carry_probe(const ShardPlan& sp, int q, unsigned rank_cin, const u64* z1, const u64* z2,
                               const u64* s_buf, unsigned* maps_buf, u64 z_out[2], cudaStream_t st) {
  if (!st) st = stream_;
  CarryArgs c = carry_args(sp.pp, z1, z2, sp.geom.local_len, nullptr);
  c.k_off = std::size_t(q) * sp.geom.local_len;
  c.tail = q == sp.geom.G - 1;
  c.s = const_cast<u64*>(s_buf);
  c.maps = maps_buf;
  lens_.ensure(2);
  u64* zd = reinterpret_cast<u64*>(lens_.ptr);
  launch_carry_shard_probe(c, rank_cin, zd, st);
  ++launches_;
  cuda_check(cudaGetLastError(), "shard probe");
  cuda_check(cudaMemcpyAsync(z_out, zd, 2 * sizeof(u64), cudaMemcpyDeviceToHost, st), "probe");
  cuda_check(cudaStreamSynchronize(st), "sync");
}

void Engine::shard_carry_emit(const ShardPlan& sp, int q, unsigned rank_cin, unsigned long long top, unsigned top_len,
                              const u64* z1, const u64* z2, const u64* s_buf, unsigned* maps_buf, char* d_out,
                              cudaStream_t st) {
  if (!st) st = stream_;
  CarryArgs c = carry_args(sp.pp, z1, z2, sp.geom.local_len, d_out);
  c.k_off = std::size_t(q) * sp.geom.local_len;
  c.tail = q == sp.geom.G - 1;
  c.s = const_cast<u64*>(s_buf);
  c.maps = maps_buf;
  const unsigned long long meta[3] = {top, top_len, top_len + top * sp.pp.base_exp};
  cuda_check(cudaMemcpyAsync(meta_.ptr, meta, sizeof meta, cudaMemcpyHostToDevice, st), "meta");
  launch_carry_shard_emit(c, rank_cin, st);
  launches_ += 2;
  cuda_check(cudaGetLastError(), "shard emit");
  check_err(st);
}

void Engine::shard_pack_compact(const ShardPlan& sp, const char* d_compact, std::size_t nd_compact, u64* d_out,
                                cudaStream_t st) {
  // the compacted slice is a digit string whose limb i (from the end) is this rank's local limb i
  launch_pack(d_compact, nd_compact, sp.pp.base_exp, d_out, sp.geom.local_len, err_.ptr, st, 63, 0, 0, false);
  ++launches_;
  cuda_check(cudaGetLastError(), "shard pack");
}

void Engine::shard_carry_begin_async(const ShardPlan& sp, int q, const u64* z1, const u64* z2, const u64 h1[2],
                                     const u64 h2[2], u64* s_buf, unsigned* maps_buf, unsigned* h_rank_map,
                                     cudaStream_t st) {
  CarryArgs c = carry_args(sp.pp, z1, z2, sp.geom.local_len, nullptr);
  c.k_off = std::size_t(q) * sp.geom.local_len;
  c.halo1[0] = h1[0];
  c.halo1[1] = h1[1];
  c.halo2[0] = h2[0];
  c.halo2[1] = h2[1];
  c.tail = q == sp.geom.G - 1;
  c.s = s_buf;
  c.maps = maps_buf;
  shard_.tmp.ensure(4);
  unsigned* rmap = reinterpret_cast<unsigned*>(shard_.tmp.ptr);
  launch_carry_shard_begin(c, rmap, st);
  launches_ += 2;
  cuda_check(cudaGetLastError(), "shard carry");
  cuda_check(cudaMemcpyAsync(h_rank_map, rmap, sizeof(unsigned), cudaMemcpyDeviceToHost, st), "rank map");
}

void Engine::shard_carry_probe_async(const ShardPlan& sp, int q, unsigned rank_cin, const u64* z1, const u64* z2,
                                     const u64* s_buf, unsigned* maps_buf, u64* h_z, cudaStream_t st) {
  CarryArgs c = carry_args(sp.pp, z1, z2, sp.geom.local_len, nullptr);
  c.k_off = std::size_t(q) * sp.geom.local_len;
  c.tail = q == sp.geom.G - 1;
  c.s = const_cast<u64*>(s_buf);
  c.maps = maps_buf;
  shard_.tmp.ensure(4);
  u64* zd = reinterpret_cast<u64*>(shard_.tmp.ptr) + 2;
  launch_carry_shard_probe(c, rank_cin, zd, st);
  ++launches_;
  cuda_check(cudaGetLastError(), "shard probe");
  cuda_check(cudaMemcpyAsync(h_z, zd, 2 * sizeof(u64), cudaMemcpyDeviceToHost, st), "probe");
}

void Engine::shard_carry_emit_async(const ShardPlan& sp, int q, unsigned rank_cin, unsigned long long top,
                                    unsigned top_len, const u64* z1, const u64* z2, const u64* s_buf,
                                    unsigned* maps_buf, char* d_out, cudaStream_t st) {
  CarryArgs c = carry_args(sp.pp, z1, z2, sp.geom.local_len, d_out);
  c.k_off = std::size_t(q) * sp.geom.local_len;
  c.tail = q == sp.geom.G - 1;
  c.s = const_cast<u64*>(s_buf);
  c.maps = maps_buf;
  const unsigned long long meta[3] = {top, top_len, top_len + top * sp.pp.base_exp};
  cuda_check(cudaMemcpyAsync(meta_.ptr, meta, sizeof meta, cudaMemcpyHostToDevice, st), "meta");
  launch_carry_shard_emit(c, rank_cin, st);
  launches_ += 2;
  cuda_check(cudaGetLastError(), "shard emit");
}

DivB div_for(u64 base) { return div_for_impl(base); }
CrtConsts crt_consts(u64 p1, u64 p2) { return crt_consts_impl(p1, p2); }

}  // namespace dmg
