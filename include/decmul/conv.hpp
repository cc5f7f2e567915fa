// decmul/conv.hpp — drop-in for the reference's convolution parity hooks
// (proj/include/decmul/conv.hpp:59-75), backed by libdecmul_gpu.so.
//
// ConvPlan here is a light handle (prime, length, six-step threshold, and the
// reference plan's shape / root / six-step factors for inspection): the device
// plan (roots chosen exactly as primitive_root_of_unity does, twiddle tables in
// HBM) is cached inside the library context, like the reference's conv_plan_for
// cache (conv.cpp:311-322). forward_transform returns the reference's documented
// storage order (conv.hpp:19-24) for the plan's threshold -- the default 2^15 or
// the one forced through build_conv_plan(ctx, n, six_step_threshold), as in
// test_conv.cpp:183-196 and selftest.cpp:109-118; inverse_transform consumes
// it; convolve_mod_p returns natural-order canonical residues.
#pragma once

#include <memory>
#include <span>
#include <stdexcept>
#include <vector>

#include "decimal.hpp"

namespace decmul {

enum class ConvShape { kDirect, kSixStep, kFourStepThreeRows };  // reference conv.hpp:11

inline constexpr std::size_t kDefaultSixStepThreshold = std::size_t(1) << 15;  // conv.hpp:15

// The reference's MontCtx (montgomery.hpp) reduced to what this boundary needs: the prime.
struct MontCtx {
  Word p = 0;
};
inline MontCtx make_ctx(Word p) { return MontCtx{p}; }

struct ConvPlan {
  Word p = 0;
  std::size_t n = 0;
  std::size_t six_step_threshold = kDefaultSixStepThreshold;
  ConvShape shape = ConvShape::kDirect;
  Word root = 0;               // plain primitive n-th root (primitive_root_of_unity, primes.cpp:99-112)
  std::size_t n1 = 0, n2 = 0;  // kSixStep: n = n1 * n2, n1 = 2^floor(k/2)
};

// build_conv_plan (conv.hpp:59-60, conv.cpp:212-271): same argument checks and messages.
inline ConvPlan build_conv_plan(const MontCtx& ctx, std::size_t n,
                                std::size_t six_step_threshold = kDefaultSixStepThreshold) {
  ConvPlan pl;
  pl.p = ctx.p;
  pl.n = n;
  pl.six_step_threshold = six_step_threshold;
  int shape = 0;
  detail::check(decmul_gpu_conv_plan_info(ctx.p, n, six_step_threshold, &shape, &pl.root, &pl.n1, &pl.n2), nullptr);
  pl.shape = ConvShape(shape);
  return pl;
}

inline std::shared_ptr<const ConvPlan> conv_plan_for(Word prime, std::size_t n, AdjustStrategy = {}) {
  return std::make_shared<const ConvPlan>(build_conv_plan(make_ctx(prime), n));
}

inline void forward_transform(const ConvPlan& plan, std::span<Word> a) {
  if (a.size() != plan.n) throw std::invalid_argument("forward_transform: size mismatch");
  decmul_gpu_ctx* ctx = detail::context();
  detail::check(decmul_gpu_forward_transform_ex(ctx, plan.p, plan.n, plan.six_step_threshold, a.data()), ctx);
}

inline void inverse_transform(const ConvPlan& plan, std::span<Word> a) {
  if (a.size() != plan.n) throw std::invalid_argument("inverse_transform: size mismatch");
  decmul_gpu_ctx* ctx = detail::context();
  detail::check(decmul_gpu_inverse_transform_ex(ctx, plan.p, plan.n, plan.six_step_threshold, a.data()), ctx);
}

inline void pointwise_product(const ConvPlan& plan, std::span<Word> a, std::span<const Word> b) {
  if (a.size() != plan.n || b.size() != plan.n) throw std::invalid_argument("pointwise_product: size mismatch");
  decmul_gpu_ctx* ctx = detail::context();
  detail::check(decmul_gpu_pointwise_product(ctx, plan.p, plan.n, a.data(), b.data()), ctx);
}

inline std::vector<Word> convolve_mod_p(const ConvPlan& plan, std::span<const Word> x, std::span<const Word> y) {
  if (x.size() > plan.n || y.size() > plan.n)
    throw std::invalid_argument("convolve_mod_p: input longer than plan length");
  std::vector<Word> out(plan.n);
  decmul_gpu_ctx* ctx = detail::context();
  detail::check(decmul_gpu_convolve_mod_p(ctx, plan.p, plan.n, x.data(), x.size(), y.data(), y.size(), out.data()),
                ctx);
  return out;
}

}  // namespace decmul
