// decmul/conv.hpp — drop-in for the reference's convolution parity hooks
// (proj/include/decmul/conv.hpp:59-75), backed by libdecmul_gpu.so.
//
// ConvPlan here is a light handle (prime, length): the device plan (roots chosen
// exactly as primitive_root_of_unity does, twiddle tables in HBM) is cached
// inside the library context, like the reference's conv_plan_for cache
// (conv.cpp:311-322). forward_transform returns the reference's documented
// storage order (conv.hpp:19-24) for its default plan; inverse_transform
// consumes it; convolve_mod_p returns natural-order canonical residues.
#pragma once

#include <memory>
#include <span>
#include <stdexcept>
#include <vector>

#include "decimal.hpp"

namespace decmul {

struct ConvPlan {
  Word p = 0;
  std::size_t n = 0;
};

inline std::shared_ptr<const ConvPlan> conv_plan_for(Word prime, std::size_t n, AdjustStrategy = {}) {
  return std::make_shared<const ConvPlan>(ConvPlan{prime, n});
}

inline void forward_transform(const ConvPlan& plan, std::span<Word> a) {
  if (a.size() != plan.n) throw std::invalid_argument("forward_transform: size mismatch");
  decmul_gpu_ctx* ctx = detail::context();
  detail::check(decmul_gpu_forward_transform(ctx, plan.p, plan.n, a.data()), ctx);
}

inline void inverse_transform(const ConvPlan& plan, std::span<Word> a) {
  if (a.size() != plan.n) throw std::invalid_argument("inverse_transform: size mismatch");
  decmul_gpu_ctx* ctx = detail::context();
  detail::check(decmul_gpu_inverse_transform(ctx, plan.p, plan.n, a.data()), ctx);
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
