// decmul/transpose.hpp — drop-in for the reference's in-place transposes
// (proj/include/decmul/transpose.hpp:11-24), executed by the device kernels
// (tile-pair swaps staged through shared memory). The scratch argument of the
// reference's rectangular forms is accepted and unused (the device stages rows
// through its own workspace).
#pragma once

#include "decimal.hpp"

namespace decmul {

inline void transpose_square_sub(Word* p, std::size_t n, std::size_t stride) {
  decmul_gpu_ctx* ctx = detail::context();
  detail::check(decmul_gpu_transpose_square_sub(ctx, p, n, stride), ctx);
}

inline void transpose_n_x_2n(Word* p, std::size_t n, Word* /*scratch*/) {
  decmul_gpu_ctx* ctx = detail::context();
  detail::check(decmul_gpu_transpose_n_x_2n(ctx, p, n), ctx);
}

inline void transpose_2n_x_n(Word* p, std::size_t n, Word* /*scratch*/) {
  decmul_gpu_ctx* ctx = detail::context();
  detail::check(decmul_gpu_transpose_2n_x_n(ctx, p, n), ctx);
}

}  // namespace decmul
