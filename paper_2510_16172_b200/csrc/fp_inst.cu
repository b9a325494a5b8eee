// Per-order instantiation unit, compiled once per (K, part) so the heavy
// unrolled kernels build in parallel:
//   -DFP_INST_K=K -DFP_INST_PART=0   dense kernels (fp32 + fp64, every op)
//   -DFP_INST_PART=1 / 2             kind-mask specialised fp32 solve /
//                                    fused solve + VJP, one kernel per mask
//   -DFP_INST_PART=3 / 4             tile kernels (solve, fused), fp32 / fp64:
//                                    every mask of the order, per-warp dispatch
#include "fp_dispatch.h"
#include "fp_kernels.cuh"

#ifndef FP_INST_K
#error "compile with -DFP_INST_K=<order>"
#endif
#ifndef FP_INST_PART
#define FP_INST_PART 0
#endif

namespace fp {

namespace {
constexpr int kK = FP_INST_K;
constexpr unsigned kDense = (1u << kK) - 1u;

template <typename R>
cudaError_t dense_by_op(const PathArgs<R>& a, int op, cudaStream_t s) {
  switch (op) {
    case OP_SOLVE: return launch_path_impl<R, kK, kDense, OP_SOLVE>(a, s);
    case OP_SOLVE_VJP: return launch_path_impl<R, kK, kDense, OP_SOLVE_VJP>(a, s);
    case OP_VJP: return launch_path_impl<R, kK, kDense, OP_VJP>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

// Compile-time chain over every mask 0 .. 2^K - 1.
template <int OP, unsigned M>
cudaError_t by_mask(unsigned mask, const PathArgs<float>& a, cudaStream_t s) {
  if (mask == M) return launch_path_impl<float, kK, M, OP>(a, s);
  if constexpr (M + 1 < (1u << kK)) {
    return by_mask<OP, M + 1>(mask, a, s);
  } else {
    return cudaErrorInvalidValue;
  }
}
}  // namespace

#if FP_INST_PART == 0
template <>
cudaError_t dispatch_dense<float, kK>(const PathArgs<float>& a, int op, cudaStream_t s) {
  return dense_by_op<float>(a, op, s);
}
template <>
cudaError_t dispatch_dense<double, kK>(const PathArgs<double>& a, int op, cudaStream_t s) {
  return dense_by_op<double>(a, op, s);
}
#elif FP_INST_PART == 1
template <>
cudaError_t dispatch_masked_solve<kK>(const PathArgs<float>& a, unsigned mask, cudaStream_t s) {
  return by_mask<OP_SOLVE, 0u>(mask, a, s);
}
#elif FP_INST_PART == 2
template <>
cudaError_t dispatch_masked_solve_vjp<kK>(const PathArgs<float>& a, unsigned mask, cudaStream_t s) {
  return by_mask<OP_SOLVE_VJP, 0u>(mask, a, s);
}
#elif FP_INST_PART == 3
// fp32 tile kernels. Orders <= FP_PAIR_MAX_K would run two paths per thread
// (fp_pair.cuh): bitwise the same results, but measured slower (K=1 0.466 vs
// 0.411 ms, K=2 0.95 vs 0.72 ms: half the warps per SM for the same
// dependency chains; profiles/r02s_ab_pair.txt), so 0 (off) by default.
#ifndef FP_PAIR_MAX_K
#define FP_PAIR_MAX_K 0
#endif
template <>
cudaError_t dispatch_tile<float, kK>(const PathArgs<float>& a, int op, cudaStream_t s) {
  constexpr bool kPair = kK <= FP_PAIR_MAX_K;
  return op == OP_SOLVE_VJP ? launch_path_impl<float, kK, kAnyMask, OP_SOLVE_VJP, kPair>(a, s)
                            : launch_path_impl<float, kK, kAnyMask, OP_SOLVE, kPair>(a, s);
}
#elif FP_INST_PART == 4
template <>
cudaError_t dispatch_tile<double, kK>(const PathArgs<double>& a, int op, cudaStream_t s) {
  return op == OP_SOLVE_VJP ? launch_path_impl<double, kK, kAnyMask, OP_SOLVE_VJP>(a, s)
                            : launch_path_impl<double, kK, kAnyMask, OP_SOLVE>(a, s);
}
#endif

}  // namespace fp
