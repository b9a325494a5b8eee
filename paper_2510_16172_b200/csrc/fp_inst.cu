// Per-order instantiation unit: compiled once per K (-DFP_INST_K=K) so the
// heavy unrolled kernels of different orders build in parallel.
#include "fp_dispatch.h"
#include "fp_kernels.cuh"

#ifndef FP_INST_K
#error "compile with -DFP_INST_K=<order>"
#endif

namespace fp {

namespace {
constexpr int kK = FP_INST_K;
constexpr unsigned kDense = (1u << kK) - 1u;

template <typename R, unsigned MASK>
cudaError_t by_op(const PathArgs<R>& a, int op, cudaStream_t s) {
  switch (op) {
    case OP_SOLVE: return launch_path_impl<R, kK, MASK, OP_SOLVE>(a, s);
    case OP_SOLVE_VJP: return launch_path_impl<R, kK, MASK, OP_SOLVE_VJP>(a, s);
    case OP_VJP: return launch_path_impl<R, kK, MASK, OP_VJP>(a, s);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace


template <>
cudaError_t dispatch_k<float, kK>(const PathArgs<float>& a, int op, unsigned mask, cudaStream_t s) {
  (void)mask;
  return by_op<float, kDense>(a, op, s);
}

template <>
cudaError_t dispatch_k<double, kK>(const PathArgs<double>& a, int op, unsigned mask, cudaStream_t s) {
  (void)mask;
  return by_op<double, kDense>(a, op, s);
}

}  // namespace fp
