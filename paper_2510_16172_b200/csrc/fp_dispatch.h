// Cross-unit declarations for the per-order kernel dispatch.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace fp {

template <typename R>
struct PathArgs;

// Dense (uniform 2K) kernels, every op; defined in fp_inst.cu (part 0).
template <typename R, int K>
cudaError_t dispatch_dense(const PathArgs<R>& a, int op, cudaStream_t s);

// Kind-mask specialised fp32 kernels for K <= 5; fp_inst.cu parts 1 (solve)
// and 2 (fused solve + VJP).
template <int K>
cudaError_t dispatch_masked_solve(const PathArgs<float>& a, unsigned mask, cudaStream_t s);
template <int K>
cudaError_t dispatch_masked_solve_vjp(const PathArgs<float>& a, unsigned mask, cudaStream_t s);

// Tile kernels (per-warp kind-mask dispatch, K <= 5); fp_inst.cu parts 3 (fp32), 4 (fp64).
template <typename R, int K>
cudaError_t dispatch_tile(const PathArgs<R>& a, int op, cudaStream_t s);

// Warp-per-path solver for orders 9..64 (fp_wide.cu), every op, fp32/fp64.
template <typename R>
cudaError_t dispatch_wide(int K, const PathArgs<R>& a, int op, cudaStream_t s);

void count_launches(uint64_t n);

}  // namespace fp
