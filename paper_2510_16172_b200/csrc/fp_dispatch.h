// Cross-unit declarations for the per-order kernel dispatch.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace fp {

template <typename R>
struct PathArgs;

// Defined in fp_inst.cu, one explicit specialisation per (R, K).
template <typename R, int K>
cudaError_t dispatch_k(const PathArgs<R>& a, int op, unsigned mask, cudaStream_t s);

void count_launches(uint64_t n);

}  // namespace fp
