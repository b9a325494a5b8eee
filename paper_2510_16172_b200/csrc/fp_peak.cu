// FP32 FFMA throughput microbenchmark: the measured SIMT roofline peak.
//
// MEASURED_PEAKS.json carries HBM and tensor-core peaks only; the Fermat
// kernels are FP32-pipe bound, so bench.py measures this peak on the same
// GPU in the same run. Every thread runs 16 independent FFMA chains (enough
// ILP to cover the 4-cycle FMA latency at full occupancy).
#include <cuda_runtime.h>

#include "../../include/fermat_b200.h"
#include "fp_dispatch.h"

namespace fp {

__global__ void __launch_bounds__(256) ffma_peak_kernel(int iters, float seed, float* out) {
  float acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = seed + float(threadIdx.x + j);
  const float x = 0.999999f + seed * 1e-9f, y = 1e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = fmaf(acc[j], x, y);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += acc[j];
  if (s == 1234.5f) out[0] = s;  // keep the chains alive
}

// The same throughput with every operand in a distinct register, paired
// (FFMA2, three register pairs per instruction) — the operand form of every
// FMA in the path kernels. Register-file bandwidth, not the pipe, limits it
// on this part (~47 TFLOP/s vs ~72 for the uniform-operand form above), so
// it is the practically attainable FP32 ceiling for register-resident
// per-path arithmetic; bench.py reports both.
__device__ __forceinline__ float2 ffma2_rr(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

__global__ void __launch_bounds__(256) ffma2_reg_peak_kernel(int iters, float seed, float* out) {
  constexpr int NC = 8;
  float2 acc[NC], a[NC], b[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    acc[j] = make_float2(seed + float(threadIdx.x + j), float(j));
    a[j] = make_float2(0.999f + 1e-6f * float(threadIdx.x ^ j), 0.998f);
    b[j] = make_float2(1e-7f * float((j + 1) * threadIdx.x), 1e-8f * float(j));
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int j = 0; j < NC; ++j) acc[j] = ffma2_rr(a[(j + r) % NC], b[(j + 3 * r) % NC], acc[j]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < NC; ++j) s += acc[j].x + acc[j].y;
  if (s == 1234.5f) out[0] = s;
}

// Benchmark gate: holds the stream until the host sets *flag (pinned host
// memory, read over the mapping), so a timed region can be enqueued in full
// before the device starts it; host-side jitter then never idles the GPU
// inside a timed step. Bounded by timeout_ns (globaltimer) so it cannot hang.
__global__ void gate_kernel(const volatile int* flag, unsigned long long timeout_ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*flag == 0) {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) break;
  }
}

}  // namespace fp

extern "C" int fp_gate_wait(const int* host_flag, double timeout_s, void* stream) {
  if (host_flag == nullptr || !(timeout_s > 0.0) || timeout_s > 60.0) return FP_ERR_INVALID_ARGUMENT;
  fp::gate_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
      host_flag, static_cast<unsigned long long>(timeout_s * 1e9));
  return cudaGetLastError() == cudaSuccess ? FP_OK : FP_ERR_CUDA;
}

// blocks x 256 threads, each iters x 8 x 8 FFMA2 = iters x 128 FMA lanes, as
// fp_peak_ffma (so bench.py times both with the same FLOP count).
extern "C" int fp_peak_ffma_reg(int blocks, int iters, float* out, void* stream) {
  if (blocks < 1 || iters < 1) return FP_ERR_INVALID_ARGUMENT;
  fp::ffma2_reg_peak_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(iters, 0.5f, out);
  fp::count_launches(1);
  return cudaGetLastError() == cudaSuccess ? FP_OK : FP_ERR_CUDA;
}

extern "C" int fp_peak_ffma(int blocks, int iters, float* out, void* stream) {
  if (blocks < 1 || iters < 1) return FP_ERR_INVALID_ARGUMENT;
  fp::ffma_peak_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(iters, 0.5f, out);
  fp::count_launches(1);
  return cudaGetLastError() == cudaSuccess ? FP_OK : FP_ERR_CUDA;
}
