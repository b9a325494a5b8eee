// FP32 pipe microbenchmark: FFMA (3 distinct registers, register+uniform)
// vs paired FFMA2 (fma.rn.f32x2). Reports FLOP/s over the whole GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_rates fma_rates.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t f2u(float2 a) { return *reinterpret_cast<uint64_t*>(&a); }
__device__ __forceinline__ float2 u2f(uint64_t a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(d);
}

constexpr int NC = 16;  // independent chains per thread

// acc_j = fma(a_j, b_j, acc_j): three distinct per-thread registers
__global__ void k_ffma_reg(int iters, float* out) {
  float acc[NC], a[NC], b[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    acc[j] = threadIdx.x + j;
    a[j] = 0.999f + 1e-6f * (threadIdx.x ^ j);
    b[j] = 1e-7f * (j + 1) * threadIdx.x;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int j = 0; j < NC; ++j) acc[j] = fmaf(a[(j + r) % NC], b[(j + 3 * r) % NC], acc[j]);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < NC; ++j) s += acc[j];
  if (s == 1234.5f) out[0] = s;
}
// acc_j = fma(acc_j, x, y): uniform operands (the fp_peak_ffma form)
__global__ void k_ffma_uni(int iters, float x, float y, float* out) {
  float acc[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) acc[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int j = 0; j < NC; ++j) acc[j] = fmaf(acc[j], x, y);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < NC; ++j) s += acc[j];
  if (s == 1234.5f) out[0] = s;
}
// paired: NC/2 float2 chains, 3 distinct register pairs
__global__ void k_ffma2_reg(int iters, float* out) {
  float2 acc[NC / 2], a[NC / 2], b[NC / 2];
#pragma unroll
  for (int j = 0; j < NC / 2; ++j) {
    acc[j] = make_float2(threadIdx.x + j, j);
    a[j] = make_float2(0.999f + 1e-6f * (threadIdx.x ^ j), 0.998f);
    b[j] = make_float2(1e-7f * (j + 1) * threadIdx.x, 1e-8f * j);
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < NC / 2; ++j) acc[j] = ffma2(a[(j + r) % (NC / 2)], b[(j + 3 * r) % (NC / 2)], acc[j]);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < NC / 2; ++j) s += acc[j].x + acc[j].y;
  if (s == 1234.5f) out[0] = s;
}
// mixed: FFMA2 interleaved with an equal number of ALU ops (IADD3/LOP3)
__global__ void k_ffma2_alu(int iters, float* out) {
  float2 acc[NC / 2], a[NC / 2], b[NC / 2];
  uint32_t ia[NC / 2];
#pragma unroll
  for (int j = 0; j < NC / 2; ++j) {
    acc[j] = make_float2(threadIdx.x + j, j);
    a[j] = make_float2(0.999f + 1e-6f * (threadIdx.x ^ j), 0.998f);
    b[j] = make_float2(1e-7f * (j + 1) * threadIdx.x, 1e-8f * j);
    ia[j] = threadIdx.x * (j + 7);
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < NC / 2; ++j) {
        acc[j] = ffma2(a[(j + r) % (NC / 2)], b[(j + 3 * r) % (NC / 2)], acc[j]);
        ia[j] = (ia[j] ^ (ia[(j + 1) % (NC / 2)] + r)) ;
      }
  }
  float s = 0;
  uint32_t t = 0;
#pragma unroll
  for (int j = 0; j < NC / 2; ++j) { s += acc[j].x + acc[j].y; t += ia[j]; }
  if (s == 1234.5f || t == 77) out[0] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int threads : {128, 256, 512}) {
    const int blocks = sms * (2048 / threads);
    const double fl_per_thread = 2.0 * iters * 8 * NC;  // every kernel does iters*8*NC fma lanes
    auto time = [&](const char* name, auto launch) {
      launch();
      cudaEventRecord(e0);
      for (int rep = 0; rep < 5; ++rep) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double tf = fl_per_thread * blocks * threads * 5 / (ms * 1e-3) / 1e12;
      printf("%-12s threads=%3d  %.1f TFLOP/s\n", name, threads, tf);
    };
    time("ffma_reg", [&] { k_ffma_reg<<<blocks, threads>>>(iters, out); });
    time("ffma_uni", [&] { k_ffma_uni<<<blocks, threads>>>(iters, 0.999999f, 1e-7f, out); });
    time("ffma2_reg", [&] { k_ffma2_reg<<<blocks, threads>>>(iters, out); });
    time("ffma2_alu", [&] { k_ffma2_alu<<<blocks, threads>>>(iters, out); });
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
