// Visibility post-processing of traced paths (the step
// after the solve in exhaustive tracing, PAPER.md:32,67 — no reference code:
// SPEC.md:11 puts occlusion out of the reference's scope).
//
// For every traced path (TX -> x_1 .. x_K -> RX, interaction points from the
// solver) two physical validity tests:
//   * BLOCKED (bit 0): some segment crosses a blocker parallelogram
//     O + a U + b V, a, b in [0, 1] (scene walls and roofs) farther than eps
//     metres from both of its ends: e < s < 1 - e with e = eps / |segment|
//     (a segment starts / ends on the surface it interacts with, s = 0 / 1,
//     up to the fp32 rounding of the interaction points, ~1e-5 m at 100 m);
//   * WRONG_SIDE (bit 1): a reflection whose incoming and outgoing segments
//     are not on the same side of the reflector's plane (a stationary point of
//     the length on the far side is a straight crossing, not a reflection).
// Arithmetic is fp64 with every operation explicit and unfused (-fmad=false),
// in the order oracle/visibility_oracle.py evaluates it, so the flags are bit
// for bit the oracle's on the same points.
#include <cuda_runtime.h>

#include "../../include/fermat_b200.h"
#include "fp_dispatch.h"

namespace fp {

namespace {

constexpr int kVisThreads = 256;
constexpr int kMaxBlockers = 2048;

struct VisArgs {
  const double* blk;  // (Q, 3, 3): O, U, V
  int Q;
  const float *tx, *rx;
  const int32_t* rec_rx;
  const float* points;  // (n, K, 3)
  const int32_t* rec_seq;
  const float* obj_basis;   // (N, 3, 2)
  const uint8_t* obj_plane;  // (N,)
  int n_obj;
  int64_t n;
  int K;
  double eps;
  uint8_t* flags;
  int32_t* first_blocker;
};

// Segment P -> P + D against parallelogram (O, U, V): Moller-Trumbore.
__device__ __forceinline__ bool crosses(const double (&P)[3], const double (&D)[3], const double* b,
                                        double e) {
  const double O0 = b[0], O1 = b[1], O2 = b[2];
  const double U0 = b[3], U1 = b[4], U2 = b[5];
  const double V0 = b[6], V1 = b[7], V2 = b[8];
  const double h0 = D[1] * V2 - D[2] * V1;
  const double h1 = D[2] * V0 - D[0] * V2;
  const double h2 = D[0] * V1 - D[1] * V0;
  const double det = U0 * h0 + U1 * h1 + U2 * h2;
  if (det == 0.0) return false;
  const double f = 1.0 / det;
  const double w0 = P[0] - O0, w1 = P[1] - O1, w2 = P[2] - O2;
  const double a = f * (w0 * h0 + w1 * h1 + w2 * h2);
  if (!(a >= 0.0 && a <= 1.0)) return false;
  const double q0 = w1 * U2 - w2 * U1;
  const double q1 = w2 * U0 - w0 * U2;
  const double q2 = w0 * U1 - w1 * U0;
  const double bb = f * (D[0] * q0 + D[1] * q1 + D[2] * q2);
  if (!(bb >= 0.0 && bb <= 1.0)) return false;
  const double s = f * (V0 * q0 + V1 * q1 + V2 * q2);
  return s > e && s < 1.0 - e;
}

template <int K>
__global__ void __launch_bounds__(kVisThreads) visibility_kernel(const VisArgs a) {
  extern __shared__ double sblk[];
  for (int e = threadIdx.x; e < a.Q * 9; e += blockDim.x) sblk[e] = a.blk[e];
  __syncthreads();
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < a.n;
       r += int64_t(gridDim.x) * blockDim.x) {
    double X[K + 2][3];
    const int rxi = a.rec_rx[r];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      X[0][c] = double(a.tx[c]);
      X[K + 1][c] = double(a.rx[3 * rxi + c]);
    }
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int c = 0; c < 3; ++c) X[i + 1][c] = double(a.points[(r * K + i) * 3 + c]);
    uint8_t fl = 0;
    int32_t first = -1;
    // reflections: both neighbours strictly on one side of the plane
    if (a.rec_seq != nullptr) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int o = a.rec_seq[r * K + i];
        if (o < 0 || o >= a.n_obj || !a.obj_plane[o]) continue;
        const float* A = a.obj_basis + size_t(o) * 6;
        const double a0 = A[0], a1 = A[2], a2 = A[4];  // column 0
        const double b0 = A[1], b1 = A[3], b2 = A[5];  // column 1
        const double n0 = a1 * b2 - a2 * b1;
        const double n1 = a2 * b0 - a0 * b2;
        const double n2 = a0 * b1 - a1 * b0;
        const double din = (X[i][0] - X[i + 1][0]) * n0 + (X[i][1] - X[i + 1][1]) * n1 +
                           (X[i][2] - X[i + 1][2]) * n2;
        const double dout = (X[i + 2][0] - X[i + 1][0]) * n0 + (X[i + 2][1] - X[i + 1][1]) * n1 +
                            (X[i + 2][2] - X[i + 1][2]) * n2;
        if (!(din * dout > 0.0)) fl |= FP_VIS_WRONG_SIDE;
      }
    }
#pragma unroll
    for (int k = 0; k <= K; ++k) {
      const double P[3] = {X[k][0], X[k][1], X[k][2]};
      const double D[3] = {X[k + 1][0] - X[k][0], X[k + 1][1] - X[k][1], X[k + 1][2] - X[k][2]};
      const double e = a.eps / sqrt(D[0] * D[0] + D[1] * D[1] + D[2] * D[2]);
      for (int q = 0; q < a.Q; ++q) {
        if (crosses(P, D, sblk + 9 * q, e)) {
          fl |= FP_VIS_BLOCKED;
          first = q;
          break;
        }
      }
      if (fl & FP_VIS_BLOCKED) break;
    }
    a.flags[r] = fl;
    if (a.first_blocker) a.first_blocker[r] = first;
  }
}

}  // namespace

}  // namespace fp

extern "C" int fp_visibility_f64(const double* blockers, int n_blockers, const float* tx,
                                 const float* rx, const int32_t* rec_rx, const float* points,
                                 const int32_t* rec_seq, const float* obj_basis,
                                 const uint8_t* obj_plane, int n_objects, int64_t n, int order,
                                 double eps, uint8_t* flags, int32_t* first_blocker, void* stream) {
  if (order < 1 || order > 3) return FP_ERR_UNSUPPORTED_ORDER;
  if (n < 0 || n_blockers < 0 || n_blockers > fp::kMaxBlockers || !(eps >= 0.0))
    return FP_ERR_INVALID_ARGUMENT;
  if (n == 0) return FP_OK;
  if (!tx || !rx || !rec_rx || !points || !flags || (n_blockers > 0 && !blockers))
    return FP_ERR_INVALID_ARGUMENT;
  if (rec_seq && (!obj_basis || !obj_plane || n_objects < 1)) return FP_ERR_INVALID_ARGUMENT;
  fp::VisArgs a{blockers, n_blockers, tx, rx, rec_rx, points, rec_seq, obj_basis, obj_plane,
                n_objects, n, order, eps, flags, first_blocker};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (n + fp::kVisThreads - 1) / fp::kVisThreads;
  if (blocks > int64_t(sms) * 16) blocks = int64_t(sms) * 16;
  const size_t smem = size_t(n_blockers) * 9 * sizeof(double);
  cudaError_t e = cudaSuccess;
  switch (order) {
    case 1:
      e = cudaFuncSetAttribute(fp::visibility_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e == cudaSuccess) fp::visibility_kernel<1><<<unsigned(blocks), fp::kVisThreads, smem, s>>>(a);
      break;
    case 2:
      e = cudaFuncSetAttribute(fp::visibility_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e == cudaSuccess) fp::visibility_kernel<2><<<unsigned(blocks), fp::kVisThreads, smem, s>>>(a);
      break;
    default:
      e = cudaFuncSetAttribute(fp::visibility_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e == cudaSuccess) fp::visibility_kernel<3><<<unsigned(blocks), fp::kVisThreads, smem, s>>>(a);
      break;
  }
  fp::count_launches(1);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? FP_OK : FP_ERR_CUDA;
}
