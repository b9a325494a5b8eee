// Comparison solvers on the GPU: the reference's
// masked damped Newton (the config-1 comparator, baselines.py:152-193) and the
// exact image method for all-plane paths (baselines.py:48-71).
#include <cuda_runtime.h>

#include "fp_dispatch.h"
#include "fp_kernels.cuh"

namespace fp {

// Unclamped total length at parameters t (batching.py:123-126).
template <typename R, int K>
__device__ __forceinline__ R length_at(const Geo<R, K>& G, const R (&t)[K][2]) {
  R prev[3] = {G.x0(0), G.x0(1), G.x0(2)};
  R L = R(0);
#pragma unroll
  for (int i = 0; i <= K; ++i) {
    R x[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      if (i < K)
        x[r] = fma(G.A(i, r, 1), t[i][1], G.A(i, r, 0) * t[i][0]) + G.b(i, r);
      else
        x[r] = G.xe(r);
    }
    const R d0 = x[0] - prev[0], d1 = x[1] - prev[1], d2 = x[2] - prev[2];
    L += Num<R>::sqrt_(fma(d2, d2, fma(d1, d1, d0 * d0)));
#pragma unroll
    for (int r = 0; r < 3; ++r) prev[r] = x[r];
  }
  return L;
}

// Reference-exact gradient with clamped norms (batching.py:95-104): IEEE
// sqrt and division (no fast reciprocal), so the comparator's residual
// gradients carry the reference's rounding, not the hot path's.
template <typename R, int K>
__device__ __forceinline__ void grad_exact(const Geo<R, K>& G, const R (&t)[2 * K], R (&s)[K + 1][3],
                                           R (&nc)[K + 1], R (&g)[2 * K]) {
  R P[K + 2][3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    P[0][r] = G.x0(r);
    P[K + 1][r] = G.xe(r);
  }
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int r = 0; r < 3; ++r) P[i + 1][r] = fma(G.A(i, r, 1), t[2 * i + 1], G.A(i, r, 0) * t[2 * i]) + G.b(i, r);
  R u[K + 1][3];
#pragma unroll
  for (int k = 0; k <= K; ++k) {
#pragma unroll
    for (int r = 0; r < 3; ++r) s[k][r] = P[k + 1][r] - P[k][r];
    nc[k] = clamp_floor(Num<R>::sqrt_(fma(s[k][2], s[k][2], fma(s[k][1], s[k][1], s[k][0] * s[k][0]))), G.eps);
#pragma unroll
    for (int r = 0; r < 3; ++r) u[k][r] = Num<R>::div(s[k][r], nc[k]);
  }
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const R q0 = u[i][0] - u[i + 1][0], q1 = u[i][1] - u[i + 1][1], q2 = u[i][2] - u[i + 1][2];
      g[2 * i + c] = fma(G.A(i, 2, c), q2, fma(G.A(i, 1, c), q1, G.A(i, 0, c) * q0));
    }
}

// Damped Newton on active coordinates with step halving (baselines.py:152-193):
// H from clamped segments (hessian_batch, baselines.py:131-149), inert rows
// and columns pinned to the identity, damping 1e-10 tr(H_a) / dim(active),
// block-tridiagonal solve, up to 20 halvings while the length increases.
template <typename R, int K>
__global__ void __launch_bounds__(kThreads) newton_kernel(const R* basis, const R* anchor,
                                                          const R* start, const R* end, const R* T0,
                                                          int64_t B, int iterations, R* T_out,
                                                          R* g_out, R* trace_gnorm) {
  constexpr unsigned MASK = (1u << K) - 1u;  // dense layout: t[i][c] = P.t[2i + c]
  (void)MASK;
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= B) return;
  Geo<R, K> G;
  load_geo<R, K, MASK>(G, basis + b * 6 * K, anchor + b * 3 * K, start + 3 * b, end + 3 * b);
  struct {
    R t[2 * K], g[2 * K], s[K + 1][3], nc[K + 1];
  } P;
#pragma unroll
  for (int j = 0; j < 2 * K; ++j) P.t[j] = T0[b * 2 * K + j];
  bool act[K][2];
  int dim = 0;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      act[i][c] = G.A(i, 0, c) != R(0) || G.A(i, 1, c) != R(0) || G.A(i, 2, c) != R(0);
      dim += act[i][c];
    }
  grad_exact<R, K>(G, P.t, P.s, P.nc, P.g);
  for (int it = 0; it < iterations; ++it) {
    // Hessian blocks at the current T as hessian_batch computes them
    // (baselines.py:131-149): M_k = (I - u_k u_k^T) / n_k with clamped norms,
    // diagonal A_i^T (M_i + M_{i+1}) A_i, off-diagonal -A_i^T M_{i+1} A_{i+1}.
    R M[K + 1][6];  // symmetric 3x3: xx, xy, xz, yy, yz, zz
#pragma unroll
    for (int k = 0; k <= K; ++k) {
      R u[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) u[r] = Num<R>::div(P.s[k][r], P.nc[k]);
      const int ri[6] = {0, 0, 0, 1, 1, 2}, ci[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
      for (int e = 0; e < 6; ++e)
        M[k][e] = Num<R>::div((ri[e] == ci[e] ? R(1) : R(0)) - u[ri[e]] * u[ci[e]], P.nc[k]);
    }
    auto mget = [&](const R* m, int r, int c) -> R {
      const int lo = r < c ? r : c, hi = r < c ? c : r;
      return m[lo == 0 ? hi : (lo == 1 ? 2 + hi : 5)];
    };
    R D[K][3], O[K][2][2];
    R tr = R(0);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      R Ms[6];
#pragma unroll
      for (int e = 0; e < 6; ++e) Ms[e] = M[i][e] + M[i + 1][e];
      R Dm[2][2];
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) {
          R acc = R(0);
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) acc = fma(G.A(i, r, x) * mget(Ms, r, c), G.A(i, c, y), acc);
          Dm[x][y] = acc;
        }
      D[i][0] = Dm[0][0];
      D[i][1] = Dm[0][1];
      D[i][2] = Dm[1][1];
      if (i + 1 < K) {
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y) {
            R acc = R(0);
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
              for (int c = 0; c < 3; ++c)
                acc = fma(G.A(i, r, x) * mget(M[i + 1], r, c), G.A(i + 1, c, y), acc);
            O[i][x][y] = (act[i][x] && act[i + 1][y]) ? -acc : R(0);
          }
      }
      if (act[i][0]) tr += D[i][0];
      if (act[i][1]) tr += D[i][2];
    }
    const R lam = R(1e-10) * tr / R(dim > 0 ? dim : 1);
    R rhs[K][2];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (!(act[i][0] && act[i][1])) D[i][1] = R(0);
      D[i][0] = act[i][0] ? D[i][0] + lam : R(1);
      D[i][2] = act[i][1] ? D[i][2] + lam : R(1);
      rhs[i][0] = act[i][0] ? -P.g[2 * i] : R(0);
      rhs[i][1] = act[i][1] ? -P.g[2 * i + 1] : R(0);
    }
    // block Thomas elimination
    R Ci[K][3], z[K][2];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      R C0 = D[i][0], C1 = D[i][1], C2 = D[i][2], z0 = rhs[i][0], z1 = rhs[i][1];
      if (i > 0) {
        R Lm[2][2];
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          Lm[x][0] = O[i - 1][0][x] * Ci[i - 1][0] + O[i - 1][1][x] * Ci[i - 1][1];
          Lm[x][1] = O[i - 1][0][x] * Ci[i - 1][1] + O[i - 1][1][x] * Ci[i - 1][2];
        }
        C0 -= Lm[0][0] * O[i - 1][0][0] + Lm[0][1] * O[i - 1][1][0];
        C1 -= Lm[0][0] * O[i - 1][0][1] + Lm[0][1] * O[i - 1][1][1];
        C2 -= Lm[1][0] * O[i - 1][0][1] + Lm[1][1] * O[i - 1][1][1];
        z0 -= Lm[0][0] * z[i - 1][0] + Lm[0][1] * z[i - 1][1];
        z1 -= Lm[1][0] * z[i - 1][0] + Lm[1][1] * z[i - 1][1];
      }
      const R id = Num<R>::rcp(C0 * C2 - C1 * C1);
      Ci[i][0] = C2 * id;
      Ci[i][1] = -C1 * id;
      Ci[i][2] = C0 * id;
      z[i][0] = z0;
      z[i][1] = z1;
    }
    R step[K][2];
    R n0 = R(0), n1 = R(0);
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
      R r0 = z[i][0], r1 = z[i][1];
      if (i + 1 < K) {
        r0 -= O[i][0][0] * n0 + O[i][0][1] * n1;
        r1 -= O[i][1][0] * n0 + O[i][1][1] * n1;
      }
      step[i][0] = act[i][0] ? Ci[i][0] * r0 + Ci[i][1] * r1 : R(0);
      step[i][1] = act[i][1] ? Ci[i][1] * r0 + Ci[i][2] * r1 : R(0);
      n0 = step[i][0];
      n1 = step[i][1];
    }
    // step halving while the length increases (baselines.py:180-191)
    R t0[K][2], cand[K][2];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      t0[i][0] = P.t[2 * i];
      t0[i][1] = P.t[2 * i + 1];
      cand[i][0] = t0[i][0] + step[i][0];
      cand[i][1] = t0[i][1] + step[i][1];
    }
    const R L0 = length_at<R, K>(G, t0);
    R Lc = length_at<R, K>(G, cand);
    R scale = R(1);
    for (int h = 0; h < 20 && Lc > L0; ++h) {
      scale *= R(0.5);
#pragma unroll
      for (int i = 0; i < K; ++i) {
        cand[i][0] = t0[i][0] + scale * step[i][0];
        cand[i][1] = t0[i][1] + scale * step[i][1];
      }
      Lc = length_at<R, K>(G, cand);
    }
    if (Lc <= L0) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        P.t[2 * i] = cand[i][0];
        P.t[2 * i + 1] = cand[i][1];
      }
    }
    grad_exact<R, K>(G, P.t, P.s, P.nc, P.g);
    if (trace_gnorm) {
      R q = R(0);
#pragma unroll
      for (int j = 0; j < 2 * K; ++j) q = fma(P.g[j], P.g[j], q);
      trace_gnorm[int64_t(it) * B + b] = Num<R>::sqrt_(q);
    }
  }
#pragma unroll
  for (int j = 0; j < 2 * K; ++j) {
    T_out[b * 2 * K + j] = P.t[j];
    if (g_out) g_out[b * 2 * K + j] = P.g[j];
  }
}

// Fixed-step gradient descent (baselines._gd_kernel, baselines.py:87-101):
// eta = 0.1 |end - start| / (1 + |g0|), T -= eta g for `iterations` steps.
template <typename R, int K>
__global__ void __launch_bounds__(kThreads) gd_kernel(const R* basis, const R* anchor, const R* start,
                                                      const R* end, const R* T0, int64_t B,
                                                      int iterations, R* T_out, R* g_out) {
  constexpr unsigned MASK = (1u << K) - 1u;
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= B) return;
  Geo<R, K> G;
  load_geo<R, K, MASK>(G, basis + b * 6 * K, anchor + b * 3 * K, start + 3 * b, end + 3 * b);
  R t[2 * K], g[2 * K], s[K + 1][3], nc[K + 1];
#pragma unroll
  for (int j = 0; j < 2 * K; ++j) t[j] = T0[b * 2 * K + j];
  grad_exact<R, K>(G, t, s, nc, g);
  R g2 = R(0), d2 = R(0);
#pragma unroll
  for (int j = 0; j < 2 * K; ++j) g2 = fma(g[j], g[j], g2);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const R d = G.xe(r) - G.x0(r);
    d2 = fma(d, d, d2);
  }
  const R eta = Num<R>::div(R(0.1) * Num<R>::sqrt_(d2), R(1) + Num<R>::sqrt_(g2));
  for (int it = 0; it < iterations; ++it) {
#pragma unroll
    for (int j = 0; j < 2 * K; ++j) t[j] = t[j] - eta * g[j];
    grad_exact<R, K>(G, t, s, nc, g);
  }
#pragma unroll
  for (int j = 0; j < 2 * K; ++j) {
    T_out[b * 2 * K + j] = t[j];
    if (g_out) g_out[b * 2 * K + j] = g[j];
  }
}

// Image method (baselines.py:48-71): mirror the start across each plane, then
// intersect the line from the last image to the end with each plane in reverse.
// status bit FP_STATUS_SINGULAR marks a sight line parallel to its plane
// (NoIntersection, |denom| <= 1e-12 |dir|).
template <typename R>
__global__ void image_kernel(const R* basis, const R* anchor, const R* start, const R* end, int64_t B,
                             int K, R* points, uint8_t* status) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= B) return;
  constexpr int kMax = 64;
  R img[kMax][3], nrm[kMax][3];
  R m[3] = {start[3 * b], start[3 * b + 1], start[3 * b + 2]};
  uint8_t st = 0;
  for (int i = 0; i < K; ++i) {
    const R* A = basis + (b * K + i) * 6;
    R n[3] = {A[2] * A[5] - A[4] * A[3], A[4] * A[1] - A[0] * A[5], A[0] * A[3] - A[2] * A[1]};
    const R inv = Num<R>::rcp(Num<R>::sqrt_(fma(n[2], n[2], fma(n[1], n[1], n[0] * n[0]))));
    const R* a = anchor + (b * K + i) * 3;
    R d = R(0);
    for (int r = 0; r < 3; ++r) {
      nrm[i][r] = n[r] * inv;
      d = fma(m[r] - a[r], nrm[i][r], d);
    }
    for (int r = 0; r < 3; ++r) {
      m[r] = m[r] - R(2) * d * nrm[i][r];
      img[i][r] = m[r];
    }
  }
  R y[3] = {end[3 * b], end[3 * b + 1], end[3 * b + 2]};
  for (int i = K - 1; i >= 0; --i) {
    const R* a = anchor + (b * K + i) * 3;
    R dir[3], den = R(0), num = R(0), dn = R(0);
    for (int r = 0; r < 3; ++r) {
      dir[r] = y[r] - img[i][r];
      den = fma(dir[r], nrm[i][r], den);
      num = fma(a[r] - img[i][r], nrm[i][r], num);
      dn = fma(dir[r], dir[r], dn);
    }
    if (fabs(den) <= R(1e-12) * Num<R>::sqrt_(dn)) st |= FP_STATUS_SINGULAR;
    const R t = Num<R>::div(num, den);
    for (int r = 0; r < 3; ++r) {
      y[r] = fma(t, dir[r], img[i][r]);
      points[(b * K + i) * 3 + r] = y[r];
    }
  }
  if (status) status[b] = st;
}

template <typename R, int K>
static cudaError_t launch_newton(const R* basis, const R* anchor, const R* start, const R* end,
                                 const R* T0, int64_t B, int it, R* T_out, R* g_out, R* trace,
                                 cudaStream_t s) {
  newton_kernel<R, K><<<unsigned((B + kThreads - 1) / kThreads), kThreads, 0, s>>>(
      basis, anchor, start, end, T0, B, it, T_out, g_out, trace);
  count_launches(1);
  return cudaGetLastError();
}

template <typename R>
static int gd_impl(const R* basis, const R* anchor, const R* start, const R* end, const R* T0,
                   int64_t B, int K, int iterations, R* T_out, R* g_out, void* stream) {
  if (B < 0 || iterations < 1 || (B > 0 && (!basis || !anchor || !start || !end || !T0 || !T_out)))
    return FP_ERR_INVALID_ARGUMENT;
  if (B == 0) return FP_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned blocks = unsigned((B + kThreads - 1) / kThreads);
  switch (K) {
    case 1: gd_kernel<R, 1><<<blocks, kThreads, 0, s>>>(basis, anchor, start, end, T0, B, iterations, T_out, g_out); break;
    case 2: gd_kernel<R, 2><<<blocks, kThreads, 0, s>>>(basis, anchor, start, end, T0, B, iterations, T_out, g_out); break;
    case 3: gd_kernel<R, 3><<<blocks, kThreads, 0, s>>>(basis, anchor, start, end, T0, B, iterations, T_out, g_out); break;
    case 4: gd_kernel<R, 4><<<blocks, kThreads, 0, s>>>(basis, anchor, start, end, T0, B, iterations, T_out, g_out); break;
    case 5: gd_kernel<R, 5><<<blocks, kThreads, 0, s>>>(basis, anchor, start, end, T0, B, iterations, T_out, g_out); break;
    default: return FP_ERR_UNSUPPORTED_ORDER;
  }
  count_launches(1);
  return cudaGetLastError() == cudaSuccess ? FP_OK : FP_ERR_CUDA;
}

template <typename R>
static int newton_impl(const R* basis, const R* anchor, const R* start, const R* end, const R* T0,
                       int64_t B, int K, int iterations, R* T_out, R* g_out, R* trace, void* stream) {
  if (B < 0 || iterations < 1 || (B > 0 && (!basis || !anchor || !start || !end || !T0 || !T_out)))
    return FP_ERR_INVALID_ARGUMENT;
  if (B == 0) return FP_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (K) {
    case 1: e = launch_newton<R, 1>(basis, anchor, start, end, T0, B, iterations, T_out, g_out, trace, s); break;
    case 2: e = launch_newton<R, 2>(basis, anchor, start, end, T0, B, iterations, T_out, g_out, trace, s); break;
    case 3: e = launch_newton<R, 3>(basis, anchor, start, end, T0, B, iterations, T_out, g_out, trace, s); break;
    case 4: e = launch_newton<R, 4>(basis, anchor, start, end, T0, B, iterations, T_out, g_out, trace, s); break;
    case 5: e = launch_newton<R, 5>(basis, anchor, start, end, T0, B, iterations, T_out, g_out, trace, s); break;
    default: return FP_ERR_UNSUPPORTED_ORDER;
  }
  return e == cudaSuccess ? FP_OK : FP_ERR_CUDA;
}

}  // namespace fp

using namespace fp;

extern "C" {

int fp_newton_f32(const float* basis, const float* anchor, const float* start, const float* end,
                  const float* T0, int64_t B, int K, int iterations, float* T_out, float* g_out,
                  float* trace_gnorm, void* stream) {
  return newton_impl<float>(basis, anchor, start, end, T0, B, K, iterations, T_out, g_out,
                            trace_gnorm, stream);
}

int fp_newton_f64(const double* basis, const double* anchor, const double* start, const double* end,
                  const double* T0, int64_t B, int K, int iterations, double* T_out, double* g_out,
                  double* trace_gnorm, void* stream) {
  return newton_impl<double>(basis, anchor, start, end, T0, B, K, iterations, T_out, g_out,
                             trace_gnorm, stream);
}

int fp_gd_f32(const float* basis, const float* anchor, const float* start, const float* end,
              const float* T0, int64_t B, int K, int iterations, float* T_out, float* g_out,
              void* stream) {
  return gd_impl<float>(basis, anchor, start, end, T0, B, K, iterations, T_out, g_out, stream);
}

int fp_gd_f64(const double* basis, const double* anchor, const double* start, const double* end,
              const double* T0, int64_t B, int K, int iterations, double* T_out, double* g_out,
              void* stream) {
  return gd_impl<double>(basis, anchor, start, end, T0, B, K, iterations, T_out, g_out, stream);
}

int fp_image_method_f64(const double* basis, const double* anchor, const double* start,
                        const double* end, int64_t B, int K, double* points, uint8_t* status,
                        void* stream) {
  if (B < 0 || K < 0 || K > 64 || (B > 0 && K > 0 && !points)) return FP_ERR_INVALID_ARGUMENT;
  if (B == 0 || K == 0) return FP_OK;
  image_kernel<double><<<unsigned((B + 63) / 64), 64, 0, static_cast<cudaStream_t>(stream)>>>(
      basis, anchor, start, end, B, K, points, status);
  count_launches(1);
  return cudaGetLastError() == cudaSuccess ? FP_OK : FP_ERR_CUDA;
}

}  // extern "C"
