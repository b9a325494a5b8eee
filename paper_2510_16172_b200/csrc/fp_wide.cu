// Warp-cooperative solver for orders 9..64.
//
// The reference accepts up to 64 interactions per path (geometry.py:23,
// MAX_INTERACTIONS); the register-resident kernels stop at order 8. Here one
// warp owns one path (two paths per warp, 16 lanes each, up to order 15 in
// fp32 / 11 in fp64): the dense 2K formulation (edges carry their zero basis
// column, geometry.py:86-90), the inverse Hessian and the per-path vectors in
// shared memory (16-byte row reads, a bank-conflict-free row stride),
// lanes striding over interactions, segments and Hessian rows, reductions as
// warp butterflies. The operations follow the reference's batched code in
// order — embed / clamped segments / gradient (batching.py:83-126), the
// fixed-point step size (solver.py:84-112), the BFGS loop with its curvature
// and finite-H' guards (solver.py:146-215) — in fp32 or fp64, with IEEE
// division and square root. The implicit VJP (objective.py:48-135,
// implicit_diff.py:39-77) assembles the block-tridiagonal Hessian in parallel
// and runs the block-Thomas solve (with the Tikhonov retry) on one lane.
// This is the long-path fallback: correct and bounded, not the tuned path.
#include <cuda_runtime.h>

#include "fp_dispatch.h"
#include "fp_kernels.cuh"

namespace fp {

namespace {

constexpr int kWideMaxOrder = 64;
constexpr int kWideThreads = 128;  // 4 paths per CTA when shared memory allows

// Reductions over the lanes of one path: a whole warp (lp = 32) or an aligned
// half (lp = 16, two paths per warp; gm masks the half).
template <typename R>
__device__ __forceinline__ R warp_sum(R v, int lp, unsigned gm) {
  for (int o = lp >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(gm, v, o);
  return v;
}
template <typename R>
__device__ __forceinline__ R warp_min(R v, int lp, unsigned gm) {
  for (int o = lp >> 1; o > 0; o >>= 1) {
    const R w = __shfl_xor_sync(gm, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// Per-warp shared-memory layout (units of R). Every array starts on a
// 16-byte boundary, so the BFGS loop reads H rows and the broadcast vectors
// with 16-byte loads; the H row stride makes those row reads bank-conflict
// free (a stride of 4 x odd words: the 8 lanes of each 128-byte phase hit
// distinct 4-bank groups).
struct WideLayout {
  int K, m, S, ld;
  int H, t, g, gn, p, st, y, hy, A, b, x, s, nc, nu, u, d, a2c, D, O, rhs, act, sol, dx, w, red;
  int total;
  __host__ __device__ static int row_stride(int m, int esize) {
    int ld = m;
    if (esize == 4)
      while (ld % 8 != 4) ++ld;  // ld words
    else
      while (ld % 4 != 2) ++ld;  // 2 ld words
    return ld;
  }
  __host__ __device__ WideLayout(int k, int esize)
      : K(k), m(2 * k), S(k + 1), ld(row_stride(2 * k, esize)) {
    int o = 0;
    auto take = [&o](int n) {
      const int r = o;
      o += (n + 3) & ~3;  // 4 elements: 16 bytes (fp32), 32 bytes (fp64)
      return r;
    };
    H = take(m * ld);
    t = take(m);
    g = take(m);
    gn = take(m);
    p = take(m);
    st = take(m);
    y = take(m);
    hy = take(m);
    A = take(6 * K);
    b = take(3 * K);
    x = take(3 * (K + 2));
    s = take(3 * S);
    nc = take(S);
    nu = take(S);
    u = take(3 * S);
    d = take(3 * S);
    a2c = take(2 * S);
    D = take(3 * K);
    O = take(4 * K);
    rhs = take(2 * K);
    act = take(2 * K);
    sol = take(2 * K);
    dx = take(3 * K);
    w = take(3 * S);
    red = take(8);
    total = o;
  }
};

// 16-byte vectors of R (four floats, two doubles).
template <typename R> struct Vec16;
template <> struct Vec16<float> { using T = float4; static constexpr int W = 4; };
template <> struct Vec16<double> { using T = double2; static constexpr int W = 2; };

template <typename R>
struct WideCtx {
  WideLayout L;
  R* sm;
  int lane;     // lane within the path's lanes
  int lp;       // lanes per path (32, or 16: two paths per warp)
  unsigned gm;  // mask of the path's lanes
  R eps;
  __device__ R* at(int off) const { return sm + off; }
  __device__ R Aij(int i, int r, int c) const { return sm[L.A + 6 * i + 2 * r + c]; }
};

// x, segments, norms and the clamped gradient of the parameters at `t`
// into `gout` (batching.py:83-120): einsum order, IEEE div / sqrt.
template <typename R>
__device__ void wide_eval(const WideCtx<R>& c, const R* t, R* gout) {
  const WideLayout& L = c.L;
  R* sm = c.sm;
  for (int q = c.lane; q < L.K + 2; q += c.lp) {
    R* X = sm + L.x + 3 * q;
    if (q == 0 || q == L.K + 1) continue;  // endpoints stored at load
    const int i = q - 1;
#pragma unroll
    for (int r = 0; r < 3; ++r)
      X[r] = (c.Aij(i, r, 0) * t[2 * i] + c.Aij(i, r, 1) * t[2 * i + 1]) + sm[L.b + 3 * i + r];
  }
  __syncwarp(c.gm);
  for (int k = c.lane; k < L.S; k += c.lp) {
    const R* lo = sm + L.x + 3 * k;
    const R* hi = lo + 3;
    R s[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) s[r] = hi[r] - lo[r];
    const R n = Num<R>::sqrt_((s[0] * s[0] + s[1] * s[1]) + s[2] * s[2]);
    const R cl = n < c.eps ? c.eps : n;  // np.maximum: NaN propagates
    sm[L.nu + k] = n;
    sm[L.nc + k] = cl;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      sm[L.s + 3 * k + r] = s[r];
      sm[L.u + 3 * k + r] = Num<R>::div(s[r], cl);
    }
  }
  __syncwarp(c.gm);
  for (int i = c.lane; i < L.K; i += c.lp) {
    R q[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) q[r] = sm[L.u + 3 * i + r] - sm[L.u + 3 * (i + 1) + r];
#pragma unroll
    for (int cc = 0; cc < 2; ++cc)
      gout[2 * i + cc] = (c.Aij(i, 0, cc) * q[0] + c.Aij(i, 1, cc) * q[1]) + c.Aij(i, 2, cc) * q[2];
  }
  __syncwarp(c.gm);
}

template <typename R>
__device__ R wide_length(const WideCtx<R>& c) {
  R l = R(0);
  for (int k = c.lane; k < c.L.S; k += c.lp) l += c.sm[c.L.nu + k];
  return warp_sum(l, c.lp, c.gm);
}

template <typename R>
__device__ R wide_dot(const WideCtx<R>& c, const R* a, const R* b) {
  R acc = R(0);
  for (int j = c.lane; j < c.L.m; j += c.lp) acc = fma(a[j], b[j], acc);
  return warp_sum(acc, c.lp, c.gm);
}

// out = H v (rows across lanes; each row and v read as 16-byte vectors, the
// products accumulated in column order). A lane's rows (j, j + lp, ...) run
// their chains side by side: independent FMA chains hide each other's latency.
template <typename R, int NR>
__device__ __forceinline__ void wide_matvec_rows(const WideCtx<R>& c, const R* v, R* out, R sign) {
  using V = typename Vec16<R>::T;
  constexpr int W = Vec16<R>::W;
  const WideLayout& L = c.L;
  const R* h[NR];
  R acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int j = c.lane + c.lp * r;
    h[r] = c.sm + L.H + (j < L.m ? j : 0) * L.ld;  // past the last row: row 0, result dropped
    acc[r] = R(0);
  }
  int q = 0;
  for (; q + W <= L.m; q += W) {
    const V vv = *reinterpret_cast<const V*>(v + q);
    const R* ve = reinterpret_cast<const R*>(&vv);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const V hv = *reinterpret_cast<const V*>(h[r] + q);
      const R* he = reinterpret_cast<const R*>(&hv);
#pragma unroll
      for (int e = 0; e < W; ++e) acc[r] = fma(he[e], ve[e], acc[r]);
    }
  }
  for (; q < L.m; ++q)
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[r] = fma(h[r][q], v[q], acc[r]);
#pragma unroll
  for (int r = 0; r < NR; ++r)
    if (c.lane + c.lp * r < L.m) out[c.lane + c.lp * r] = sign * acc[r];
}

// NRMAX: the most rows a lane owns in this kernel instantiation (m <= lp NRMAX).
template <typename R, int NRMAX>
__device__ void wide_matvec(const WideCtx<R>& c, const R* v, R* out, R sign) {
  const int nr = (c.L.m + c.lp - 1) / c.lp;  // rows per lane, the same on every lane of the path
  if (nr == 1) wide_matvec_rows<R, 1>(c, v, out, sign);
  if constexpr (NRMAX >= 2) if (nr == 2) wide_matvec_rows<R, 2>(c, v, out, sign);
  if constexpr (NRMAX >= 3) if (nr == 3) wide_matvec_rows<R, 3>(c, v, out, sign);
  if constexpr (NRMAX >= 4) if (nr == 4) wide_matvec_rows<R, 4>(c, v, out, sign);
  __syncwarp(c.gm);
}

// The BFGS update of the rows of this lane, the reference's expression per
// entry (solver.py:186-195), rows side by side.
template <typename R, int NR>
__device__ __forceinline__ void wide_update_rows(const WideCtx<R>& c, const R* stp, const R* hy, R rho,
                                                 R coef) {
  using V = typename Vec16<R>::T;
  constexpr int W = Vec16<R>::W;
  const WideLayout& L = c.L;
  R* h[NR];
  R sj[NR], hj[NR];
  bool live[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int j0 = c.lane + c.lp * r;
    live[r] = j0 < L.m;
    const int j = live[r] ? j0 : 0;  // past the last row: row 0, computed, never stored
    h[r] = c.sm + L.H + j * L.ld;
    sj[r] = stp[j];
    hj[r] = hy[j];
  }
  int q = 0;
  for (; q + W <= L.m; q += W) {
    const V sv = *reinterpret_cast<const V*>(stp + q);
    const V yv = *reinterpret_cast<const V*>(hy + q);
    const R* se = reinterpret_cast<const R*>(&sv);
    const R* ye = reinterpret_cast<const R*>(&yv);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      V hv = *reinterpret_cast<const V*>(h[r] + q);
      R* he = reinterpret_cast<R*>(&hv);
#pragma unroll
      for (int e = 0; e < W; ++e)
        he[e] = (he[e] - rho * (sj[r] * ye[e] + se[e] * hj[r])) + coef * (sj[r] * se[e]);
      if (live[r]) *reinterpret_cast<V*>(h[r] + q) = hv;
    }
  }
  for (; q < L.m; ++q)
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const R v = (h[r][q] - rho * (sj[r] * hy[q] + stp[q] * hj[r])) + coef * (sj[r] * stp[q]);
      if (live[r]) h[r][q] = v;
    }
}

template <typename R, int NRMAX>
__device__ void wide_update(const WideCtx<R>& c, const R* stp, const R* hy, R rho, R coef) {
  const int nr = (c.L.m + c.lp - 1) / c.lp;
  if (nr == 1) wide_update_rows<R, 1>(c, stp, hy, rho, coef);
  if constexpr (NRMAX >= 2) if (nr == 2) wide_update_rows<R, 2>(c, stp, hy, rho, coef);
  if constexpr (NRMAX >= 3) if (nr == 3) wide_update_rows<R, 3>(c, stp, hy, rho, coef);
  if constexpr (NRMAX >= 4) if (nr == 4) wide_update_rows<R, 4>(c, stp, hy, rho, coef);
}

template <typename R>
__device__ __forceinline__ R warp_absmax(R v, int lp, unsigned gm) {
  for (int o = lp >> 1; o > 0; o >>= 1) v = absmax_nan(v, __shfl_xor_sync(gm, v, o));
  return v;
}

// Fixed-point step size along p (solver.py:84-112); sets `zero`.
template <typename R>
__device__ R wide_step_size(const WideCtx<R>& c, const R* p, int fp_iters, bool& zero) {
  const WideLayout& L = c.L;
  R* sm = c.sm;
  R a2sum = R(0);
  for (int k = c.lane; k < L.S; k += c.lp) {
    R dd[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const R hi = k < L.K ? c.Aij(k, r, 0) * p[2 * k] + c.Aij(k, r, 1) * p[2 * k + 1] : R(0);
      const R lo = k > 0 ? c.Aij(k - 1, r, 0) * p[2 * k - 2] + c.Aij(k - 1, r, 1) * p[2 * k - 1] : R(0);
      dd[r] = hi - lo;
      sm[L.d + 3 * k + r] = dd[r];
    }
    const R* s = sm + L.s + 3 * k;
    const R a2 = (dd[0] * dd[0] + dd[1] * dd[1]) + dd[2] * dd[2];
    const R cc = (dd[0] * s[0] + dd[1] * s[1]) + dd[2] * s[2];
    sm[L.a2c + 2 * k] = a2;
    sm[L.a2c + 2 * k + 1] = cc;
    a2sum += a2;
  }
  zero = warp_sum(a2sum, c.lp, c.gm) <= Num<R>::tiny();
  R alpha = R(0);
  for (int f = 0; f < fp_iters; ++f) {
    R num = R(0), den = R(0);
    for (int k = c.lane; k < L.S; k += c.lp) {
      const R* s = sm + L.s + 3 * k;
      const R* dd = sm + L.d + 3 * k;
      R e[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) e[r] = s[r] + alpha * dd[r];
      R n = Num<R>::sqrt_((e[0] * e[0] + e[1] * e[1]) + e[2] * e[2]);
      n = n < c.eps ? c.eps : n;
      num += Num<R>::div(sm[L.a2c + 2 * k + 1], n);
      den += Num<R>::div(sm[L.a2c + 2 * k], n);
    }
    num = warp_sum(num, c.lp, c.gm);
    den = warp_sum(den, c.lp, c.gm);
    const R cand = -Num<R>::div(num, zero ? R(1) : den);
    alpha = (zero || !finite(cand)) ? alpha : cand;
  }
  __syncwarp(c.gm);
  return alpha;
}

// Implicit VJP at the current state (same mathematics as implicit_vjp in
// fp_path.cuh): outputs to the path's records directly.
template <typename R>
__device__ uint8_t wide_vjp(const WideCtx<R>& c, const PathArgs<R>& a, int64_t row, const R* t) {
  const WideLayout& L = c.L;
  R* sm = c.sm;
  const int K = L.K;
  uint8_t st = 0;
  const R wl = a.wL ? a.wL[row] : a.wL_scale;
  const bool full = a.mode == FP_VJP_FULL, mixed = a.mode == FP_VJP_MIXED;
  const bool has_v = a.vT != nullptr;
  const bool need_solve = !mixed && (has_v || (full && wl != R(0)));
  const R* vT = has_v ? a.vT + row * 2 * K : nullptr;
  // per interaction: active flags, Hessian blocks, rhs
  R trace = R(0);
  for (int i = c.lane; i < K; i += c.lp) {
    bool act[2];
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      act[cc] = c.Aij(i, 0, cc) != R(0) || c.Aij(i, 1, cc) != R(0) || c.Aij(i, 2, cc) != R(0);
      sm[L.act + 2 * i + cc] = act[cc] ? R(1) : R(0);
      const R v = vT ? vT[2 * i + cc] : R(0);
      sm[L.sol + 2 * i + cc] = mixed ? v : R(0);
      const R gv = full ? fma(wl, sm[L.g + 2 * i + cc], v) : v;
      sm[L.rhs + 2 * i + cc] = act[cc] ? -gv : R(0);
    }
    if (!need_solve) continue;
    const R* ui = sm + L.u + 3 * i;
    const R* uo = ui + 3;
    const R ri = R(1) / sm[L.nc + i], ro = R(1) / sm[L.nc + i + 1];
    R ain[2], aout[2], gii[3];
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      ain[cc] = fma(c.Aij(i, 2, cc), ui[2], fma(c.Aij(i, 1, cc), ui[1], c.Aij(i, 0, cc) * ui[0]));
      aout[cc] = fma(c.Aij(i, 2, cc), uo[2], fma(c.Aij(i, 1, cc), uo[1], c.Aij(i, 0, cc) * uo[0]));
    }
    gii[0] = fma(c.Aij(i, 2, 0), c.Aij(i, 2, 0), fma(c.Aij(i, 1, 0), c.Aij(i, 1, 0), c.Aij(i, 0, 0) * c.Aij(i, 0, 0)));
    gii[1] = fma(c.Aij(i, 2, 0), c.Aij(i, 2, 1), fma(c.Aij(i, 1, 0), c.Aij(i, 1, 1), c.Aij(i, 0, 0) * c.Aij(i, 0, 1)));
    gii[2] = fma(c.Aij(i, 2, 1), c.Aij(i, 2, 1), fma(c.Aij(i, 1, 1), c.Aij(i, 1, 1), c.Aij(i, 0, 1) * c.Aij(i, 0, 1)));
    R D0 = (gii[0] - ain[0] * ain[0]) * ri + (gii[0] - aout[0] * aout[0]) * ro;
    R D1 = (gii[1] - ain[0] * ain[1]) * ri + (gii[1] - aout[0] * aout[1]) * ro;
    R D2 = (gii[2] - ain[1] * ain[1]) * ri + (gii[2] - aout[1] * aout[1]) * ro;
    if (act[0]) trace += D0;
    if (act[1]) trace += D2;
    if (!act[0]) { D0 = R(1); D1 = R(0); }
    if (!act[1]) { D2 = R(1); D1 = R(0); }
    sm[L.D + 3 * i] = D0;
    sm[L.D + 3 * i + 1] = D1;
    sm[L.D + 3 * i + 2] = D2;
    if (i + 1 < K) {
      R ain1[2];  // A_{i+1}^T u_{i+1}
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
        ain1[cc] = fma(c.Aij(i + 1, 2, cc), uo[2], fma(c.Aij(i + 1, 1, cc), uo[1], c.Aij(i + 1, 0, cc) * uo[0]));
#pragma unroll
      for (int aa = 0; aa < 2; ++aa)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) {
          const R gij = fma(c.Aij(i, 2, aa), c.Aij(i + 1, 2, bb),
                            fma(c.Aij(i, 1, aa), c.Aij(i + 1, 1, bb), c.Aij(i, 0, aa) * c.Aij(i + 1, 0, bb)));
          sm[L.O + 4 * i + 2 * aa + bb] = -(gij - aout[aa] * ain1[bb]) * ro;
        }
    }
  }
  trace = warp_sum(trace, c.lp, c.gm);
  __syncwarp(c.gm);
  if (need_solve) {
    if (c.lane == 0) {
      // _solve_sym (implicit_diff.py:55-71): block-Thomas elimination, accepted
      // when |H_a x - rhs| <= tol (1 + |rhs|) — after one step of iterative
      // refinement if the first solution misses (fp_path.cuh explains why) —
      // else (or on a zero pivot / a non-finite solution) one Tikhonov retry,
      // accepted when finite. Scratch: Ci in dx (3K), z in w (2K of 3S), the
      // residual in y (2K) and the correction in hy (2K) (BFGS scratch, free
      // here).
      R* Ci = sm + L.dx;
      R* z = sm + L.w;
      R* res = sm + L.y;
      R* dxs = sm + L.hy;
      const R* O_ = sm + L.O;
      auto factor = [&](R lam) {
        bool ok = true;
        for (int i = 0; i < K; ++i) {
          const R* D = sm + L.D + 3 * i;
          const bool a0 = sm[L.act + 2 * i] != R(0), a1 = sm[L.act + 2 * i + 1] != R(0);
          R C0 = D[0] + (a0 ? lam : R(0)), C1 = D[1], C2 = D[2] + (a1 ? lam : R(0));
          if (i > 0) {
            const R* O = O_ + 4 * (i - 1);  // O[a][b] = O[2a + b]
            const R* Cp = Ci + 3 * (i - 1);
            R Lm[2][2];
            for (int aa = 0; aa < 2; ++aa) {
              Lm[aa][0] = O[aa] * Cp[0] + O[2 + aa] * Cp[1];
              Lm[aa][1] = O[aa] * Cp[1] + O[2 + aa] * Cp[2];
            }
            C0 -= Lm[0][0] * O[0] + Lm[0][1] * O[2];
            C1 -= Lm[0][0] * O[1] + Lm[0][1] * O[3];
            C2 -= Lm[1][0] * O[1] + Lm[1][1] * O[3];
          }
          const R det = C0 * C2 - C1 * C1;
          ok = ok && det != R(0) && finite(det);  // LinAlgError: exactly singular pivot
          const R id = R(1) / det;
          Ci[3 * i] = C2 * id;
          Ci[3 * i + 1] = -C1 * id;
          Ci[3 * i + 2] = C0 * id;
        }
        return ok;
      };
      auto substitute = [&](const R* b, R* x) {
        for (int i = 0; i < K; ++i) {
          R z0 = b[2 * i], z1 = b[2 * i + 1];
          if (i > 0) {
            const R* O = O_ + 4 * (i - 1);
            const R* Cp = Ci + 3 * (i - 1);
            R Lm[2][2];
            for (int aa = 0; aa < 2; ++aa) {
              Lm[aa][0] = O[aa] * Cp[0] + O[2 + aa] * Cp[1];
              Lm[aa][1] = O[aa] * Cp[1] + O[2 + aa] * Cp[2];
            }
            z0 -= Lm[0][0] * z[2 * (i - 1)] + Lm[0][1] * z[2 * (i - 1) + 1];
            z1 -= Lm[1][0] * z[2 * (i - 1)] + Lm[1][1] * z[2 * (i - 1) + 1];
          }
          z[2 * i] = z0;
          z[2 * i + 1] = z1;
        }
        bool ok = true;
        R nx0 = R(0), nx1 = R(0);
        for (int i = K - 1; i >= 0; --i) {
          R r0 = z[2 * i], r1 = z[2 * i + 1];
          if (i + 1 < K) {
            const R* O = O_ + 4 * i;
            r0 -= O[0] * nx0 + O[1] * nx1;
            r1 -= O[2] * nx0 + O[3] * nx1;
          }
          const R v0 = Ci[3 * i] * r0 + Ci[3 * i + 1] * r1;
          const R v1 = Ci[3 * i + 1] * r0 + Ci[3 * i + 2] * r1;
          nx0 = sm[L.act + 2 * i] != R(0) ? v0 : R(0);
          nx1 = sm[L.act + 2 * i + 1] != R(0) ? v1 : R(0);
          x[2 * i] = nx0;
          x[2 * i + 1] = nx1;
          ok = ok && finite(v0) && finite(v1);
        }
        return ok;
      };
      auto residual = [&](const R* x) {  // res = rhs - H_a x; returns |res|^2
        const R* rh = sm + L.rhs;
        R rr = R(0);
        for (int i = 0; i < K; ++i) {
          const R* D = sm + L.D + 3 * i;
          R r0 = D[0] * x[2 * i] + D[1] * x[2 * i + 1];
          R r1 = D[1] * x[2 * i] + D[2] * x[2 * i + 1];
          if (i > 0) {
            const R* O = O_ + 4 * (i - 1);
            r0 += O[0] * x[2 * i - 2] + O[2] * x[2 * i - 1];
            r1 += O[1] * x[2 * i - 2] + O[3] * x[2 * i - 1];
          }
          if (i + 1 < K) {
            const R* O = O_ + 4 * i;
            r0 += O[0] * x[2 * i + 2] + O[1] * x[2 * i + 3];
            r1 += O[2] * x[2 * i + 2] + O[3] * x[2 * i + 3];
          }
          res[2 * i] = rh[2 * i] - r0;
          res[2 * i + 1] = rh[2 * i + 1] - r1;
          rr = fma(res[2 * i + 1], res[2 * i + 1], fma(res[2 * i], res[2 * i], rr));
        }
        return rr;
      };
      R* x = sm + L.sol;
      bool solved = false;
      if (factor(R(0)) && substitute(sm + L.rhs, x)) {
        R bb = R(0);
        for (int i = 0; i < 2 * K; ++i) bb = fma(sm[L.rhs + i], sm[L.rhs + i], bb);
        const R tol = Num<R>::resid_tol() * (R(1) + Num<R>::sqrt_(bb));
        solved = Num<R>::sqrt_(residual(x)) <= tol;  // NaN: not solved
        if (!solved && substitute(res, dxs)) {
          for (int i = 0; i < 2 * K; ++i) x[i] += dxs[i];
          solved = Num<R>::sqrt_(residual(x)) <= tol;
        }
      }
      if (!solved) solved = factor(R(1e-12) * trace) && substitute(sm + L.rhs, x);
      if (!solved)
        for (int i = 0; i < 2 * K; ++i) sm[L.sol + i] = R(0);
      sm[L.red] = solved ? R(1) : R(0);
    }
    __syncwarp(c.gm);
    if (sm[L.red] == R(0)) st |= FP_STATUS_SINGULAR;
  }
  // param_vjp with the solution + wl * length partials (objective.py:89-135)
  for (int i = c.lane; i < K; i += c.lp)
#pragma unroll
    for (int r = 0; r < 3; ++r)
      sm[L.dx + 3 * i + r] = fma(c.Aij(i, r, 1), sm[L.sol + 2 * i + 1], c.Aij(i, r, 0) * sm[L.sol + 2 * i]);
  __syncwarp(c.gm);
  for (int k = c.lane; k < L.S; k += c.lp) {
    const R* u = sm + L.u + 3 * k;
    R ds[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const R hi = k < K ? sm[L.dx + 3 * k + r] : R(0);
      const R lo = k > 0 ? sm[L.dx + 3 * (k - 1) + r] : R(0);
      ds[r] = hi - lo;
    }
    const R ud = fma(u[2], ds[2], fma(u[1], ds[1], u[0] * ds[0]));
    const R rk = R(1) / sm[L.nc + k];
#pragma unroll
    for (int r = 0; r < 3; ++r) sm[L.w + 3 * k + r] = (ds[r] - u[r] * ud) * rk;
  }
  __syncwarp(c.gm);
  bool fin = true;
  for (int i = c.lane; i < K; i += c.lp) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const R q = sm[L.u + 3 * i + r] - sm[L.u + 3 * (i + 1) + r];
      const R zi = sm[L.w + 3 * i + r] - sm[L.w + 3 * (i + 1) + r];
      const R e = fma(wl, q, zi);
      const R b0 = fma(e, t[2 * i], q * sm[L.sol + 2 * i]);
      const R b1 = fma(e, t[2 * i + 1], q * sm[L.sol + 2 * i + 1]);
      fin = fin && finite(e) && finite(b0) && finite(b1);
      if (a.d_anchor) a.d_anchor[(row * K + i) * 3 + r] = e;
      if (a.d_basis) {
        a.d_basis[(row * K + i) * 6 + 2 * r] = b0;
        a.d_basis[(row * K + i) * 6 + 2 * r + 1] = b1;
      }
    }
    if (a.u_out) {
      a.u_out[(row * K + i) * 2] = sm[L.sol + 2 * i];
      a.u_out[(row * K + i) * 2 + 1] = sm[L.sol + 2 * i + 1];
    }
  }
  if (c.lane < 3) {
    const int r = c.lane;
    const R d0 = -fma(wl, sm[L.u + r], sm[L.w + r]);
    const R d1 = fma(wl, sm[L.u + 3 * K + r], sm[L.w + 3 * K + r]);
    fin = fin && finite(d0) && finite(d1);
    if (a.d_start) a.d_start[row * 3 + r] = d0;
    if (a.d_end) a.d_end[row * 3 + r] = d1;
  }
  if (!__all_sync(c.gm, fin)) st |= FP_STATUS_NONFINITE;
  return st;
}

// One instantiation per bound on the rows a lane owns (NRMAX = 1: K <= 16,
// 2: K <= 32, 4: K <= 64), so short orders do not pay the registers of the
// four-row loops. CTAs per SM requested from ptxas: FP_WIDE_MIN_BLOCKS_R<n>
// (A/B builds; K = 33..64 is shared-memory bound at one CTA per SM).
#ifndef FP_WIDE_MIN_BLOCKS_R1
#define FP_WIDE_MIN_BLOCKS_R1 6  // 80 registers; measured: K=16 fp32 3.97 -> 2.90 ms vs uncapped (153)
#endif
#ifndef FP_WIDE_MIN_BLOCKS_R2
#define FP_WIDE_MIN_BLOCKS_R2 1
#endif
#ifndef FP_WIDE_MIN_BLOCKS_L16
#define FP_WIDE_MIN_BLOCKS_L16 6
#endif
template <int NRMAX, int LP>
struct WideMin {
  static constexpr int value = LP == 16     ? FP_WIDE_MIN_BLOCKS_L16
                               : NRMAX == 1 ? FP_WIDE_MIN_BLOCKS_R1
                               : NRMAX == 2 ? FP_WIDE_MIN_BLOCKS_R2
                                            : 1;
};
// LP lanes per path: 32 (one path per warp) or 16 (two paths per warp, for
// orders whose segment and row loops leave most of a warp idle).
template <typename R, int OP, int NRMAX, int LP>
__global__ void __launch_bounds__(kWideThreads, (WideMin<NRMAX, LP>::value))
    wide_kernel(const __grid_constant__ PathArgs<R> a, int K, int ppb) {
  static_assert(LP == 16 || LP == 32, "16 or 32 lanes per path");
  extern __shared__ __align__(16) unsigned char wide_smem[];
  const int slot = int(threadIdx.x) / LP, lane = int(threadIdx.x) & (LP - 1);
  const unsigned gm = LP == 32 ? 0xffffffffu : (0xffffu << (threadIdx.x & 16));
  if (slot >= ppb) return;
  const WideLayout L(K, int(sizeof(R)));
  const int64_t row = a.row_begin + int64_t(blockIdx.x) * ppb + slot;
  if (row >= a.B) return;  // the path's lanes leave together: only path-level sync below
  R* sm = reinterpret_cast<R*>(wide_smem) + size_t(slot) * L.total;
  const int m = L.m;
  // ---- load ----------------------------------------------------------------
  for (int e = lane; e < 6 * K; e += LP) sm[L.A + e] = a.basis[row * 6 * K + e];
  for (int e = lane; e < 3 * K; e += LP) sm[L.b + e] = a.anchor[row * 3 * K + e];
  for (int e = lane; e < m; e += LP) sm[L.t + e] = a.T[row * m + e];
  if (lane < 3) {
    sm[L.x + lane] = a.start[row * 3 + lane];
    sm[L.x + 3 * (K + 1) + lane] = a.end[row * 3 + lane];
  }
  __syncwarp(gm);
  R eps;
  {
    const double dx = double(sm[L.x + 3 * (K + 1)]) - double(sm[L.x]);
    const double dy = double(sm[L.x + 3 * (K + 1) + 1]) - double(sm[L.x + 1]);
    const double dz = double(sm[L.x + 3 * (K + 1) + 2]) - double(sm[L.x + 2]);
    eps = R(1e-12 * (1.0 + __dsqrt_rn(__fma_rn(dz, dz, __fma_rn(dy, dy, dx * dx)))));
  }
  const WideCtx<R> c{L, sm, lane, LP, gm, eps};
  R* t = sm + L.t;
  R* g = sm + L.g;
  wide_eval(c, t, g);
  uint8_t st = 0;
  if (OP != OP_VJP) {
    R n0 = Num<R>::inf();
    for (int k = lane; k < L.S; k += LP) n0 = sm[L.nu + k] < n0 ? sm[L.nu + k] : n0;
    if (warp_min(n0, LP, gm) <= eps) st |= FP_STATUS_DEGENERATE_ENTRY;  // checked_segments (solver.py:166)
    R* H = sm + L.H;
    for (int j = lane; j < m; j += LP)
      for (int q = 0; q < m; ++q) H[j * L.ld + q] = j == q ? R(1) : R(0);
    R hbound = R(1);  // >= max |H_ij| (the update's overflow pre-check)
    const bool last_dead = a.H_out == nullptr && a.trace_len == nullptr;
    R* p = sm + L.p;
    R* stp = sm + L.st;
    R* gn = sm + L.gn;
    R* y = sm + L.y;
    R* hy = sm + L.hy;
    __syncwarp(gm);
    for (int it = 0; it < a.iterations; ++it) {
      wide_matvec<R, NRMAX>(c, g, p, R(-1));  // p = -H g
      bool zero;
      const R alpha = wide_step_size(c, p, a.fp_iters, zero);
      if (zero) st |= FP_STATUS_ZERO_DIRECTION;
      uint8_t fate = zero ? FP_FATE_ZERO_DIRECTION : 0;
      for (int j = lane; j < m; j += LP) {
        stp[j] = alpha * p[j];
        t[j] = t[j] + stp[j];
      }
      __syncwarp(gm);
      wide_eval(c, t, gn);
      if (last_dead && it == a.iterations - 1) {
        // the last update and its curvature test feed nothing read afterwards
        for (int j = lane; j < m; j += LP) g[j] = gn[j];
        __syncwarp(gm);
        break;
      }
      for (int j = lane; j < m; j += LP) y[j] = gn[j] - g[j];
      __syncwarp(gm);
      const R sy = wide_dot(c, stp, y);
      const R sn = Num<R>::sqrt_(wide_dot(c, stp, stp));
      const R yn = Num<R>::sqrt_(wide_dot(c, y, y));
      if (!(sy > (R(1e-12) * sn) * yn)) fate |= FP_FATE_CURVATURE_SKIP;
      if (sy > (R(1e-12) * sn) * yn) {
        const R rho = R(1) / sy;
        wide_matvec<R, NRMAX>(c, y, hy, R(1));
        const R yHy = wide_dot(c, y, hy);
        const R coef = rho * rho * yHy + rho;
        // The reference skips the update when any entry of H' is not finite
        // (solver.py:196-199). With ms = max|s|, mh = max|Hy| and bound >=
        // max|H|, every intermediate of an entry is at most 2 ms mh, ms^2,
        // 2 |rho| ms mh, |coef| ms^2 or bound + 2 |rho| ms mh + |coef| ms^2;
        // below Num<R>::suspect() (340x / 1800x under the largest finite
        // value) none can overflow, so the entry-by-entry check runs only
        // above it (or on a NaN, which the NaN-propagating maxima carry).
        // Same verdicts as checking every entry.
        R ms = R(0), mh = R(0);
        for (int j = lane; j < m; j += LP) {
          ms = absmax_nan(ms, stp[j]);
          mh = absmax_nan(mh, hy[j]);
        }
        ms = warp_absmax(ms, LP, gm);
        mh = warp_absmax(mh, LP, gm);
        const R am = ms * mh, ss = ms * ms;
        const R r2a = R(2) * fabs(rho) * am, cs = fabs(coef) * ss;
        const R nb = (hbound + r2a) + cs;
        const R big = absmax_nan(absmax_nan(R(2) * am, ss), absmax_nan(absmax_nan(r2a, cs), nb));
        bool fin = true;
        R mx = R(0);
        const bool checked = !(big < Num<R>::suspect());
        if (checked) {
          for (int j = lane; j < m; j += LP) {
            const R* h = H + j * L.ld;
            for (int q = 0; q < m; ++q) {
              const R v = (h[q] - rho * (stp[j] * hy[q] + stp[q] * hy[j])) + coef * (stp[j] * stp[q]);
              fin = fin && finite(v);
              mx = fabs(v) > mx ? fabs(v) : mx;
            }
          }
          fin = __all_sync(gm, fin);
          mx = warp_absmax(mx, LP, gm);
        }
        if (checked) fate |= FP_FATE_ENTRY_CHECK;
        if (!fin) fate |= FP_FATE_NONFINITE_SKIP;
        if (fin) {
          wide_update<R, NRMAX>(c, stp, hy, rho, coef);
          hbound = checked ? mx * R(1.0009765625) : nb;
        }
        __syncwarp(gm);
      }
      for (int j = lane; j < m; j += LP) g[j] = gn[j];
      __syncwarp(gm);
      if (a.trace_len != nullptr) {
        const R len = wide_length(c);
        const R gq = wide_dot(c, g, g);
        if (lane == 0) {
          a.trace_len[int64_t(it) * a.ld + row] = len;
          a.trace_gnorm[int64_t(it) * a.ld + row] = Num<R>::sqrt_(gq);
          if (a.trace_fate != nullptr) a.trace_fate[int64_t(it) * a.ld + row] = fate;
        }
      }
    }
    if (a.H_out != nullptr)
      for (int j = lane; j < m; j += LP)
        for (int q = 0; q < m; ++q) a.H_out[(row * m + j) * m + q] = H[j * L.ld + q];
  }
  // ---- final classification (as final_status) ------------------------------------
  const R len = wide_length(c);
  R nmin = Num<R>::inf();
  for (int k = lane; k < L.S; k += LP) nmin = sm[L.nu + k] < nmin ? sm[L.nu + k] : nmin;
  nmin = warp_min(nmin, LP, gm);
  const R gq = wide_dot(c, g, g);
  if (!(Num<R>::sqrt_(gq) < R(1e-5) * (R(1) + len))) st |= FP_STATUS_NOT_STATIONARY;
  if (nmin <= eps) st |= FP_STATUS_DEGENERATE_FINAL;
  if (nmin < R(1e-3)) st |= FP_STATUS_SHORT_SEGMENT;
  bool fin = finite(len);
  for (int j = lane; j < m; j += LP) fin = fin && finite(t[j]) && finite(g[j]);
  if (!__all_sync(gm, fin)) st |= FP_STATUS_NONFINITE;
  if (OP != OP_VJP) {
    for (int j = lane; j < m; j += LP) {
      if (a.T_out) a.T_out[row * m + j] = t[j];
      if (a.g_out) a.g_out[row * m + j] = g[j];
    }
    if (a.points_out)
      for (int e = lane; e < 3 * K; e += LP) a.points_out[row * 3 * K + e] = sm[L.x + 3 + e];
    if (a.length_out && lane == 0) a.length_out[row] = len;
  }
  if (OP != OP_SOLVE) st |= wide_vjp(c, a, row, t);
  if (a.status_out && lane == 0) a.status_out[row] = st;
}

}  // namespace

size_t wide_smem_per_path(int K, size_t elem) { return size_t(WideLayout(K, int(elem)).total) * elem; }

template <typename R, int NRMAX, int LP>
cudaError_t launch_wide(int op, const PathArgs<R>& a, int K, int ppb, int64_t blocks, int threads,
                        size_t smem, cudaStream_t s);

// Orders up to FP_WIDE_LP16_MAX_K_F32 / _F64 run two paths per warp (16 lanes
// each); 0 keeps one path per warp (A/B builds). Measured (profiles/
// r02x_ab_wide_lp16.txt, fused step, 20 iterations): fp32 K=9 4.77 -> 3.02
// ms, K=12 3.69 -> 2.47, K=15 3.39 -> 3.03, K=16 2.90 -> 3.03; fp64 K=9 6.31
// -> 5.76, K=11 5.54 -> 4.96, K=12 5.19 -> 6.42 (shared memory per path
// doubles, fewer CTAs fit).
#ifndef FP_WIDE_LP16_MAX_K_F32
#define FP_WIDE_LP16_MAX_K_F32 15
#endif
#ifndef FP_WIDE_LP16_MAX_K_F64
#define FP_WIDE_LP16_MAX_K_F64 11
#endif

template <typename R>
cudaError_t dispatch_wide(int K, const PathArgs<R>& a, int op, cudaStream_t s) {
  if (K <= 8 || K > kWideMaxOrder) return cudaErrorInvalidValue;
  const int64_t rows = a.B - a.row_begin;
  if (rows <= 0) return cudaSuccess;
  const size_t per = wide_smem_per_path(K, sizeof(R));
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int lp = K <= (sizeof(R) == 4 ? FP_WIDE_LP16_MAX_K_F32 : FP_WIDE_LP16_MAX_K_F64) ? 16 : 32;
  int ppb = int(size_t(optin) / per);  // paths per CTA
  ppb = ppb > kWideThreads / lp ? kWideThreads / lp : ppb;
  if (ppb < 1) return cudaErrorInvalidValue;
  const size_t smem = per * size_t(ppb);
  const int64_t blocks = (rows + ppb - 1) / ppb;
  const int threads = (ppb * lp + 31) / 32 * 32;
  const int nrmax = (2 * K + lp - 1) / lp;
  if (lp == 16) return launch_wide<R, 2, 16>(op, a, K, ppb, blocks, threads, smem, s);
  switch (nrmax) {
    case 1: return launch_wide<R, 1, 32>(op, a, K, ppb, blocks, threads, smem, s);
    case 2: return launch_wide<R, 2, 32>(op, a, K, ppb, blocks, threads, smem, s);
    default: return launch_wide<R, 4, 32>(op, a, K, ppb, blocks, threads, smem, s);
  }
}

template <typename R, int NRMAX, int LP>
cudaError_t launch_wide(int op, const PathArgs<R>& a, int K, int ppb, int64_t blocks, int threads,
                        size_t smem, cudaStream_t s) {
  cudaError_t e;
  switch (op) {
    case OP_SOLVE:
      e = cudaFuncSetAttribute(wide_kernel<R, OP_SOLVE, NRMAX, LP>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e == cudaSuccess)
        wide_kernel<R, OP_SOLVE, NRMAX, LP><<<unsigned(blocks), threads, smem, s>>>(a, K, ppb);
      break;
    case OP_SOLVE_VJP:
      e = cudaFuncSetAttribute(wide_kernel<R, OP_SOLVE_VJP, NRMAX, LP>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e == cudaSuccess)
        wide_kernel<R, OP_SOLVE_VJP, NRMAX, LP><<<unsigned(blocks), threads, smem, s>>>(a, K, ppb);
      break;
    case OP_VJP:
      e = cudaFuncSetAttribute(wide_kernel<R, OP_VJP, NRMAX, LP>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e == cudaSuccess)
        wide_kernel<R, OP_VJP, NRMAX, LP><<<unsigned(blocks), threads, smem, s>>>(a, K, ppb);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template cudaError_t dispatch_wide<float>(int, const PathArgs<float>&, int, cudaStream_t);
template cudaError_t dispatch_wide<double>(int, const PathArgs<double>&, int, cudaStream_t);

}  // namespace fp
