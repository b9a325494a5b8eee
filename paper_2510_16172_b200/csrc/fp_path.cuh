// Per-path register-resident Fermat path state and math (sm_100a).
//
// One thread owns one path. The unknowns live in a compressed vector of the
// active coordinates of the kind mask MASK (bit i set: interaction i is a
// plane with two unknowns; clear: an edge with one). MASK = all ones is the
// "dense" uniform 2K formulation of the reference (geometry.py:86-90): edges
// carry a zero second basis column, which produces exact zeros, so it is
// valid for every batch; specialised masks skip the inert lanes and give the
// same bits for those paths.
//
// Reference semantics reproduced (file:line under /root/reference/pkg/src/fermatpath):
//   embed / segments / clamped norms / gradient   batching.py:83-120
//   fixed-point step size (paper Eq. 6)           solver.py:84-112
//   BFGS loop, curvature skip, finite-H skip      solver.py:146-215
//   unclamped length                               batching.py:123-126
//   Hessian blocks, param_vjp, length partials     objective.py:48-135
//   stationarity gate, active solve, Tikhonov     implicit_diff.py:25-77
#pragma once

#include "fp_common.cuh"

namespace fp {

template <typename R, int K>
struct Geo {
  R A[K][3][2];  // basis, row r, column c
  R b[K][3];     // anchor
  R x0[3], xe[3];
  R eps;         // 1e-12 (1 + |end - start|), fp64 then cast (batching.py:67-72)
  R reps;        // 1 / eps
};

// Load one path's geometry from a record in the reference layout.
template <typename R, int K, unsigned MASK>
__device__ __forceinline__ void load_geo(Geo<R, K>& G, const R* basis, const R* anchor,
                                         const R* start, const R* end) {
  using L = Lay<K, MASK>;
#pragma unroll
  for (int i = 0; i < K; ++i) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      G.A[i][r][0] = basis[i * 6 + r * 2 + 0];
      G.A[i][r][1] = L::plane(i) ? basis[i * 6 + r * 2 + 1] : R(0);
      G.b[i][r] = anchor[i * 3 + r];
    }
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    G.x0[r] = start[r];
    G.xe[r] = end[r];
  }
  const double dx = double(G.xe[0]) - double(G.x0[0]);
  const double dy = double(G.xe[1]) - double(G.x0[1]);
  const double dz = double(G.xe[2]) - double(G.x0[2]);
  const double nrm = __dsqrt_rn(__fma_rn(dz, dz, __fma_rn(dy, dy, dx * dx)));
  G.eps = R(1e-12 * (1.0 + nrm));
  G.reps = Num<R>::rcp(G.eps);
}

template <typename R, int K, unsigned MASK>
struct PathState {
  using L = Lay<K, MASK>;
  static constexpr int S = L::S;
  static constexpr int NA = L::NA;

  R t[NA];     // active unknowns
  R g[NA];     // clamped-norm gradient at t
  R s[S][3];   // segments at t
  R rn[S];     // 1 / max(|s_k|, eps)
  R nu[S];     // |s_k| (unclamped)

  // Path length: sum of unclamped norms (batching.py:123-126).
  __device__ __forceinline__ R length() const {
    R l = nu[0];
#pragma unroll
    for (int k = 1; k < S; ++k) l += nu[k];
    return l;
  }
  // Shortest segment (NaN-blind like the reference's `norms <= eps` test).
  __device__ __forceinline__ R min_norm() const {
    R m = nu[0];
#pragma unroll
    for (int k = 1; k < S; ++k) m = nu[k] < m ? nu[k] : m;
    return m;
  }

  // x_i = A_i t_i + b_i (geometry.py:153-165)
  __device__ __forceinline__ void points(const Geo<R, K>& G, R (&P)[K + 2][3]) const {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      P[0][r] = G.x0[r];
      P[K + 1][r] = G.xe[r];
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        R v = G.A[i][r][0] * t[L::idx(i, 0)];
        if (L::plane(i)) v = fma(G.A[i][r][1], t[L::idx(i, 1)], v);
        P[i + 1][r] = v + G.b[i][r];
      }
    }
  }

  // Embed, segments, norms, clamped gradient into `gout` (batching.py:95-104).
  __device__ __forceinline__ void eval(const Geo<R, K>& G, R (&gout)[NA]) {
    R P[K + 2][3];
    points(G, P);
    R u[S][3];
#pragma unroll
    for (int k = 0; k < S; ++k) {
#pragma unroll
      for (int r = 0; r < 3; ++r) s[k][r] = P[k + 1][r] - P[k][r];
      R q = s[k][0] * s[k][0];
      q = fma(s[k][1], s[k][1], q);
      q = fma(s[k][2], s[k][2], q);
      R nc;
      norm_rcp(q, G.eps, G.reps, nu[k], nc, rn[k]);
#pragma unroll
      for (int r = 0; r < 3; ++r) u[k][r] = s[k][r] * rn[k];
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const R q0 = u[i][0] - u[i + 1][0];
      const R q1 = u[i][1] - u[i + 1][1];
      const R q2 = u[i][2] - u[i + 1][2];
      gout[L::idx(i, 0)] = fma(G.A[i][2][0], q2, fma(G.A[i][1][0], q1, G.A[i][0][0] * q0));
      if (L::plane(i))
        gout[L::idx(i, 1)] = fma(G.A[i][2][1], q2, fma(G.A[i][1][1], q1, G.A[i][0][1] * q0));
    }
  }

  // Fixed-point step size along p (solver.py:84-112). Returns alpha; sets
  // `zero` when the direction moves no interaction point. The first fixed-
  // point iterate starts at alpha = 0, where the trial segments are exactly
  // the current ones, so it reuses their clamped norms.
  __device__ __forceinline__ R step_size(const Geo<R, K>& G, const R (&p)[NA], int fp_iters,
                                         bool& zero) const {
    R w[K][3];
#pragma unroll
    for (int i = 0; i < K; ++i) {
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        R v = G.A[i][r][0] * p[L::idx(i, 0)];
        if (L::plane(i)) v = fma(G.A[i][r][1], p[L::idx(i, 1)], v);
        w[i][r] = v;
      }
    }
    R d[S][3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      d[0][r] = w[0][r];
      d[K][r] = -w[K - 1][r];
    }
#pragma unroll
    for (int k = 1; k < K; ++k) {
#pragma unroll
      for (int r = 0; r < 3; ++r) d[k][r] = w[k][r] - w[k - 1][r];
    }
    R a2[S], c[S];
    R total;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      a2[k] = fma(d[k][2], d[k][2], fma(d[k][1], d[k][1], d[k][0] * d[k][0]));
      c[k] = fma(d[k][2], s[k][2], fma(d[k][1], s[k][1], d[k][0] * s[k][0]));
      total = k == 0 ? a2[0] : total + a2[k];
    }
    zero = total <= Num<R>::tiny();
    R alpha = R(0);
    {
      R num = c[0] * rn[0], den = a2[0] * rn[0];
#pragma unroll
      for (int k = 1; k < S; ++k) {
        num = fma(c[k], rn[k], num);
        den = fma(a2[k], rn[k], den);
      }
      const R cand = -div_fast(num, zero ? R(1) : den);
      alpha = (zero || !finite(cand)) ? alpha : cand;
    }
    for (int f = 1; f < fp_iters; ++f) {
      R num = R(0), den = R(0);
#pragma unroll
      for (int k = 0; k < S; ++k) {
        const R e0 = fma(alpha, d[k][0], s[k][0]);
        const R e1 = fma(alpha, d[k][1], s[k][1]);
        const R e2 = fma(alpha, d[k][2], s[k][2]);
        R n0, n, ri;
        norm_rcp(fma(e2, e2, fma(e1, e1, e0 * e0)), G.eps, G.reps, n0, n, ri);
        num = k == 0 ? c[0] * ri : fma(c[k], ri, num);
        den = k == 0 ? a2[0] * ri : fma(a2[k], ri, den);
      }
      const R cand = -div_fast(num, zero ? R(1) : den);
      alpha = (zero || !finite(cand)) ? alpha : cand;
    }
    return alpha;
  }
};

// Dot product over the active unknowns as two FMA chains, one per basis
// column c (half the dependent latency of one chain). Grouping by column, not
// by compressed position, keeps the kind-specialised kernels bit-identical to
// the dense one: an edge's inert term only adds an exact zero to chain 1.
template <typename R, int K, unsigned MASK, int NA>
__device__ __forceinline__ R dot(const R (&a)[NA], const R (&b)[NA]) {
  using L = Lay<K, MASK>;
  R c0 = a[L::idx(0, 0)] * b[L::idx(0, 0)];
#pragma unroll
  for (int i = 1; i < K; ++i) c0 = fma(a[L::idx(i, 0)], b[L::idx(i, 0)], c0);
  bool any = false;
  R c1 = R(0);
#pragma unroll
  for (int i = 0; i < K; ++i) {
    if (!L::plane(i)) continue;
    c1 = any ? fma(a[L::idx(i, 1)], b[L::idx(i, 1)], c1) : a[L::idx(i, 1)] * b[L::idx(i, 1)];
    any = true;
  }
  return any ? c0 + c1 : c0;
}

// Packed symmetric inverse-Hessian approximation with the BFGS update.
//
// The reference update (solver.py:180-199)
//   H' = H - rho (s Hy^T + Hy s^T) + (rho^2 yHy + rho) s s^T
// is applied in the equivalent symmetric two-term form H' = H + s z^T + z s^T
// with z = -rho Hy + (rho^2 yHy + rho)/2 s (two FMAs per packed entry), and
// the next direction -H' g_new is obtained from H g_new by the same rank-two
// formula, so each iteration needs one matrix-vector product: H y follows
// from H g_new + p (p = -H g_old).
template <typename R, int K, unsigned MASK>
struct InvHess {
  using L = Lay<K, MASK>;
  static constexpr int NA = L::NA;
  static constexpr int NH = NA * (NA + 1) / 2;
  R h[NH];
  R bound;  // upper bound on max |h_ij| (for the overflow pre-check)

  __device__ static constexpr int id(int i, int j) {
    return i <= j ? i * NA - i * (i - 1) / 2 + (j - i) : j * NA - j * (j - 1) / 2 + (i - j);
  }
  __device__ __forceinline__ void identity() {
#pragma unroll
    for (int i = 0; i < NA; ++i)
#pragma unroll
      for (int j = i; j < NA; ++j) h[id(i, j)] = i == j ? R(1) : R(0);
    bound = R(1);
  }
  // out = H v, each row as the column-grouped two-chain dot product.
  __device__ __forceinline__ void mul(const R (&v)[NA], R (&out)[NA]) const {
#pragma unroll
    for (int r = 0; r < NA; ++r) {
      R c0 = h[id(r, L::idx(0, 0))] * v[L::idx(0, 0)];
#pragma unroll
      for (int i = 1; i < K; ++i) c0 = fma(h[id(r, L::idx(i, 0))], v[L::idx(i, 0)], c0);
      bool any = false;
      R c1 = R(0);
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (!L::plane(i)) continue;
        const int j = L::idx(i, 1);
        c1 = any ? fma(h[id(r, j)], v[j], c1) : h[id(r, j)] * v[j];
        any = true;
      }
      out[r] = any ? c0 + c1 : c0;
    }
  }
  // One BFGS step. In: step sg, gradient change y, new gradient gn, old
  // direction p (= -H g_old), curvature flag ok and sy = sg.y. Out: p =
  // -H' gn with H' the updated matrix (or the old one when the update is
  // skipped: failed curvature test or a non-finite H', solver.py:184,198).
  __device__ __forceinline__ void step(const R (&sg)[NA], const R (&y)[NA], const R (&gn)[NA],
                                       R (&p)[NA], bool ok, R sy) {
    R Hg[NA];
    mul(gn, Hg);
    if (ok) {
      R Hy[NA];
#pragma unroll
      for (int i = 0; i < NA; ++i) Hy[i] = Hg[i] + p[i];
      const R rho = rcp_fast(sy);
      const R yHy = dot<R, K, MASK, NA>(y, Hy);
      const R half = R(0.5) * fma(rho * rho, yHy, rho);
      R z[NA];
      R ss = R(0), sz = R(0);
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        z[i] = fma(half, sg[i], -(rho * Hy[i]));
        ss += fabs(sg[i]);
        sz += fabs(z[i]);
      }
      // |H'_ij| <= bound + 2 sum|s| sum|z|; NaN/inf propagate into nb.
      const R nb = fma(R(2) * ss, sz, bound) * R(1.0009765625);
      bool take = true;
      if (!(nb < R(1e36))) {
        // Rare: possible overflow. Check every entry before committing.
        R mx = R(0);
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
          for (int j = i; j < NA; ++j) {
            const R v = fma(z[i], sg[j], fma(sg[i], z[j], h[id(i, j)]));
            take = take && finite(v);
            mx = fabs(v) > mx ? fabs(v) : mx;
          }
        if (take) bound = mx * R(1.0009765625);
      } else {
        bound = nb;
      }
      if (take) {
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
          for (int j = i; j < NA; ++j) h[id(i, j)] = fma(z[i], sg[j], fma(sg[i], z[j], h[id(i, j)]));
        const R zg = dot<R, K, MASK, NA>(z, gn), sgn = dot<R, K, MASK, NA>(sg, gn);
#pragma unroll
        for (int i = 0; i < NA; ++i) p[i] = -fma(sg[i], zg, fma(z[i], sgn, Hg[i]));
        return;
      }
    }
#pragma unroll
    for (int i = 0; i < NA; ++i) p[i] = -Hg[i];
  }
};

// Stationarity gate |g| < 1e-5 (1 + L) (implicit_diff.py:25,30-36).
template <typename R, int NA>
__device__ __forceinline__ bool stationary(const R (&g)[NA], R len) {
  R q = R(0);
#pragma unroll
  for (int i = 0; i < NA; ++i) q = fma(g[i], g[i], q);
  return Num<R>::sqrt_(q) < R(1e-5) * (R(1) + len);
}


// The fixed-iteration BFGS loop (solver.py:146-215) from the state P (which
// must hold t and its evaluation). Returns DEGENERATE_ENTRY / ZERO_DIRECTION
// status bits; optional per-iteration trace (solver.py:202-206) and final
// inverse Hessian (return_state) in the dense 2K layout.
template <typename R, int K, unsigned MASK>
__device__ __forceinline__ uint8_t bfgs_solve(const Geo<R, K>& G, PathState<R, K, MASK>& P,
                                              int iterations, int fp_iters, R* trace_len,
                                              R* trace_gnorm, int64_t trace_ld, int64_t row,
                                              R* H_out) {
  using L = Lay<K, MASK>;
  constexpr int NA = L::NA;
  uint8_t st = 0;
  if (P.min_norm() <= G.eps) st |= FP_STATUS_DEGENERATE_ENTRY;  // checked_segments (solver.py:166)
  InvHess<R, K, MASK> H;
  H.identity();
  R p[NA];
#pragma unroll
  for (int j = 0; j < NA; ++j) p[j] = -P.g[j];  // H = I
  for (int it = 0; it < iterations; ++it) {
    bool zero;
    const R alpha = P.step_size(G, p, fp_iters, zero);
    if (zero) st |= FP_STATUS_ZERO_DIRECTION;
    R sg[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      sg[j] = alpha * p[j];
      P.t[j] = P.t[j] + sg[j];
    }
    R gn[NA];
    P.eval(G, gn);
    R y[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) y[j] = gn[j] - P.g[j];
    const R sy = dot<R, K, MASK, NA>(sg, y);
    const R ss = dot<R, K, MASK, NA>(sg, sg);
    const R yy = dot<R, K, MASK, NA>(y, y);
    const bool ok = sy > (R(1e-12) * sqrt_test(ss)) * sqrt_test(yy);
    H.step(sg, y, gn, p, ok, sy);
#pragma unroll
    for (int j = 0; j < NA; ++j) P.g[j] = gn[j];
    if (trace_len != nullptr) {
      R q = R(0);
#pragma unroll
      for (int j = 0; j < NA; ++j) q = fma(P.g[j], P.g[j], q);
      trace_len[int64_t(it) * trace_ld + row] = P.length();
      trace_gnorm[int64_t(it) * trace_ld + row] = Num<R>::sqrt_(q);
    }
  }
  if (H_out != nullptr) {
    R* Ho = H_out + row * (4 * K * K);
#pragma unroll
    for (int i = 0; i < 2 * K; ++i)
#pragma unroll
      for (int j = 0; j < 2 * K; ++j) {
        const int ii = i >> 1, ci = i & 1, jj = j >> 1, cj = j & 1;
        const bool ai = ci == 0 || L::plane(ii), aj = cj == 0 || L::plane(jj);
        R v = (i == j) ? R(1) : R(0);
        if (ai && aj) v = H.h[InvHess<R, K, MASK>::id(L::idx(ii, ci), L::idx(jj, cj))];
        Ho[i * 2 * K + j] = v;
      }
  }
  return st;
}

// Classification at the returned T: stationarity gate, degenerate or short
// segments, non-finite state.
template <typename R, int K, unsigned MASK>
__device__ __forceinline__ uint8_t final_status(const Geo<R, K>& G, const PathState<R, K, MASK>& P) {
  constexpr int NA = Lay<K, MASK>::NA;
  uint8_t st = 0;
  const R len = P.length(), nmin = P.min_norm();
  if (!stationary<R, NA>(P.g, len)) st |= FP_STATUS_NOT_STATIONARY;
  if (nmin <= G.eps) st |= FP_STATUS_DEGENERATE_FINAL;
  if (nmin < R(1e-3)) st |= FP_STATUS_SHORT_SEGMENT;
  bool fin = finite(len);
#pragma unroll
  for (int j = 0; j < NA; ++j) fin = fin && finite(P.t[j]) && finite(P.g[j]);
  if (!fin) st |= FP_STATUS_NONFINITE;
  return st;
}

// ---------------------------------------------------------------------------
// Implicit-gradient VJP at the current state (objective.py:48-135,
// implicit_diff.py:39-77). `vT` is the cotangent on T in the compressed
// layout (may be all zero), `wl` the weight on L. With `full`, the rhs of the
// stationarity system includes wl * g (the chain-rule correction).
template <typename R, int K>
struct SceneGrad {
  R db[K][3][2];
  R da[K][3];
  R d0[3], d1[3];
  R u[K][2];  // solve_stationary_system solution (full 2K layout, inert 0)
};

template <typename R, int K, unsigned MASK>
__device__ __forceinline__ uint8_t implicit_vjp(const Geo<R, K>& G, const PathState<R, K, MASK>& P,
                                                const R (&tf)[K][2], const R (&vf)[K][2], R wl,
                                                bool full, bool need_solve, bool mixed,
                                                SceneGrad<R, K>& out) {
  using L = Lay<K, MASK>;
  constexpr int S = L::S;
  uint8_t st = 0;
  // Active flags: a coordinate is active when its basis column is nonzero
  // (geometry.py:74-77).
  bool act[K][2];
#pragma unroll
  for (int i = 0; i < K; ++i) {
#pragma unroll
    for (int c = 0; c < 2; ++c)
      act[i][c] = (G.A[i][0][c] != R(0)) || (G.A[i][1][c] != R(0)) || (G.A[i][2][c] != R(0));
  }
  R u[S][3];
#pragma unroll
  for (int k = 0; k < S; ++k)
#pragma unroll
    for (int r = 0; r < 3; ++r) u[k][r] = P.s[k][r] * P.rn[k];
  R q[K][3];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int r = 0; r < 3; ++r) q[i][r] = u[i][r] - u[i + 1][r];

  // `mixed`: use vf itself as the direction u (objective.param_vjp,
  // objective.py:101-135) — no stationarity solve.
  R sol[K][2];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    sol[i][0] = mixed ? vf[i][0] : R(0);
    sol[i][1] = mixed ? vf[i][1] : R(0);
  }

  if (need_solve) {
    // Hessian blocks: A_i^T M_k A_j = (G_ij - (A_i^T u_k)(A_j^T u_k)^T) / n_k.
    R D[K][3];      // symmetric 2x2: (00, 01, 11)
    R O[K][2][2];   // O_i couples interaction i and i+1
    R au_in[K][2], au_out[K][2];  // A_i^T u_i, A_i^T u_{i+1}
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        au_in[i][c] = fma(G.A[i][2][c], u[i][2], fma(G.A[i][1][c], u[i][1], G.A[i][0][c] * u[i][0]));
        au_out[i][c] =
            fma(G.A[i][2][c], u[i + 1][2], fma(G.A[i][1][c], u[i + 1][1], G.A[i][0][c] * u[i + 1][0]));
      }
    R rhs[K][2];
    R trace = R(0);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      R gii[3];
      gii[0] = fma(G.A[i][2][0], G.A[i][2][0], fma(G.A[i][1][0], G.A[i][1][0], G.A[i][0][0] * G.A[i][0][0]));
      gii[1] = fma(G.A[i][2][0], G.A[i][2][1], fma(G.A[i][1][0], G.A[i][1][1], G.A[i][0][0] * G.A[i][0][1]));
      gii[2] = fma(G.A[i][2][1], G.A[i][2][1], fma(G.A[i][1][1], G.A[i][1][1], G.A[i][0][1] * G.A[i][0][1]));
      const R ri = P.rn[i], ro = P.rn[i + 1];
      D[i][0] = (gii[0] - au_in[i][0] * au_in[i][0]) * ri + (gii[0] - au_out[i][0] * au_out[i][0]) * ro;
      D[i][1] = (gii[1] - au_in[i][0] * au_in[i][1]) * ri + (gii[1] - au_out[i][0] * au_out[i][1]) * ro;
      D[i][2] = (gii[2] - au_in[i][1] * au_in[i][1]) * ri + (gii[2] - au_out[i][1] * au_out[i][1]) * ro;
      if (i + 1 < K) {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const R gij = fma(G.A[i][2][a], G.A[i + 1][2][b],
                              fma(G.A[i][1][a], G.A[i + 1][1][b], G.A[i][0][a] * G.A[i + 1][0][b]));
            O[i][a][b] = -(gij - au_out[i][a] * au_in[i + 1][b]) * ro;
          }
      }
      // rhs = -(wl g + vT) on active coordinates, 0 on inert ones
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const R gc = (c == 0 || L::plane(i)) ? P.g[L::idx(i, c)] : R(0);
        const R vc = vf[i][c];
        const R v = full ? fma(wl, gc, vc) : vc;
        rhs[i][c] = act[i][c] ? -v : R(0);
      }
      if (act[i][0]) trace += D[i][0];
      if (act[i][1]) trace += D[i][2];
      // pin inert coordinates: their rows/columns are exactly zero
      if (!act[i][0]) { D[i][0] = R(1); D[i][1] = R(0); }
      if (!act[i][1]) { D[i][2] = R(1); D[i][1] = R(0); }
    }
    // Block Thomas elimination, with a Tikhonov retry (implicit_diff.py:64-71).
    bool solved = false;
    for (int attempt = 0; attempt < 2 && !solved; ++attempt) {
      const R lam = attempt == 0 ? R(0) : R(1e-12) * trace;
      R Ci[K][3];  // inverse pivot blocks
      R z[K][2];
      bool ok = true;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        R C0 = D[i][0] + (act[i][0] ? lam : R(0));
        R C1 = D[i][1];
        R C2 = D[i][2] + (act[i][1] ? lam : R(0));
        R z0 = rhs[i][0], z1 = rhs[i][1];
        if (i > 0) {
          // Lm = O_{i-1}^T Cinv_{i-1}; C -= Lm O_{i-1}; z -= Lm z_{i-1}
          R Lm[2][2];
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            Lm[a][0] = O[i - 1][0][a] * Ci[i - 1][0] + O[i - 1][1][a] * Ci[i - 1][1];
            Lm[a][1] = O[i - 1][0][a] * Ci[i - 1][1] + O[i - 1][1][a] * Ci[i - 1][2];
          }
          C0 -= Lm[0][0] * O[i - 1][0][0] + Lm[0][1] * O[i - 1][1][0];
          C1 -= Lm[0][0] * O[i - 1][0][1] + Lm[0][1] * O[i - 1][1][1];
          C2 -= Lm[1][0] * O[i - 1][0][1] + Lm[1][1] * O[i - 1][1][1];
          z0 -= Lm[0][0] * z[i - 1][0] + Lm[0][1] * z[i - 1][1];
          z1 -= Lm[1][0] * z[i - 1][0] + Lm[1][1] * z[i - 1][1];
        }
        const R det = C0 * C2 - C1 * C1;
        ok = ok && (det > R(0)) && finite(det);
        const R id = rcp_fast(det);
        Ci[i][0] = C2 * id;
        Ci[i][1] = -C1 * id;
        Ci[i][2] = C0 * id;
        z[i][0] = z0;
        z[i][1] = z1;
      }
      if (!ok) continue;
      // back substitution
      R nxt0 = R(0), nxt1 = R(0);
#pragma unroll
      for (int i = K - 1; i >= 0; --i) {
        R r0 = z[i][0], r1 = z[i][1];
        if (i + 1 < K) {
          r0 -= O[i][0][0] * nxt0 + O[i][0][1] * nxt1;
          r1 -= O[i][1][0] * nxt0 + O[i][1][1] * nxt1;
        }
        const R v0 = Ci[i][0] * r0 + Ci[i][1] * r1;
        const R v1 = Ci[i][1] * r0 + Ci[i][2] * r1;
        sol[i][0] = act[i][0] ? v0 : R(0);
        sol[i][1] = act[i][1] ? v1 : R(0);
        nxt0 = sol[i][0];
        nxt1 = sol[i][1];
        ok = ok && finite(v0) && finite(v1);
      }
      solved = ok;
    }
    if (!solved) {
      st |= FP_STATUS_SINGULAR;
#pragma unroll
      for (int i = 0; i < K; ++i) sol[i][0] = sol[i][1] = R(0);
    }
  }

  // param_vjp with the solution (objective.py:101-135) + wl * length partials
  // (objective.py:89-98).
  R dx[K][3];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int r = 0; r < 3; ++r) dx[i][r] = fma(G.A[i][r][1], sol[i][1], G.A[i][r][0] * sol[i][0]);
  R w[S][3];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    R ds[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const R hi = k < K ? dx[k][r] : R(0);
      const R lo = k > 0 ? dx[k - 1][r] : R(0);
      ds[r] = hi - lo;
    }
    const R ud = fma(u[k][2], ds[2], fma(u[k][1], ds[1], u[k][0] * ds[0]));
#pragma unroll
    for (int r = 0; r < 3; ++r) w[k][r] = (ds[r] - u[k][r] * ud) * P.rn[k];
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const R zi = w[i][r] - w[i + 1][r];
      const R e = fma(wl, q[i][r], zi);
      out.da[i][r] = e;
      out.db[i][r][0] = fma(e, tf[i][0], q[i][r] * sol[i][0]);
      out.db[i][r][1] = fma(e, tf[i][1], q[i][r] * sol[i][1]);
    }
    out.u[i][0] = sol[i][0];
    out.u[i][1] = sol[i][1];
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    out.d0[r] = -fma(wl, u[0][r], w[0][r]);
    out.d1[r] = fma(wl, u[K][r], w[K][r]);
  }
  return st;
}

}  // namespace fp
