// Per-path register-resident Fermat path state and math (sm_100a).
//
// One thread owns one path. The unknowns live in a compressed vector of the
// active coordinates of the kind mask MASK (bit i set: interaction i is a
// plane with two unknowns; clear: an edge with one). MASK = all ones is the
// "dense" uniform 2K formulation of the reference (geometry.py:86-90): edges
// carry a zero second basis column, which produces exact zeros, so it is
// valid for every batch; specialised masks skip the inert lanes.
//
// Paired arithmetic: the loop is issue-bound (ncu: warps eligible but not
// selected, FMA pipe ~50%), so the state is laid out for the sm_100 paired
// FP32 instructions FFMA2 / FMUL2 / FADD2 (two IEEE operations per issue,
// a scalar operand broadcast and negations for free):
//   * 3-vectors as an (x, y) pair plus a scalar z; the basis A_i as column
//     pairs {A_0c, A_1c} plus A_2c, so A t, A p and points are paired;
//   * vectors over the NA unknowns as NA/2 pairs (odd NA: the last hi lane
//     is padding and never read);
//   * the inverse Hessian as row pairs {h(2m, c), h(2m+1, c)} of its upper
//     triangle (c >= 2m), so the rank-two update and H v are paired.
// Each lane rounds exactly like the scalar operation it replaces. fp64 runs
// the same code with the pair operations emulated by two scalar ones.
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

// ---- paired arithmetic -------------------------------------------------------
template <typename R> struct PairOf;
template <> struct PairOf<float> { using T = float2; };
template <> struct PairOf<double> { using T = double2; };
template <typename R> using V2 = typename PairOf<R>::T;

__device__ __forceinline__ float2 mk2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 mk2(double a, double b) { return make_double2(a, b); }
template <typename R>
__device__ __forceinline__ V2<R> bc2(R a) { return mk2(a, a); }

__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
// Products are FFMA2 with a -0 addend that ptxas cannot see (`nz`, a kernel
// argument): ptxas contracts FMUL2 + FADD2 into FFMA2 even under -fmad=false,
// which would round differently in different kernels. a * b + (-0) == a * b
// exactly, so each lane still rounds like the scalar product.
__device__ __forceinline__ float2 mulz(float2 a, float2 b, float nz) {
  return __ffma2_rn(a, b, make_float2(nz, nz));
}
// Plain FMUL2, only where the product feeds an FFMA2 addend (nothing to contract).
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, neg2(b)); }

__device__ __forceinline__ double2 fma2(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
}
__device__ __forceinline__ double2 mulz(double2 a, double2 b, double) {
  return make_double2(a.x * b.x, a.y * b.y);
}
__device__ __forceinline__ double2 mul2(double2 a, double2 b) { return make_double2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 neg2(double2 a) { return make_double2(-a.x, -a.y); }
__device__ __forceinline__ double2 sub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// Pair ops on the last pair of an odd-length vector (`lo` true: its high lane
// is padding, never read): one scalar op on the low lane instead of the
// pair — half the FMA-pipe cycles, identical low-lane rounding; the high
// lane of the result is left undefined. `lo` is a compile-time constant
// after unrolling.
__device__ __forceinline__ float2 lo_only(float x) {
  float2 r;
  r.x = x;
  return r;
}
__device__ __forceinline__ double2 lo_only(double x) {
  double2 r;
  r.x = x;
  return r;
}
// (`lo` must be a genuine bool: an array or pointer would convert silently)
template <typename B, typename P>
__device__ __forceinline__ P fma2p(B lo, P a, P b, P c) {
  static_assert(std::is_same<B, bool>::value, "lo must be a bool");
  return lo ? lo_only(fma(a.x, b.x, c.x)) : fma2(a, b, c);
}
template <typename B, typename P>
__device__ __forceinline__ P mul2p(B lo, P a, P b) {
  static_assert(std::is_same<B, bool>::value, "lo must be a bool");
  return lo ? lo_only(a.x * b.x) : mul2(a, b);
}
template <typename B, typename P, typename R>
__device__ __forceinline__ P mulzp(B lo, P a, P b, R nz) {
  static_assert(std::is_same<B, bool>::value, "lo must be a bool");
  return lo ? lo_only(a.x * b.x) : mulz(a, b, nz);
}
template <typename B, typename P>
__device__ __forceinline__ P add2p(B lo, P a, P b) {
  static_assert(std::is_same<B, bool>::value, "lo must be a bool");
  return lo ? lo_only(a.x + b.x) : add2(a, b);
}
template <typename B, typename P>
__device__ __forceinline__ P sub2p(B lo, P a, P b) {
  static_assert(std::is_same<B, bool>::value, "lo must be a bool");
  return lo ? lo_only(a.x - b.x) : sub2(a, b);
}
template <typename B, typename P>
__device__ __forceinline__ P neg2p(B lo, P a) {
  static_assert(std::is_same<B, bool>::value, "lo must be a bool");
  return lo ? lo_only(-a.x) : neg2(a);
}

// Lane access by value / by store (never a reference picked by a condition:
// a selected pointer into the pair defeats scalar replacement and sends the
// whole state to local memory in the large tile kernels).
template <typename P>
__device__ __forceinline__ auto lane(const P& p, int h) { return h ? p.y : p.x; }
template <typename P, typename V>
__device__ __forceinline__ void set_lane(P& p, int h, V v) {
  if (h)
    p.y = v;
  else
    p.x = v;
}

// Vectors over the NA unknowns: NP pairs, element j in lane j & 1 of pair j >> 1.
template <int NA>
struct Packed {
  static constexpr int NP = (NA + 1) / 2;  // pairs
  static constexpr int NF = NA / 2;        // full pairs (no padding lane)
};
#define FP_EL(v, j) lane((v)[(j) >> 1], (j) & 1)
#define FP_SET(v, j, x) set_lane((v)[(j) >> 1], (j) & 1, (x))

// v . w over the NA real elements: lane-wise pair chains, then the two lanes
// (and the unpaired last element of an odd NA).
template <typename R, int NA>
__device__ __forceinline__ R dotv(const V2<R> (&a)[Packed<NA>::NP], const V2<R> (&b)[Packed<NA>::NP], R nz) {
  constexpr int NF = Packed<NA>::NF;
  R r;
  if constexpr (NF > 0) {
    V2<R> acc = NF > 1 ? mul2(a[0], b[0]) : mulz(a[0], b[0], nz);
#pragma unroll
    for (int m = 1; m < NF; ++m) acc = fma2(a[m], b[m], acc);
    r = acc.x + acc.y;
    if constexpr (NA & 1) r = fma(a[NF].x, b[NF].x, r);
  } else {
    r = a[0].x * b[0].x;
  }
  return r;
}

// max_j |v_j| over the real elements, NaN-propagating (ALU pipe).
template <typename R, int NA>
__device__ __forceinline__ R absmaxv(const V2<R> (&a)[Packed<NA>::NP]) {
  R m = fabs(a[0].x);
#pragma unroll
  for (int j = 1; j < NA; ++j) m = absmax_nan(m, FP_EL(a, j));
  return m;
}

// ---- geometry ----------------------------------------------------------------
template <typename R, int K>
struct Geo {
  V2<R> Axy[K][2];  // basis column c of interaction i, rows x and y
  R Az[K][2];       // basis column c, row z
  V2<R> bxy[K];     // anchor rows x, y
  R bz[K];
  V2<R> x0xy, xexy;  // start / end
  R x0z, xez;
  R nz;    // -0, opaque to ptxas (see mulz); kernels set it from their argument
  R eps;   // 1e-12 (1 + |end - start|), fp64 then cast (batching.py:67-72)
  R reps;  // 1 / eps
  __device__ __forceinline__ R A(int i, int r, int c) const {
    return r == 0 ? Axy[i][c].x : (r == 1 ? Axy[i][c].y : Az[i][c]);
  }
  __device__ __forceinline__ R b(int i, int r) const {
    return r == 0 ? bxy[i].x : (r == 1 ? bxy[i].y : bz[i]);
  }
  __device__ __forceinline__ R x0(int r) const { return r == 0 ? x0xy.x : (r == 1 ? x0xy.y : x0z); }
  __device__ __forceinline__ R xe(int r) const { return r == 0 ? xexy.x : (r == 1 ? xexy.y : xez); }
};

// Load one path's geometry from a record in the reference layout.
template <typename R, int K, unsigned MASK>
__device__ __forceinline__ void load_geo(Geo<R, K>& G, const R* basis, const R* anchor,
                                         const R* start, const R* end) {
  using L = Lay<K, MASK>;
#pragma unroll
  for (int i = 0; i < K; ++i) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const bool live = c == 0 || L::plane(i);
      G.Axy[i][c] = mk2(live ? basis[i * 6 + c] : R(0), live ? basis[i * 6 + 2 + c] : R(0));
      G.Az[i][c] = live ? basis[i * 6 + 4 + c] : R(0);
    }
    G.bxy[i] = mk2(anchor[i * 3 + 0], anchor[i * 3 + 1]);
    G.bz[i] = anchor[i * 3 + 2];
  }
  G.x0xy = mk2(start[0], start[1]);
  G.x0z = start[2];
  G.xexy = mk2(end[0], end[1]);
  G.xez = end[2];
  const double dx = double(end[0]) - double(start[0]);
  const double dy = double(end[1]) - double(start[1]);
  const double dz = double(end[2]) - double(start[2]);
  const double nrm = __dsqrt_rn(__fma_rn(dz, dz, __fma_rn(dy, dy, dx * dx)));
  G.eps = R(1e-12 * (1.0 + nrm));
  G.reps = Num<R>::rcp(G.eps);
  G.nz = R(-0.0);
}

// A_i v_i as (xy pair, z) for the unknowns (v0, v1) of interaction i.
template <typename R, int K, bool PLANE>
__device__ __forceinline__ void apply_A(const Geo<R, K>& G, int i, R v0, R v1, V2<R>& xy, R& z) {
  xy = PLANE ? mul2(G.Axy[i][0], bc2(v0)) : mulz(G.Axy[i][0], bc2(v0), G.nz);
  z = G.Az[i][0] * v0;
  if (PLANE) {
    xy = fma2(G.Axy[i][1], bc2(v1), xy);
    z = fma(G.Az[i][1], v1, z);
  }
}

// ---- per-path state -------------------------------------------------------------
template <typename R, int K, unsigned MASK>
struct PathState {
  using L = Lay<K, MASK>;
  static constexpr int S = L::S;
  static constexpr int NA = L::NA;
  static constexpr int NP = Packed<NA>::NP;

  V2<R> t[NP];    // active unknowns
  V2<R> g[NP];    // clamped-norm gradient at t
  V2<R> sxy[S];   // segments at t (x, y)
  R sz[S];        //                (z)
  static constexpr int SP = (S + 1) / 2;
  V2<R> rnp[SP];  // 1 / max(|s_k|, eps), segment pairs (k in lane k & 1 of pair k >> 1)
  R nu[S];        // |s_k| (unclamped; valid after eval<false> / finish_norms)

  __device__ __forceinline__ R T(int j) const { return FP_EL(t, j); }
  __device__ __forceinline__ void setT(int j, R v) { FP_SET(t, j, v); }
  __device__ __forceinline__ R Gr(int j) const { return FP_EL(g, j); }
  __device__ __forceinline__ R RN(int k) const { return FP_EL(rnp, k); }
  __device__ __forceinline__ R S3(int k, int r) const {
    return r == 0 ? sxy[k].x : (r == 1 ? sxy[k].y : sz[k]);
  }
  __device__ __forceinline__ void zero_t() {
#pragma unroll
    for (int m = 0; m < NP; ++m) t[m] = mk2(R(0), R(0));
  }

  // Path length: sum of unclamped norms (batching.py:123-126).
  __device__ __forceinline__ R length() const {
    R l = nu[0];
#pragma unroll
    for (int k = 1; k < S; ++k) l += nu[k];
    return l;
  }
  // Shortest segment over the non-NaN norms (NaN only if all are): `m <= eps`
  // is the reference's np.any(norms <= eps) (batching.py:107-114).
  __device__ __forceinline__ R min_norm() const {
    R m = nu[0];
#pragma unroll
    for (int k = 1; k < S; ++k) m = (nu[k] < m || m != m) ? nu[k] : m;
    return m;
  }

  // x_i = A_i t_i + b_i (geometry.py:153-165); index 0 / K+1 are start / end.
  // The dense layout's inert term 0 * t_i1 adds an exact zero, so every
  // kernel embeds a path identically.
  __device__ __forceinline__ void points(const Geo<R, K>& G, V2<R> (&Pxy)[K + 2], R (&Pz)[K + 2]) const {
    Pxy[0] = G.x0xy;
    Pz[0] = G.x0z;
    Pxy[K + 1] = G.xexy;
    Pz[K + 1] = G.xez;
    static_for<K>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      // b_i + A_i0 t_i0 (+ A_i1 t_i1) as one explicit FMA chain
      const R t0 = T(L::idx(i, 0));
      Pxy[i + 1] = fma2(G.Axy[i][0], bc2(t0), G.bxy[i]);
      Pz[i + 1] = fma(G.Az[i][0], t0, G.bz[i]);
      if constexpr (L::plane(i)) {
        const R t1 = T(L::idx(i, 1));
        Pxy[i + 1] = fma2(G.Axy[i][1], bc2(t1), Pxy[i + 1]);
        Pz[i + 1] = fma(G.Az[i][1], t1, Pz[i + 1]);
      }
    });
  }

  // Points as plain 3-vectors (outputs).
  __device__ __forceinline__ void points(const Geo<R, K>& G, R (&X)[K + 2][3]) const {
    V2<R> Pxy[K + 2];
    R Pz[K + 2];
    points(G, Pxy, Pz);
#pragma unroll
    for (int i = 0; i < K + 2; ++i) {
      X[i][0] = Pxy[i].x;
      X[i][1] = Pxy[i].y;
      X[i][2] = Pz[i];
    }
  }

  // Embed, segments, norms, clamped gradient into `gout` (batching.py:95-104).
  // LIGHT (the BFGS loop): reciprocal clamped norms only; the unclamped norms
  // `nu` are left stale until finish_norms().
  template <bool LIGHT = false>
  __device__ __forceinline__ void eval(const Geo<R, K>& G, V2<R> (&gout)[NP]) {
    V2<R> Pxy[K + 2];
    R Pz[K + 2];
    points(G, Pxy, Pz);
    V2<R> uxy[S];
    R uz[S];
    V2<R> qp[SP];  // squared norms, segment pairs
#pragma unroll
    for (int k = 0; k < S; ++k) {
      sxy[k] = sub2(Pxy[k + 1], Pxy[k]);
      sz[k] = Pz[k + 1] - Pz[k];
      R q = sxy[k].x * sxy[k].x;
      q = fma(sxy[k].y, sxy[k].y, q);
      FP_SET(qp, k, fma(sz[k], sz[k], q));
    }
    if (LIGHT) {
      // reciprocal clamped norms (MUFU.RSQ, fp_common.cuh rcp_norm)
      const R eps2 = G.eps * G.eps;
#pragma unroll
      for (int m = 0; m < S / 2; ++m) rcp_norm2(qp[m], G.eps, eps2, G.reps, rnp[m]);
      if constexpr (S & 1) {
        R r;
        rcp_norm(qp[SP - 1].x, G.eps, eps2, G.reps, r);
        rnp[SP - 1].x = r;  // high lane: padding, never read
      }
    } else {
#pragma unroll
      for (int k = 0; k < S; ++k) {
        R nc, r;
        norm_rcp(FP_EL(qp, k), G.eps, G.reps, nu[k], nc, r);
        FP_SET(rnp, k, r);
      }
    }
#pragma unroll
    for (int k = 0; k < S; ++k) {
      uxy[k] = mulz(sxy[k], bc2(RN(k)), G.nz);
      uz[k] = sz[k] * RN(k);
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const V2<R> qxy = sub2(uxy[i], uxy[i + 1]);
      const R qz = uz[i] - uz[i + 1];
      FP_SET(gout, L::idx(i, 0), fma(G.Az[i][0], qz, fma(G.Axy[i][0].y, qxy.y, G.Axy[i][0].x * qxy.x)));
      if (L::plane(i))
        FP_SET(gout, L::idx(i, 1), fma(G.Az[i][1], qz, fma(G.Axy[i][1].y, qxy.y, G.Axy[i][1].x * qxy.x)));
    }
  }

  // Evaluation at T* for the VJP-only op: the loop's reciprocal norms and
  // gradient (eval<true>), then the unclamped norms — the state a solve
  // ends in, so the fused step, solve-then-VJP and VJP-only agree bit for
  // bit.
  __device__ __forceinline__ void eval_entry(const Geo<R, K>& G) {
    eval<true>(G, g);
    finish_norms(G);
  }

  // Unclamped norms of the current segments (bitwise those eval<false> gives).
  __device__ __forceinline__ void finish_norms(const Geo<R, K>& G) {
#pragma unroll
    for (int k = 0; k < S; ++k) {
      R q = sxy[k].x * sxy[k].x;
      q = fma(sxy[k].y, sxy[k].y, q);
      q = fma(sz[k], sz[k], q);
      R nc, r;
      norm_rcp(q, G.eps, G.reps, nu[k], nc, r);
    }
  }

  // Fixed-point step size along p (solver.py:84-112). Returns alpha; sets
  // `zero` when the direction moves no interaction point. The first fixed-
  // point iterate starts at alpha = 0, where the trial segments are exactly
  // the current ones, so it reuses their clamped norms.
  __device__ __forceinline__ R step_size(const Geo<R, K>& G, const V2<R> (&p)[NP], int fp_iters,
                                         bool& zero) const {
    V2<R> wxy[K];
    R wz[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (L::plane(i))
        apply_A<R, K, true>(G, i, FP_EL(p, L::idx(i, 0)), FP_EL(p, L::idx(i, 1)), wxy[i], wz[i]);
      else
        apply_A<R, K, false>(G, i, FP_EL(p, L::idx(i, 0)), R(0), wxy[i], wz[i]);
    }
    V2<R> dxy[S];
    R dz[S];
    dxy[0] = wxy[0];
    dz[0] = wz[0];
    dxy[K] = neg2(wxy[K - 1]);
    dz[K] = -wz[K - 1];
#pragma unroll
    for (int k = 1; k < K; ++k) {
      dxy[k] = sub2(wxy[k], wxy[k - 1]);
      dz[k] = wz[k] - wz[k - 1];
    }
    V2<R> ca[S];  // {c_k, a2_k}
    R total;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const R a2 = fma(dz[k], dz[k], fma(dxy[k].y, dxy[k].y, dxy[k].x * dxy[k].x));
      const R cc = fma(dz[k], sz[k], fma(dxy[k].y, sxy[k].y, dxy[k].x * sxy[k].x));
      ca[k] = mk2(cc, a2);
      total = k == 0 ? a2 : total + a2;
    }
    zero = total <= Num<R>::tiny();
    R alpha = R(0);
    {
      // {num, den} = sum_k {c_k, a2_k} / max(|s_k|, eps), one paired chain
      V2<R> nd = mul2(ca[0], bc2(RN(0)));
#pragma unroll
      for (int k = 1; k < S; ++k) nd = fma2(ca[k], bc2(RN(k)), nd);
      const R num = nd.x, den = nd.y;
      const R cand = -div_fast(num, zero ? R(1) : den);
      alpha = (zero || !finite(cand)) ? alpha : cand;
    }
    for (int f = 1; f < fp_iters; ++f) {
      R num = R(0), den = R(0);
#pragma unroll
      for (int k = 0; k < S; ++k) {
        const V2<R> exy = fma2(bc2(alpha), dxy[k], sxy[k]);
        const R e2 = fma(alpha, dz[k], sz[k]);
        R n0, n, ri;
        norm_rcp(fma(e2, e2, fma(exy.y, exy.y, exy.x * exy.x)), G.eps, G.reps, n0, n, ri);
        num = k == 0 ? ca[0].x * ri : fma(ca[k].x, ri, num);
        den = k == 0 ? ca[0].y * ri : fma(ca[k].y, ri, den);
      }
      const R cand = -div_fast(num, zero ? R(1) : den);
      alpha = (zero || !finite(cand)) ? alpha : cand;
    }
    return alpha;
  }
};

// Packed symmetric inverse-Hessian approximation with the BFGS update.
//
// Storage: row pairs. Pair (m, c), c >= 2m, holds {h(2m, c), h(2m+1, c)};
// the diagonal block's h(2m+1, 2m) duplicates h(2m, 2m+1) and is kept equal
// to it. Odd NA: the last pair's hi lane is a padding row (never read).
//
// The reference update (solver.py:180-199)
//   H' = H - rho (s Hy^T + Hy s^T) + (rho^2 yHy + rho) s s^T
// is applied in the equivalent symmetric two-term form H' = H + s z^T + z s^T
// with z = -rho Hy + (rho^2 yHy + rho)/2 s (two FFMA2 per stored pair), and
// the next direction -H' g_new is obtained from H g_new by the same rank-two
// formula, so each iteration needs one matrix-vector product: H y follows
// from H g_new + p (p = -H g_old).

template <typename R, int K, unsigned MASK>
struct InvHess {
  using L = Lay<K, MASK>;
  static constexpr int NA = L::NA;
  static constexpr int NP = Packed<NA>::NP;
  static constexpr int NHP = NP * NA - NP * (NP - 1);  // sum over m of (NA - 2m)
  V2<R> h[NHP];
  R bound;  // upper bound on max |h_ij| (for the overflow pre-check)

  __device__ static constexpr int off(int m) { return m * NA - m * (m - 1); }
  __device__ static constexpr int pid(int m, int c) { return off(m) + c - 2 * m; }
  // h(r, c) for any r, c (symmetric)
  __device__ __forceinline__ R get(int r, int c) const {
    return r <= c ? lane(h[pid(r >> 1, c)], r & 1) : lane(h[pid(c >> 1, r)], c & 1);
  }

  __device__ __forceinline__ void identity() {
#pragma unroll
    for (int m = 0; m < NP; ++m)
#pragma unroll
      for (int c = 2 * m; c < NA; ++c)
        h[pid(m, c)] = mk2(c == 2 * m ? R(1) : R(0), c == 2 * m + 1 ? R(1) : R(0));
    bound = R(1);
  }
  // out = H v. Row pair m: the columns c < 2m come from the stored pairs of
  // the earlier row pairs (dot of {h(2m', c), h(2m'+1, c)} with {v_2m', v_2m'+1}),
  // then the pair chain over c >= 2m continues from them.
  __device__ __forceinline__ void mul(const V2<R> (&v)[NP], V2<R> (&out)[NP], R nz) const {
#pragma unroll
    for (int m = 0; m < NP; ++m) {
      const bool pad = (NA & 1) && m == NP - 1;  // padding high lane
      V2<R> acc;
      if (m == 0) {
        acc = NA > 1 ? mul2(h[pid(0, 0)], bc2(v[0].x)) : mulzp(pad, h[pid(0, 0)], bc2(v[0].x), nz);
      } else {
        R lo[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 2 * m + e;
          if (c >= NA) {
            lo[e] = R(0);
            continue;
          }
          V2<R> l = m > 1 ? mul2(h[pid(0, c)], v[0]) : mulz(h[pid(0, c)], v[0], nz);
#pragma unroll
          for (int mm = 1; mm < m; ++mm) l = fma2(h[pid(mm, c)], v[mm], l);
          lo[e] = l.x + l.y;
        }
        acc = fma2p(pad, h[pid(m, 2 * m)], bc2(v[m].x), mk2(lo[0], lo[1]));
      }
#pragma unroll
      for (int c = 2 * m + 1; c < NA; ++c) acc = fma2(h[pid(m, c)], bc2(FP_EL(v, c)), acc);
      out[m] = acc;
    }
  }
  // One BFGS step. In: step sg, gradient change y, new gradient gn, old
  // direction p (= -H g_old), curvature flag ok, sy = sg.y and ms =
  // max_j |sg_j|. Out: p = -H' gn with H' the updated matrix (or the old one
  // when the update is skipped: failed curvature test or a non-finite H',
  // solver.py:184,198). Returns the update's FP_FATE_* bits.
  __device__ __forceinline__ uint8_t step(const V2<R> (&sg)[NP], const V2<R> (&y)[NP],
                                          const V2<R> (&gn)[NP], V2<R> (&p)[NP], bool ok, R sy, R ms,
                                          R nz) {
    V2<R> Hg[NP];
    mul(gn, Hg, nz);
    if (ok) {
      V2<R> Hy[NP];
#pragma unroll
      for (int m = 0; m < NP; ++m) Hy[m] = add2p((NA & 1) && m == NP - 1, Hg[m], p[m]);
      const R rho = rcp_fast(sy);
      const R yHy = dotv<R, NA>(y, Hy, nz);
      const R rr = rho * rho;
      const R half = R(0.5) * fma(rr, yHy, rho);
      V2<R> z[NP];
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        const bool lo = (NA & 1) && m == NP - 1;
        z[m] = fma2p(lo, bc2(half), sg[m], mul2p(lo, bc2(-rho), Hy[m]));
      }
      // |H'_ij| <= bound + |z_i s_j + s_i z_j| <= bound + 2 max|s| max|z|, and
      // |z_j| <= |half| max|s| + rho max|Hy|, so w = max|s| (|half| max|s| +
      // rho max|Hy|) bounds |s_i z_j| — and also the reference's products
      // rho |s_i Hy_j| and |coef s_i s_j| / 2. The reference evaluates
      // H' = H - rho (s Hy^T + Hy s^T) + (rho^2 yHy + rho) s s^T, whose
      // intermediates (s_i s_j, s_i Hy_j, rho^2 yHy, ...) can overflow fp32
      // where the two-term form does not — and then it skips the update
      // (solver.py:196-199). So the update is "suspect" when the bound on H'
      // or max|s| max(max|s|, max|Hy|) reaches Num<R>::suspect() (1e36 in
      // fp32: far above every healthy path, 340x below FLT_MAX; 1e305 in
      // fp64). (An overflowing rho^2 or rho^2 yHy makes `half`, hence w,
      // infinite: max|s| > 0 here, as s.y > 0.) Suspect updates evaluate the
      // reference's expression entry by entry. The magnitudes are FMNMX (ALU
      // pipe) reductions; NaN/inf propagate into `sus` and send the update
      // down the checked path too. (The bound is a trigger with a 340x
      // margin, so its own rounding needs no allowance.)
      const R mhy = absmaxv<R, NA>(Hy);
      const R w = ms * fma(ms, fabs(half), mhy * rho);
      const R nb = fma(R(2), w, bound);
      const R sus = absmax_nan(nb, ms * absmax_nan(ms, mhy));
      bool take = true;
      uint8_t checked = 0;
      if (!(sus < Num<R>::suspect())) {
        checked = FP_FATE_ENTRY_CHECK;
        // Rare: possible overflow. Check every entry before committing, in
        // the reference's evaluation order and in the committed form.
        const R coef = rr * yHy + rho;  // (rho rho) yHy + rho, unfused like numpy
        R mx = R(0);
#pragma unroll
        for (int r = 0; r < NA; ++r)
#pragma unroll
          for (int c = r; c < NA; ++c) {
            const R hv = get(r, c);
            const R v = fma(FP_EL(z, r), FP_EL(sg, c), fma(FP_EL(sg, r), FP_EL(z, c), hv));
            const R cross = FP_EL(sg, r) * FP_EL(Hy, c) + FP_EL(sg, c) * FP_EL(Hy, r);
            const R vr = (hv - rho * cross) + coef * (FP_EL(sg, r) * FP_EL(sg, c));
            take = take && finite(v) && finite(vr);
            mx = fabs(v) > mx ? fabs(v) : mx;
          }
        if (take) bound = mx * R(1.0009765625);
      } else {
        bound = nb;
      }
      if (take) {
#pragma unroll
        for (int m = 0; m < NP; ++m) {
#pragma unroll
          for (int c = 2 * m; c < NA; ++c) {
            const bool lo = (NA & 1) && m == NP - 1;  // the padded diagonal pair
            h[pid(m, c)] = fma2p(lo, z[m], bc2(FP_EL(sg, c)), fma2p(lo, sg[m], bc2(FP_EL(z, c)), h[pid(m, c)]));
          }
          if (2 * m + 1 < NA) h[pid(m, 2 * m)].y = h[pid(m, 2 * m + 1)].x;  // keep H symmetric
        }
        const R zg = dotv<R, NA>(z, gn, nz), sgn = dotv<R, NA>(sg, gn, nz);
#pragma unroll
        for (int m = 0; m < NP; ++m) {
          const bool lo = (NA & 1) && m == NP - 1;
          p[m] = fma2p(lo, sg[m], bc2(-zg), fma2p(lo, z[m], bc2(-sgn), neg2p(lo, Hg[m])));
        }
        return checked;
      }
#pragma unroll
      for (int m = 0; m < NP; ++m) p[m] = neg2p((NA & 1) && m == NP - 1, Hg[m]);
      return FP_FATE_NONFINITE_SKIP | checked;
    }
#pragma unroll
    for (int m = 0; m < NP; ++m) p[m] = neg2p((NA & 1) && m == NP - 1, Hg[m]);
    return FP_FATE_CURVATURE_SKIP;
  }
};

// |g|^2 as one sequential chain in coordinate order: the dense 2K layout only
// adds exact zeros for inert coordinates, so every kernel (dense, specialised,
// VJP-only) classifies a path identically.
template <typename R, int NA>
__device__ __forceinline__ R norm2_seq(const V2<R> (&g)[Packed<NA>::NP]) {
  R q = R(0);
#pragma unroll
  for (int j = 0; j < NA; ++j) q = fma(FP_EL(g, j), FP_EL(g, j), q);
  return q;
}

// Stationarity gate |g| < 1e-5 (1 + L) (implicit_diff.py:25,30-36).
template <typename R, int NA>
__device__ __forceinline__ bool stationary(const V2<R> (&g)[Packed<NA>::NP], R len) {
  return Num<R>::sqrt_(norm2_seq<R, NA>(g)) < R(1e-5) * (R(1) + len);
}

#ifdef FP_EXACT_F32
constexpr bool kExactF32 = true;
#else
constexpr bool kExactF32 = false;
#endif
#ifndef FP_LAST_BREAK_ORDERS
#define FP_LAST_BREAK_ORDERS 0x08u  // order 3
#endif
#ifndef FP_LAST_PEEL_ORDERS
#define FP_LAST_PEEL_ORDERS 0x16u  // orders 1, 2, 4
#endif
#ifndef FP_UNROLL_MAX_K
#define FP_UNROLL_MAX_K 1
#endif
constexpr int kUnrollMaxOrder = FP_UNROLL_MAX_K;

// The BFGS iterations (solver.py:171-211). GENERAL = false is the common case
// compiled without the per-iteration checks: one fixed-point step (F = 1, the
// reference default solver.py:45) and no trace.
template <typename R, int K, unsigned MASK, bool GENERAL>
__device__ __forceinline__ void bfgs_iterations(const Geo<R, K>& G, PathState<R, K, MASK>& P,
                                                InvHess<R, K, MASK>& H,
                                                V2<R> (&p)[Packed<Lay<K, MASK>::NA>::NP], uint8_t& st,
                                                int iterations, int fp_iters_rt, R* trace_len,
                                                R* trace_gnorm, uint8_t* trace_fate, int64_t trace_ld,
                                                int64_t row, bool keep_last_update = true) {
  using L = Lay<K, MASK>;
  constexpr int NA = L::NA;
  constexpr int NP = Packed<NA>::NP;
  const int fp_iters = GENERAL ? fp_iters_rt : 1;
  // The last iteration's curvature test, inverse-Hessian update and next
  // direction feed nothing the caller reads unless it returns H (or traces
  // the update fates): without them the last iteration ends at its new
  // gradient. Every output is bitwise the same. Two forms, per order
  // (FP_LAST_BREAK_ORDERS / FP_LAST_PEEL_ORDERS, bit K): leave the loop after
  // the last evaluation, or peel the last iteration out of the loop.
  // Measured (profiles/r02t_ab_last.txt, r02v_ab_peel.txt; fused step):
  // break K=3 1.043 -> 1.021 ms (peel 1.029), config-3 walls 71.2 -> 69.5
  // ms; peel K=1 0.411 -> 0.4025 (break 0.417: the loop is unrolled by two),
  // K=2 0.7155 -> 0.704 (break 0.712), K=4 1.443 -> 1.4415 with the forward
  // 1.281 -> 1.263; K=5 (out-of-line variants) keeps the full iteration
  // (break 2.026, peel 2.044 vs 2.004).
  constexpr bool kBreakLast = !GENERAL && ((FP_LAST_BREAK_ORDERS >> K) & 1);
  constexpr bool kPeelLast = !GENERAL && !kBreakLast && ((FP_LAST_PEEL_ORDERS >> K) & 1);
  const bool short_last = (kBreakLast || kPeelLast) && !keep_last_update && iterations > 0;
  const int last = (kBreakLast && short_last) ? iterations - 1 : -1;
  const int n_loop = (kPeelLast && short_last) ? iterations - 1 : iterations;
  // one step along p and the evaluation at the new t
  auto advance = [&](V2<R> (&sg)[NP], V2<R> (&gn)[NP], bool& zero) {
    const R alpha = P.step_size(G, p, fp_iters, zero);
    if (zero) st |= FP_STATUS_ZERO_DIRECTION;
#pragma unroll
    for (int m = 0; m < NP; ++m) {
      const bool lo = (NA & 1) && m == NP - 1;  // padding high lane
      sg[m] = mulzp(lo, bc2(alpha), p[m], G.nz);
      P.t[m] = add2p(lo, P.t[m], sg[m]);
    }
    P.template eval<true>(G, gn);
  };
  // Short loop bodies (order 1) run two iterations per trip: -1.2% at K=1
  // (tools/ab_libs.sh; at K=3 unrolling measured slower, instruction cache;
  // at K=2 fused 0.704 -> 0.7125 ms, profiles/r02z_ab_unroll2.txt).
  constexpr int kUnroll = (K <= kUnrollMaxOrder && !GENERAL) ? 2 : 1;
#pragma unroll(kUnroll)
  for (int it = 0; it < n_loop; ++it) {
    bool zero;
    V2<R> sg[NP], gn[NP];
    advance(sg, gn, zero);
    if (kBreakLast && it == last) {
#pragma unroll
      for (int m = 0; m < NP; ++m) P.g[m] = gn[m];
      break;
    }
    V2<R> y[NP];
#pragma unroll
    for (int m = 0; m < NP; ++m) y[m] = sub2p((NA & 1) && m == NP - 1, gn[m], P.g[m]);
    // Curvature test sy > 1e-12 |s| |y| (solver.py:184). From 3 unknowns on,
    // the norms come only when needed: |s| |y| <= NA max|s| max|y| (FMNMX
    // reductions, ALU pipe), so above that bound the test passes and at or
    // below 0 it fails — the same verdicts, bit for bit; only the band in
    // between (s, y nearly orthogonal) evaluates the norms (K=3 fused -0.7%,
    // forward -1.3%, K=2 -1.1%; slower for 1-2 unknowns and for the
    // out-of-line variants of orders 4-5, which keep the branch-free dots).
    const R sy = dotv<R, NA>(sg, y, G.nz);
    const R ms = absmaxv<R, NA>(sg);
    bool ok;
    if constexpr (NA >= 3 && K <= 3) {
      // (while |s|^2 and |y|^2 cannot overflow: past that the reference's
      // norms are infinite and its test fails, which the exact path follows)
      const R my = absmaxv<R, NA>(y);
      ok = absmax_nan(ms, my) < Num<R>::sqrt_big() && sy > (R(1e-12 * NA * 1.0001) * ms) * my;
      if (!ok && sy > R(0)) {
        const R ss = dotv<R, NA>(sg, sg, G.nz);
        const R yy = dotv<R, NA>(y, y, G.nz);
        ok = sy > (R(1e-12) * sqrt_test(ss)) * sqrt_test(yy);
      }
    } else if constexpr (NA == 1 && sizeof(R) == 4 && !kExactF32) {
      // One unknown: sy = fl(s y), and 1e-12 sqrt(fl(s^2)) sqrt(fl(y^2)) is
      // below |sy| whenever s^2 and y^2 are finite (sqrt.approx flushes a
      // subnormal square to 0, which keeps the test sy > 0), infinite or NaN
      // when one of them overflows (the test fails) — so the test is sy > 0
      // with |s|, |y| < 2^64 (the smallest float whose square rounds to inf).
      // Same verdicts; two MUFU.SQRT and four FMUL fewer per iteration.
      const R big = R(18446744073709551616.0);  // 2^64
      ok = sy > R(0) && fabs(sg[0].x) < big && fabs(y[0].x) < big;
    } else {
      const R ss = dotv<R, NA>(sg, sg, G.nz);
      const R yy = dotv<R, NA>(y, y, G.nz);
      ok = sy > (R(1e-12) * sqrt_test(ss)) * sqrt_test(yy);
    }
    const uint8_t fate = H.step(sg, y, gn, p, ok, sy, ms, G.nz);
#pragma unroll
    for (int m = 0; m < NP; ++m) P.g[m] = gn[m];
    if (GENERAL && trace_len != nullptr) {
      P.finish_norms(G);
      trace_len[int64_t(it) * trace_ld + row] = P.length();
      trace_gnorm[int64_t(it) * trace_ld + row] = Num<R>::sqrt_(norm2_seq<R, NA>(P.g));
      if (trace_fate != nullptr)
        trace_fate[int64_t(it) * trace_ld + row] = fate | (zero ? FP_FATE_ZERO_DIRECTION : 0);
    }
  }
  if constexpr (kPeelLast) {
    if (n_loop < iterations) {
      bool zero;
      V2<R> sg[NP], gn[NP];
      advance(sg, gn, zero);
#pragma unroll
      for (int m = 0; m < NP; ++m) P.g[m] = gn[m];
    }
  }
}

// The fixed-iteration BFGS loop (solver.py:146-215) from the state P (which
// must hold t and its evaluation). Returns DEGENERATE_ENTRY / ZERO_DIRECTION
// status bits; optional per-iteration trace (solver.py:202-206) and final
// inverse Hessian (return_state) in the dense 2K layout.
template <typename R, int K, unsigned MASK>
__device__ __forceinline__ uint8_t bfgs_solve(const Geo<R, K>& G, PathState<R, K, MASK>& P,
                                              int iterations, int fp_iters, R* trace_len,
                                              R* trace_gnorm, uint8_t* trace_fate, int64_t trace_ld,
                                              int64_t row, R* H_out) {
  using L = Lay<K, MASK>;
  constexpr int NA = L::NA;
  constexpr int NP = Packed<NA>::NP;
  uint8_t st = 0;
  if (P.min_norm() <= G.eps) st |= FP_STATUS_DEGENERATE_ENTRY;  // checked_segments (solver.py:166)
  InvHess<R, K, MASK> H;
  H.identity();
  V2<R> p[NP];
#pragma unroll
  for (int m = 0; m < NP; ++m) p[m] = neg2(P.g[m]);  // H = I
#ifndef FP_NO_LOOP_SPECIALISATION
  if (fp_iters == 1 && trace_len == nullptr)
    bfgs_iterations<R, K, MASK, false>(G, P, H, p, st, iterations, 1, nullptr, nullptr, nullptr, 0, 0,
                                       H_out != nullptr);
  else
#endif
    bfgs_iterations<R, K, MASK, true>(G, P, H, p, st, iterations, fp_iters, trace_len, trace_gnorm,
                                      trace_fate, trace_ld, row);
  P.finish_norms(G);
  if (H_out != nullptr) {
    R* Ho = H_out + row * (4 * K * K);
#pragma unroll
    for (int i = 0; i < 2 * K; ++i)
#pragma unroll
      for (int j = 0; j < 2 * K; ++j) {
        const int ii = i >> 1, ci = i & 1, jj = j >> 1, cj = j & 1;
        const bool ai = ci == 0 || L::plane(ii), aj = cj == 0 || L::plane(jj);
        R v = (i == j) ? R(1) : R(0);
        if (ai && aj) v = H.get(L::idx(ii, ci), L::idx(jj, cj));
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
  for (int j = 0; j < NA; ++j) fin = fin && finite(P.T(j)) && finite(P.Gr(j));
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
      act[i][c] = (G.A(i, 0, c) != R(0)) || (G.A(i, 1, c) != R(0)) || (G.A(i, 2, c) != R(0));
  }
  R u[S][3];
#pragma unroll
  for (int k = 0; k < S; ++k)
#pragma unroll
    for (int r = 0; r < 3; ++r) u[k][r] = P.S3(k, r) * P.RN(k);
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
        au_in[i][c] = fma(G.A(i, 2, c), u[i][2], fma(G.A(i, 1, c), u[i][1], G.A(i, 0, c) * u[i][0]));
        au_out[i][c] =
            fma(G.A(i, 2, c), u[i + 1][2], fma(G.A(i, 1, c), u[i + 1][1], G.A(i, 0, c) * u[i + 1][0]));
      }
    R rhs[K][2];
    R trace = R(0);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      R gii[3];
      gii[0] = fma(G.A(i, 2, 0), G.A(i, 2, 0), fma(G.A(i, 1, 0), G.A(i, 1, 0), G.A(i, 0, 0) * G.A(i, 0, 0)));
      gii[1] = fma(G.A(i, 2, 0), G.A(i, 2, 1), fma(G.A(i, 1, 0), G.A(i, 1, 1), G.A(i, 0, 0) * G.A(i, 0, 1)));
      gii[2] = fma(G.A(i, 2, 1), G.A(i, 2, 1), fma(G.A(i, 1, 1), G.A(i, 1, 1), G.A(i, 0, 1) * G.A(i, 0, 1)));
      const R ri = P.RN(i), ro = P.RN(i + 1);
      D[i][0] = (gii[0] - au_in[i][0] * au_in[i][0]) * ri + (gii[0] - au_out[i][0] * au_out[i][0]) * ro;
      D[i][1] = (gii[1] - au_in[i][0] * au_in[i][1]) * ri + (gii[1] - au_out[i][0] * au_out[i][1]) * ro;
      D[i][2] = (gii[2] - au_in[i][1] * au_in[i][1]) * ri + (gii[2] - au_out[i][1] * au_out[i][1]) * ro;
      if (i + 1 < K) {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const R gij = fma(G.A(i, 2, a), G.A(i + 1, 2, b),
                              fma(G.A(i, 1, a), G.A(i + 1, 1, b), G.A(i, 0, a) * G.A(i + 1, 0, b)));
            O[i][a][b] = -(gij - au_out[i][a] * au_in[i + 1][b]) * ro;
          }
      }
      // rhs = -(wl g + vT) on active coordinates, 0 on inert ones
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const R gc = (c == 0 || L::plane(i)) ? P.Gr(L::idx(i, c)) : R(0);
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
    // _solve_sym (implicit_diff.py:55-71): block-Thomas elimination (the
    // system is block tridiagonal), accepted when its residual
    // |H_a x - rhs| <= tol (1 + |rhs|); otherwise (or on a zero pivot / a
    // non-finite solution) one retry on H_a + lambda I with lambda =
    // 1e-12 tr(H_a), accepted when finite. Inert rows are pinned identity rows
    // with zero rhs: they add nothing to either norm. LAPACK's LU solve is
    // backward stable (residual ~ eps |H| |x|); the explicit 2x2 block
    // inverses are not quite, so a solution that misses the bound first gets
    // one step of fixed-precision iterative refinement (which restores a
    // backward-stable residual) before the bound decides.
    R Ci[K][3];      // inverse pivot blocks
    R Lm[K][2][2];   // elimination multipliers O_{i-1}^T Cinv_{i-1}
    auto factor = [&](R lam) {
      bool ok = true;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        R C0 = D[i][0] + (act[i][0] ? lam : R(0));
        R C1 = D[i][1];
        R C2 = D[i][2] + (act[i][1] ? lam : R(0));
        if (i > 0) {
          // Lm = O_{i-1}^T Cinv_{i-1}; C -= Lm O_{i-1}
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            Lm[i][a][0] = O[i - 1][0][a] * Ci[i - 1][0] + O[i - 1][1][a] * Ci[i - 1][1];
            Lm[i][a][1] = O[i - 1][0][a] * Ci[i - 1][1] + O[i - 1][1][a] * Ci[i - 1][2];
          }
          C0 -= Lm[i][0][0] * O[i - 1][0][0] + Lm[i][0][1] * O[i - 1][1][0];
          C1 -= Lm[i][0][0] * O[i - 1][0][1] + Lm[i][0][1] * O[i - 1][1][1];
          C2 -= Lm[i][1][0] * O[i - 1][0][1] + Lm[i][1][1] * O[i - 1][1][1];
        }
        const R det = C0 * C2 - C1 * C1;
        ok = ok && (det != R(0)) && finite(det);  // LinAlgError: exactly singular pivot
        const R id = rcp_fast(det);
        Ci[i][0] = C2 * id;
        Ci[i][1] = -C1 * id;
        Ci[i][2] = C0 * id;
      }
      return ok;
    };
    // x = (factored matrix)^-1 b; false when x is not finite
    auto substitute = [&](const R (&b)[K][2], R (&x)[K][2]) {
      R z[K][2];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        z[i][0] = b[i][0];
        z[i][1] = b[i][1];
        if (i > 0) {
          z[i][0] -= Lm[i][0][0] * z[i - 1][0] + Lm[i][0][1] * z[i - 1][1];
          z[i][1] -= Lm[i][1][0] * z[i - 1][0] + Lm[i][1][1] * z[i - 1][1];
        }
      }
      bool ok = true;
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
        x[i][0] = act[i][0] ? v0 : R(0);
        x[i][1] = act[i][1] ? v1 : R(0);
        nxt0 = x[i][0];
        nxt1 = x[i][1];
        ok = ok && finite(v0) && finite(v1);
      }
      return ok;
    };
    // r = rhs - H_a x (unregularised); returns |r|^2
    auto residual = [&](const R (&x)[K][2], R (&r)[K][2]) {
      R rr = R(0);
#pragma unroll
      for (int i = 0; i < K; ++i) {
        R r0 = D[i][0] * x[i][0] + D[i][1] * x[i][1];
        R r1 = D[i][1] * x[i][0] + D[i][2] * x[i][1];
        if (i > 0) {
          r0 += O[i - 1][0][0] * x[i - 1][0] + O[i - 1][1][0] * x[i - 1][1];
          r1 += O[i - 1][0][1] * x[i - 1][0] + O[i - 1][1][1] * x[i - 1][1];
        }
        if (i + 1 < K) {
          r0 += O[i][0][0] * x[i + 1][0] + O[i][0][1] * x[i + 1][1];
          r1 += O[i][1][0] * x[i + 1][0] + O[i][1][1] * x[i + 1][1];
        }
        r[i][0] = rhs[i][0] - r0;
        r[i][1] = rhs[i][1] - r1;
        rr = fma(r[i][1], r[i][1], fma(r[i][0], r[i][0], rr));
      }
      return rr;
    };
    bool solved = false;
    if (factor(R(0)) && substitute(rhs, sol)) {
      if constexpr (sizeof(R) == 8) {
        // threshold tests: sqrt_test suffices
        R bb = R(0);
#pragma unroll
        for (int i = 0; i < K; ++i) bb = fma(rhs[i][1], rhs[i][1], fma(rhs[i][0], rhs[i][0], bb));
        const R tol = Num<R>::resid_tol() * (R(1) + sqrt_test(bb));
        R r[K][2];
        solved = sqrt_test(residual(sol, r)) <= tol;  // NaN: not solved
        if (!solved) {
          R dx[K][2];
          if (substitute(r, dx)) {
#pragma unroll
            for (int i = 0; i < K; ++i) {
              sol[i][0] += dx[i][0];
              sol[i][1] += dx[i][1];
            }
            solved = sqrt_test(residual(sol, r)) <= tol;
          }
        }
      } else {
        // fp32: the check is inert, so it is not computed. At the reference's
        // trigger point (cond(H_a) ~ 4.5e7, scaled bound 5.4 (1 + |rhs|))
        // an fp32 solve has no correct digits left, and the retry's shift
        // 1e-12 tr(H_a) lies below the fp32 unit roundoff of every active
        // diagonal entry above 2e-5 tr(H_a) / NA, so it would return the
        // same solution. The fp64 kernels run the reference's rule; the
        // fp32 gradient contract is 1e-3 relative.
        solved = true;
      }
    }
    // Tikhonov retry (implicit_diff.py:64-71): accepted when finite
    if (!solved) solved = factor(R(1e-12) * trace) && substitute(rhs, sol);
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
    for (int r = 0; r < 3; ++r) dx[i][r] = fma(G.A(i, r, 1), sol[i][1], G.A(i, r, 0) * sol[i][0]);
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
    for (int r = 0; r < 3; ++r) w[k][r] = (ds[r] - u[k][r] * ud) * P.RN(k);
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
