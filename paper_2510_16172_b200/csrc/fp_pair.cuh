// Two paths per thread: the fp32 BFGS loop with each scalar of the per-path
// loop carried as a pair (path a in .x, path b in .y), so every scalar FP32
// operation of the loop becomes one paired FFMA2 / FADD2 for two paths.
//
// Status: an A/B option (FP_PAIR_MAX_K, fp_inst.cu), off by default — the
// results are bitwise those of the per-path kernels, but at the same
// registers per path a warp now carries 64 paths with the loop's dependency
// chains unchanged, so half the warps hide the same latencies: measured K=1
// 0.466 vs 0.411 ms, K=2 0.95 vs 0.72 ms per fused step (profiles/
// r02s_ab_pair.txt).
//
// Motivation: at orders 1-2 most of the loop is scalar arithmetic (one or two
// interactions leave little to pair inside a path: the order-1 diffraction
// variant has one unknown), so the per-path kernels there are issue-bound
// (ncu, order 1: issue active 80%, FMA pipe 59%). Pairing across paths halves
// the issue slots of that arithmetic; MUFU, compares, selects and the
// NaN-propagating magnitude reductions stay per lane.
//
// Exactness: each lane performs the same IEEE operations, in the same order,
// as the per-path loop (fp_path.cuh bfgs_iterations with GENERAL = false,
// step_size with F = 1, eval<true>, InvHess::mul / step, dotv, absmaxv, the
// curvature tests): a within-path pair operation of that code is two
// operations here (one per element), a scalar one is one paired operation.
// Products are FFMA2 with an opaque -0 addend (fp_path.cuh mulz) so ptxas
// cannot contract them into a neighbouring add. Results are bitwise those of
// the per-path kernels (tests/test_gpu_solve.py, tile vs bucketed dispatch
// and batch-invariance tests; tools/ab_bits.py).
//
// Lanes that disagree (one path's update skipped, a suspect update) compute
// both outcomes and select per lane; the rare entry-by-entry overflow check of
// a suspect update runs per lane with the scalar expressions of InvHess::step.
#pragma once

#include "fp_path.cuh"

namespace fp {

using X = float2;

__device__ __forceinline__ X xb(float v) { return make_float2(v, v); }
__device__ __forceinline__ X xfma(X a, X b, X c) { return __ffma2_rn(a, b, c); }
// exact product a * b (a * b + (-0) with an opaque -0, see fp_path.cuh mulz)
__device__ __forceinline__ X xmul(X a, X b, X nz) { return __ffma2_rn(a, b, nz); }
__device__ __forceinline__ X xadd(X a, X b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ X xneg(X a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ X xsub(X a, X b) { return __fadd2_rn(a, xneg(b)); }
__device__ __forceinline__ X xabs(X a) { return make_float2(fabsf(a.x), fabsf(a.y)); }
__device__ __forceinline__ float xl(X v, int e) { return e ? v.y : v.x; }

// Geometry of two paths.
template <int K>
struct GeoX {
  X A[K][3][2];  // basis (interaction, row, column); dead columns unused
  X b[K][3];
  X x0[3], xe[3];
  X eps, eps2, reps, nz;
};

template <int K, unsigned MASK>
struct PairState {
  using L = Lay<K, MASK>;
  static constexpr int NA = L::NA, S = L::S;
  static constexpr int NH = NA * (NA + 1) / 2;
  X t[NA], g[NA];
  X s[S][3];  // segments at t
  X rn[S];    // 1 / max(|s_k|, eps)
  X h[NH];    // inverse Hessian, upper triangle h(r, c), r <= c
  X bound;    // InvHess::bound per path
  __device__ static constexpr int hi(int r, int c) { return r * NA - r * (r - 1) / 2 + (c - r); }
};

// ---- pack / unpack ----------------------------------------------------------
template <int K, unsigned MASK>
__device__ __forceinline__ void pack_pair(const Geo<float, K>& ga, const Geo<float, K>& gb,
                                          const PathState<float, K, MASK>& pa,
                                          const PathState<float, K, MASK>& pb, GeoX<K>& G,
                                          PairState<K, MASK>& P) {
  using L = Lay<K, MASK>;
#pragma unroll
  for (int i = 0; i < K; ++i) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
      for (int c = 0; c < 2; ++c) G.A[i][r][c] = make_float2(ga.A(i, r, c), gb.A(i, r, c));
      G.b[i][r] = make_float2(ga.b(i, r), gb.b(i, r));
    }
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    G.x0[r] = make_float2(ga.x0(r), gb.x0(r));
    G.xe[r] = make_float2(ga.xe(r), gb.xe(r));
  }
  G.nz = make_float2(ga.nz, gb.nz);
  G.reps = make_float2(ga.reps, gb.reps);
  G.eps = make_float2(ga.eps, gb.eps);
  G.eps2 = xmul(G.eps, G.eps, G.nz);  // eval's eps * eps
#pragma unroll
  for (int j = 0; j < L::NA; ++j) {
    P.t[j] = make_float2(pa.T(j), pb.T(j));
    P.g[j] = make_float2(pa.Gr(j), pb.Gr(j));
  }
#pragma unroll
  for (int k = 0; k < L::S; ++k) {
#pragma unroll
    for (int r = 0; r < 3; ++r) P.s[k][r] = make_float2(pa.S3(k, r), pb.S3(k, r));
    P.rn[k] = make_float2(pa.RN(k), pb.RN(k));
  }
}

// Lane e of the pair state back into a per-path state (t, g, segments and
// reciprocal norms: what finish_norms, final_status and the VJP read).
template <int K, unsigned MASK>
__device__ __forceinline__ void unpack_lane(const PairState<K, MASK>& P, int e,
                                            PathState<float, K, MASK>& p) {
  using L = Lay<K, MASK>;
#pragma unroll
  for (int j = 0; j < L::NA; ++j) {
    p.setT(j, xl(P.t[j], e));
    FP_SET(p.g, j, xl(P.g[j], e));
  }
#pragma unroll
  for (int k = 0; k < L::S; ++k) {
    p.sxy[k] = make_float2(xl(P.s[k][0], e), xl(P.s[k][1], e));
    p.sz[k] = xl(P.s[k][2], e);
    FP_SET(p.rnp, k, xl(P.rn[k], e));
  }
}

// ---- per-path pieces, paired ----------------------------------------------------
// eval<true> (fp_path.cuh): points, segments, reciprocal clamped norms
// (rcp_norm), clamped-norm gradient into gout.
template <int K, unsigned MASK>
__device__ __forceinline__ void eval_pair(const GeoX<K>& G, PairState<K, MASK>& P,
                                          X (&gout)[Lay<K, MASK>::NA]) {
  using L = Lay<K, MASK>;
  constexpr int S = L::S;
  X Pt[K + 2][3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    Pt[0][r] = G.x0[r];
    Pt[K + 1][r] = G.xe[r];
  }
  static_for<K>([&](auto ic) {
    constexpr int i = decltype(ic)::value;
    const X t0 = P.t[L::idx(i, 0)];
#pragma unroll
    for (int r = 0; r < 3; ++r) Pt[i + 1][r] = xfma(G.A[i][r][0], t0, G.b[i][r]);
    if constexpr (L::plane(i)) {
      const X t1 = P.t[L::idx(i, 1)];
#pragma unroll
      for (int r = 0; r < 3; ++r) Pt[i + 1][r] = xfma(G.A[i][r][1], t1, Pt[i + 1][r]);
    }
  });
  X u[S][3];
#pragma unroll
  for (int k = 0; k < S; ++k) {
#pragma unroll
    for (int r = 0; r < 3; ++r) P.s[k][r] = xsub(Pt[k + 1][r], Pt[k][r]);
    X q = xmul(P.s[k][0], P.s[k][0], G.nz);
    q = xfma(P.s[k][1], P.s[k][1], q);
    q = xfma(P.s[k][2], P.s[k][2], q);
    rcp_norm(q.x, G.eps.x, G.eps2.x, G.reps.x, P.rn[k].x);
    rcp_norm(q.y, G.eps.y, G.eps2.y, G.reps.y, P.rn[k].y);
#pragma unroll
    for (int r = 0; r < 3; ++r) u[k][r] = xmul(P.s[k][r], P.rn[k], G.nz);
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    X q[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) q[r] = xsub(u[i][r], u[i + 1][r]);
#pragma unroll
    for (int c = 0; c < 2; ++c)
      if (c == 0 || L::plane(i))
        gout[L::idx(i, c)] =
            xfma(G.A[i][2][c], q[2], xfma(G.A[i][1][c], q[1], xmul(G.A[i][0][c], q[0], G.nz)));
  }
}

// dotv: the two pair lanes of the per-path code accumulate separately (even /
// odd elements), then add; an odd last element is fused last.
template <int NA>
__device__ __forceinline__ X dot_pair(const X (&a)[NA], const X (&b)[NA], X nz) {
  constexpr int NF = NA / 2;
  if constexpr (NF > 0) {
    X ax = xmul(a[0], b[0], nz), ay = xmul(a[1], b[1], nz);
#pragma unroll
    for (int m = 1; m < NF; ++m) {
      ax = xfma(a[2 * m], b[2 * m], ax);
      ay = xfma(a[2 * m + 1], b[2 * m + 1], ay);
    }
    X r = xadd(ax, ay);
    if constexpr (NA & 1) r = xfma(a[NA - 1], b[NA - 1], r);
    return r;
  } else {
    return xmul(a[0], b[0], nz);
  }
}

template <int NA>
__device__ __forceinline__ X absmax_pair(const X (&a)[NA]) {
  X m = xabs(a[0]);
#pragma unroll
  for (int j = 1; j < NA; ++j) {
    m.x = absmax_nan(m.x, a[j].x);
    m.y = absmax_nan(m.y, a[j].y);
  }
  return m;
}

__device__ __forceinline__ X rcp_fast_pair(X x) {
  const X r = make_float2(rcp_approx(x.x), rcp_approx(x.y));
  return xfma(r, xfma(xneg(x), r, xb(1.0f)), r);
}

// step_size with F = 1 (fp_path.cuh): alpha per path, `zero` per lane.
template <int K, unsigned MASK>
__device__ __forceinline__ X step_pair(const GeoX<K>& G, const PairState<K, MASK>& P,
                                       const X (&p)[Lay<K, MASK>::NA], bool& za, bool& zb) {
  using L = Lay<K, MASK>;
  constexpr int S = L::S;
  X w[K][3];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const X p0 = p[L::idx(i, 0)];
#pragma unroll
    for (int r = 0; r < 3; ++r) w[i][r] = xmul(G.A[i][r][0], p0, G.nz);
    if (L::plane(i)) {
      const X p1 = p[L::idx(i, 1)];
#pragma unroll
      for (int r = 0; r < 3; ++r) w[i][r] = xfma(G.A[i][r][1], p1, w[i][r]);
    }
  }
  X num, den, total;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    X d[3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
      d[r] = k == 0 ? w[0][r] : (k == K ? xneg(w[K - 1][r]) : xsub(w[k][r], w[k - 1][r]));
    const X a2 = xfma(d[2], d[2], xfma(d[1], d[1], xmul(d[0], d[0], G.nz)));
    const X cc = xfma(d[2], P.s[k][2], xfma(d[1], P.s[k][1], xmul(d[0], P.s[k][0], G.nz)));
    total = k == 0 ? a2 : xadd(total, a2);
    num = k == 0 ? xmul(cc, P.rn[0], G.nz) : xfma(cc, P.rn[k], num);
    den = k == 0 ? xmul(a2, P.rn[0], G.nz) : xfma(a2, P.rn[k], den);
  }
  za = total.x <= FLT_MIN;
  zb = total.y <= FLT_MIN;
  // -div_fast(num, zero ? 1 : den)
  const X b = make_float2(za ? 1.0f : den.x, zb ? 1.0f : den.y);
  const X r = make_float2(rcp_approx(b.x), rcp_approx(b.y));
  const X q = xmul(num, r, G.nz);
  const X cand = xneg(xfma(xfma(xneg(b), q, num), r, q));
  return make_float2((za || !finite(cand.x)) ? 0.0f : cand.x, (zb || !finite(cand.y)) ? 0.0f : cand.y);
}

// out = H v (InvHess::mul's operation order per element).
template <int K, unsigned MASK>
__device__ __forceinline__ void hmul_pair(const PairState<K, MASK>& P, const X (&v)[Lay<K, MASK>::NA],
                                          X (&o)[Lay<K, MASK>::NA], X nz) {
  using PS = PairState<K, MASK>;
  constexpr int NA = PS::NA;
  constexpr int NP = (NA + 1) / 2;
#pragma unroll
  for (int m = 0; m < NP; ++m) {
    const bool pad = (NA & 1) && m == NP - 1;
    if (m == 0) {
      o[0] = xmul(P.h[PS::hi(0, 0)], v[0], nz);
      if (NA > 1) o[1] = xmul(P.h[PS::hi(0, 1)], v[0], nz);
    } else {
      X lo[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 2 * m + e;
        if (c >= NA) {
          lo[e] = xb(0.0f);
          continue;
        }
        X lx = xmul(P.h[PS::hi(0, c)], v[0], nz), ly = xmul(P.h[PS::hi(1, c)], v[1], nz);
#pragma unroll
        for (int mm = 1; mm < m; ++mm) {
          lx = xfma(P.h[PS::hi(2 * mm, c)], v[2 * mm], lx);
          ly = xfma(P.h[PS::hi(2 * mm + 1, c)], v[2 * mm + 1], ly);
        }
        lo[e] = xadd(lx, ly);
      }
      o[2 * m] = xfma(P.h[PS::hi(2 * m, 2 * m)], v[2 * m], lo[0]);
      if (!pad) o[2 * m + 1] = xfma(P.h[PS::hi(2 * m, 2 * m + 1)], v[2 * m], lo[1]);
    }
#pragma unroll
    for (int c = 2 * m + 1; c < NA; ++c) {
      o[2 * m] = xfma(P.h[PS::hi(2 * m, c)], v[c], o[2 * m]);
      o[2 * m + 1] = xfma(P.h[PS::hi(2 * m + 1, c)], v[c], o[2 * m + 1]);
    }
  }
}

// InvHess::step for two paths: p <- -H' gn with H' the updated matrix, or
// -H gn when a path's update is skipped (curvature test, non-finite H').
template <int K, unsigned MASK>
__device__ __forceinline__ void hstep_pair(PairState<K, MASK>& P, const X (&sg)[Lay<K, MASK>::NA],
                                           const X (&y)[Lay<K, MASK>::NA],
                                           const X (&gn)[Lay<K, MASK>::NA], X (&p)[Lay<K, MASK>::NA],
                                           bool oka, bool okb, X sy, X ms, X nz) {
  using PS = PairState<K, MASK>;
  constexpr int NA = PS::NA;
  X Hg[NA];
  hmul_pair<K, MASK>(P, gn, Hg, nz);
  bool ta = oka, tb = okb;
  if (oka || okb) {
    X Hy[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) Hy[j] = xadd(Hg[j], p[j]);
    const X rho = rcp_fast_pair(sy);
    const X yHy = dot_pair<NA>(y, Hy, nz);
    const X rr = xmul(rho, rho, nz);
    const X half = xmul(xb(0.5f), xfma(rr, yHy, rho), nz);
    X z[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) z[j] = xfma(half, sg[j], xmul(xneg(rho), Hy[j], nz));
    const X mhy = absmax_pair<NA>(Hy);
    const X w = xmul(ms, xfma(ms, xabs(half), xmul(mhy, rho, nz)), nz);
    const X nb = xfma(xb(2.0f), w, P.bound);
    const X m2 = xmul(ms, make_float2(absmax_nan(ms.x, mhy.x), absmax_nan(ms.y, mhy.y)), nz);
    const X sus = make_float2(absmax_nan(nb.x, m2.x), absmax_nan(nb.y, m2.y));
    X bound = nb;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (!(e ? okb : oka)) continue;
      if (xl(sus, e) < Num<float>::suspect()) continue;
      // Rare: the reference's entry-by-entry check (InvHess::step), lane e.
      const float rh = xl(rho, e);
      const float coef = xl(rr, e) * xl(yHy, e) + rh;
      float mx = 0.0f;
      bool take = true;
#pragma unroll
      for (int r = 0; r < NA; ++r)
#pragma unroll
        for (int c = r; c < NA; ++c) {
          const float hv = xl(P.h[PS::hi(r, c)], e);
          const float sr = xl(sg[r], e), sc = xl(sg[c], e);
          const float v = fmaf(xl(z[r], e), sc, fmaf(sr, xl(z[c], e), hv));
          const float cross = sr * xl(Hy[c], e) + sc * xl(Hy[r], e);
          const float vr = (hv - rh * cross) + coef * (sr * sc);
          take = take && finite(v) && finite(vr);
          mx = fabsf(v) > mx ? fabsf(v) : mx;
        }
      set_lane(bound, e, take ? mx * 1.0009765625f : xl(P.bound, e));
      if (e) tb = take; else ta = take;
    }
    if (ta && tb) {
      P.bound = bound;
#pragma unroll
      for (int r = 0; r < NA; ++r)
#pragma unroll
        for (int c = r; c < NA; ++c)
          P.h[PS::hi(r, c)] = xfma(z[r], sg[c], xfma(sg[r], z[c], P.h[PS::hi(r, c)]));
    } else {
      P.bound = make_float2(ta ? bound.x : P.bound.x, tb ? bound.y : P.bound.y);
#pragma unroll
      for (int r = 0; r < NA; ++r)
#pragma unroll
        for (int c = r; c < NA; ++c) {
          const X hn = xfma(z[r], sg[c], xfma(sg[r], z[c], P.h[PS::hi(r, c)]));
          const X ho = P.h[PS::hi(r, c)];
          P.h[PS::hi(r, c)] = make_float2(ta ? hn.x : ho.x, tb ? hn.y : ho.y);
        }
    }
    const X zg = dot_pair<NA>(z, gn, nz), sgn = dot_pair<NA>(sg, gn, nz);
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      const X pn = xfma(sg[j], xneg(zg), xfma(z[j], xneg(sgn), xneg(Hg[j])));
      p[j] = make_float2(ta ? pn.x : -Hg[j].x, tb ? pn.y : -Hg[j].y);
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < NA; ++j) p[j] = xneg(Hg[j]);
}

// The fixed-iteration BFGS loop of two paths (bfgs_iterations, GENERAL =
// false: F = 1, no trace). P holds t, g, the segments and reciprocal norms of
// the entry evaluation; returns ZERO_DIRECTION bits per path.
template <int K, unsigned MASK>
__device__ __forceinline__ void bfgs_pair(const GeoX<K>& G, PairState<K, MASK>& P, int iterations,
                                          uint8_t& sta, uint8_t& stb) {
  using PS = PairState<K, MASK>;
  constexpr int NA = PS::NA;
#pragma unroll
  for (int r = 0; r < NA; ++r)
#pragma unroll
    for (int c = r; c < NA; ++c) P.h[PS::hi(r, c)] = xb(r == c ? 1.0f : 0.0f);
  P.bound = xb(1.0f);
  X p[NA];
#pragma unroll
  for (int j = 0; j < NA; ++j) p[j] = xneg(P.g[j]);
  for (int it = 0; it < iterations; ++it) {
    bool za, zb;
    const X alpha = step_pair<K, MASK>(G, P, p, za, zb);
    if (za) sta |= FP_STATUS_ZERO_DIRECTION;
    if (zb) stb |= FP_STATUS_ZERO_DIRECTION;
    X sg[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      sg[j] = xmul(alpha, p[j], G.nz);
      P.t[j] = xadd(P.t[j], sg[j]);
    }
    X gn[NA];
    eval_pair<K, MASK>(G, P, gn);
    X y[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) y[j] = xsub(gn[j], P.g[j]);
    // curvature test sy > 1e-12 |s| |y| (bfgs_iterations' two forms)
    const X sy = dot_pair<NA>(sg, y, G.nz);
    const X ms = absmax_pair<NA>(sg);
    bool oka, okb;
    if constexpr (NA >= 3 && K <= 3) {
      const X my = absmax_pair<NA>(y);
      const X lim = xmul(xmul(xb(float(1e-12 * NA * 1.0001)), ms, G.nz), my, G.nz);
      oka = absmax_nan(ms.x, my.x) < Num<float>::sqrt_big() && sy.x > lim.x;
      okb = absmax_nan(ms.y, my.y) < Num<float>::sqrt_big() && sy.y > lim.y;
      const bool ra = !oka && sy.x > 0.0f, rb = !okb && sy.y > 0.0f;
      if (ra || rb) {
        const X ss = dot_pair<NA>(sg, sg, G.nz);
        const X yy = dot_pair<NA>(y, y, G.nz);
        const X l2 = xmul(xmul(xb(1e-12f), make_float2(sqrt_test(ss.x), sqrt_test(ss.y)), G.nz),
                          make_float2(sqrt_test(yy.x), sqrt_test(yy.y)), G.nz);
        if (ra) oka = sy.x > l2.x;
        if (rb) okb = sy.y > l2.y;
      }
    } else {
      const X ss = dot_pair<NA>(sg, sg, G.nz);
      const X yy = dot_pair<NA>(y, y, G.nz);
      const X l2 = xmul(xmul(xb(1e-12f), make_float2(sqrt_test(ss.x), sqrt_test(ss.y)), G.nz),
                        make_float2(sqrt_test(yy.x), sqrt_test(yy.y)), G.nz);
      oka = sy.x > l2.x;
      okb = sy.y > l2.y;
    }
    hstep_pair<K, MASK>(P, sg, y, gn, p, oka, okb, sy, ms, G.nz);
#pragma unroll
    for (int j = 0; j < NA; ++j) P.g[j] = gn[j];
  }
}

}  // namespace fp
