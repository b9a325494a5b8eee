// Kernel templates: batched forward solve, fused solve + implicit VJP, and
// VJP-only, one path per thread.
//
// Data movement: each CTA owns kThreads consecutive paths. Their input
// records are contiguous in the reference layout, so a full CTA stages its
// slabs (basis, anchor, start, end, T) into shared memory with one TMA bulk
// copy each (cp.async.bulk + mbarrier complete_tx); partial or unaligned
// CTAs fall back to coalesced vector loads. Outputs are gathered per slab in
// shared memory and written back with coalesced stores. With a row index
// (bucketed dispatch), threads read and write their records directly.
#pragma once

#include <atomic>

#include "fp_pair.cuh"
#include "fp_path.cuh"

namespace fp {

enum Op { OP_SOLVE = 0, OP_SOLVE_VJP = 1, OP_VJP = 2 };

template <typename R>
struct PathArgs {
  const R *basis, *anchor, *start, *end;
  const R* T;       // T0 for the solve, T* for VJP-only
  const R* vT;      // VJP-only: cotangent on T (B,K,2), may be null
  const R* wL;      // per-path weight on L, may be null
  R wL_scale;       // weight used when wL is null
  R nz;             // -0 (Geo::nz: keeps ptxas from contracting paired products)
  int mode;         // fp_vjp_mode
  int64_t B;        // staged mode: rows [row_begin, B) of the batch
  int64_t row_begin;
  int64_t ld;       // leading dimension of the (iterations, batch) trace arrays
  int iterations, fp_iters;
  R *T_out, *g_out, *points_out, *length_out;
  uint8_t* status_out;
  R *trace_len, *trace_gnorm, *H_out;
  uint8_t* trace_fate;  // (iterations, batch) FP_FATE_* bits of each BFGS update (with the trace)
  R *d_basis, *d_anchor, *d_start, *d_end, *u_out;
  // Gathered dispatch (fp_bucket.cu): rows[0 .. n_rows) are this launch's
  // paths (a kind-mask bucket that is not one contiguous range).
  const int32_t* rows;
  int64_t n_rows;
  // Tile kernels: count of warps whose paths have different kind masks (nullable).
  unsigned long long* mixed_warps;
};

// Per-path output destinations (shared-memory slab slots or global records).
template <typename R>
struct Outs {
  R *T, *g, *pts, *len, *db, *da, *d0, *d1, *u;
  uint8_t* st;
};

// Slab layout of one tile (kThreads paths) in shared memory, per op. Inputs:
// basis, anchor, start, end, T (+ vT for OP_VJP), each a contiguous run of
// records. Outputs (the same slab, after the inputs are in registers): only
// the arrays the op can write — T, g (OP_SOLVE), points, L for solves;
// the scene gradient (+ u for OP_VJP) for VJPs — then one status byte per
// path.
template <int K, int OP = OP_SOLVE_VJP>
struct W {
  static constexpr int basis = 6 * K, anchor = 3 * K, vec = 3, T = 2 * K, pts = 3 * K;
  static constexpr bool has_v = OP == OP_VJP;
  static constexpr bool w_T = OP != OP_VJP, w_g = OP == OP_SOLVE, w_pts = OP != OP_VJP,
                        w_len = OP != OP_VJP, w_grad = OP != OP_SOLVE, w_u = OP == OP_VJP;
  static constexpr int in_elems = basis + anchor + 2 * vec + T + (has_v ? T : 0);
  static constexpr int oT = 0;
  static constexpr int og = oT + (w_T ? T : 0);
  static constexpr int oP = og + (w_g ? T : 0);
  static constexpr int oL = oP + (w_pts ? pts : 0);
  static constexpr int oDB = oL + (w_len ? 1 : 0);
  static constexpr int oDA = oDB + (w_grad ? basis : 0);
  static constexpr int oD0 = oDA + (w_grad ? anchor : 0);
  static constexpr int oD1 = oD0 + (w_grad ? vec : 0);
  static constexpr int oU = oD1 + (w_grad ? vec : 0);
  static constexpr int out_elems = oU + (w_u ? T : 0);
  static constexpr int slab_elems = in_elems > out_elems ? in_elems : out_elems;
};

// Bytes of one slab (+ status bytes), 128-byte aligned so two slabs stack.
template <typename R, int K, int OP>
constexpr size_t slab_bytes() {
  return (size_t(W<K, OP>::slab_elems) * kThreads * sizeof(R) + kThreads + 127) / 128 * 128;
}
template <typename R, int K, int OP>
constexpr size_t smem_bytes() {
  return slab_bytes<R, K, OP>();
}

extern __shared__ __align__(128) unsigned char fp_smem[];

// Output destinations of one path, computed only when results are written
// (keeps ten 64-bit pointers out of the registers live across the solve).
template <typename R, int K, int OP>
__device__ __forceinline__ Outs<R> make_outs(const PathArgs<R>& a, int64_t row, int tid, bool staged,
                                             unsigned char* slab) {
  using Wk = W<K, OP>;
  Outs<R> o;
  if (!staged) {
    o.T = a.T_out ? a.T_out + row * Wk::T : nullptr;
    o.g = a.g_out ? a.g_out + row * Wk::T : nullptr;
    o.pts = a.points_out ? a.points_out + row * Wk::pts : nullptr;
    o.len = a.length_out ? a.length_out + row : nullptr;
    o.db = a.d_basis ? a.d_basis + row * Wk::basis : nullptr;
    o.da = a.d_anchor ? a.d_anchor + row * Wk::anchor : nullptr;
    o.d0 = a.d_start ? a.d_start + row * 3 : nullptr;
    o.d1 = a.d_end ? a.d_end + row * 3 : nullptr;
    o.u = a.u_out ? a.u_out + row * Wk::T : nullptr;
    o.st = a.status_out ? a.status_out + row : nullptr;
    return o;
  }
  R* sl = reinterpret_cast<R*>(slab);
  o.T = (Wk::w_T && a.T_out) ? sl + kThreads * Wk::oT + tid * Wk::T : nullptr;
  o.g = (Wk::w_g && a.g_out) ? sl + kThreads * Wk::og + tid * Wk::T : nullptr;
  o.pts = (Wk::w_pts && a.points_out) ? sl + kThreads * Wk::oP + tid * Wk::pts : nullptr;
  o.len = (Wk::w_len && a.length_out) ? sl + kThreads * Wk::oL + tid : nullptr;
  o.db = (Wk::w_grad && a.d_basis) ? sl + kThreads * Wk::oDB + tid * Wk::basis : nullptr;
  o.da = (Wk::w_grad && a.d_anchor) ? sl + kThreads * Wk::oDA + tid * Wk::anchor : nullptr;
  o.d0 = (Wk::w_grad && a.d_start) ? sl + kThreads * Wk::oD0 + tid * 3 : nullptr;
  o.d1 = (Wk::w_grad && a.d_end) ? sl + kThreads * Wk::oD1 + tid * 3 : nullptr;
  o.u = (Wk::w_u && a.u_out) ? sl + kThreads * Wk::oU + tid * Wk::T : nullptr;
  o.st = reinterpret_cast<uint8_t*>(slab + size_t(Wk::slab_elems) * kThreads * sizeof(R)) + tid;
  return o;
}

// ---- TMA bulk copy helpers -------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// TMA bulk store shared -> global (bulk_group completion) for the output slabs.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

template <typename R>
__device__ __forceinline__ void coop_copy(R* dst, const R* src, int count) {
  for (int e = threadIdx.x; e < count; e += blockDim.x) dst[e] = src[e];
}

// One path's inputs, held in registers.
template <typename R, int K>
struct Rec {
  R b[6 * K], a[3 * K], x0[3], x1[3], T[2 * K], v[2 * K];
};

template <typename R, int K>
__device__ __forceinline__ void load_rec(Rec<R, K>& r, const R* b, const R* a, const R* x0,
                                         const R* x1, const R* T, const R* v) {
#pragma unroll
  for (int e = 0; e < 6 * K; ++e) r.b[e] = b[e];
#pragma unroll
  for (int e = 0; e < 3 * K; ++e) r.a[e] = a[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    r.x0[e] = x0[e];
    r.x1[e] = x1[e];
  }
#pragma unroll
  for (int e = 0; e < 2 * K; ++e) {
    r.T[e] = T[e];
    r.v[e] = v ? v[e] : R(0);
  }
}

// ---- the per-path body -------------------------------------------------------
// Stage 1: geometry, the initial unknowns and their evaluation. The solve
// starts from the refined evaluation; the VJP-only op evaluates T* the way
// the loop's last iteration did (eval_entry), so a fused step and
// solve-then-VJP agree bit for bit.
template <typename R, int K, unsigned MASK, int OP>
__device__ __forceinline__ void begin_path(const PathArgs<R>& a, const Rec<R, K>& in, Geo<R, K>& G,
                                           PathState<R, K, MASK>& P, R (&tin)[K]) {
  using L = Lay<K, MASK>;
  load_geo<R, K, MASK>(G, in.b, in.a, in.x0, in.x1);
  G.nz = a.nz;
  P.zero_t();
#pragma unroll
  for (int i = 0; i < K; ++i) {
    P.setT(L::idx(i, 0), in.T[2 * i]);
    if (L::plane(i)) P.setT(L::idx(i, 1), in.T[2 * i + 1]);
    tin[i] = in.T[2 * i + 1];
  }
  if (OP == OP_VJP)
    P.eval_entry(G);
  else
    P.eval(G, P.g);
}

// Stage 3: classification at the returned T, outputs and (VJP ops) the
// implicit VJP.
template <typename R, int K, unsigned MASK, int OP>
__device__ __forceinline__ void finish_path(const PathArgs<R>& a, int64_t row, const Rec<R, K>& in,
                                            bool has_v, int tid, bool staged, unsigned char* slab,
                                            const Geo<R, K>& G, const PathState<R, K, MASK>& P,
                                            const R (&tin)[K], uint8_t st) {
  using L = Lay<K, MASK>;
  st |= final_status<R, K, MASK>(G, P);
  bool fin = (st & FP_STATUS_NONFINITE) == 0;

  R tf[K][2];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    tf[i][0] = P.T(L::idx(i, 0));
    tf[i][1] = L::plane(i) ? P.T(L::idx(i, 1)) : tin[i];
  }
  const Outs<R> o = make_outs<R, K, OP>(a, row, tid, staged, slab);
  if (OP != OP_VJP) {
    if (o.T)
#pragma unroll
      for (int i = 0; i < K; ++i) {
        o.T[2 * i] = tf[i][0];
        o.T[2 * i + 1] = tf[i][1];
      }
    if (o.g)
#pragma unroll
      for (int i = 0; i < K; ++i) {
        o.g[2 * i] = P.Gr(L::idx(i, 0));
        o.g[2 * i + 1] = L::plane(i) ? P.Gr(L::idx(i, 1)) : R(0);
      }
    if (o.pts) {
      R X[K + 2][3];
      P.points(G, X);
#pragma unroll
      for (int i = 0; i < K; ++i)
#pragma unroll
        for (int r = 0; r < 3; ++r) o.pts[3 * i + r] = X[i + 1][r];
    }
    if (o.len) o.len[0] = P.length();
  }
  if (OP != OP_SOLVE) {
    R vf[K][2];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      vf[i][0] = in.v[2 * i];
      vf[i][1] = in.v[2 * i + 1];
    }
    const R wl = a.wL ? a.wL[row] : a.wL_scale;
    const bool full = a.mode == FP_VJP_FULL;
    const bool mixed = a.mode == FP_VJP_MIXED;
    const bool need_solve = !mixed && (has_v || (full && wl != R(0)));
    SceneGrad<R, K> sg;
    st |= implicit_vjp<R, K, MASK>(G, P, tf, vf, wl, full, need_solve, mixed, sg);
#pragma unroll
    for (int i = 0; i < K; ++i) {
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        fin = fin && finite(sg.da[i][r]) && finite(sg.db[i][r][0]) && finite(sg.db[i][r][1]);
        if (o.da) o.da[3 * i + r] = sg.da[i][r];
        if (o.db) {
          o.db[6 * i + 2 * r] = sg.db[i][r][0];
          o.db[6 * i + 2 * r + 1] = sg.db[i][r][1];
        }
      }
      if (o.u) {
        o.u[2 * i] = sg.u[i][0];
        o.u[2 * i + 1] = sg.u[i][1];
      }
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      fin = fin && finite(sg.d0[r]) && finite(sg.d1[r]);
      if (o.d0) o.d0[r] = sg.d0[r];
      if (o.d1) o.d1[r] = sg.d1[r];
    }
  }
  if (!fin) st |= FP_STATUS_NONFINITE;
  if (o.st) o.st[0] = st;
}

template <typename R, int K, unsigned MASK, int OP>
__device__ __forceinline__ void run_path(const PathArgs<R>& a, int64_t row, const Rec<R, K>& in,
                                         bool has_v, int tid, bool staged, unsigned char* slab) {
  Geo<R, K> G;
  PathState<R, K, MASK> P;
  R tin[K];
  begin_path<R, K, MASK, OP>(a, in, G, P, tin);
  uint8_t st = 0;
  if (OP != OP_VJP)
    st |= bfgs_solve<R, K, MASK>(G, P, a.iterations, a.fp_iters, a.trace_len, a.trace_gnorm,
                                 a.trace_fate, a.ld, row, a.H_out);
  finish_path<R, K, MASK, OP>(a, row, in, has_v, tid, staged, slab, G, P, tin, st);
}

// Two paths of the same kind mask through the paired loop (fp_pair.cuh):
// stages 1 and 3 per path, the BFGS iterations for both at once. Only the
// loop's common form (F = 1, no trace, no final H): the caller checks.
template <int K, unsigned MASK, int OP>
__device__ __forceinline__ void run_pair(const PathArgs<float>& a, int64_t rowa, int64_t rowb,
                                         const Rec<float, K>& ina, const Rec<float, K>& inb,
                                         bool has_v, int tida, int tidb, unsigned char* slab) {
  static_assert(OP != OP_VJP, "the VJP-only op has no loop");
  Geo<float, K> ga, gb;
  PathState<float, K, MASK> pa, pb;
  float tina[K], tinb[K];
  begin_path<float, K, MASK, OP>(a, ina, ga, pa, tina);
  begin_path<float, K, MASK, OP>(a, inb, gb, pb, tinb);
  // checked_segments (bfgs_solve)
  uint8_t sta = pa.min_norm() <= ga.eps ? FP_STATUS_DEGENERATE_ENTRY : 0;
  uint8_t stb = pb.min_norm() <= gb.eps ? FP_STATUS_DEGENERATE_ENTRY : 0;
  {
    GeoX<K> G;
    PairState<K, MASK> P;
    pack_pair<K, MASK>(ga, gb, pa, pb, G, P);
    bfgs_pair<K, MASK>(G, P, a.iterations, sta, stb);
    unpack_lane<K, MASK>(P, 0, pa);
    unpack_lane<K, MASK>(P, 1, pb);
  }
  pa.finish_norms(ga);
  pb.finish_norms(gb);
  finish_path<float, K, MASK, OP>(a, rowa, ina, has_v, tida, true, slab, ga, pa, tina, sta);
  finish_path<float, K, MASK, OP>(a, rowb, inb, has_v, tidb, true, slab, gb, pb, tinb, stb);
}

// ---- per-warp kind-mask dispatch (the "tile" kernels) -------------------------
// MASK == kAnyMask instantiates path_kernel with every specialised variant of
// order K inlined: each thread derives its path's kind mask from the staged
// record (bit i set when interaction i has a nonzero second basis column,
// geometry.py:74-77 — the classify_kernel rule) and runs that variant. Warps
// whose paths share a mask (ordering-major batches, every warp but the
// boundaries) run one variant; a mixed warp runs each lane's own variant under
// SIMT divergence, so a path's bits never depend on its neighbours. No
// classification pass, no host round trip, one launch.
constexpr unsigned kAnyMask = 0xFFFFFFFFu;

template <typename R, int K>
__device__ __forceinline__ unsigned rec_mask(const Rec<R, K>& in) {
  unsigned m = 0;
#pragma unroll
  for (int i = 0; i < K; ++i)
    m |= unsigned(in.b[6 * i + 1] != R(0) || in.b[6 * i + 3] != R(0) || in.b[6 * i + 5] != R(0)) << i;
  return m;
}

// Orders above kInlineTileMaxOrder keep each variant a separate (noinline)
// function: ptxas compiles 2^K inlined solvers in one function too slowly.
constexpr int kInlineTileMaxOrder = 3;

template <typename R, int K, int OP, unsigned M>
__device__ __noinline__ void run_variant(const PathArgs<R>& a, int64_t row, const Rec<R, K>& in,
                                         bool has_v, int tid, unsigned char* slab) {
  run_path<R, K, M, OP>(a, row, in, has_v, tid, true, slab);
}

template <typename R, int K, int OP, unsigned M = 0>
__device__ __forceinline__ void run_any_mask(unsigned m, const PathArgs<R>& a, int64_t row,
                                             const Rec<R, K>& in, bool has_v, int tid,
                                             unsigned char* slab) {
  if (m == M) {
    if constexpr (K <= kInlineTileMaxOrder)
      run_path<R, K, M, OP>(a, row, in, has_v, tid, true, slab);
    else
      run_variant<R, K, OP, M>(a, row, in, has_v, tid, slab);
    return;
  }
  if constexpr (M + 1 < (1u << K)) run_any_mask<R, K, OP, M + 1>(m, a, row, in, has_v, tid, slab);
}

template <int K, int OP, unsigned M = 0>
__device__ __forceinline__ void run_pair_any_mask(unsigned m, const PathArgs<float>& a, int64_t rowa,
                                                  int64_t rowb, const Rec<float, K>& ina,
                                                  const Rec<float, K>& inb, bool has_v, int tida,
                                                  int tidb, unsigned char* slab) {
  if (m == M) {
    run_pair<K, M, OP>(a, rowa, rowb, ina, inb, has_v, tida, tidb, slab);
    return;
  }
  if constexpr (M + 1 < (1u << K))
    run_pair_any_mask<K, OP, M + 1>(m, a, rowa, rowb, ina, inb, has_v, tida, tidb, slab);
}

// Copy `width`-element records of the tile from global to shared memory with
// asynchronous copies (cp.async, LDGSTS): every element's load is in flight
// at once instead of one load latency per loop trip. Gathered tiles move each
// record as a run of consecutive lanes (one or two cache lines per record).
// Completion: cp_async_wait_all() + __syncthreads() by the caller.
template <typename R>
__device__ __forceinline__ void cp_async_elem(R* dst, const R* src) {
  static_assert(sizeof(R) == 4 || sizeof(R) == 8, "4- or 8-byte elements");
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src),
               "n"(int(sizeof(R)))
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
template <typename R, int WD>
__device__ __forceinline__ void tile_in(R* dst, const R* src, const int32_t* srow, int64_t base, int n) {
  for (int e = threadIdx.x; e < n * WD; e += blockDim.x) {
    const int r = e / WD, c = e - r * WD;
    const int64_t row = srow ? int64_t(srow[r]) : base + r;
    cp_async_elem(dst + e, src + row * WD + c);
  }
}
template <typename R, int WD>
__device__ __forceinline__ void tile_out(R* dst, const R* src, const int32_t* srow, int64_t base, int n) {
  if (srow == nullptr) {
    for (int e = threadIdx.x; e < n * WD; e += blockDim.x) dst[base * WD + e] = src[e];
    return;
  }
  for (int e = threadIdx.x; e < n * WD; e += blockDim.x) {
    const int r = e / WD, c = e - r * WD;
    dst[int64_t(srow[r]) * WD + c] = src[e];
  }
}

// ---- one tile of up to kThreads paths ----------------------------------------
// Input slab pointers of a tile (see W).
template <typename R, int K, int OP>
struct InSlab {
  R *b, *a, *x0, *x1, *T, *v;
  __device__ __forceinline__ explicit InSlab(unsigned char* slab) {
    using Wk = W<K, OP>;
    b = reinterpret_cast<R*>(slab);
    a = b + kThreads * Wk::basis;
    x0 = a + kThreads * Wk::anchor;
    x1 = x0 + kThreads * 3;
    T = x1 + kThreads * 3;
    v = T + kThreads * Wk::T;
  }
};

// Can the full contiguous tile at `base` move with TMA bulk copies (every
// input / output run 16-byte aligned)?
template <typename R, int K, int OP>
__device__ __forceinline__ bool tile_in_aligned(const PathArgs<R>& a, int64_t base) {
  using Wk = W<K, OP>;
  return aligned16(a.basis + base * Wk::basis) && aligned16(a.anchor + base * Wk::anchor) &&
         aligned16(a.start + base * 3) && aligned16(a.end + base * 3) &&
         aligned16(a.T + base * Wk::T) && (!Wk::has_v || !a.vT || aligned16(a.vT + base * Wk::T));
}
template <typename R, int K, int OP>
__device__ __forceinline__ bool tile_out_aligned(const PathArgs<R>& a, int64_t base) {
  using Wk = W<K, OP>;
  return (!a.T_out || aligned16(a.T_out + base * Wk::T)) && (!a.g_out || aligned16(a.g_out + base * Wk::T)) &&
         (!a.points_out || aligned16(a.points_out + base * Wk::pts)) &&
         (!a.length_out || aligned16(a.length_out + base)) &&
         (!a.d_basis || aligned16(a.d_basis + base * Wk::basis)) &&
         (!a.d_anchor || aligned16(a.d_anchor + base * Wk::anchor)) &&
         (!a.d_start || aligned16(a.d_start + base * 3)) && (!a.d_end || aligned16(a.d_end + base * 3)) &&
         (!a.u_out || aligned16(a.u_out + base * Wk::T)) && (!a.status_out || aligned16(a.status_out + base));
}

// One thread: TMA bulk loads of a full aligned tile into `slab`, completing on `bar`.
template <typename R, int K, int OP>
__device__ __forceinline__ void tile_load_tma(const PathArgs<R>& a, int64_t base, unsigned char* slab,
                                              uint64_t* bar) {
  using Wk = W<K, OP>;
  const InSlab<R, K, OP> in(slab);
  const bool has_v = Wk::has_v && a.vT != nullptr;
  const uint32_t bb = kThreads * Wk::basis * sizeof(R), ba = kThreads * Wk::anchor * sizeof(R),
                 bv = kThreads * 3 * sizeof(R), bt = kThreads * Wk::T * sizeof(R);
  mbar_expect_tx(bar, bb + ba + 2 * bv + bt + (has_v ? bt : 0));
  bulk_g2s(in.b, a.basis + base * Wk::basis, bb, bar);
  bulk_g2s(in.a, a.anchor + base * Wk::anchor, ba, bar);
  bulk_g2s(in.x0, a.start + base * 3, bv, bar);
  bulk_g2s(in.x1, a.end + base * 3, bv, bar);
  bulk_g2s(in.T, a.T + base * Wk::T, bt, bar);
  if (has_v) bulk_g2s(in.v, a.vT + base * Wk::T, bt, bar);
}

// All threads: cp.async element copies of a partial / unaligned / gathered tile.
template <typename R, int K, int OP>
__device__ __forceinline__ void tile_load_async(const PathArgs<R>& a, const int32_t* srow, int64_t base,
                                                int n, unsigned char* slab) {
  using Wk = W<K, OP>;
  const InSlab<R, K, OP> in(slab);
  tile_in<R, Wk::basis>(in.b, a.basis, srow, base, n);
  tile_in<R, Wk::anchor>(in.a, a.anchor, srow, base, n);
  tile_in<R, 3>(in.x0, a.start, srow, base, n);
  tile_in<R, 3>(in.x1, a.end, srow, base, n);
  tile_in<R, Wk::T>(in.T, a.T, srow, base, n);
  if (Wk::has_v && a.vT) tile_in<R, Wk::T>(in.v, a.vT, srow, base, n);
  cp_async_wait_all();
}

// All threads, inputs staged in `slab`: each thread takes its record into
// registers, the slab is reused for the outputs, every path is solved (its
// own kind-mask variant under kAnyMask) and its results land in the slab.
// Ends with the slab complete and visible to the TMA (async) proxy.
template <typename R, int K, unsigned MASK, int OP>
__device__ __forceinline__ void tile_compute(const PathArgs<R>& a, const int32_t* srow, int64_t base,
                                             int n, unsigned char* slab) {
  using Wk = W<K, OP>;
  const int tid = threadIdx.x;
  const bool has_v = Wk::has_v && a.vT != nullptr;
  const InSlab<R, K, OP> sl(slab);
  Rec<R, K> in;
  if (tid < n)
    load_rec(in, sl.b + tid * Wk::basis, sl.a + tid * Wk::anchor, sl.x0 + tid * 3, sl.x1 + tid * 3,
             sl.T + tid * Wk::T, has_v ? sl.v + tid * Wk::T : nullptr);
  __syncthreads();
  if (tid < n) {
    const int64_t row = srow ? int64_t(srow[tid]) : base + tid;
    if constexpr (MASK == kAnyMask) {
      const unsigned m = rec_mask<R, K>(in);
      if (a.mixed_warps != nullptr) {
        const unsigned act = __activemask();
        if (__match_any_sync(act, m) != act && (tid & 31) == __ffs(act) - 1)
          atomicAdd(a.mixed_warps, 1ull);
      }
      run_any_mask<R, K, OP>(m, a, row, in, has_v, tid, slab);
    } else {
      run_path<R, K, MASK, OP>(a, row, in, has_v, tid, true, slab);
    }
  }
  fence_async_smem();  // make the slab writes visible to the TMA (async) proxy
  __syncthreads();
}

// Paired tile (kThreads / 2 threads): thread t takes the tile's paths t and
// t + kThreads / 2. When both exist, share a kind mask and the loop is the
// common form, they run the paired loop (run_pair); otherwise each runs its
// own per-path variant in turn. A path's bits are the same either way.
template <int K, int OP>
__device__ __forceinline__ void tile_compute_pair(const PathArgs<float>& a, const int32_t* srow,
                                                  int64_t base, int n, unsigned char* slab) {
  using Wk = W<K, OP>;
  constexpr int NT = kThreads / 2;
  const int ta = threadIdx.x, tb = threadIdx.x + NT;
  const bool has_v = Wk::has_v && a.vT != nullptr;
  const InSlab<float, K, OP> sl(slab);
  Rec<float, K> ra, rb;
  if (ta < n)
    load_rec(ra, sl.b + ta * Wk::basis, sl.a + ta * Wk::anchor, sl.x0 + ta * 3, sl.x1 + ta * 3,
             sl.T + ta * Wk::T, has_v ? sl.v + ta * Wk::T : nullptr);
  if (tb < n)
    load_rec(rb, sl.b + tb * Wk::basis, sl.a + tb * Wk::anchor, sl.x0 + tb * 3, sl.x1 + tb * 3,
             sl.T + tb * Wk::T, has_v ? sl.v + tb * Wk::T : nullptr);
  __syncthreads();
  if (ta < n) {
    const int64_t rowa = srow ? int64_t(srow[ta]) : base + ta;
    const unsigned ma = rec_mask<float, K>(ra);
    const bool two = tb < n;
    const unsigned mb = two ? rec_mask<float, K>(rb) : ma;
    if (a.mixed_warps != nullptr) {
      // one warp covers 64 paths: count it twice (the host's fraction is per 32 paths)
      const unsigned act = __activemask();
      const unsigned key = (two && ma != mb) ? 0xFFFFFFFFu : ma;
      if ((__match_any_sync(act, key) != act || key == 0xFFFFFFFFu) && (threadIdx.x & 31) == __ffs(act) - 1)
        atomicAdd(a.mixed_warps, 2ull);
    }
    const bool loop_common = a.fp_iters == 1 && a.trace_len == nullptr && a.H_out == nullptr;
    if (two && ma == mb && loop_common) {
      const int64_t rowb = srow ? int64_t(srow[tb]) : base + tb;
      run_pair_any_mask<K, OP>(ma, a, rowa, rowb, ra, rb, has_v, ta, tb, slab);
    } else {
      run_any_mask<float, K, OP>(ma, a, rowa, ra, has_v, ta, slab);
      if (two) {
        const int64_t rowb = srow ? int64_t(srow[tb]) : base + tb;
        run_any_mask<float, K, OP>(mb, a, rowb, rb, has_v, tb, slab);
      }
    }
  }
  fence_async_smem();
  __syncthreads();
}

// One thread: TMA bulk stores of a full aligned tile's output runs (committed
// as one bulk group; the caller waits for the reads before reusing the slab).
template <typename R, int K, int OP>
__device__ __forceinline__ void tile_store_tma(const PathArgs<R>& a, int64_t base, unsigned char* slab) {
  using Wk = W<K, OP>;
  R* sl = reinterpret_cast<R*>(slab);
  uint8_t* ost = slab + size_t(Wk::slab_elems) * kThreads * sizeof(R);
  constexpr uint32_t bT = kThreads * Wk::T * sizeof(R), bP = kThreads * Wk::pts * sizeof(R),
                     bL = kThreads * sizeof(R), bB = kThreads * Wk::basis * sizeof(R),
                     bA = kThreads * Wk::anchor * sizeof(R), bV = kThreads * 3 * sizeof(R);
  if (Wk::w_T && a.T_out) bulk_s2g(a.T_out + base * Wk::T, sl + kThreads * Wk::oT, bT);
  if (Wk::w_g && a.g_out) bulk_s2g(a.g_out + base * Wk::T, sl + kThreads * Wk::og, bT);
  if (Wk::w_pts && a.points_out) bulk_s2g(a.points_out + base * Wk::pts, sl + kThreads * Wk::oP, bP);
  if (Wk::w_len && a.length_out) bulk_s2g(a.length_out + base, sl + kThreads * Wk::oL, bL);
  if (Wk::w_grad && a.d_basis) bulk_s2g(a.d_basis + base * Wk::basis, sl + kThreads * Wk::oDB, bB);
  if (Wk::w_grad && a.d_anchor) bulk_s2g(a.d_anchor + base * Wk::anchor, sl + kThreads * Wk::oDA, bA);
  if (Wk::w_grad && a.d_start) bulk_s2g(a.d_start + base * 3, sl + kThreads * Wk::oD0, bV);
  if (Wk::w_grad && a.d_end) bulk_s2g(a.d_end + base * 3, sl + kThreads * Wk::oD1, bV);
  if (Wk::w_u && a.u_out) bulk_s2g(a.u_out + base * Wk::T, sl + kThreads * Wk::oU, bT);
  if (a.status_out) bulk_s2g(a.status_out + base, ost, kThreads);
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// All threads: cooperative (scattering) stores of a partial / gathered tile.
template <typename R, int K, int OP>
__device__ __forceinline__ void tile_store_coop(const PathArgs<R>& a, const int32_t* srow, int64_t base,
                                                int n, unsigned char* slab) {
  using Wk = W<K, OP>;
  R* sl = reinterpret_cast<R*>(slab);
  uint8_t* ost = slab + size_t(Wk::slab_elems) * kThreads * sizeof(R);
  if (Wk::w_T && a.T_out) tile_out<R, Wk::T>(a.T_out, sl + kThreads * Wk::oT, srow, base, n);
  if (Wk::w_g && a.g_out) tile_out<R, Wk::T>(a.g_out, sl + kThreads * Wk::og, srow, base, n);
  if (Wk::w_pts && a.points_out) tile_out<R, Wk::pts>(a.points_out, sl + kThreads * Wk::oP, srow, base, n);
  if (Wk::w_len && a.length_out) tile_out<R, 1>(a.length_out, sl + kThreads * Wk::oL, srow, base, n);
  if (Wk::w_grad && a.d_basis) tile_out<R, Wk::basis>(a.d_basis, sl + kThreads * Wk::oDB, srow, base, n);
  if (Wk::w_grad && a.d_anchor) tile_out<R, Wk::anchor>(a.d_anchor, sl + kThreads * Wk::oDA, srow, base, n);
  if (Wk::w_grad && a.d_start) tile_out<R, 3>(a.d_start, sl + kThreads * Wk::oD0, srow, base, n);
  if (Wk::w_grad && a.d_end) tile_out<R, 3>(a.d_end, sl + kThreads * Wk::oD1, srow, base, n);
  if (Wk::w_u && a.u_out) tile_out<R, Wk::T>(a.u_out, sl + kThreads * Wk::oU, srow, base, n);
  if (a.status_out) tile_out<uint8_t, 1>(a.status_out, ost, srow, base, n);
}

// One tile per CTA: stage inputs (TMA bulk copies for full aligned contiguous
// tiles, cp.async otherwise), compute in registers, stage the outputs and
// write them back (TMA bulk stores when full and aligned).
template <typename R, int K, unsigned MASK, int OP, bool PAIR = false>
__device__ __forceinline__ void process_tile(const PathArgs<R>& a, const int32_t* srow, int64_t base,
                                             int n, uint64_t* bar) {
  const int tid = threadIdx.x;
  unsigned char* slab = fp_smem;
  const bool full = srow == nullptr && n == kThreads;
  if (full && tile_in_aligned<R, K, OP>(a, base)) {
    if (tid == 0) mbar_init(bar, 1);
    __syncthreads();
    if (tid == 0) tile_load_tma<R, K, OP>(a, base, slab, bar);
    mbar_wait(bar, 0);
  } else {
    tile_load_async<R, K, OP>(a, srow, base, n, slab);
    __syncthreads();
  }
  if constexpr (PAIR)
    tile_compute_pair<K, OP>(a, srow, base, n, slab);
  else
    tile_compute<R, K, MASK, OP>(a, srow, base, n, slab);
  if (full && tile_out_aligned<R, K, OP>(a, base)) {
    if (tid == 0) {
      tile_store_tma<R, K, OP>(a, base, slab);
      bulk_wait_read_all();
    }
    return;
  }
  tile_store_coop<R, K, OP>(a, srow, base, n, slab);
}

// Minimum co-resident CTAs per SM requested from ptxas (caps registers at
// 65536 / (128 * n)). Measured on B200 at K = 3: 4 CTAs (<= 128 registers)
// beats ptxas' unconstrained choice (140-170 registers, 3 CTAs) by 7-10%;
// larger active sets get more registers. FP_MIN_BLOCKS overrides (A/B runs).
template <typename R, int NA>
struct MinBlocks {
#ifdef FP_MIN_BLOCKS
  static constexpr int value = FP_MIN_BLOCKS;
#else
  static constexpr int value = sizeof(R) == 8 ? 1 : (NA <= 6 ? 4 : (NA <= 8 ? 3 : 2));
#endif
};

// Tile kernels (MASK == kAnyMask): one register budget for all variants of
// the order. Measured on B200: order 1 runs 8 CTAs/SM (64 registers, no
// spills), order 2 runs 5 (96 registers), order 5 runs 3 (168 registers;
// its spills stay in L1) instead of the NA rule;
// FP_TILE_MIN_BLOCKS_K<k> overrides.
#ifndef FP_TILE_MIN_BLOCKS_K1
#define FP_TILE_MIN_BLOCKS_K1 8
#endif
#ifndef FP_TILE_MIN_BLOCKS_K2
#define FP_TILE_MIN_BLOCKS_K2 5
#endif
#ifndef FP_TILE_MIN_BLOCKS_K3
#define FP_TILE_MIN_BLOCKS_K3 4
#endif
#ifndef FP_TILE_MIN_BLOCKS_K4
#define FP_TILE_MIN_BLOCKS_K4 3
#endif
#ifndef FP_TILE_MIN_BLOCKS_K5
#define FP_TILE_MIN_BLOCKS_K5 3  // 2 before the per-op slab layout; 3: fused 2.230 -> 2.066 ms
#endif
// fp64 tile kernels (registers are pairs). Measured on B200 (tools/f64_ab.py,
// 2^20 paths, fused): uncapped (254 registers at K=3, 2 CTAs/SM) vs capped —
// K=1 6 CTAs 0.325 -> 0.319 ms, K=2 4 CTAs 0.680 -> 0.534 ms, K=3 3 CTAs
// 0.881 -> 0.853 ms (the spills stay in L1); K=4/5 uncapped is best.
#ifndef FP_TILE_MIN_BLOCKS_F64_K1
#define FP_TILE_MIN_BLOCKS_F64_K1 6
#endif
#ifndef FP_TILE_MIN_BLOCKS_F64_K2
#define FP_TILE_MIN_BLOCKS_F64_K2 4
#endif
#ifndef FP_TILE_MIN_BLOCKS_F64_K3
#define FP_TILE_MIN_BLOCKS_F64_K3 3
#endif
template <typename R, int K, unsigned MASK>
struct LaunchMin {
  static constexpr int value =
      MASK != kAnyMask ? MinBlocks<R, Lay<K, MASK>::NA>::value
      : sizeof(R) == 8 ? (K == 1   ? FP_TILE_MIN_BLOCKS_F64_K1
                          : K == 2 ? FP_TILE_MIN_BLOCKS_F64_K2
                          : K == 3 ? FP_TILE_MIN_BLOCKS_F64_K3
                                   : 1)
                       : (K == 1   ? FP_TILE_MIN_BLOCKS_K1
                          : K == 2 ? FP_TILE_MIN_BLOCKS_K2
                          : K == 3 ? FP_TILE_MIN_BLOCKS_K3
                          : K == 4 ? FP_TILE_MIN_BLOCKS_K4
                                   : FP_TILE_MIN_BLOCKS_K5);
};

// Paired tile kernels (fp32, kThreads / 2 threads, two paths per thread;
// fp_pair.cuh): CTAs per SM requested from ptxas. FP_PAIR_MIN_BLOCKS_K<k>
// overrides.
#ifndef FP_PAIR_MIN_BLOCKS_K1
#define FP_PAIR_MIN_BLOCKS_K1 8
#endif
#ifndef FP_PAIR_MIN_BLOCKS_K2
#define FP_PAIR_MIN_BLOCKS_K2 4
#endif
template <int K>
struct PairMin {
  static constexpr int value = K == 1 ? FP_PAIR_MIN_BLOCKS_K1 : K == 2 ? FP_PAIR_MIN_BLOCKS_K2 : 4;
};

template <typename R, int K, unsigned MASK, int OP, bool PAIR>
struct KernelShape {
  static constexpr int threads = PAIR ? kThreads / 2 : kThreads;
  static constexpr int min_blocks = PAIR ? PairMin<K>::value : LaunchMin<R, K, MASK>::value;
};

template <typename R, int K, unsigned MASK, int OP, bool PAIR = false>
__global__ void __launch_bounds__((KernelShape<R, K, MASK, OP, PAIR>::threads),
                                  (KernelShape<R, K, MASK, OP, PAIR>::min_blocks))
    path_kernel(const __grid_constant__ PathArgs<R> a) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ int32_t srow[kThreads];
  const int tid = threadIdx.x;
  if (a.rows != nullptr) {
    const int64_t t0 = int64_t(blockIdx.x) * kThreads;
    if (t0 >= a.n_rows) return;
    const int n = int(a.n_rows - t0 < kThreads ? a.n_rows - t0 : int64_t(kThreads));
    for (int i = tid; i < n; i += blockDim.x) srow[i] = a.rows[t0 + i];
    __syncthreads();
    process_tile<R, K, MASK, OP, PAIR>(a, srow, 0, n, &bar);
    return;
  }
  const int64_t base = a.row_begin + int64_t(blockIdx.x) * kThreads;
  if (base >= a.B) return;
  const int n = int(a.B - base < kThreads ? a.B - base : int64_t(kThreads));
  process_tile<R, K, MASK, OP, PAIR>(a, nullptr, base, n, &bar);
}

// Host-side launcher (defined per K in fp_inst.cu).
template <typename R, int K, unsigned MASK, int OP>
cudaError_t launch_path(const PathArgs<R>& a, cudaStream_t stream);

template <typename R, int K, unsigned MASK, int OP, bool PAIR = false>
cudaError_t launch_path_impl(const PathArgs<R>& a, cudaStream_t stream) {
  static_assert(!PAIR || (std::is_same<R, float>::value && MASK == kAnyMask && OP != OP_VJP),
                "paired kernels: fp32 tile solves only");
  const int64_t rows = a.rows ? a.n_rows : a.B - a.row_begin;
  if (rows <= 0) return cudaSuccess;
  constexpr size_t smem = smem_bytes<R, K, OP>();
  // The dynamic shared-memory attribute is per device: one bit per device
  // ordinal records that this instantiation was configured there.
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    e = cudaFuncSetAttribute(path_kernel<R, K, MASK, OP, PAIR>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit, std::memory_order_acq_rel);
  }
  const int64_t blocks = (rows + kThreads - 1) / kThreads;
  path_kernel<R, K, MASK, OP, PAIR>
      <<<dim3(unsigned(blocks)), dim3(KernelShape<R, K, MASK, OP, PAIR>::threads), smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace fp
