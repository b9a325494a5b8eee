// C ABI of the B200 Fermat path solver (include/fermat_b200.h).
//
// Validation mirrors the reference's host-side checks (SolveOptions
// iterations/fixed_point_iters >= 1, solver.py:51-55; interaction count
// bounds, geometry.py:23); everything per path is reported in status bytes.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <algorithm>
#include <vector>

#include "fp_bucket.h"
#include "fp_dispatch.h"
#include "fp_kernels.cuh"

namespace fp {

static std::atomic<uint64_t> g_launches{0};
static std::atomic<int> g_last_cuda{0};

void count_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return FP_OK;
  g_last_cuda.store(int(e));
  return FP_ERR_CUDA;
}

// ---- K = 0: no interactions (solver.py:160-164); length |end - start| ------
template <typename R>
__global__ void order0_kernel(const R* start, const R* end, int64_t B, R* length_out,
                              const R* wL, R wL_scale, R* d_start, R* d_end, uint8_t* status) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= B) return;
  R s[3];
  R q = R(0);
  for (int r = 0; r < 3; ++r) {
    s[r] = end[3 * b + r] - start[3 * b + r];
    q = fma(s[r], s[r], q);
  }
  const R n = Num<R>::sqrt_(q);
  if (length_out) length_out[b] = n;
  const R w = wL ? wL[b] : wL_scale;
  for (int r = 0; r < 3; ++r) {
    const R u = Num<R>::div(s[r], n);
    if (d_start) d_start[3 * b + r] = -w * u;
    if (d_end) d_end[3 * b + r] = w * u;
  }
  if (status) status[b] = finite(n) ? 0 : FP_STATUS_NONFINITE;
}

template <typename R>
static int run_order0(const R* start, const R* end, int64_t B, R* length_out, const R* wL,
                      R wL_scale, R* d_start, R* d_end, uint8_t* status, cudaStream_t s) {
  if (B == 0) return FP_OK;
  const int t = 256;
  order0_kernel<R><<<unsigned((B + t - 1) / t), t, 0, s>>>(start, end, B, length_out, wL, wL_scale,
                                                          d_start, d_end, status);
  count_launches(1);
  return cuda_status(cudaGetLastError());
}

static std::atomic<int> g_policy{FP_POLICY_AUTO};

template <typename R>
static int dispatch_dense_k(int K, const PathArgs<R>& a, int op, cudaStream_t s) {
  cudaError_t e;
  switch (K) {
    case 1: e = dispatch_dense<R, 1>(a, op, s); break;
    case 2: e = dispatch_dense<R, 2>(a, op, s); break;
    case 3: e = dispatch_dense<R, 3>(a, op, s); break;
    case 4: e = dispatch_dense<R, 4>(a, op, s); break;
    case 5: e = dispatch_dense<R, 5>(a, op, s); break;
    case 6: e = dispatch_dense<R, 6>(a, op, s); break;
    case 7: e = dispatch_dense<R, 7>(a, op, s); break;
    case 8: e = dispatch_dense<R, 8>(a, op, s); break;
    default:
      if (K > FP_MAX_ORDER) return FP_ERR_UNSUPPORTED_ORDER;
      e = dispatch_wide<R>(K, a, op, s);
      break;
  }
  if (a.B > 0) count_launches(1);
  return cuda_status(e);
}

static cudaError_t masked_k(int K, const PathArgs<float>& a, int op, unsigned m, cudaStream_t s) {
  const bool v = op == OP_SOLVE_VJP;
  switch (K) {
    case 1: return v ? dispatch_masked_solve_vjp<1>(a, m, s) : dispatch_masked_solve<1>(a, m, s);
    case 2: return v ? dispatch_masked_solve_vjp<2>(a, m, s) : dispatch_masked_solve<2>(a, m, s);
    case 3: return v ? dispatch_masked_solve_vjp<3>(a, m, s) : dispatch_masked_solve<3>(a, m, s);
    case 4: return v ? dispatch_masked_solve_vjp<4>(a, m, s) : dispatch_masked_solve<4>(a, m, s);
    case 5: return v ? dispatch_masked_solve_vjp<5>(a, m, s) : dispatch_masked_solve<5>(a, m, s);
    default: return cudaErrorInvalidValue;
  }
}

// ---- tile kernels and their layout probe ------------------------------------
// The tile kernel (order <= kMaxTileOrder) counts warps whose paths carry
// different kind masks; that count comes back asynchronously (pinned copy +
// event, read by a later call once the event has completed — no sync). The
// bucketed path learns the same number from its classification. AUTO keeps
// using the tile kernel while the last known mixed fraction is small.
constexpr int kMaxTileOrder = 5;
#ifndef FP_AUTO_TILE_MAX_ORDER
#define FP_AUTO_TILE_MAX_ORDER 5
#endif
constexpr int kAutoTileMaxOrder = FP_AUTO_TILE_MAX_ORDER;  // orders AUTO sends to the tile kernel
constexpr double kMaxMixedFraction = 0.125;

// Probe the layout on every tile call of an order whose previous probe has
// come back (a counter the kernel bumps per mixed-mask warp, read back by a
// one-thread kernel): a change to a scattered layout costs one divergent
// call, not up to kProbeEvery of them (fp64 order 5: ~30x the sorted time
// each). Calls enqueued while a probe is in flight launch the kernel alone.
constexpr int kProbeEvery = 1;

struct LayoutProbe {
  std::mutex mu;
  bool init[kMaxTileOrder + 1] = {};
  bool pending[kMaxTileOrder + 1] = {};
  cudaEvent_t ev[kMaxTileOrder + 1];
  unsigned long long* host = nullptr;  // pinned, one slot per order
  unsigned long long* dev = nullptr;   // device counters, one per order
  int64_t warps[kMaxTileOrder + 1] = {};
  double frac[kMaxTileOrder + 1] = {};
  int since[kMaxTileOrder + 1] = {};   // tile calls since the last probe
};
// One probe per device: its counters, pinned slots and events belong to the
// device the tile kernels run on, and each device sees its own layouts.
constexpr int kMaxDevices = 64;
static LayoutProbe& probe() {
  static LayoutProbe p[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return p[dev];
}

static bool tile_preferred(int K) {
  LayoutProbe& p = probe();
  std::lock_guard<std::mutex> lk(p.mu);
  if (p.pending[K] && cudaEventQuery(p.ev[K]) == cudaSuccess) {
    p.frac[K] = p.warps[K] ? double(p.host[K]) / double(p.warps[K]) : 0.0;
    p.pending[K] = false;
  }
  return p.frac[K] <= kMaxMixedFraction;
}

static void record_mixed_fraction(int K, int64_t mixed, int64_t B) {
  if (K > kMaxTileOrder) return;
  LayoutProbe& p = probe();
  std::lock_guard<std::mutex> lk(p.mu);
  p.frac[K] = B > 0 ? double(mixed) / double((B + 31) / 32) : 0.0;
  p.pending[K] = false;
}

__global__ void publish_counter(unsigned long long* dev, volatile unsigned long long* host) {
  *host = *dev;
  *dev = 0;
}

template <typename R>
static cudaError_t run_tile(int K, const PathArgs<R>& a0, int op, cudaStream_t s) {
  PathArgs<R> a = a0;
  LayoutProbe& p = probe();
  cudaError_t e = cudaSuccess;
  bool probing = false;
  {
    std::lock_guard<std::mutex> lk(p.mu);
    if (!p.init[K]) {
      if (p.host == nullptr)
        e = cudaMallocHost(&p.host, sizeof(unsigned long long) * (kMaxTileOrder + 1));
      if (e == cudaSuccess && p.dev == nullptr) {
        e = cudaMalloc(&p.dev, sizeof(unsigned long long) * (kMaxTileOrder + 1));
        if (e == cudaSuccess) e = cudaMemset(p.dev, 0, sizeof(unsigned long long) * (kMaxTileOrder + 1));
      }
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.ev[K], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
      p.init[K] = true;
      p.since[K] = kProbeEvery;
    }
    // (a permuted launch says nothing about the caller's layout: no probe)
    probing = a.rows == nullptr && !p.pending[K] && ++p.since[K] >= kProbeEvery;
    if (probing) {
      p.since[K] = 0;
      a.mixed_warps = p.dev + K;  // zero here: publish_counter resets it
    }
  }
  switch (K) {
    case 1: e = dispatch_tile<R, 1>(a, op, s); break;
    case 2: e = dispatch_tile<R, 2>(a, op, s); break;
    case 3: e = dispatch_tile<R, 3>(a, op, s); break;
    case 4: e = dispatch_tile<R, 4>(a, op, s); break;
    default: e = dispatch_tile<R, 5>(a, op, s); break;
  }
  count_launches(1);
  if (e == cudaSuccess && probing) {
    std::lock_guard<std::mutex> lk(p.mu);
    // A one-thread kernel stores the counter into the pinned (UVA-mapped) host
    // slot: a device-to-host memcpy would queue behind every copy already on
    // the copy engine (the host-buffer pipeline's outputs) and stall this stream.
    publish_counter<<<1, 1, 0, s>>>(p.dev + K, p.host + K);
    count_launches(1);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaEventRecord(p.ev[K], s);
    p.warps[K] = (a.B - a.row_begin + 31) / 32;
    p.pending[K] = e == cudaSuccess;
  }
  return e;
}

// Solve / fused step for K <= 5. Tile path (see run_tile; fp32 and fp64), or
// bucketed (fp32): classify paths by kind mask on the device, then one
// specialised kernel per non-empty mask (the staged TMA kernel on the mask's
// row range when it is contiguous, the gathering kernel over a row
// permutation otherwise) on side streams so tails overlap. fp64 batches with
// a scattered layout run the dense kernel.
// Routes: any kernel the policy picks; never one that synchronises the
// stream (tile or dense, for enqueue loops like the host-buffer pipeline);
// dense only.
enum Route { kRouteAny = 0, kRouteNoSync = 1, kRouteDense = 2 };

template <typename R>
static int dispatch(int K, const PathArgs<R>& a, int op, cudaStream_t s, int route = kRouteAny) {
  constexpr bool is_f32 = sizeof(R) == sizeof(float);
  const int64_t B = a.B;
  const int policy = g_policy.load();
  const bool special = route != kRouteDense && policy != FP_POLICY_DENSE && K >= 1 &&
                       K <= kMaxSpecialisedOrder && (op == OP_SOLVE || op == OP_SOLVE_VJP) &&
                       B > 0 && B < (int64_t(1) << 31) && a.rows == nullptr;
  if (!special) return dispatch_dense_k<R>(K, a, op, s);
  const bool tile = (K <= kMaxTileOrder && policy == FP_POLICY_TILE) ||
                    (K <= kAutoTileMaxOrder && policy == FP_POLICY_AUTO &&
                     (route == kRouteNoSync || tile_preferred(K)));
  if (tile) return cuda_status(run_tile<R>(K, a, op, s));
  if (route == kRouteNoSync || K > kMaxTileOrder) return dispatch_dense_k<R>(K, a, op, s);
  if (!is_f32 || (policy == FP_POLICY_AUTO && K <= kAutoTileMaxOrder)) {
    // Scattered layout under AUTO (and fp64 under every bucketed policy):
    // classify, sort the rows by kind mask, and run the tile kernel over that
    // permutation, so warps are uniform and each path still runs its own
    // mask's variant (bitwise what the tile kernel gives it in any layout;
    // never the dense kernel, whose rounding differs). One launch, no
    // per-mask tails.
    BucketScratch sc;
    BucketPlan plan;
    cudaError_t e = bucket_plan<R>(a.basis, B, K, sc, plan, s);
    if (e == cudaSuccess) record_mixed_fraction(K, plan.mixed_warps, B);
    if (e == cudaSuccess && !plan.all_contiguous) e = bucket_scatter(B, plan, sc, s);
    if (e == cudaSuccess) {
      PathArgs<R> b = a;
      if (!plan.all_contiguous) {
        b.rows = sc.rows;
        b.n_rows = B;
      }
      e = run_tile<R>(K, b, op, s);
    }
    bucket_free(sc, s);
    return cuda_status(e);
  }
  if constexpr (is_f32) {
    BucketScratch sc;
    BucketPlan plan;
    cudaError_t e = bucket_plan<float>(a.basis, B, K, sc, plan, s);
    if (e == cudaSuccess) record_mixed_fraction(K, plan.mixed_warps, B);
    if (e == cudaSuccess && !plan.all_contiguous) e = bucket_scatter(B, plan, sc, s);
    int live = 0;
    for (int m = 0; m < plan.nb; ++m) live += plan.count[m] > 0;
    SideStreams& ss = side_streams();
    const bool fan = live > 1 && g_policy.load() != FP_POLICY_AUTO_SERIAL;
    // the device's side streams serve one caller at a time, fork through join
    std::unique_lock<std::mutex> fan_lock(ss.mu, std::defer_lock);
    if (fan) fan_lock.lock();
    if (e == cudaSuccess && fan) e = ss.fork(s, live);
    int k = 0;
    for (unsigned m = 0; m < unsigned(plan.nb) && e == cudaSuccess; ++m) {
      if (plan.count[m] == 0) continue;
      PathArgs<float> b = a;
      if (plan.contiguous[m]) {
        b.row_begin = plan.lo[m];
        b.B = plan.hi[m] + 1;
      } else {
        b.rows = sc.rows + plan.offset[m];
        b.n_rows = plan.count[m];
      }
      cudaStream_t st = fan ? ss.st[k++ % SideStreams::kSide] : s;
      e = masked_k(K, b, op, m, st);
      count_launches(1);
    }
    if (e == cudaSuccess && fan) e = ss.join(s);
    bucket_free(sc, s);
    return cuda_status(e);
  }
  return FP_ERR_INVALID_ARGUMENT;
}

template <typename R>
static PathArgs<R> blank_args() {
  PathArgs<R> a;
  std::memset(&a, 0, sizeof(a));
  a.nz = R(-0.0);
  return a;
}

template <typename R>
static void finish_args(PathArgs<R>& a) {
  a.row_begin = 0;
  a.ld = a.B;
}

template <typename R>
static int solve_impl(const R* basis, const R* anchor, const R* start, const R* end, const R* T0,
                      int64_t B, int K, int iterations, int fp_iters, R* T_out, R* g_out,
                      R* points_out, R* length_out, uint8_t* status_out, R* trace_len,
                      R* trace_gnorm, uint8_t* trace_fate, R* H_out, void* stream) {
  if (B < 0 || iterations < 1 || fp_iters < 1) return FP_ERR_INVALID_ARGUMENT;
  if (K < 0 || K > FP_MAX_ORDER) return FP_ERR_UNSUPPORTED_ORDER;
  if ((trace_len == nullptr) != (trace_gnorm == nullptr)) return FP_ERR_INVALID_ARGUMENT;
  if (trace_fate != nullptr && trace_len == nullptr) return FP_ERR_INVALID_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (K == 0) {
    if (B > 0 && (start == nullptr || end == nullptr)) return FP_ERR_INVALID_ARGUMENT;
    return run_order0<R>(start, end, B, length_out, nullptr, R(0), nullptr, nullptr, status_out, s);
  }
  if (B > 0 && (!basis || !anchor || !start || !end || !T0)) return FP_ERR_INVALID_ARGUMENT;
  PathArgs<R> a = blank_args<R>();
  a.basis = basis; a.anchor = anchor; a.start = start; a.end = end; a.T = T0;
  a.B = B; a.iterations = iterations; a.fp_iters = fp_iters;
  a.T_out = T_out; a.g_out = g_out; a.points_out = points_out; a.length_out = length_out;
  a.status_out = status_out; a.trace_len = trace_len; a.trace_gnorm = trace_gnorm; a.H_out = H_out;
  a.trace_fate = trace_fate;
  finish_args(a);
  return dispatch<R>(K, a, OP_SOLVE, s);
}

template <typename R>
static int vjp_impl(const R* basis, const R* anchor, const R* start, const R* end, const R* T,
                    const R* v_T, const R* w_L, R w_L_scale, int mode, int64_t B, int K, R* d_basis,
                    R* d_anchor, R* d_start, R* d_end, R* u_out, uint8_t* status_out, void* stream) {
  if (B < 0) return FP_ERR_INVALID_ARGUMENT;
  if (mode != FP_VJP_FULL && mode != FP_VJP_ENVELOPE && mode != FP_VJP_MIXED)
    return FP_ERR_UNSUPPORTED_MODE;
  if (K < 0 || K > FP_MAX_ORDER) return FP_ERR_UNSUPPORTED_ORDER;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (K == 0)
    return run_order0<R>(start, end, B, nullptr, w_L, w_L_scale, d_start, d_end, status_out, s);
  if (B > 0 && (!basis || !anchor || !start || !end || !T)) return FP_ERR_INVALID_ARGUMENT;
  PathArgs<R> a = blank_args<R>();
  a.basis = basis; a.anchor = anchor; a.start = start; a.end = end; a.T = T; a.vT = v_T;
  a.wL = w_L; a.wL_scale = w_L_scale; a.mode = mode; a.B = B; a.iterations = 1; a.fp_iters = 1;
  a.d_basis = d_basis; a.d_anchor = d_anchor; a.d_start = d_start; a.d_end = d_end;
  a.u_out = u_out; a.status_out = status_out;
  finish_args(a);
  return dispatch<R>(K, a, OP_VJP, s);
}

template <typename R>
static int solve_vjp_impl(const R* basis, const R* anchor, const R* start, const R* end,
                          const R* T0, int64_t B, int K, int iterations, int fp_iters, const R* w_L,
                          R w_L_scale, int mode, R* T_out, R* points_out, R* length_out, R* d_basis,
                          R* d_anchor, R* d_start, R* d_end, uint8_t* status_out, cudaStream_t s,
                          int route = kRouteAny) {
  if (B < 0 || iterations < 1 || fp_iters < 1) return FP_ERR_INVALID_ARGUMENT;
  if (mode != FP_VJP_FULL && mode != FP_VJP_ENVELOPE) return FP_ERR_UNSUPPORTED_MODE;
  if (K < 0 || K > FP_MAX_ORDER) return FP_ERR_UNSUPPORTED_ORDER;
  if (K == 0)
    return run_order0<R>(start, end, B, length_out, w_L, w_L_scale, d_start, d_end, status_out, s);
  if (B > 0 && (!basis || !anchor || !start || !end || !T0)) return FP_ERR_INVALID_ARGUMENT;
  PathArgs<R> a = blank_args<R>();
  a.basis = basis; a.anchor = anchor; a.start = start; a.end = end; a.T = T0;
  a.wL = w_L; a.wL_scale = w_L_scale; a.mode = mode;
  a.B = B; a.iterations = iterations; a.fp_iters = fp_iters;
  a.T_out = T_out; a.points_out = points_out; a.length_out = length_out;
  a.d_basis = d_basis; a.d_anchor = d_anchor; a.d_start = d_start; a.d_end = d_end;
  a.status_out = status_out;
  finish_args(a);
  return dispatch<R>(K, a, OP_SOLVE_VJP, s, route);
}

// ---- generic-order helpers (scalar API; any K <= 64) ------------------------
constexpr int kGenMax = 64;

// objective.path_length / gradient / hessian with unclamped norms.
template <typename R>
__global__ void objective_kernel(const R* basis, const R* anchor, const R* start, const R* end,
                                 const R* T, int64_t B, int K, R* length_out, R* grad_out,
                                 R* hess_out, uint8_t* status) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const R* A = basis + b * 6 * K;
  R P[kGenMax + 2][3];
  for (int r = 0; r < 3; ++r) {
    P[0][r] = start[3 * b + r];
    P[K + 1][r] = end[3 * b + r];
  }
  for (int i = 0; i < K; ++i)
    for (int r = 0; r < 3; ++r)
      P[i + 1][r] = fma(A[6 * i + 2 * r + 1], T[b * 2 * K + 2 * i + 1],
                        A[6 * i + 2 * r] * T[b * 2 * K + 2 * i]) + anchor[b * 3 * K + 3 * i + r];
  const double dx = double(P[K + 1][0]) - double(P[0][0]), dy = double(P[K + 1][1]) - double(P[0][1]),
               dz = double(P[K + 1][2]) - double(P[0][2]);
  const R eps = R(1e-12 * (1.0 + sqrt(dz * dz + (dy * dy + dx * dx))));
  R u[kGenMax + 1][3], n[kGenMax + 1];
  R L = R(0);
  uint8_t st = 0;
  for (int k = 0; k <= K; ++k) {
    R q = R(0);
    for (int r = 0; r < 3; ++r) {
      u[k][r] = P[k + 1][r] - P[k][r];
      q = fma(u[k][r], u[k][r], q);
    }
    n[k] = Num<R>::sqrt_(q);
    L += n[k];
    if (n[k] <= eps) st |= FP_STATUS_DEGENERATE_FINAL;
    for (int r = 0; r < 3; ++r) u[k][r] = Num<R>::div(u[k][r], n[k]);
  }
  if (length_out) length_out[b] = L;
  if (grad_out)
    for (int i = 0; i < K; ++i)
      for (int c = 0; c < 2; ++c) {
        R acc = R(0);
        for (int r = 0; r < 3; ++r) acc = fma(A[6 * i + 2 * r + c], u[i][r] - u[i + 1][r], acc);
        grad_out[b * 2 * K + 2 * i + c] = acc;
      }
  if (hess_out) {
    const int m = 2 * K;
    R* H = hess_out + b * m * m;
    for (int e = 0; e < m * m; ++e) H[e] = R(0);
    // block(i, j) = A_i^T M_k A_j with M_k = (I - u_k u_k^T) / n_k
    auto amb = [&](int i, int j, int k, int ci, int cj) {
      R au_i = R(0), au_j = R(0), aa = R(0);
      for (int r = 0; r < 3; ++r) {
        au_i = fma(A[6 * i + 2 * r + ci], u[k][r], au_i);
        au_j = fma(A[6 * j + 2 * r + cj], u[k][r], au_j);
        aa = fma(A[6 * i + 2 * r + ci], A[6 * j + 2 * r + cj], aa);
      }
      return Num<R>::div(aa - au_i * au_j, n[k]);
    };
    for (int i = 0; i < K; ++i)
      for (int ci = 0; ci < 2; ++ci)
        for (int cj = 0; cj < 2; ++cj) {
          H[(2 * i + ci) * m + 2 * i + cj] = amb(i, i, i, ci, cj) + amb(i, i, i + 1, ci, cj);
          if (i + 1 < K) {
            const R off = -amb(i, i + 1, i + 1, ci, cj);
            H[(2 * i + ci) * m + 2 * (i + 1) + cj] = off;
            H[(2 * (i + 1) + cj) * m + 2 * i + ci] = off;
          }
        }
  }
  if (status) status[b] = st | (finite(L) ? 0 : FP_STATUS_NONFINITE);
}

// solver.line_search_alpha with caller alpha0 and k iterations (unclamped
// denominators: a collapsed one reports FP_STATUS_DEGENERATE_ENTRY).
template <typename R>
__global__ void line_search_kernel(const R* basis, const R* anchor, const R* start, const R* end,
                                   const R* T, const R* Pd, const R* alpha0, int64_t B, int K,
                                   int k_iters, R* alpha_out, uint8_t* status) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const R* A = basis + b * 6 * K;
  R X[kGenMax + 2][3], Wd[kGenMax + 2][3];
  for (int r = 0; r < 3; ++r) {
    X[0][r] = start[3 * b + r];
    X[K + 1][r] = end[3 * b + r];
    Wd[0][r] = Wd[K + 1][r] = R(0);
  }
  for (int i = 0; i < K; ++i)
    for (int r = 0; r < 3; ++r) {
      const R* t = T + b * 2 * K + 2 * i;
      const R* p = Pd + b * 2 * K + 2 * i;
      X[i + 1][r] = fma(A[6 * i + 2 * r + 1], t[1], A[6 * i + 2 * r] * t[0]) + anchor[b * 3 * K + 3 * i + r];
      Wd[i + 1][r] = fma(A[6 * i + 2 * r + 1], p[1], A[6 * i + 2 * r] * p[0]);
    }
  const double dx = double(X[K + 1][0]) - double(X[0][0]), dy = double(X[K + 1][1]) - double(X[0][1]),
               dz = double(X[K + 1][2]) - double(X[0][2]);
  const R eps = R(1e-12 * (1.0 + sqrt(dz * dz + (dy * dy + dx * dx))));
  uint8_t st = 0;
  R total = R(0);
  for (int k = 0; k <= K; ++k) {
    R q = R(0), a2 = R(0);
    for (int r = 0; r < 3; ++r) {
      const R s = X[k + 1][r] - X[k][r];
      const R d = Wd[k + 1][r] - Wd[k][r];
      q = fma(s, s, q);
      a2 = fma(d, d, a2);
    }
    if (Num<R>::sqrt_(q) <= eps) st |= FP_STATUS_DEGENERATE_ENTRY;
    total += a2;
  }
  R alpha = alpha0 ? alpha0[b] : R(0);
  if (total <= Num<R>::tiny()) {
    st |= FP_STATUS_ZERO_DIRECTION;
  } else if (!(st & FP_STATUS_DEGENERATE_ENTRY)) {
    for (int it = 0; it < k_iters; ++it) {
      R num = R(0), den = R(0);
      for (int k = 0; k <= K; ++k) {
        R c = R(0), a2 = R(0), q = R(0);
        for (int r = 0; r < 3; ++r) {
          const R s = X[k + 1][r] - X[k][r];
          const R d = Wd[k + 1][r] - Wd[k][r];
          const R e = fma(alpha, d, s);
          c = fma(d, s, c);
          a2 = fma(d, d, a2);
          q = fma(e, e, q);
        }
        const R n = Num<R>::sqrt_(q);
        if (n <= eps) st |= FP_STATUS_DEGENERATE_ENTRY;
        num += Num<R>::div(c, n);
        den += Num<R>::div(a2, n);
      }
      if (st & FP_STATUS_DEGENERATE_ENTRY) break;
      alpha = -Num<R>::div(num, den);
    }
  }
  alpha_out[b] = alpha;
  if (status) status[b] = st;
}

// solver.init_params: least-squares projection of the start/end midpoint onto
// each surface's active span (2x2 or 1x1 normal equations).
template <typename R>
__global__ void init_params_kernel(const R* basis, const R* anchor, const R* start, const R* end,
                                   int64_t B, int K, R* T_out) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= B * K) return;
  const int64_t b = idx / K;
  const int i = int(idx % K);
  const R* A = basis + b * 6 * K + 6 * i;
  R mid[3], c0[3], c1[3];
  for (int r = 0; r < 3; ++r) {
    mid[r] = R(0.5) * (start[3 * b + r] + end[3 * b + r]) - anchor[b * 3 * K + 3 * i + r];
    c0[r] = A[2 * r];
    c1[r] = A[2 * r + 1];
  }
  const bool a0 = c0[0] != R(0) || c0[1] != R(0) || c0[2] != R(0);
  const bool a1 = c1[0] != R(0) || c1[1] != R(0) || c1[2] != R(0);
  R g00 = 0, g01 = 0, g11 = 0, r0 = 0, r1 = 0;
  for (int r = 0; r < 3; ++r) {
    g00 = fma(c0[r], c0[r], g00);
    g01 = fma(c0[r], c1[r], g01);
    g11 = fma(c1[r], c1[r], g11);
    r0 = fma(c0[r], mid[r], r0);
    r1 = fma(c1[r], mid[r], r1);
  }
  R t0 = R(0), t1 = R(0);
  if (a0 && a1) {
    const R det = g00 * g11 - g01 * g01;
    t0 = Num<R>::div(g11 * r0 - g01 * r1, det);
    t1 = Num<R>::div(g00 * r1 - g01 * r0, det);
  } else if (a0) {
    t0 = Num<R>::div(r0, g00);
  } else if (a1) {
    t1 = Num<R>::div(r1, g11);
  }
  T_out[b * 2 * K + 2 * i] = t0;
  T_out[b * 2 * K + 2 * i + 1] = t1;
}

// ---- host-buffer pipeline for the fused step ---------------------------------
// Three streams: copy-in, compute, copy-out. A ring of `depth` chunk slots,
// each with an input region and an output region on the device; cross-stream
// events order only what shares memory:
//   copy-in  of chunk c  waits for the kernel of chunk c - depth (input region free)
//   kernel   of chunk c  waits for its copy-in and for the copy-out of c - depth
//   copy-out of chunk c  waits for its kernel
// so host-to-device copies run ahead of the device-to-host ones instead of
// queueing behind them (one stream per slot serialises the two directions).
struct HostPipe {
  std::mutex mu;
  cudaStream_t s_in = nullptr, s_k = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_k, ev_out;
  std::vector<void*> bufs;
  size_t buf_bytes = 0;
  int device = -1;
  int64_t chunks = 0;   // chunks enqueued since setup: the ring position carries across calls
  uint64_t layout = 0;  // slot layout of the last call (order, chunk, element size)
  // Completion of submitted calls: ticket t records on job_ev[t % kJobs];
  // at most kJobs calls are in flight (a submit first waits for ticket t - kJobs).
  static constexpr int kJobs = 16;
  cudaEvent_t job_ev[kJobs] = {};
  uint64_t next_ticket = 1;
  void drain() {
    for (cudaStream_t s : {s_in, s_k, s_out})
      if (s) cudaStreamSynchronize(s);
  }
  void release() {
    drain();
    for (void* p : bufs) cudaFree(p);
    for (auto* v : {&ev_in, &ev_k, &ev_out})
      for (cudaEvent_t e : *v) cudaEventDestroy(e);
    for (cudaStream_t s : {s_in, s_k, s_out})
      if (s) cudaStreamDestroy(s);
    bufs.clear();
    ev_in.clear();
    ev_k.clear();
    ev_out.clear();
    s_in = s_k = s_out = nullptr;
    buf_bytes = 0;
    device = -1;
    chunks = 0;
    layout = 0;
  }
  cudaError_t setup(int dev, int depth, size_t slot) {
    release();
    cudaError_t e;
    for (cudaStream_t* s : {&s_in, &s_k, &s_out})
      if ((e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking)) != cudaSuccess) return e;
    for (int i = 0; i < depth; ++i) {
      for (auto* v : {&ev_in, &ev_k, &ev_out}) {
        cudaEvent_t ev;
        if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
        v->push_back(ev);
      }
      void* p = nullptr;
      if ((e = cudaMalloc(&p, slot)) != cudaSuccess) return e;
      bufs.push_back(p);
    }
    buf_bytes = slot;
    device = dev;
    return cudaSuccess;
  }
};
// One pipeline per device (streams, slots and events live on that device);
// tickets carry the device ordinal in their top byte.
static HostPipe g_pipes[kMaxDevices];
constexpr int kTicketShift = 56;

// The copies of one chunk in one direction, one cudaMemcpyAsync per array.
static cudaError_t copy_arrays(void** dst, void** src, size_t* bytes, size_t n, cudaMemcpyKind kind,
                               cudaStream_t s) {
  for (size_t i = 0; i < n; ++i) {
    cudaError_t e = cudaMemcpyAsync(dst[i], src[i], bytes[i], kind, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <typename R>
static int host_submit(const R* basis, const R* anchor, const R* start, const R* end, const R* T0,
                       int64_t B, int K, int iterations, int fp_iters, R w_L_scale, int mode,
                       R* T_out, R* points_out, R* length_out, R* d_basis, R* d_anchor,
                       R* d_start, R* d_end, uint8_t* status_out, int64_t chunk, int depth,
                       uint64_t* ticket) {
  if (ticket) *ticket = 0;  // 0: nothing in flight
  if (B < 0 || iterations < 1 || fp_iters < 1 || depth < 1 || depth > 8)
    return FP_ERR_INVALID_ARGUMENT;
  if (mode != FP_VJP_FULL && mode != FP_VJP_ENVELOPE) return FP_ERR_UNSUPPORTED_MODE;
  if (K < 0 || K > FP_MAX_ORDER) return FP_ERR_UNSUPPORTED_ORDER;
  if (B == 0) return FP_OK;
  // Required inputs (the same contract as the device entries); T0 == NULL
  // means zero initialisation, done on the device (no host-to-device copy).
  if (start == nullptr || end == nullptr) return FP_ERR_INVALID_ARGUMENT;
  if (K > 0 && (basis == nullptr || anchor == nullptr)) return FP_ERR_INVALID_ARGUMENT;
  if (chunk <= 0) chunk = 1 << 18;
  chunk = (chunk + kThreads - 1) / kThreads * kThreads;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e);
  if (dev < 0 || dev >= kMaxDevices) return FP_ERR_INVALID_ARGUMENT;
  HostPipe& g_pipe = g_pipes[dev];
  std::lock_guard<std::mutex> lock(g_pipe.mu);
  // Per slot: inputs then outputs for `chunk` paths, 256-byte aligned pieces.
  const int64_t w_in[5] = {6 * K, 3 * K, 3, 3, 2 * K};
  const int64_t w_out[7] = {2 * K, 3 * K, 1, 6 * K, 3 * K, 3, 3};
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  size_t slot = al(size_t(chunk));  // status
  for (int i = 0; i < 5; ++i) slot += al(size_t(chunk * w_in[i]) * sizeof(R));
  for (int i = 0; i < 7; ++i) slot += al(size_t(chunk * w_out[i]) * sizeof(R));
  if (g_pipe.device != dev || int(g_pipe.bufs.size()) != depth || g_pipe.buf_bytes < slot) {
    if ((e = g_pipe.setup(dev, depth, slot)) != cudaSuccess) {
      g_pipe.release();
      return cuda_status(e);
    }
  }
  // Calls with the same slot layout chain through the ring (the event waits
  // below keep every region's reuse ordered); a layout change first lets the
  // previous calls finish, since their input and output regions differ.
  const uint64_t layout = (uint64_t(K) << 48) ^ (uint64_t(chunk) << 8) ^ sizeof(R);
  if (g_pipe.layout != layout) {
    g_pipe.drain();
    g_pipe.layout = layout;
  }
  const R* hin[5] = {basis, anchor, start, end, T0};
  R* hout[7] = {T_out, points_out, length_out, d_basis, d_anchor, d_start, d_end};
  // Chunk schedule: ramp up from chunk/8 (the first copy-out starts after one
  // small copy-in + solve) and back down at the end (short drain); full
  // chunks in between.
  std::vector<int64_t> sizes;
  {
    const int64_t r[3] = {chunk / 8, chunk / 4, chunk / 2};
    std::vector<int64_t> head, tail;
    int64_t left = B;
    for (int i = 0; i < 3 && left > 0; ++i) {
      const int64_t h = std::min<int64_t>((r[i] + kThreads - 1) / kThreads * kThreads, left);
      head.push_back(h);
      left -= h;
      if (left <= 0) break;
      const int64_t t = std::min<int64_t>((r[i] + kThreads - 1) / kThreads * kThreads, left);
      tail.push_back(t);
      left -= t;
    }
    sizes = head;
    for (; left > 0; left -= std::min(left, chunk)) sizes.push_back(std::min(left, chunk));
    sizes.insert(sizes.end(), tail.rbegin(), tail.rend());
  }
  cudaStream_t s_in = g_pipe.s_in, s_k = g_pipe.s_k, s_out = g_pipe.s_out;
  // Enqueue every chunk; on an error stop enqueuing but still drain the
  // streams below, so no copy or kernel of this call is in flight when the
  // next call reuses (or reallocates) the slots.
  auto enqueue = [&]() -> int {
    cudaError_t e;
    int64_t c = g_pipe.chunks, lo = 0;
    for (const int64_t n : sizes) {
      const int j = int(c % depth);
      char* p = static_cast<char*>(g_pipe.bufs[j]);
      R* din[5];
      R* dout[7];
      for (int i = 0; i < 5; ++i) {
        din[i] = reinterpret_cast<R*>(p);
        p += al(size_t(chunk * w_in[i]) * sizeof(R));
      }
      for (int i = 0; i < 7; ++i) {
        dout[i] = reinterpret_cast<R*>(p);
        p += al(size_t(chunk * w_out[i]) * sizeof(R));
      }
      uint8_t* dst = reinterpret_cast<uint8_t*>(p);
      // copy in (the slot's input region is free once chunk c - depth's kernel ran)
      if (c >= depth && (e = cudaStreamWaitEvent(s_in, g_pipe.ev_k[j], 0)) != cudaSuccess)
        return cuda_status(e);
      {
        void *dv[5], *sv[5];
        size_t nb[5], m = 0;
        for (int i = 0; i < 5; ++i) {
          if (w_in[i] == 0 || hin[i] == nullptr) continue;
          dv[m] = din[i];
          sv[m] = const_cast<R*>(hin[i] + lo * w_in[i]);
          nb[m++] = size_t(n * w_in[i]) * sizeof(R);
        }
        if ((e = copy_arrays(dv, sv, nb, m, cudaMemcpyHostToDevice, s_in)) != cudaSuccess)
          return cuda_status(e);
        if (T0 == nullptr && K > 0 &&
            (e = cudaMemsetAsync(din[4], 0, size_t(n * w_in[4]) * sizeof(R), s_in)) != cudaSuccess)
          return cuda_status(e);
      }
      if ((e = cudaEventRecord(g_pipe.ev_in[j], s_in)) != cudaSuccess) return cuda_status(e);
      // solve + VJP (the output region is free once chunk c - depth was copied out)
      if ((e = cudaStreamWaitEvent(s_k, g_pipe.ev_in[j], 0)) != cudaSuccess) return cuda_status(e);
      if (c >= depth && (e = cudaStreamWaitEvent(s_k, g_pipe.ev_out[j], 0)) != cudaSuccess)
        return cuda_status(e);
      // Tile kernel (no host round trip): the bucketed plan would synchronise
      // its stream and stall this enqueue loop.
      int rc = solve_vjp_impl<R>(din[0], din[1], din[2], din[3], din[4], n, K, iterations, fp_iters,
                                     nullptr, w_L_scale, mode, hout[0] ? dout[0] : nullptr,
                                     hout[1] ? dout[1] : nullptr, hout[2] ? dout[2] : nullptr,
                                     hout[3] ? dout[3] : nullptr, hout[4] ? dout[4] : nullptr,
                                     hout[5] ? dout[5] : nullptr, hout[6] ? dout[6] : nullptr,
                                     status_out ? dst : nullptr, s_k, kRouteNoSync);
      if (rc != FP_OK) return rc;
      if ((e = cudaEventRecord(g_pipe.ev_k[j], s_k)) != cudaSuccess) return cuda_status(e);
      // copy out
      if ((e = cudaStreamWaitEvent(s_out, g_pipe.ev_k[j], 0)) != cudaSuccess) return cuda_status(e);
      {
        void *dv[8], *sv[8];
        size_t nb[8], m = 0;
        for (int i = 0; i < 7; ++i) {
          if (w_out[i] == 0 || hout[i] == nullptr) continue;
          dv[m] = hout[i] + lo * w_out[i];
          sv[m] = dout[i];
          nb[m++] = size_t(n * w_out[i]) * sizeof(R);
        }
        if (status_out) {
          dv[m] = status_out + lo;
          sv[m] = dst;
          nb[m++] = size_t(n);
        }
        if ((e = copy_arrays(dv, sv, nb, m, cudaMemcpyDeviceToHost, s_out)) != cudaSuccess)
          return cuda_status(e);
      }
      if ((e = cudaEventRecord(g_pipe.ev_out[j], s_out)) != cudaSuccess) return cuda_status(e);
      lo += n;
      ++c;
      g_pipe.chunks = c;
    }
    return FP_OK;
  };
  int rc = enqueue();
  if (rc != FP_OK) {
    g_pipe.drain();
    return rc;
  }
  // completion ticket: an event after this call's last copy-out
  const uint64_t t = g_pipe.next_ticket++;
  cudaEvent_t& ev = g_pipe.job_ev[t % HostPipe::kJobs];
  if (ev == nullptr) {
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return cuda_status(e);
  } else if ((e = cudaEventSynchronize(ev)) != cudaSuccess) {  // ticket t - kJobs
    return cuda_status(e);
  }
  if ((e = cudaEventRecord(ev, s_out)) != cudaSuccess) return cuda_status(e);
  if (ticket) *ticket = t | (uint64_t(dev) << kTicketShift);
  return FP_OK;
}

// Wait until the outputs of submitted call `ticket` are in host memory.
static int host_wait(uint64_t ticket_in) {
  if (ticket_in == 0) return FP_OK;
  const int dev = int(ticket_in >> kTicketShift);
  const uint64_t ticket = ticket_in & ((uint64_t(1) << kTicketShift) - 1);
  if (dev >= kMaxDevices || ticket == 0) return FP_ERR_INVALID_ARGUMENT;
  HostPipe& g_pipe = g_pipes[dev];
  cudaEvent_t ev = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_pipe.mu);
    if (ticket >= g_pipe.next_ticket) return FP_ERR_INVALID_ARGUMENT;
    if (ticket + HostPipe::kJobs < g_pipe.next_ticket) return FP_OK;  // its slot was reused: done
    ev = g_pipe.job_ev[ticket % HostPipe::kJobs];
  }
  return cuda_status(cudaEventSynchronize(ev));
}

}  // namespace fp

using namespace fp;

extern "C" {

int fp_solve_f32(const float* basis, const float* anchor, const float* start, const float* end,
                 const float* T0, int64_t B, int K, int iterations, int fp_iters, float* T_out,
                 float* g_out, float* points_out, float* length_out, uint8_t* status_out,
                 float* trace_len, float* trace_gnorm, uint8_t* trace_fate, float* H_out,
                 void* stream) {
  return solve_impl<float>(basis, anchor, start, end, T0, B, K, iterations, fp_iters, T_out, g_out,
                           points_out, length_out, status_out, trace_len, trace_gnorm, trace_fate,
                           H_out, stream);
}

int fp_solve_f64(const double* basis, const double* anchor, const double* start, const double* end,
                 const double* T0, int64_t B, int K, int iterations, int fp_iters, double* T_out,
                 double* g_out, double* points_out, double* length_out, uint8_t* status_out,
                 double* trace_len, double* trace_gnorm, uint8_t* trace_fate, double* H_out,
                 void* stream) {
  return solve_impl<double>(basis, anchor, start, end, T0, B, K, iterations, fp_iters, T_out, g_out,
                            points_out, length_out, status_out, trace_len, trace_gnorm, trace_fate,
                            H_out, stream);
}

int fp_vjp_f32(const float* basis, const float* anchor, const float* start, const float* end,
               const float* T, const float* v_T, const float* w_L, float w_L_scale, int mode,
               int64_t B, int K, float* d_basis, float* d_anchor, float* d_start, float* d_end,
               float* u_out, uint8_t* status_out, void* stream) {
  return vjp_impl<float>(basis, anchor, start, end, T, v_T, w_L, w_L_scale, mode, B, K, d_basis,
                         d_anchor, d_start, d_end, u_out, status_out, stream);
}

int fp_vjp_f64(const double* basis, const double* anchor, const double* start, const double* end,
               const double* T, const double* v_T, const double* w_L, double w_L_scale, int mode,
               int64_t B, int K, double* d_basis, double* d_anchor, double* d_start, double* d_end,
               double* u_out, uint8_t* status_out, void* stream) {
  return vjp_impl<double>(basis, anchor, start, end, T, v_T, w_L, w_L_scale, mode, B, K, d_basis,
                          d_anchor, d_start, d_end, u_out, status_out, stream);
}

int fp_solve_vjp_f32(const float* basis, const float* anchor, const float* start, const float* end,
                     const float* T0, int64_t B, int K, int iterations, int fp_iters,
                     const float* w_L, float w_L_scale, int mode, float* T_out, float* points_out,
                     float* length_out, float* d_basis, float* d_anchor, float* d_start,
                     float* d_end, uint8_t* status_out, void* stream) {
  return solve_vjp_impl<float>(basis, anchor, start, end, T0, B, K, iterations, fp_iters, w_L,
                               w_L_scale, mode, T_out, points_out, length_out, d_basis, d_anchor,
                               d_start, d_end, status_out, static_cast<cudaStream_t>(stream));
}

int fp_solve_vjp_f64(const double* basis, const double* anchor, const double* start,
                     const double* end, const double* T0, int64_t B, int K, int iterations,
                     int fp_iters, const double* w_L, double w_L_scale, int mode, double* T_out,
                     double* points_out, double* length_out, double* d_basis, double* d_anchor,
                     double* d_start, double* d_end, uint8_t* status_out, void* stream) {
  return solve_vjp_impl<double>(basis, anchor, start, end, T0, B, K, iterations, fp_iters, w_L,
                                w_L_scale, mode, T_out, points_out, length_out, d_basis, d_anchor,
                                d_start, d_end, status_out, static_cast<cudaStream_t>(stream));
}

int fp_solve_vjp_host_f32(const float* basis, const float* anchor, const float* start,
                          const float* end, const float* T0, int64_t B, int K, int iterations,
                          int fp_iters, float w_L_scale, int mode, float* T_out, float* points_out,
                          float* length_out, float* d_basis, float* d_anchor, float* d_start,
                          float* d_end, uint8_t* status_out, int64_t chunk, int depth) {
  uint64_t t = 0;
  const int rc = host_submit<float>(basis, anchor, start, end, T0, B, K, iterations, fp_iters,
                                    w_L_scale, mode, T_out, points_out, length_out, d_basis, d_anchor,
                                    d_start, d_end, status_out, chunk, depth, &t);
  return rc != FP_OK ? rc : host_wait(t);
}

int fp_solve_vjp_host_f64(const double* basis, const double* anchor, const double* start,
                          const double* end, const double* T0, int64_t B, int K, int iterations,
                          int fp_iters, double w_L_scale, int mode, double* T_out,
                          double* points_out, double* length_out, double* d_basis,
                          double* d_anchor, double* d_start, double* d_end, uint8_t* status_out,
                          int64_t chunk, int depth) {
  uint64_t t = 0;
  const int rc = host_submit<double>(basis, anchor, start, end, T0, B, K, iterations, fp_iters,
                                     w_L_scale, mode, T_out, points_out, length_out, d_basis,
                                     d_anchor, d_start, d_end, status_out, chunk, depth, &t);
  return rc != FP_OK ? rc : host_wait(t);
}

int fp_solve_vjp_host_submit_f32(const float* basis, const float* anchor, const float* start,
                                 const float* end, const float* T0, int64_t B, int K, int iterations,
                                 int fp_iters, float w_L_scale, int mode, float* T_out,
                                 float* points_out, float* length_out, float* d_basis,
                                 float* d_anchor, float* d_start, float* d_end, uint8_t* status_out,
                                 int64_t chunk, int depth, uint64_t* ticket) {
  if (ticket == nullptr) return FP_ERR_INVALID_ARGUMENT;
  return host_submit<float>(basis, anchor, start, end, T0, B, K, iterations, fp_iters, w_L_scale,
                            mode, T_out, points_out, length_out, d_basis, d_anchor, d_start, d_end,
                            status_out, chunk, depth, ticket);
}

int fp_solve_vjp_host_submit_f64(const double* basis, const double* anchor, const double* start,
                                 const double* end, const double* T0, int64_t B, int K,
                                 int iterations, int fp_iters, double w_L_scale, int mode,
                                 double* T_out, double* points_out, double* length_out,
                                 double* d_basis, double* d_anchor, double* d_start, double* d_end,
                                 uint8_t* status_out, int64_t chunk, int depth, uint64_t* ticket) {
  if (ticket == nullptr) return FP_ERR_INVALID_ARGUMENT;
  return host_submit<double>(basis, anchor, start, end, T0, B, K, iterations, fp_iters, w_L_scale,
                             mode, T_out, points_out, length_out, d_basis, d_anchor, d_start, d_end,
                             status_out, chunk, depth, ticket);
}

int fp_host_wait(uint64_t ticket) { return host_wait(ticket); }

int fp_objective_f64(const double* basis, const double* anchor, const double* start,
                     const double* end, const double* T, int64_t B, int K, double* length_out,
                     double* grad_out, double* hess_out, uint8_t* status_out, void* stream) {
  if (B < 0) return FP_ERR_INVALID_ARGUMENT;
  if (K < 0 || K > kGenMax) return FP_ERR_UNSUPPORTED_ORDER;
  if (B == 0) return FP_OK;
  const int t = 64;
  objective_kernel<double><<<unsigned((B + t - 1) / t), t, 0, static_cast<cudaStream_t>(stream)>>>(
      basis, anchor, start, end, T, B, K, length_out, grad_out, hess_out, status_out);
  count_launches(1);
  return cuda_status(cudaGetLastError());
}

int fp_line_search_f64(const double* basis, const double* anchor, const double* start,
                       const double* end, const double* T, const double* P, const double* alpha0,
                       int64_t B, int K, int k, double* alpha_out, uint8_t* status_out,
                       void* stream) {
  if (B < 0 || k < 1 || alpha_out == nullptr) return FP_ERR_INVALID_ARGUMENT;
  if (K < 0 || K > kGenMax) return FP_ERR_UNSUPPORTED_ORDER;
  if (B == 0) return FP_OK;
  const int t = 64;
  line_search_kernel<double><<<unsigned((B + t - 1) / t), t, 0, static_cast<cudaStream_t>(stream)>>>(
      basis, anchor, start, end, T, P, alpha0, B, K, k, alpha_out, status_out);
  count_launches(1);
  return cuda_status(cudaGetLastError());
}

int fp_init_params_f64(const double* basis, const double* anchor, const double* start,
                       const double* end, int64_t B, int K, double* T_out, void* stream) {
  if (B < 0 || T_out == nullptr) return FP_ERR_INVALID_ARGUMENT;
  if (K < 0 || K > kGenMax) return FP_ERR_UNSUPPORTED_ORDER;
  if (B == 0 || K == 0) return FP_OK;
  const int t = 128;
  const int64_t n = B * K;
  init_params_kernel<double><<<unsigned((n + t - 1) / t), t, 0, static_cast<cudaStream_t>(stream)>>>(
      basis, anchor, start, end, B, K, T_out);
  count_launches(1);
  return cuda_status(cudaGetLastError());
}

uint64_t fp_launch_count(void) { return g_launches.load(); }

int fp_set_kernel_policy(int policy) {
  if (policy != FP_POLICY_AUTO && policy != FP_POLICY_DENSE && policy != FP_POLICY_AUTO_SERIAL &&
      policy != FP_POLICY_BUCKET && policy != FP_POLICY_TILE)
    return FP_ERR_INVALID_ARGUMENT;
  g_policy.store(policy);
  return FP_OK;
}
int fp_last_cuda_error(void) { return g_last_cuda.load(); }

const char* fp_error_string(int code) {
  switch (code) {
    case FP_OK: return "ok";
    case FP_ERR_INVALID_ARGUMENT: return "invalid argument";
    case FP_ERR_UNSUPPORTED_ORDER: return "unsupported interaction count";
    case FP_ERR_CUDA: return cudaGetErrorString(static_cast<cudaError_t>(g_last_cuda.load()));
    case FP_ERR_UNSUPPORTED_MODE: return "unsupported VJP mode";
    default: return "unknown error";
  }
}

int fp_version(void) { return 1; }

}  // extern "C"
