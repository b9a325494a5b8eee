// Exhaustive candidate tracing: enumeration, solve, bounds mask, compaction,
// and the inverse-design gradient step (BASELINE configs 3 and 4).
//
// The reference solves given sequences only; enumeration and the bounds mask
// are new (prose at PAPER.md:67). Specification:
//   * objects are planes (reflectors: wall quads, centroid anchor, half-extent
//     basis) or edges (diffraction: midpoint anchor, half-length direction);
//   * a candidate is (RX index, ordered object sequence o_1..o_k) with no
//     immediate repeat; candidates are grouped by kind pattern p (bit j set:
//     position j is a plane) so each launch runs one kind-specialised solver;
//   * within (order, pattern): radices r_0 = n_{p_0}, r_j = n_{p_j} - [p_j ==
//     p_{j-1}]; sequence index s -> digits d (most significant first) ->
//     list positions o_0 = d_0, o_j = d_j + [p_j == p_{j-1} and d_j >= o_{j-1}]
//     (lexicographic order of the list positions); candidate c -> rx = c /
//     count_p, s = c % count_p (RX-major);
//   * a solved path is VALID when it converged (FP_STATUS_UNCONVERGED_MASK
//     clear) and every interaction point is inside its object: |t_0| <= 1 and,
//     for planes, |t_1| <= 1;
//   * valid paths are compacted with warp-aggregated atomics.
// With gradients (config 4): loss = sum over valid paths of 1 / L^2, the
// cotangent on L is -2 / L^3, the full implicit VJP runs for valid paths only,
// and object / TX / RX gradients are accumulated with atomics (TX reduced
// across the warp first).
#include <cuda_runtime.h>

#include <cstring>

#include "fp_dispatch.h"
#include "fp_kernels.cuh"

namespace fp {

struct EnumArgs {
  const float *obj_basis, *obj_anchor;  // (N,3,2), (N,3)
  float nz;                             // -0 (Geo::nz)
  const int32_t *plane_ids, *edge_ids;
  int n_planes, n_edges;
  const float *tx, *rx;  // (3), (n_rx,3)
  int n_rx;
  int64_t cand_begin, cand_end;
  int64_t count_p;       // sequences of this pattern per RX
  int64_t place[4];      // place value of digit j (product of later radices)
  int iterations, fp_iters;
  unsigned long long* counters;  // [candidates, converged, in-bounds, valid]
  int64_t capacity;
  int32_t *rec_rx, *rec_seq;
  float *rec_T, *rec_L, *rec_points;
  double *obj_grad, *tx_grad, *rx_grad, *loss;  // fp64 accumulators (config 4)
};

template <int K, unsigned MASK>
__device__ __forceinline__ void decode(const EnumArgs& a, int64_t c, int& rx, int (&obj)[K]) {
  using L = Lay<K, MASK>;
  rx = int(c / a.count_p);
  int64_t s = c - int64_t(rx) * a.count_p;
  int prev = -1;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int64_t d = s / a.place[j];
    s -= d * a.place[j];
    int o = int(d);
    if (j > 0 && L::plane(j) == L::plane(j - 1) && o >= prev) ++o;
    prev = o;
    obj[j] = L::plane(j) ? __ldg(a.plane_ids + o) : __ldg(a.edge_ids + o);
  }
}

// Register budget: the path kernels' NA rule; FP_ENUM_MIN_BLOCKS overrides
// (A/B builds).
template <int NA>
struct EnumMinBlocks {
#ifdef FP_ENUM_MIN_BLOCKS
  static constexpr int value = FP_ENUM_MIN_BLOCKS;
#else
  static constexpr int value = MinBlocks<float, NA>::value;
#endif
};

template <int K, unsigned MASK, bool GRAD>
__global__ void __launch_bounds__(kThreads, (EnumMinBlocks<Lay<K, MASK>::NA>::value))
    enum_kernel(const EnumArgs a) {
  using L = Lay<K, MASK>;
  constexpr int NA = L::NA;
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  // candidates / converged / in-bounds: per-CTA shared counters, one global
  // atomic each per CTA (not per warp: 8M warps on three addresses)
  __shared__ unsigned int cta_count[3];
  // config 4: per-warp staging of each lane's object gradients ([i][lane][9])
  __shared__ float gstage[GRAD ? kThreads / 32 : 1][GRAD ? K * 32 * 9 : 1];
  if (threadIdx.x < 3) cta_count[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t c0 = a.cand_begin + int64_t(blockIdx.x) * blockDim.x; c0 < a.cand_end; c0 += stride) {
    const int64_t c = c0 + threadIdx.x;
    const bool live = c < a.cand_end;
    bool conv = false, inb = false;
    float wl = 0.f, len = 0.f;
    int rx = 0;
    int obj[K];
    Geo<float, K> G;
    PathState<float, K, MASK> P;
    if (live) {
      decode<K, MASK>(a, c, rx, obj);
      float bb[6 * K], aa[3 * K], x0[3], x1[3];
#pragma unroll
      for (int i = 0; i < K; ++i) {
#pragma unroll
        for (int e = 0; e < 6; ++e) bb[6 * i + e] = __ldg(a.obj_basis + 6 * obj[i] + e);
#pragma unroll
        for (int e = 0; e < 3; ++e) aa[3 * i + e] = __ldg(a.obj_anchor + 3 * obj[i] + e);
      }
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        x0[e] = __ldg(a.tx + e);
        x1[e] = __ldg(a.rx + 3 * rx + e);
      }
      load_geo<float, K, MASK>(G, bb, aa, x0, x1);
      G.nz = a.nz;
      P.zero_t();
      P.eval(G, P.g);
      uint8_t st = bfgs_solve<float, K, MASK>(G, P, a.iterations, a.fp_iters, nullptr, nullptr, nullptr, 0, 0,
                                              nullptr);
      st |= final_status<float, K, MASK>(G, P);
      conv = (st & FP_STATUS_UNCONVERGED_MASK) == 0;
      inb = true;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        inb = inb && fabsf(P.T(L::idx(i, 0))) <= 1.f;
        if (L::plane(i)) inb = inb && fabsf(P.T(L::idx(i, 1))) <= 1.f;
      }
      len = P.length();
    }
    const bool valid = live && conv && inb;
    // ---- counters and compaction (warp-aggregated) -------------------------
    const unsigned bl = __ballot_sync(0xffffffffu, live), bc = __ballot_sync(0xffffffffu, live && conv),
                   bi = __ballot_sync(0xffffffffu, live && inb), bv = __ballot_sync(0xffffffffu, valid);
    unsigned long long base = 0;
    if (lane == 0) {
      atomicAdd_block(&cta_count[0], unsigned(__popc(bl)));
      if (bc) atomicAdd_block(&cta_count[1], unsigned(__popc(bc)));
      if (bi) atomicAdd_block(&cta_count[2], unsigned(__popc(bi)));
      if (bv) base = atomicAdd(&a.counters[3], (unsigned long long)__popc(bv));
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    if (valid) {
      const int64_t pos = int64_t(base) + __popc(bv & ((1u << lane) - 1u));
      if (pos < a.capacity) {
        if (a.rec_rx) a.rec_rx[pos] = rx;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (a.rec_seq) a.rec_seq[pos * K + i] = obj[i];
          if (a.rec_T) {
            a.rec_T[pos * 2 * K + 2 * i] = P.T(L::idx(i, 0));
            a.rec_T[pos * 2 * K + 2 * i + 1] = L::plane(i) ? P.T(L::idx(i, 1)) : 0.f;
          }
        }
        if (a.rec_L) a.rec_L[pos] = len;
        if (a.rec_points) {
          float X[K + 2][3];
          P.points(G, X);
#pragma unroll
          for (int i = 0; i < K; ++i)
#pragma unroll
            for (int r = 0; r < 3; ++r) a.rec_points[pos * 3 * K + 3 * i + r] = X[i + 1][r];
        }
      }
    }
    if (GRAD) {
      // ---- config 4: loss sum 1/L^2, cotangent -2/L^3, full implicit VJP ----
      // Per-path terms are fp32 (the solve's precision) and so are the sums
      // over one warp (<= 32 terms); the global sums over up to ~1e8 valid
      // paths accumulate in fp64 (fp32 atomics drift by ~1e-3 relative at
      // that count).
      float lossv = 0.f, g0[3] = {0.f, 0.f, 0.f};
      bool contrib = false;
      float* wg = gstage[threadIdx.x >> 5];
      if (valid) {
        const float il = 1.f / len;
        const float l2 = il * il;
        wl = -2.f * l2 * il;
        float tf[K][2], vf[K][2];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          tf[i][0] = P.T(L::idx(i, 0));
          tf[i][1] = L::plane(i) ? P.T(L::idx(i, 1)) : 0.f;
          vf[i][0] = vf[i][1] = 0.f;
        }
        SceneGrad<float, K> sg;
        const uint8_t vs = implicit_vjp<float, K, MASK>(G, P, tf, vf, wl, true, true, false, sg);
        if ((vs & FP_STATUS_SINGULAR) == 0) {
          contrib = true;
          lossv = l2;
          // park this path's (basis 6, anchor 3) gradients per interaction in
          // shared memory ([i][lane][9]) so its registers die here
#pragma unroll
          for (int i = 0; i < K; ++i)
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              wg[(i * 32 + lane) * 9 + 2 * r] = sg.db[i][r][0];
              wg[(i * 32 + lane) * 9 + 2 * r + 1] = sg.db[i][r][1];
              wg[(i * 32 + lane) * 9 + 6 + r] = sg.da[i][r];
            }
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            g0[r] = sg.d0[r];
            if (a.rx_grad) atomicAdd(a.rx_grad + 3 * rx + r, double(sg.d1[r]));
          }
        }
      }
      const unsigned cm = __ballot_sync(0xffffffffu, contrib);
      if (cm) {
        // Candidates of a warp are consecutive sequences: they share their
        // leading objects (the last digit varies fastest). For interactions
        // 0 .. K-2 the lanes that hit the same object are summed from the
        // staged gradients (lanes 0..8 each take one element, in lane order)
        // and added with one atomic per element; the last interaction,
        // spread over many objects, adds per lane. (Per-lane atomics on the
        // shared leading objects cost 7% of the config-4 step on the
        // 192-object alphabet.)
        __syncwarp();
        const bool live_e = lane < 9;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          // element `lane` of interaction i is inert for edges' second column
          const bool elem_ok = live_e && (lane >= 6 || (lane & 1) == 0 || L::plane(i));
          if (i == K - 1) {
            if (contrib) {
              double* og = a.obj_grad + int64_t(obj[i]) * 9;
#pragma unroll
              for (int e = 0; e < 9; ++e)
                if (e >= 6 || (e & 1) == 0 || L::plane(i))
                  atomicAdd(og + e, double(wg[(i * 32 + lane) * 9 + e]));
            }
            continue;
          }
          unsigned pending = cm;
          while (pending) {
            const int leader = __ffs(pending) - 1;
            const int o = __shfl_sync(0xffffffffu, obj[i], leader);
            const unsigned grp = __ballot_sync(0xffffffffu, ((pending >> lane) & 1u) && obj[i] == o);
            pending &= ~grp;
            if (elem_ok) {
              float v = 0.f;
              for (unsigned m = grp; m; m &= m - 1) v += wg[(i * 32 + __ffs(m) - 1) * 9 + lane];
              atomicAdd(a.obj_grad + int64_t(o) * 9 + lane, double(v));
            }
          }
        }
        __syncwarp();
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          lossv += __shfl_xor_sync(0xffffffffu, lossv, off);
#pragma unroll
          for (int r = 0; r < 3; ++r) g0[r] += __shfl_xor_sync(0xffffffffu, g0[r], off);
        }
        if (lane == 0) {
          atomicAdd(a.loss, double(lossv));
#pragma unroll
          for (int r = 0; r < 3; ++r) atomicAdd(a.tx_grad + r, double(g0[r]));
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < 3 && cta_count[threadIdx.x])
    atomicAdd(&a.counters[threadIdx.x], (unsigned long long)cta_count[threadIdx.x]);
}

// Decode-only kernel (enumeration parity tests, `enumerate_candidates`).
template <int K, unsigned MASK>
__global__ void decode_kernel(const EnumArgs a, int32_t* rx_out, int32_t* seq_out) {
  const int64_t c = a.cand_begin + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= a.cand_end) return;
  int rx, obj[K];
  decode<K, MASK>(a, c, rx, obj);
  const int64_t i = c - a.cand_begin;
  if (rx_out) rx_out[i] = rx;
#pragma unroll
  for (int j = 0; j < K; ++j) seq_out[i * K + j] = obj[j];
}

template <int K, unsigned MASK>
static cudaError_t launch_enum(const EnumArgs& a, bool grad, cudaStream_t s) {
  const int64_t n = a.cand_end - a.cand_begin;
  if (n <= 0) return cudaSuccess;
  const void* fn = grad ? reinterpret_cast<const void*>(enum_kernel<K, MASK, true>)
                        : reinterpret_cast<const void*>(enum_kernel<K, MASK, false>);
  // One CTA per 128 candidates (the kernel's grid-stride loop then runs once):
  // the block scheduler balances the uneven per-candidate cost; a persistent
  // grid of resident CTAs was 6-7% slower (config 3, both alphabets).
  (void)fn;
  int64_t blocks = (n + kThreads - 1) / kThreads;
  if (blocks > int64_t(0x7fffffff)) blocks = 0x7fffffff;
  if (grad)
    enum_kernel<K, MASK, true><<<unsigned(blocks), kThreads, 0, s>>>(a);
  else
    enum_kernel<K, MASK, false><<<unsigned(blocks), kThreads, 0, s>>>(a);
  count_launches(1);
  return cudaGetLastError();
}

template <int K, unsigned M = 0>
static cudaError_t enum_by_mask(unsigned mask, const EnumArgs& a, bool grad, bool decode_only,
                                int32_t* rx_out, int32_t* seq_out, cudaStream_t s) {
  if (mask == M) {
    if (!decode_only) return launch_enum<K, M>(a, grad, s);
    const int64_t n = a.cand_end - a.cand_begin;
    if (n <= 0) return cudaSuccess;
    decode_kernel<K, M><<<unsigned((n + 255) / 256), 256, 0, s>>>(a, rx_out, seq_out);
    count_launches(1);
    return cudaGetLastError();
  }
  if constexpr (M + 1 < (1u << K)) {
    return enum_by_mask<K, M + 1>(mask, a, grad, decode_only, rx_out, seq_out, s);
  } else {
    return cudaErrorInvalidValue;
  }
}

// Per-RX count of pattern-p sequences and the digit place values.
static int64_t pattern_layout(int n_planes, int n_edges, int order, unsigned pattern, int64_t* place) {
  int64_t radix[4];
  for (int j = 0; j < order; ++j) {
    const bool pl = (pattern >> j) & 1u;
    int64_t r = pl ? n_planes : n_edges;
    if (j > 0 && pl == bool((pattern >> (j - 1)) & 1u)) r -= 1;
    radix[j] = r < 0 ? 0 : r;
  }
  int64_t cnt = 1;
  for (int j = order - 1; j >= 0; --j) {
    if (place) place[j] = cnt;
    cnt *= radix[j];
  }
  return cnt;
}

static int fill_args(EnumArgs& a, const float* obj_basis, const float* obj_anchor,
                     const int32_t* plane_ids, int n_planes, const int32_t* edge_ids, int n_edges,
                     const float* tx, const float* rx, int n_rx, int order, unsigned pattern,
                     int64_t cand_begin, int64_t cand_end) {
  if (order < 1 || order > 3) return FP_ERR_UNSUPPORTED_ORDER;
  if (pattern >= (1u << order) || n_planes < 0 || n_edges < 0 || n_rx < 1 || cand_begin < 0 ||
      cand_end < cand_begin)
    return FP_ERR_INVALID_ARGUMENT;
  std::memset(&a, 0, sizeof(a));
  a.nz = -0.0f;
  a.obj_basis = obj_basis;
  a.obj_anchor = obj_anchor;
  a.plane_ids = plane_ids;
  a.edge_ids = edge_ids;
  a.n_planes = n_planes;
  a.n_edges = n_edges;
  a.tx = tx;
  a.rx = rx;
  a.n_rx = n_rx;
  a.count_p = pattern_layout(n_planes, n_edges, order, pattern, a.place);
  if (cand_end > a.count_p * n_rx) return FP_ERR_INVALID_ARGUMENT;
  a.cand_begin = cand_begin;
  a.cand_end = cand_end;
  return FP_OK;
}

// Chain rule from object parameters to wall-vertex coordinates (config 4):
// every object parameter block (anchor, basis column 0, basis column 1) is a
// linear combination of at most four vertices, coef (N, 3, 4) x vert_ids (N, 4).
__global__ void vertex_chain_kernel(const double* __restrict__ obj_grad, int n_objects,
                                    const int32_t* __restrict__ vert_ids, const float* __restrict__ coef,
                                    double* __restrict__ vertex_grad) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n_objects) return;
  const double* g = obj_grad + 9 * o;
  double dp[3][3];
  for (int r = 0; r < 3; ++r) {
    dp[0][r] = g[6 + r];      // anchor
    dp[1][r] = g[2 * r];      // basis column 0
    dp[2][r] = g[2 * r + 1];  // basis column 1
  }
  for (int v = 0; v < 4; ++v) {
    const int vid = vert_ids[4 * o + v];
    if (vid < 0) continue;
    for (int r = 0; r < 3; ++r) {
      double acc = 0.0;
      for (int p = 0; p < 3; ++p) acc = fma(double(coef[12 * o + 4 * p + v]), dp[p][r], acc);
      atomicAdd(vertex_grad + 3 * vid + r, acc);
    }
  }
}

}  // namespace fp

using namespace fp;

extern "C" {

int64_t fp_enum_pattern_count(int n_planes, int n_edges, int order, unsigned pattern) {
  if (order < 1 || order > 3 || pattern >= (1u << order)) return -1;
  return pattern_layout(n_planes, n_edges, order, pattern, nullptr);
}

int fp_enum_decode(const int32_t* plane_ids, int n_planes, const int32_t* edge_ids, int n_edges,
                   int n_rx, int order, unsigned pattern, int64_t cand_begin, int64_t cand_end,
                   int32_t* rx_out, int32_t* seq_out, void* stream) {
  EnumArgs a;
  int rc = fill_args(a, nullptr, nullptr, plane_ids, n_planes, edge_ids, n_edges, nullptr, nullptr,
                     n_rx, order, pattern, cand_begin, cand_end);
  if (rc != FP_OK) return rc;
  if (seq_out == nullptr) return FP_ERR_INVALID_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (order) {
    case 1: e = enum_by_mask<1>(pattern, a, false, true, rx_out, seq_out, s); break;
    case 2: e = enum_by_mask<2>(pattern, a, false, true, rx_out, seq_out, s); break;
    default: e = enum_by_mask<3>(pattern, a, false, true, rx_out, seq_out, s); break;
  }
  return e == cudaSuccess ? FP_OK : FP_ERR_CUDA;
}

int fp_enum_trace_f32(const float* obj_basis, const float* obj_anchor, const int32_t* plane_ids,
                      int n_planes, const int32_t* edge_ids, int n_edges, const float* tx,
                      const float* rx, int n_rx, int order, unsigned pattern, int64_t cand_begin,
                      int64_t cand_end, int iterations, int fp_iters,
                      unsigned long long* counters, int64_t capacity, int32_t* rec_rx,
                      int32_t* rec_seq, float* rec_T, float* rec_L, float* rec_points,
                      double* obj_grad, double* tx_grad, double* rx_grad, double* loss, void* stream) {
  EnumArgs a;
  int rc = fill_args(a, obj_basis, obj_anchor, plane_ids, n_planes, edge_ids, n_edges, tx, rx, n_rx,
                     order, pattern, cand_begin, cand_end);
  if (rc != FP_OK) return rc;
  if (iterations < 1 || fp_iters < 1 || counters == nullptr || capacity < 0)
    return FP_ERR_INVALID_ARGUMENT;
  const bool grad = obj_grad != nullptr;
  if (grad && (tx_grad == nullptr || loss == nullptr)) return FP_ERR_INVALID_ARGUMENT;
  a.iterations = iterations;
  a.fp_iters = fp_iters;
  a.counters = counters;
  a.capacity = capacity;
  a.rec_rx = rec_rx;
  a.rec_seq = rec_seq;
  a.rec_T = rec_T;
  a.rec_L = rec_L;
  a.rec_points = rec_points;
  a.obj_grad = obj_grad;
  a.tx_grad = tx_grad;
  a.rx_grad = rx_grad;
  a.loss = loss;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (order) {
    case 1: e = enum_by_mask<1>(pattern, a, grad, false, nullptr, nullptr, s); break;
    case 2: e = enum_by_mask<2>(pattern, a, grad, false, nullptr, nullptr, s); break;
    default: e = enum_by_mask<3>(pattern, a, grad, false, nullptr, nullptr, s); break;
  }
  return e == cudaSuccess ? FP_OK : FP_ERR_CUDA;
}

int fp_vertex_chain_f32(const double* obj_grad, int n_objects, const int32_t* vert_ids,
                        const float* coef, double* vertex_grad, void* stream) {
  if (n_objects < 0 || (n_objects > 0 && (!obj_grad || !vert_ids || !coef || !vertex_grad)))
    return FP_ERR_INVALID_ARGUMENT;
  if (n_objects == 0) return FP_OK;
  vertex_chain_kernel<<<(n_objects + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      obj_grad, n_objects, vert_ids, coef, vertex_grad);
  count_launches(1);
  return cudaGetLastError() == cudaSuccess ? FP_OK : FP_ERR_CUDA;
}

}  // extern "C"
