// Kind-pattern bucketing for the specialised solver kernels.
//
// Each path's kind mask (bit i set when interaction i has a nonzero second
// basis column, i.e. is a plane; geometry.py:74-77) selects a kernel
// instantiation that carries only the active unknowns.
//
//   1. classify: one pass writes each path's mask and, per mask, the count and
//      the first/last row (warp-aggregated atomics); 2^K * 3 numbers come back
//      to the host (one small copy + stream sync).
//   2. masks whose rows form one contiguous range (config 2's ordering-major
//      layout, uniform batches) run the staged TMA kernel on that sub-range;
//   3. only if some mask is scattered, offsets + scatter build a row
//      permutation and those masks run the gathering kernel.
#include <cuda_runtime.h>

#include <mutex>

#include "fp_bucket.h"
#include "fp_dispatch.h"

namespace fp {

template <typename R>
__global__ void classify_kernel(const R* __restrict__ basis, int64_t B, int K,
                                uint8_t* __restrict__ codes, unsigned long long* __restrict__ stats) {
  // stats: [0, nb) counts, [nb, 2nb) min row, [2nb, 3nb) max row, [3nb] mixed warps
  __shared__ unsigned int hist[kMaxBuckets];
  __shared__ unsigned long long lo[kMaxBuckets], hi[kMaxBuckets];
  __shared__ unsigned int mixed;
  const int nb = 1 << K;
  if (threadIdx.x == 0) mixed = 0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    hist[i] = 0;
    lo[i] = ~0ull;
    hi[i] = 0;
  }
  __syncthreads();
  for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b - threadIdx.x < B;
       b += int64_t(gridDim.x) * blockDim.x) {
    unsigned code = 0;
    const bool live = b < B;
    if (live) {
      const R* A = basis + b * 6 * K;
      for (int i = 0; i < K; ++i) {
        const bool plane = A[6 * i + 1] != R(0) || A[6 * i + 3] != R(0) || A[6 * i + 5] != R(0);
        code |= unsigned(plane) << i;
      }
      codes[b] = uint8_t(code);
    }
    const unsigned live_mask = __ballot_sync(0xffffffffu, live);
    if (live) {
      const unsigned same = __match_any_sync(live_mask, code);
      const int lane = threadIdx.x & 31;
      const int leader = __ffs(same) - 1;
      const int last = 31 - __clz(same);
      // lanes are consecutive rows: the group's first/last rows are its end lanes
      const unsigned long long first = __shfl_sync(same, (unsigned long long)b, leader);
      const unsigned long long lastrow = __shfl_sync(same, (unsigned long long)b, last);
      if (lane == leader) {
        atomicAdd(&hist[code], unsigned(__popc(same)));
        atomicMin(&lo[code], first);
        atomicMax(&hi[code], lastrow);
      }
      if (lane == __ffs(live_mask) - 1 && same != live_mask) atomicAdd(&mixed, 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && mixed) atomicAdd(&stats[3 * nb], (unsigned long long)mixed);
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    if (!hist[i]) continue;
    atomicAdd(&stats[i], (unsigned long long)hist[i]);
    atomicMin(&stats[nb + i], lo[i]);
    atomicMax(&stats[2 * nb + i], hi[i]);
  }
}

__global__ void stats_init_kernel(unsigned long long* stats, int nb) {
  const int i = threadIdx.x;
  if (i < nb) {
    stats[i] = 0;
    stats[nb + i] = ~0ull;
    stats[2 * nb + i] = 0;
  }
  if (i == 0) stats[3 * nb] = 0;
}

__global__ void scatter_kernel(const uint8_t* __restrict__ codes, int64_t B,
                               unsigned long long* __restrict__ cursor, int32_t* __restrict__ rows) {
  for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b - threadIdx.x < B;
       b += int64_t(gridDim.x) * blockDim.x) {
    const bool live = b < B;
    const unsigned live_mask = __ballot_sync(0xffffffffu, live);
    if (!live) continue;
    const unsigned code = codes[b];
    const unsigned same = __match_any_sync(live_mask, code);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(same) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(&cursor[code], (unsigned long long)__popc(same));
    base = __shfl_sync(same, base, leader);
    const unsigned rank = __popc(same & ((1u << lane) - 1u));
    rows[base + rank] = int32_t(b);
  }
}

static int grid_for(int64_t B, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (B + threads - 1) / threads;
  if (blocks > int64_t(sms) * 8) blocks = int64_t(sms) * 8;
  return int(blocks < 1 ? 1 : blocks);
}

// Stream-ordered scratch comes from a pool of our own that keeps its memory
// (release threshold: unlimited). The default pool returns freed memory to
// the system at every synchronisation, and bucket_plan synchronises, so
// each call paid a fresh device allocation (0.5-18 ms per call measured).
static cudaError_t scratch_pool(cudaMemPool_t& pool) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(mu);
  if (pools[dev] == nullptr) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if ((e = cudaMemPoolCreate(&pools[dev], &props)) != cudaSuccess) return e;
    uint64_t keep = ~0ull;
    if ((e = cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep)) != cudaSuccess)
      return e;
  }
  pool = pools[dev];
  return cudaSuccess;
}

template <typename T>
static cudaError_t scratch_alloc(T** p, size_t bytes, cudaStream_t s) {
  cudaMemPool_t pool;
  cudaError_t e = scratch_pool(pool);
  if (e != cudaSuccess) return e;
  return cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, pool, s);
}

template <typename R>
cudaError_t bucket_plan(const R* basis, int64_t B, int K, BucketScratch& sc, BucketPlan& plan,
                        cudaStream_t s) {
  const int nb = 1 << K;
  plan.nb = nb;
  cudaError_t e;
  if ((e = scratch_alloc(&sc.codes, size_t(B), s)) != cudaSuccess) return e;
  if ((e = scratch_alloc(&sc.small, sizeof(unsigned long long) * (4 * kMaxBuckets + 1), s)) != cudaSuccess)
    return e;
  static unsigned long long* host = nullptr;  // pinned staging for the 3 x nb + 1 stats
  static std::mutex host_mu;                  // one caller at a time reads it back
  std::lock_guard<std::mutex> lk(host_mu);
  if (host == nullptr) {
    if ((e = cudaMallocHost(&host, sizeof(unsigned long long) * (3 * kMaxBuckets + 1))) != cudaSuccess)
      return e;
  }
  stats_init_kernel<<<1, kMaxBuckets, 0, s>>>(sc.small, nb);
  classify_kernel<R><<<grid_for(B, 256), 256, 0, s>>>(basis, B, K, sc.codes, sc.small);
  count_launches(2);
  if ((e = cudaMemcpyAsync(host, sc.small, sizeof(unsigned long long) * (3 * nb + 1),
                           cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  plan.all_contiguous = true;
  plan.mixed_warps = int64_t(host[3 * nb]);
  int64_t off = 0;
  for (int m = 0; m < nb; ++m) {
    plan.count[m] = int64_t(host[m]);
    plan.lo[m] = plan.count[m] ? int64_t(host[nb + m]) : 0;
    plan.hi[m] = plan.count[m] ? int64_t(host[2 * nb + m]) : -1;
    plan.offset[m] = off;
    off += plan.count[m];
    plan.contiguous[m] = plan.count[m] == 0 || plan.hi[m] - plan.lo[m] + 1 == plan.count[m];
    plan.all_contiguous = plan.all_contiguous && plan.contiguous[m];
  }
  return cudaSuccess;
}

struct Offsets {
  unsigned long long v[kMaxBuckets];
};

// Bucket cursors from the plan's offsets, passed by value (no host copy, no sync).
__global__ void cursor_init_kernel(unsigned long long* cursor, const Offsets off, int nb) {
  const int i = threadIdx.x;
  if (i < nb) cursor[i] = off.v[i];
}

cudaError_t bucket_scatter(int64_t B, const BucketPlan& plan, BucketScratch& sc, cudaStream_t s) {
  cudaError_t e;
  if ((e = scratch_alloc(&sc.rows, size_t(B) * sizeof(int32_t), s)) != cudaSuccess) return e;
  Offsets off = {};
  for (int m = 0; m < plan.nb; ++m) off.v[m] = (unsigned long long)plan.offset[m];
  unsigned long long* cursor = sc.small + 3 * kMaxBuckets + 1;
  cursor_init_kernel<<<1, kMaxBuckets, 0, s>>>(cursor, off, plan.nb);
  scatter_kernel<<<grid_for(B, 256), 256, 0, s>>>(sc.codes, B, cursor, sc.rows);
  count_launches(2);
  return cudaGetLastError();
}

void bucket_free(BucketScratch& sc, cudaStream_t s) {
  if (sc.codes) cudaFreeAsync(sc.codes, s);
  if (sc.rows) cudaFreeAsync(sc.rows, s);
  if (sc.small) cudaFreeAsync(sc.small, s);
  sc = BucketScratch{};
}

template cudaError_t bucket_plan<float>(const float*, int64_t, int, BucketScratch&, BucketPlan&,
                                        cudaStream_t);
template cudaError_t bucket_plan<double>(const double*, int64_t, int, BucketScratch&, BucketPlan&,
                                         cudaStream_t);

// ---- side streams: overlap the tails of the per-mask launches ----------------
SideStreams& side_streams() {
  static SideStreams ss[64];  // per device: the streams and events belong to it
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  return ss[dev];
}

cudaError_t SideStreams::fork(cudaStream_t parent, int n) {
  cudaError_t e;
  if (!ready) {
    for (int i = 0; i < kSide; ++i) {
      if ((e = cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    if ((e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming)) != cudaSuccess) return e;
    ready = true;
  }
  used = n < kSide ? n : kSide;
  if ((e = cudaEventRecord(start, parent)) != cudaSuccess) return e;
  for (int i = 0; i < used; ++i)
    if ((e = cudaStreamWaitEvent(st[i], start, 0)) != cudaSuccess) return e;
  return cudaSuccess;
}

cudaError_t SideStreams::join(cudaStream_t parent) {
  cudaError_t e;
  for (int i = 0; i < used; ++i) {
    if ((e = cudaEventRecord(done[i], st[i])) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(parent, done[i], 0)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace fp
