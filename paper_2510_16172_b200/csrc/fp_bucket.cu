// Kind-pattern bucketing for the specialised solver kernels.
//
// Each path's kind mask (bit i set when interaction i has a nonzero second
// basis column, i.e. is a plane; geometry.py:74-77) selects a kernel
// instantiation that carries only the active unknowns. One pass classifies
// and histograms, a 32-thread pass turns counts into bucket ranges, and a
// scatter pass writes the row permutation with warp-aggregated atomics (one
// atomic per warp and mask). Everything stays on the device: no host sync.
#include <cuda_runtime.h>

#include "fp_bucket.h"
#include "fp_dispatch.h"

namespace fp {

template <typename R>
__global__ void classify_kernel(const R* __restrict__ basis, int64_t B, int K,
                                uint8_t* __restrict__ codes, unsigned long long* __restrict__ counts) {
  __shared__ unsigned int hist[kMaxBuckets];
  const int nb = 1 << K;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) hist[i] = 0;
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
      const int leader = __ffs(same) - 1;
      if ((threadIdx.x & 31) == leader) atomicAdd(&hist[code], unsigned(__popc(same)));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    if (hist[i]) atomicAdd(&counts[i], (unsigned long long)hist[i]);
}

// buckets[2m] = offset, buckets[2m+1] = count; cursor[m] = offset.
__global__ void offsets_kernel(const unsigned long long* counts, int nb, int64_t* buckets,
                               unsigned long long* cursor) {
  if (threadIdx.x != 0) return;
  unsigned long long off = 0;
  for (int m = 0; m < nb; ++m) {
    buckets[2 * m] = int64_t(off);
    buckets[2 * m + 1] = int64_t(counts[m]);
    cursor[m] = off;
    off += counts[m];
  }
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

template <typename R>
cudaError_t bucket_rows(const R* basis, int64_t B, int K, BucketScratch& sc, cudaStream_t s) {
  const int nb = 1 << K;
  cudaError_t e;
  if ((e = cudaMallocAsync(&sc.codes, size_t(B), s)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&sc.rows, size_t(B) * sizeof(int32_t), s)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&sc.small, sizeof(unsigned long long) * 4 * kMaxBuckets, s)) != cudaSuccess)
    return e;
  unsigned long long* counts = sc.small;
  unsigned long long* cursor = sc.small + kMaxBuckets;
  sc.buckets = reinterpret_cast<int64_t*>(sc.small + 2 * kMaxBuckets);
  if ((e = cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * kMaxBuckets, s)) != cudaSuccess)
    return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 256;
  int64_t blocks = (B + threads - 1) / threads;
  if (blocks > int64_t(sms) * 8) blocks = int64_t(sms) * 8;
  classify_kernel<R><<<unsigned(blocks), threads, 0, s>>>(basis, B, K, sc.codes, counts);
  offsets_kernel<<<1, 32, 0, s>>>(counts, nb, sc.buckets, cursor);
  scatter_kernel<<<unsigned(blocks), threads, 0, s>>>(sc.codes, B, cursor, sc.rows);
  count_launches(3);
  return cudaGetLastError();
}

void bucket_free(BucketScratch& sc, cudaStream_t s) {
  if (sc.codes) cudaFreeAsync(sc.codes, s);
  if (sc.rows) cudaFreeAsync(sc.rows, s);
  if (sc.small) cudaFreeAsync(sc.small, s);
  sc = BucketScratch{};
}

template cudaError_t bucket_rows<float>(const float*, int64_t, int, BucketScratch&, cudaStream_t);
template cudaError_t bucket_rows<double>(const double*, int64_t, int, BucketScratch&, cudaStream_t);

}  // namespace fp
