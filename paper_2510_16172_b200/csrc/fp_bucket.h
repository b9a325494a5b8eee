// Device-side bucketing of paths by interaction-kind mask (fp_bucket.cu).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <mutex>

namespace fp {

// Largest order with per-mask specialised kernels (2^5 = 32 masks).
constexpr int kMaxSpecialisedOrder = 5;
constexpr int kMaxBuckets = 1 << kMaxSpecialisedOrder;

struct BucketScratch {
  uint8_t* codes = nullptr;
  int32_t* rows = nullptr;              // permutation, bucket-major
  unsigned long long* small = nullptr;  // stats (3 x kMaxBuckets + 1) | cursor
};

struct BucketPlan {
  int nb = 0;
  int64_t count[kMaxBuckets], lo[kMaxBuckets], hi[kMaxBuckets], offset[kMaxBuckets];
  bool contiguous[kMaxBuckets];
  bool all_contiguous = true;
  int64_t mixed_warps = 0;  // warps of 32 consecutive rows with more than one mask
};

// Classify + per-mask statistics; synchronises `s` to bring the plan home.
template <typename R>
cudaError_t bucket_plan(const R* basis, int64_t B, int K, BucketScratch& sc, BucketPlan& plan,
                        cudaStream_t s);
// Bucket-major row permutation in sc.rows (for non-contiguous masks).
cudaError_t bucket_scatter(int64_t B, const BucketPlan& plan, BucketScratch& sc, cudaStream_t s);
void bucket_free(BucketScratch& sc, cudaStream_t s);

// A small pool of non-blocking streams: the per-mask kernels run
// concurrently so that their tail waves overlap.
struct SideStreams {
  static constexpr int kSide = 4;
  cudaStream_t st[kSide];
  cudaEvent_t done[kSide];
  cudaEvent_t start;
  bool ready = false;
  int used = 0;
  std::mutex mu;  // held by the caller from fork through join
  cudaError_t fork(cudaStream_t parent, int n);
  cudaError_t join(cudaStream_t parent);
};
SideStreams& side_streams();  // the current device's

}  // namespace fp
