// Device-side bucketing of paths by interaction-kind mask (fp_bucket.cu).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace fp {

// Largest order with per-mask specialised kernels (2^5 = 32 masks).
constexpr int kMaxSpecialisedOrder = 5;
constexpr int kMaxBuckets = 1 << kMaxSpecialisedOrder;

struct BucketScratch {
  uint8_t* codes = nullptr;
  int32_t* rows = nullptr;              // permutation, bucket-major
  unsigned long long* small = nullptr;  // counts | cursor | buckets
  int64_t* buckets = nullptr;           // (offset, count) per mask, device
};

template <typename R>
cudaError_t bucket_rows(const R* basis, int64_t B, int K, BucketScratch& sc, cudaStream_t s);
void bucket_free(BucketScratch& sc, cudaStream_t s);

}  // namespace fp
