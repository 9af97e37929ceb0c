#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace dgpu {

cudaError_t launch_pair_scores(const float* A, const float* B, int k, const int64_t* u,
                               const int64_t* v, int64_t m, int symmetric, double* out,
                               cudaStream_t st, int nsm);
cudaError_t topk_indices(const double* scores, int64_t m, int64_t K, int64_t* idx_out,
                         double* score_out, cudaStream_t st);

}  // namespace dgpu
