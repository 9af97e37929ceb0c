#pragma once
#include "common.cuh"

namespace dgpu {

// Z[:, :k2] = X[:, :k] * F with F supplied transposed (FT[c][m], fp64, device).
cudaError_t launch_materialize(const float* X, int64_t n, int k, int ldx, const double* FT,
                               int ldf, int k2, float* Z, int ldz, cudaStream_t s, int nsm);
size_t materialize_smem(int k);

}  // namespace dgpu
