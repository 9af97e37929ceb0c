#pragma once
#include "common.cuh"

namespace dgpu {

// Z[:, :k2] = X[:, :k] * F with F supplied transposed (FT[c][m], fp64, device).
cudaError_t launch_materialize(const float* X, int64_t n, int k, int ldx, const double* FT,
                               int ldf, int k2, float* Z, int ldz, cudaStream_t s, int nsm);
size_t materialize_smem(int k);

// tcgen05 path (d in {32, 64, 128}); Fhi/Flo are k x k fp32 in FT layout.
bool materialize_tc_supported(int k, int ldx, int ldz, const void* X, const void* Z);
cudaError_t launch_materialize_precise(const float* X, int64_t n, int k, int ldx,
                                       const double* FT, int ldf, int k2, float* Z, int ldz,
                                       cudaStream_t s, int nsm);
cudaError_t launch_materialize_tc(const float* X, int64_t n, int k, int ldx, const float* Fhi,
                                  const float* Flo, float* Z, int ldz, cudaStream_t s, int nsm);

}  // namespace dgpu
