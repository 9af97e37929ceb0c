#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace dgpu {

// Compact device CSR of A (rows = out-arcs) and of A^T (same arrays when A is
// symmetric); weights may be null (all 1.0).
struct TsvdGraph {
  int64_t n, arcs;
  const int64_t* off;
  const int32_t* ids;
  const double* wts;
  const int64_t* toff;
  const int32_t* tids;
  const double* twts;
};

struct TsvdResult {
  int k = 0;
  int status = 0;                  // 0 ok, else damf status (6 ZeroMatrix, 101 unsupported)
  int omega = 0;                   // 0: reference Gaussian stream, 1: device Philox stream
  int gs_fallbacks = 0;            // QRs that took the Gram-Schmidt path (rank-deficient sketch)
  std::vector<double> sigma;       // k
  float* xb_dev = nullptr;         // n x k device (randomized path), caller frees
  float* yb_dev = nullptr;
  std::vector<float> xb_host, yb_host;  // n x k host (exact small path)
};

// FactorState::init_from_graph (factor_state.cpp:84-102) on the device.
cudaError_t tsvd_init(const TsvdGraph& g, int d, uint64_t seed, cudaStream_t st, int nsm,
                      TsvdResult* res, bool exact_stream);

}  // namespace dgpu
