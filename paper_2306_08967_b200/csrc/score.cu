// Batched link scoring and top-K over pair sets: the
// consumers of the materialised embeddings in the reference's evaluation,
// pair_score (eval.cpp:211-215: score = <Z[u], Y[v]> or <X[u], Y[v]>,
// max over both orders when undirected; Engine::score, engine.cpp:49-52) and
// the streaming top-K of run_graph_reconstruction (eval.cpp:336-371: best
// pairs by score descending, pair index ascending on ties).
//
// Current rows are materialised once per call (query_all, the fast HBM-bound
// path or the fp64 fold when P is ill-conditioned), pair scores are fp64 dot
// products of fp32 rows (warp per pair, 128-bit loads), and the top-K is a
// stable radix sort of (-score, index) (CUB, the toolkit's device sort).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "score.cuh"

namespace dgpu {

namespace {

__global__ void pair_scores(const float* __restrict__ A, const float* __restrict__ B, int k,
                            const int64_t* __restrict__ u, const int64_t* __restrict__ v, int64_t m,
                            int symmetric, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = warp; q < m; q += nw) {
    const int64_t a = u[q], b = v[q];
    const float* au = A + a * k;
    const float* bv = B + b * k;
    double s1 = 0.0, s2 = 0.0;
    for (int j = lane; j < k; j += 32) {
      s1 += (double)au[j] * (double)bv[j];
      if (symmetric) s2 += (double)A[b * k + j] * (double)B[a * k + j];
    }
    for (int o = 16; o > 0; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) out[q] = symmetric ? fmax(s1, s2) : s1;
  }
}

__global__ void negate(double* x, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = -x[i];
}

__global__ void neg_and_iota(const double* s, int64_t m, double* key, int64_t* idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = -s[i];
    idx[i] = i;
  }
}

}  // namespace

cudaError_t launch_pair_scores(const float* A, const float* B, int k, const int64_t* u,
                               const int64_t* v, int64_t m, int symmetric, double* out,
                               cudaStream_t st, int nsm) {
  if (m <= 0) return cudaSuccess;
  const int64_t blocks = (m * 32 + 255) / 256;
  pair_scores<<<(int)(blocks < nsm * 32 ? blocks : nsm * 32), 256, 0, st>>>(A, B, k, u, v, m,
                                                                          symmetric, out);
  return cudaGetLastError();
}

// idx_out[0..K) = indices of the K best scores, (score desc, index asc).
cudaError_t topk_indices(const double* scores, int64_t m, int64_t K, int64_t* idx_out,
                         double* score_out, cudaStream_t st) {
  if (m <= 0 || K <= 0) return cudaSuccess;
  double *k_in = nullptr, *k_out = nullptr;
  int64_t *i_in = nullptr, *i_out = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e;
  if ((e = cudaMallocAsync(&k_in, m * 8, st)) || (e = cudaMallocAsync(&k_out, m * 8, st)) ||
      (e = cudaMallocAsync(&i_in, m * 8, st)) || (e = cudaMallocAsync(&i_out, m * 8, st)))
    return e;
  neg_and_iota<<<256, 256, 0, st>>>(scores, m, k_in, i_in);
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, i_in, i_out, (int64_t)m, 0, 64,
                                  st);
  if ((e = cudaMallocAsync(&tmp, tmp_bytes, st))) return e;
  // radix sort is stable: equal keys keep ascending pair index
  e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, i_in, i_out, (int64_t)m, 0, 64,
                                      st);
  const int64_t kk = K < m ? K : m;
  if (!e) e = cudaMemcpyAsync(idx_out, i_out, kk * 8, cudaMemcpyDefault, st);
  if (!e && score_out) {
    negate<<<64, 256, 0, st>>>(k_out, kk);
    e = cudaMemcpyAsync(score_out, k_out, kk * 8, cudaMemcpyDefault, st);
  }
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(k_in, st);
  cudaFreeAsync(k_out, st);
  cudaFreeAsync(i_in, st);
  cudaFreeAsync(i_out, st);
  return e;
}

}  // namespace dgpu
