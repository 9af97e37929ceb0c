// Micro-benchmark: achievable HBM throughput of random 512-byte row gathers
// (the PPR pull's delta reads) as a function of rows in flight per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_gather micro_gather.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <random>

template <int H>
__global__ void gather(const float4* __restrict__ rows, const int* __restrict__ idx, int64_t m,
                       float4* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t i = warp * H; i < m; i += nwarps * H) {
    float4 v[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int r = idx[i + h];
      v[h] = rows[(int64_t)r * 32 + lane];  // 32 lanes x 16 B = 512 B row
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
      acc.x += v[h].x; acc.y += v[h].y; acc.z += v[h].z; acc.w += v[h].w;
    }
  }
  if (acc.x == 12345.f) out[0] = acc;
}

int main() {
  const int64_t nrows = 1ll << 23;          // 4.3 GB of 512 B rows
  const int64_t m = 1ll << 26;              // 64 M gathers (34 GB)
  float4* rows; int* idx; float4* out;
  cudaMalloc(&rows, nrows * 512); cudaMemset(rows, 0, nrows * 512);
  cudaMalloc(&idx, (m + 64) * 4); cudaMalloc(&out, 64);
  std::vector<int> h(m + 64);
  std::mt19937_64 g(1);
  for (auto& x : h) x = (int)(g() % nrows);
  cudaMemcpy(idx, h.data(), (m + 64) * 4, cudaMemcpyHostToDevice);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, int H, int bps, int threads) {
    kern<<<nsm * bps, threads>>>(rows, idx, m, out);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) kern<<<nsm * bps, threads>>>(rows, idx, m, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
    printf("H=%2d blocks/SM=%d threads=%d warps/SM=%2d: %.1f GB/s\n", H, bps, threads, bps * threads / 32,
           m * 512.0 / (ms * 1e-3) / 1e9);
  };
  for (int bps : {1, 2, 3, 4, 8}) {
    run(gather<1>, 1, bps, 256);
    run(gather<2>, 2, bps, 256);
    run(gather<4>, 4, bps, 256);
    run(gather<8>, 8, bps, 256);
  }
  return 0;
}
