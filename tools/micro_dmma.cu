// Dev microbenchmark: the event kernel's per-CTA GEMM shape (nt = 8 rows,
// M = J = 128, operands in shared memory) on FP64 tensor cores (DMMA
// m8n8k4), 16 CTAs x 8 warps: cycles per GEMM for 2 / 4 / 8 independent
// accumulator chains per warp. Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NT = 256, LD = 132;
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>  // accumulator sets (chains per tile)
__global__ void k(const double* In, double* Out, int reps, long long* cyc) {
  extern __shared__ double sm[];
  double* sb = sm;              // 128 x LD
  double* co = sm + 128 * LD;   // 8 x LD
  for (int x = threadIdx.x; x < 136 * LD; x += NT) sm[x] = In[x % (128 * LD)] * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, ar = lane >> 2, ac = lane & 3;
  long long c0 = clock64();
  double tot = 0;
  for (int r = 0; r < reps; ++r) {
    double d0[CH][2], d1[CH][2];
#pragma unroll
    for (int u = 0; u < CH; ++u) d0[u][0] = d0[u][1] = d1[u][0] = d1[u][1] = 0;
    const int bc0 = (warp << 3) + ar, bc1 = ((warp + 8) << 3) + ar;
    for (int m0 = 0; m0 < 128; m0 += 16) {
      double a[4], b[4][2];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int m = m0 + 4 * u + ac;
        a[u] = co[ar * LD + m];
        b[u][0] = sb[m * LD + bc0];
        b[u][1] = sb[m * LD + bc1];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int p = 0; p < 2; ++p) dmma(d0[u % CH][p], d1[u % CH][p], a[u], b[u][p]);
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) tot += d0[u][0] + d1[u][1] + d0[u][1] + d1[u][0];
    __syncthreads();
  }
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  if (tot == 12345.0) Out[threadIdx.x] = tot;
}
int main() {
  double *I, *O; long long* cyc;
  cudaMalloc(&I, 128 * LD * 8); cudaMalloc(&O, 4096 * 8); cudaMalloc(&cyc, 64 * 8);
  cudaMemset(I, 0, 128 * LD * 8);
  const int smem = 136 * LD * 8, reps = 200;
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h[64];
  for (int ch : {1, 2, 4}) {
    for (int it = 0; it < 3; ++it) {
      if (ch == 1) k<1><<<16, NT, smem>>>(I, O, reps, cyc);
      if (ch == 2) k<2><<<16, NT, smem>>>(I, O, reps, cyc);
      if (ch == 4) k<4><<<16, NT, smem>>>(I, O, reps, cyc);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
    const double cpg = (double)h[0] / reps;
    printf("chains/tile %d: %.0f cycles per GEMM (8x128x128 fp64, 512 DMMA), %.2f us, %.1f FMA/clk/SM; %s\n", ch,
           cpg, cpg / 1965.0, 8.0 * 128 * 128 / cpg, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
