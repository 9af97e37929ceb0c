// Dev microbenchmark: fp64 "Out[t][:] = sum_m Coef[t][m] In[m][:]" on 16 CTAs
// (the per-CTA shape of the update GEMMs: nt=8 rows, M=J=128), to measure
// B200 fp64 + L2 streaming behaviour. Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NT = 256, TCH = 8;
template <int MODE>
__global__ void k_gemm(const double* __restrict__ Coef, const double* __restrict__ In, double* Out,
                       int M, int J, int ld, int reps, long long* cyc) {
  __shared__ double coef[TCH * 132];
  __shared__ double red[NT * TCH];
  const int t0 = blockIdx.x * TCH;
  for (int x = threadIdx.x; x < TCH * M; x += NT) coef[(x / M) * 132 + x % M] = Coef[(t0 + x / M) * ld + x % M];
  __syncthreads();
  long long c0 = clock64();
  const int jt = 128, G = NT / jt, j = threadIdx.x % jt, g = threadIdx.x / jt;
  for (int r = 0; r < reps; ++r) {
    double acc[TCH];
#pragma unroll
    for (int t = 0; t < TCH; ++t) acc[t] = 0;
    if (MODE == 0) {
      for (int m = g; m < M; m += G) {
        const double x = In[m * ld + j];
#pragma unroll
        for (int t = 0; t < TCH; ++t) acc[t] = fma(coef[t * 132 + m], x, acc[t]);
      }
    } else if (MODE == 1) {
      for (int m = g; m < M; m += 8 * G) {
        double x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = In[(m + q * G) * ld + j];
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int t = 0; t < TCH; ++t) acc[t] = fma(coef[t * 132 + m + q * G], x[q], acc[t]);
      }
    } else if (MODE == 3) {  // registers only: coef in registers, x synthetic
      double c[TCH];
#pragma unroll
      for (int t = 0; t < TCH; ++t) c[t] = coef[t * 132 + g];
      for (int m = g; m < M; m += G) {
        const double x = (double)(m + j);
#pragma unroll
        for (int t = 0; t < TCH; ++t) acc[t] = fma(c[t], x, acc[t]);
      }
    } else if (MODE == 4) {  // 8 rows x 4 columns per thread, [m][t] smem layout, split-m
      // emulate: 32 column-groups x 8 m-groups; LDS.128 x4 + LDG x2 per 32 FMA
      __shared__ __align__(16) double cT[132 * TCH];
      for (int x = threadIdx.x; x < TCH * M; x += NT) cT[(x % M) * TCH + x / M] = coef[(x / M) * 132 + x % M];
      __syncthreads();
      const int cg = threadIdx.x & 31, mg = threadIdx.x >> 5;
      double a4[TCH][4];
#pragma unroll
      for (int t = 0; t < TCH; ++t)
#pragma unroll
        for (int q = 0; q < 4; ++q) a4[t][q] = 0;
      for (int m = mg; m < M; m += 8) {
        const double2 x01 = *reinterpret_cast<const double2*>(In + m * ld + 4 * cg);
        const double2 x23 = *reinterpret_cast<const double2*>(In + m * ld + 4 * cg + 2);
#pragma unroll
        for (int t2 = 0; t2 < TCH; t2 += 2) {
          const double2 cc = *reinterpret_cast<const double2*>(cT + m * TCH + t2);
          a4[t2][0] = fma(cc.x, x01.x, a4[t2][0]); a4[t2][1] = fma(cc.x, x01.y, a4[t2][1]);
          a4[t2][2] = fma(cc.x, x23.x, a4[t2][2]); a4[t2][3] = fma(cc.x, x23.y, a4[t2][3]);
          a4[t2+1][0] = fma(cc.y, x01.x, a4[t2+1][0]); a4[t2+1][1] = fma(cc.y, x01.y, a4[t2+1][1]);
          a4[t2+1][2] = fma(cc.y, x23.x, a4[t2+1][2]); a4[t2+1][3] = fma(cc.y, x23.y, a4[t2+1][3]);
        }
      }
#pragma unroll
      for (int t = 0; t < TCH; ++t) acc[t] = a4[t][0] + a4[t][1] + a4[t][2] + a4[t][3];
    } else {  // MODE 2: compute only (In from smem-less constant)
      for (int m = g; m < M; m += G) {
        const double x = (double)(m + j);
#pragma unroll
        for (int t = 0; t < TCH; ++t) acc[t] = fma(coef[t * 132 + m], x, acc[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < TCH; ++t) red[(t * G + g) * jt + j] = acc[t];
    __syncthreads();
    if (g == 0)
#pragma unroll
      for (int t = 0; t < TCH; ++t) Out[(t0 + t) * ld + j] = red[(t * G) * jt + j] + red[(t * G + 1) * jt + j];
    __syncthreads();
  }
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}
int main() {
  const int M = 128, J = 128, ld = 132, reps = 50;
  double *C, *I, *O; long long* cyc;
  cudaMalloc(&C, 132 * ld * 8); cudaMalloc(&I, 132 * ld * 8); cudaMalloc(&O, 132 * ld * 8); cudaMalloc(&cyc, 64 * 8);
  cudaMemset(C, 0, 132 * ld * 8); cudaMemset(I, 0, 132 * ld * 8);
  long long h[64];
  for (int mode = 0; mode < 5; ++mode) {
    for (int it = 0; it < 3; ++it) {
      if (mode == 0) k_gemm<0><<<16, NT>>>(C, I, O, M, J, ld, reps, cyc);
      if (mode == 1) k_gemm<1><<<16, NT>>>(C, I, O, M, J, ld, reps, cyc);
      if (mode == 2) k_gemm<2><<<16, NT>>>(C, I, O, M, J, ld, reps, cyc);
      if (mode == 3) k_gemm<3><<<16, NT>>>(C, I, O, M, J, ld, reps, cyc);
      if (mode == 4) k_gemm<4><<<16, NT>>>(C, I, O, M, J, ld, reps, cyc);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
    printf("mode %d: %.0f cycles per GEMM (CTA 0), %.2f us @1.965GHz; err=%s\n", mode, (double)h[0] / reps,
           h[0] / reps / 1965.0, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
