// Dev microbenchmark: the staged per-CTA GEMM (8 x 128 x 128 fp64 DMMA) with
// the event kernel's chunk structure -- 32-row chunks of the streamed operand
// bulk-copied from global into a two-slot ring (mbarrier), __syncthreads per
// chunk -- vs everything resident. 16 CTAs x 8 warps. Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NT = 256, LD = 132, CR = 32;
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int MODE>  // 0: resident, 1: resident + syncthreads per chunk, 2: bulk-copied chunks
__global__ void k(const double* In, double* Out, int reps, long long* cyc) {
  extern __shared__ __align__(128) double sm[];
  double* co = sm;                     // 8 x LD
  double* buf = sm + 8 * LD;           // MODE 0/1: 128 x LD resident; MODE 2: 2 x CR x LD
  __shared__ unsigned long long bar[2];
  for (int x = threadIdx.x; x < 8 * LD; x += NT) co[x] = 1e-3 * (x % 7);
  if (MODE != 2) for (int x = threadIdx.x; x < 128 * LD; x += NT) buf[x] = In[x];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, ar = lane >> 2, ac = lane & 3;
  const int bc0 = (warp << 3) + ar, bc1 = ((warp + 8) << 3) + ar;
  unsigned ph[2] = {0, 0};
  long long c0 = clock64();
  double tot = 0;
  for (int r = 0; r < reps; ++r) {
    double d0[2][2] = {{0, 0}, {0, 0}}, d1[2][2] = {{0, 0}, {0, 0}};
    auto issue = [&](int c) {
      const unsigned b = su(&bar[c & 1]), bytes = CR * LD * 8;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su(buf + (c & 1) * CR * LD)), "l"(In + (size_t)c * CR * LD), "r"(bytes), "r"(b) : "memory");
    };
    if (MODE == 2 && threadIdx.x == 0) { issue(0); issue(1); }
    for (int c = 0; c < 4; ++c) {
      const double* sb = MODE == 2 ? buf + (c & 1) * CR * LD : buf + c * CR * LD;
      if (MODE == 2) {
        asm volatile("{\n\t.reg .pred p;\n\tW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n\t}" ::"r"(su(&bar[c & 1])), "r"(ph[c & 1]) : "memory");
        ph[c & 1] ^= 1;
      }
#pragma unroll
      for (int mm = 0; mm < CR; mm += 16) {
        double a[4], b[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int mr = mm + 4 * u + ac;
          a[u] = co[ar * LD + c * CR + mr];
          b[u][0] = sb[mr * LD + bc0];
          b[u][1] = sb[mr * LD + bc1];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int p = 0; p < 2; ++p) dmma(d0[u & 1][p], d1[u & 1][p], a[u], b[u][p]);
      }
      if (MODE >= 1) __syncthreads();
      if (MODE == 2 && threadIdx.x == 0 && c + 2 < 4) issue(c + 2);
    }
    tot += d0[0][0] + d0[1][1] + d1[0][1] + d1[1][0];
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
  const int smem = (8 + 128) * LD * 8, reps = 200;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h[64];
  for (int mode = 0; mode < 3; ++mode) {
    for (int it = 0; it < 3; ++it) {
      if (mode == 0) k<0><<<16, NT, smem>>>(I, O, reps, cyc);
      if (mode == 1) k<1><<<16, NT, smem>>>(I, O, reps, cyc);
      if (mode == 2) k<2><<<16, NT, smem>>>(I, O, reps, cyc);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
    const double cpg = (double)h[0] / reps;
    printf("mode %d: %.0f cycles per GEMM, %.2f us; %s\n", mode, cpg, cpg / 1965.0, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
