// Dev microbenchmark: cost of a 16-CTA (and 8-CTA) cluster barrier on B200,
// with and without outstanding global stores before it. Not product code.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
template <int MODE>
__global__ void k(double* buf, long long* out, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 1) buf[(blockIdx.x * 256 + threadIdx.x) * 4 + (i & 3)] = i;  // 8 KB of stores per CTA
    if (MODE == 2) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::);
      asm volatile("barrier.cluster.wait.aligned;\n" ::);
    } else {
      cl.sync();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = (t1 - t0) / iters;
}
template <int MODE, int C>
void run(double* buf, long long* d) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C); cfg.blockDim = dim3(256);
  cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = C; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a; cfg.numAttrs = 1;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int r = 0; r < 3; ++r) cudaLaunchKernelEx(&cfg, k<MODE>, buf, d, 1000);
  long long h; cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("C=%2d mode %d: %lld cycles per cluster barrier (%s)\n", C, MODE, h, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  double* buf; long long* d; cudaMalloc(&buf, 1 << 24); cudaMalloc(&d, 8);
  run<0, 16>(buf, d); run<1, 16>(buf, d); run<2, 16>(buf, d);
  run<0, 8>(buf, d); run<1, 8>(buf, d); run<2, 8>(buf, d);
  run<0, 4>(buf, d); run<0, 2>(buf, d);
  return 0;
}
