// Dev microbenchmark: cycles of secular_root (event_kernel.cu) on a config-5-like
// problem (129 poles in a tight cluster plus a heavy pole), for 1 group alone,
// 2 groups in one warp, and 9 groups (the in-kernel layout). Not product.
#include "../paper_2306_08967_b200/csrc/event_kernel.cu"
#include <cstdio>
#include <algorithm>
#include <cmath>
#include <vector>
using namespace dgpu;
__global__ void k(const double* kd, const double* kz2, int K, double rho, double sz2, int heavy,
                  int ngroups, int j0, long long* out, double* taus, int reps) {
  __shared__ double skd[260], skz[260];
  for (int i = threadIdx.x; i < K; i += blockDim.x) { skd[i] = kd[i]; skz[i] = kz2[i]; }
  __syncthreads();
  const int grp = threadIdx.x >> 4;
  long long best = 1ll << 60; int its = 0;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const long long t0 = clock64();
    if (grp < ngroups) {
      double t; int o;
      its = secular_root(skd, skz, K, rho, 1.0 / rho, sz2, j0 + grp, heavy, t, o);
      if ((threadIdx.x & 15) == 0) taus[grp] = t;
    }
    __syncthreads();
    const long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
    if (r == 0 && threadIdx.x == 0) out[30] = t1 - t0;
  }
  if ((threadIdx.x & 15) == 0 && grp < ngroups) { out[1 + grp] = its; }
  if (threadIdx.x == 0) out[0] = best;
}
int main(int argc, char** argv) {
  if (argc > 1) {
    // dumped problems (tools/dump_secular.py -> secular_problems.bin: records of 800 doubles:
    // K, rho, sum z^2, ..., kd at 8, kz2 at 268): every rank's 9 roots, as in the kernel
    FILE* f = fopen(argv[1], "rb");
    if (!f) { printf("cannot open %s\n", argv[1]); return 1; }
    std::vector<double> rec(800);
    double *dkd, *dkz, *dt; long long* dout;
    cudaMalloc(&dkd, 260 * 8); cudaMalloc(&dkz, 260 * 8); cudaMalloc(&dt, 64 * 8); cudaMalloc(&dout, 64 * 8);
    for (int p = 0; p < 4 && fread(rec.data(), 8, 800, f) == 800; ++p) {
      const int K = (int)rec[0];
      int heavy = -1; for (int i = 0; i < K; ++i) if (rec[268 + i] > 0.5 * rec[2]) heavy = i;
      cudaMemcpy(dkd, rec.data() + 8, K * 8, cudaMemcpyHostToDevice);
      cudaMemcpy(dkz, rec.data() + 268, K * 8, cudaMemcpyHostToDevice);
      printf("problem %d: K=%d rho=%.6f heavy=%d\n", p, K, rec[1], heavy);
      for (int j1 : {K - 1, K - 2, K - 3, 5}) {
        k<<<1, 256>>>(dkd, dkz, K, rec[1], rec[2], heavy, 1, j1, dout, dt, 20);
        long long h[20];
        cudaMemcpy(h, dout, 20 * 8, cudaMemcpyDeviceToHost);
        printf("  single root %3d cycles=%6lld its=%lld\n", j1, h[0], h[1]);
      }
      const int per = (K + 15) / 16;
      for (int r = 0; r * per < K; ++r) {
        const int ng = std::min(per, K - r * per);
        k<<<1, 256>>>(dkd, dkz, K, rec[1], rec[2], heavy, ng, r * per, dout, dt, 20);
        long long h[20];
        cudaMemcpy(h, dout, 20 * 8, cudaMemcpyDeviceToHost);
        printf("  rank %2d roots %3d..%3d cycles=%6lld its:", r, r * per, r * per + ng - 1, h[0]);
        for (int g = 0; g < ng; ++g) printf(" %lld", h[1 + g]);
        printf("\n");
      }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
  }

  const int K = 129;
  std::vector<double> d(K), z(K);
  // old spectrum squared: sigma_i = i^-1/2 -> lambda = 1/i, ascending canonical order
  for (int i = 0; i < K - 1; ++i) d[i] = 1.0 / (K - 1 - i);
  d[K - 1] = 1.0; for (int i = 0; i < K - 1; ++i) d[i] = 1.0 / (K - i);
  d[0] = 0.0;
  std::sort(d.begin(), d.end());
  double s = 0; unsigned x = 12345;
  for (int i = 0; i < K; ++i) { x = x * 1664525u + 1013904223u; z[i] = 1e-3 * ((x >> 8) / 16777216.0 + 0.01); z[i] *= z[i]; }
  z[40] = 0.7;  // heavy pole
  for (int i = 0; i < K; ++i) s += z[i];
  for (int i = 0; i < K; ++i) z[i] /= s;
  double *dkd, *dkz, *dt; long long* dout;
  cudaMalloc(&dkd, K * 8); cudaMalloc(&dkz, K * 8); cudaMalloc(&dt, 64 * 8); cudaMalloc(&dout, 64 * 8);
  cudaMemcpy(dkd, d.data(), K * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dkz, z.data(), K * 8, cudaMemcpyHostToDevice);
  for (int heavy : {-1, 40})
    for (int j0 : {10, 60, 120})
      for (int ng : {1, 2, 9, 16}) {
        if (j0 + ng > K) continue;
        k<<<1, 256>>>(dkd, dkz, K, 2.0, 1.0, heavy, ng, j0, dout, dt, 20);
        long long h[20], h30;
        cudaMemcpy(h, dout, 20 * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&h30, dout + 30, 8, cudaMemcpyDeviceToHost);
        printf("heavy=%3d j0=%3d groups=%2d  cycles=%6lld  first-rep=%6lld  its:", heavy, j0, ng, h[0], h30);
        for (int g = 0; g < ng; ++g) printf(" %lld", h[1 + g]);
        printf("\n");
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
