// Dev microbenchmark: dependent-chain latencies of the fp64 operations the
// event kernel's serial phases are made of (one warp, one CTA). Not product.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double frcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  return r;
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int OP>
__global__ void k(double* out, long long* cyc, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-9, y = 1.0000001, z = 0.5;
  double x2 = x + 1, x3 = x + 2, x4 = x + 3;
  __shared__ double sm[64];
  sm[threadIdx.x] = x; sm[threadIdx.x + 32] = y;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = fma(x, y, z);
    if (OP == 1) x = x + y;
    if (OP == 2) x = y / x;
    if (OP == 3) x = sqrt(x) + y;
    if (OP == 4) x = frcp(x) + y;
    if (OP == 5) x += __shfl_xor_sync(0xffffffffu, x, 1);
    if (OP == 6) { dmma(x, z, y, y); }
    if (OP == 7) { x = frcp(x) + y; x2 = frcp(x2) + y; x3 = frcp(x3) + y; x4 = frcp(x4) + y; }
    if (OP == 8) { x = y / x; x2 = y / x2; x3 = y / x3; x4 = y / x4; }
    if (OP == 9) x = rsqrt(x) + y;
    if (OP == 10) { x = sm[((int)x) & 31] + y; }
    if (OP == 11) { float f = (float)x; f = fmaf(f, 1.0001f, 0.5f); x = f; }
    if (OP == 12) { dmma(x, z, y, y); dmma(x2, x3, y, y); }
    if (OP == 14) { out[1024 + threadIdx.x + 32 * (i & 7)] = x; __syncthreads(); x += 1.0; }
    if (OP == 15) { __syncthreads(); x += 1.0; }
    if (OP == 16) { out[1024 + threadIdx.x + 32 * (i & 7)] = x; x += 1.0; }
    if (OP == 17) { out[1024 + threadIdx.x + 32 * (i & 7)] = x; __syncthreads(); x += sm[threadIdx.x]; __syncthreads(); }
    if (OP == 18) { sm[threadIdx.x] = x; __syncthreads(); x += sm[(threadIdx.x + 1) & 31]; __syncthreads(); }
    if (OP == 19) { out[1024 + threadIdx.x + 32 * (i & 7)] = x; __threadfence_block(); x += 1.0; }
    if (OP == 20) { out[1024 + threadIdx.x + 32 * (i & 7)] = x; __threadfence(); x += 1.0; }
    if (OP == 13) { dmma(x, z, y, y); dmma(x2, x3, y, y); dmma(x4, y, z, z); dmma(sm[0], sm[1], z, z);}
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x + x2 + x3 + x4 + z + sm[0];
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 65536); cudaMalloc(&c, 64);
  const char* names[] = {"dfma", "dadd", "ddiv (IEEE)", "dsqrt + dadd", "frcp + dadd", "shfl(f64) + dadd", "dmma m8n8k4 (dependent)",
                         "4 x (frcp + dadd) interleaved", "4 x ddiv interleaved", "rsqrt + dadd", "lds + dadd (+cvt)", "cvt f64->f32, ffma, cvt back",
                         "2 independent dmma", "4 independent dmma", "stg + syncthreads", "syncthreads", "stg only", "stg + sync + lds + sync", "sts + sync + lds + sync", "stg + threadfence_block", "stg + threadfence"};
  const int n = 4096;
  long long h;
#define RUN(OP) k<OP><<<1, 32>>>(o, c, 1.5, n); k<OP><<<1, 32>>>(o, c, 1.5, n); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("%-36s %7.1f cycles/iter\n", names[OP], (double)h / n);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9) RUN(10) RUN(11) RUN(12) RUN(13) RUN(14) RUN(15) RUN(16) RUN(17) RUN(18) RUN(19) RUN(20)
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
