// Dev microbenchmark: operand streaming variants for the event kernel's
// per-CTA row GEMM (8 x 128 x 128 fp64 DMMA per CTA, 16-CTA cluster, the
// 128 x 128 operand streamed from L2 into a shared-memory ring).
//   mode 0: 2 slots x 32 rows, every CTA copies the whole operand (current)
//   mode 1: as 0 but a distinct operand per CTA (same-address contention?)
//   mode 2: 4 slots x 16 rows
//   mode 3: 8 slots x 8 rows
//   mode 4: copies only (no DMMA): per-SM bulk-copy throughput, 2 x 32
//   mode 5: multicast: each CTA copies 1/16 of every chunk to all 16 CTAs,
//           slot reuse ordered by split cluster barriers (arrive / wait)
//   mode 6: multicast, copies only
//   mode 7: DMMA only (operand resident)
// Not part of the product.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
constexpr int NT = 256, LD = 132, CL = 16;
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mwait(unsigned bar, unsigned ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n\t}" ::"r"(bar), "r"(ph) : "memory");
}
// SLOTS x CR rows ring; MC: multicast; NOMMA: copies only; RES: resident operand
template <int SLOTS, int CR, bool MC, bool NOMMA, bool RES, bool DISTINCT>
__global__ void __cluster_dims__(CL, 1, 1) k(const double* In0, double* Out, int reps, long long* cyc) {
  extern __shared__ __align__(128) double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  double* co = sm;            // 8 x LD
  double* buf = sm + 8 * LD;  // SLOTS x CR x LD (RES: 128 x LD)
  __shared__ unsigned long long bar[8];
  const double* In = In0 + (DISTINCT ? (size_t)rank * 128 * LD : 0);
  for (int x = threadIdx.x; x < 8 * LD; x += NT) co[x] = 1e-3 * (x % 7);
  if (RES) for (int x = threadIdx.x; x < 128 * LD; x += NT) buf[x] = In[x];
  if (threadIdx.x == 0) {
    for (int i = 0; i < SLOTS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cl.sync();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, ar = lane >> 2, ac = lane & 3;
  const int bc0 = (warp << 3) + ar, bc1 = ((warp + 8) << 3) + ar;
  constexpr int NCH = 128 / CR;
  unsigned ph[SLOTS];
#pragma unroll
  for (int i = 0; i < SLOTS; ++i) ph[i] = 0;
  long long c0 = clock64();
  double tot = 0;
  auto issue = [&](int c) {  // chunk c (global chunk counter within a rep)
    const int s = c % SLOTS;
    const unsigned b = su(&bar[s]), bytes = CR * LD * 8;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    if (!MC) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su(buf + s * CR * LD)), "l"(In + (size_t)c * CR * LD), "r"(bytes), "r"(b) : "memory");
    } else {
      // this CTA's 1/16 of the chunk, to every CTA of the cluster
      const unsigned part = bytes / CL;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
              su(buf + s * CR * LD) + rank * part), "l"((const char*)(In + (size_t)c * CR * LD) + rank * part), "r"(part),
          "r"(b), "h"((unsigned short)0xFFFF) : "memory");
    }
  };
  for (int r = 0; r < reps; ++r) {
    double d0[2][2] = {{0, 0}, {0, 0}}, d1[2][2] = {{0, 0}, {0, 0}};
    if (!RES && threadIdx.x == 0) {
      for (int c = 0; c < SLOTS && c < NCH; ++c) issue(c);
    }
    for (int c = 0; c < NCH; ++c) {
      const int s = c % SLOTS;
      const double* sb = RES ? buf + c * CR * LD : buf + s * CR * LD;
      if (!RES) {
        mwait(su(&bar[s]), ph[s]);
        ph[s] ^= 1;
      }
      if (!NOMMA) {
#pragma unroll
        for (int mm = 0; mm < CR; mm += 8) {
          double a[2], b[2][2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int mr = mm + 4 * u + ac;
            a[u] = co[ar * LD + c * CR + mr];
            b[u][0] = sb[mr * LD + bc0];
            b[u][1] = sb[mr * LD + bc1];
          }
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int p = 0; p < 2; ++p) dmma(d0[u & 1][p], d1[u & 1][p], a[u], b[u][p]);
        }
      }
      if (!RES) {
        __syncthreads();
        if (MC) {
          // every CTA must be done with slot s before anyone overwrites it
          if (c + SLOTS < NCH) {
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
          }
        }
        if (threadIdx.x == 0 && c + SLOTS < NCH) issue(c + SLOTS);
      }
    }
    tot += d0[0][0] + d0[1][1] + d1[0][1] + d1[1][0];
    __syncthreads();
    if (MC) cl.sync();
  }
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  if (tot == 12345.0) Out[threadIdx.x] = tot;
}
template <class K>
void run(const char* name, K kern, int smem, const double* I, double* O, long long* cyc) {
  const int reps = 200;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int it = 0; it < 3; ++it) kern<<<CL, NT, smem>>>(I, O, reps, cyc);
  cudaDeviceSynchronize();
  long long h[CL];
  cudaMemcpy(h, cyc, CL * 8, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < CL; ++i) mx = h[i] > mx ? h[i] : mx;
  const double cpg = (double)mx / reps;
  printf("%-44s %7.0f cycles per GEMM, %.2f us, %.1f B/clk; %s\n", name, cpg, cpg / 1965.0, 128.0 * LD * 8 / cpg,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  double *I, *O; long long* cyc;
  cudaMalloc(&I, (size_t)CL * 128 * LD * 8); cudaMalloc(&O, 4096 * 8); cudaMalloc(&cyc, 64 * 8);
  cudaMemset(I, 0, (size_t)CL * 128 * LD * 8);
  const int ring = (8 + 64) * LD * 8, res = (8 + 128) * LD * 8;
  run("0: 2x32 unicast", k<2, 32, false, false, false, false>, ring, I, O, cyc);
  run("1: 2x32 unicast, distinct operand per CTA", k<2, 32, false, false, false, true>, ring, I, O, cyc);
  run("2: 4x16 unicast", k<4, 16, false, false, false, false>, ring, I, O, cyc);
  run("3: 8x8 unicast", k<8, 8, false, false, false, false>, ring, I, O, cyc);
  run("4: 2x32 unicast, copies only", k<2, 32, false, true, false, false>, ring, I, O, cyc);
  run("4b: 8x8 unicast, copies only", k<8, 8, false, true, false, false>, ring, I, O, cyc);
  run("4c: 4x32 unicast (whole operand), copies only", k<4, 32, false, true, false, false>, res, I, O, cyc);
  run("4d: 4x32 unicast (whole operand)", k<4, 32, false, false, false, false>, res, I, O, cyc);
  run("5: 2x32 multicast", k<2, 32, true, false, false, false>, ring, I, O, cyc);
  run("5b: 4x16 multicast", k<4, 16, true, false, false, false>, ring, I, O, cyc);
  run("5c: 4x32 multicast (whole operand)", k<4, 32, true, false, false, false>, res, I, O, cyc);
  run("6: 2x32 multicast, copies only", k<2, 32, true, true, false, false>, ring, I, O, cyc);
  run("6c: 4x32 multicast (whole operand), copies only", k<4, 32, true, true, false, false>, res, I, O, cyc);
  run("7: resident operand, DMMA only", k<2, 32, false, false, true, false>, res, I, O, cyc);
  return 0;
}
