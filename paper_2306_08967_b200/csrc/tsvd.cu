// Device randomized truncated SVD of the adjacency: the reference's
// FactorState::init_from_graph (factor_state.cpp:84-102) over
// randomized_tsvd (svd.cpp:47-96), so Engine(g, cfg) starts on the GPU.
//
//   l = min_dim <= 600 ? min_dim : min(min_dim, d + 10)
//   Y = A Omega, Q = qr(Y); 4 x { Q = qr(A^T Q); Q = qr(A Q) } (l < min_dim)
//   B^T = A^T Q = Q2 R2;  R2^T = Uc S Vc^T;  U = Q Uc, V = Q2 Vc
//   keep k = min(d, rank) columns above 1e-12 s_1;  X_b = U sqrt(S), Y_b = V sqrt(S)
//
// Omega is the reference's stream (mt19937_64 + Box-Muller, rng.hpp),
// generated on the host, so the device init reproduces the reference's
// subspace; everything else is fp64 on the device:
//   spmm_gather_f64   y[u] = sum_{p in row u} w_p x[ids_p]   (warp per row; rows above
//                     256 arcs by spmm_heavy_f64, a block per 2,048-arc chunk)
//   gram_dmma         G = Y^T Y, upper triangle  (row tiles in shared memory, FP64
//                     tensor cores, fp64 atomics)
//   chol_f64          G = R^T R, R^-1 (one CTA)  -> CholeskyQR2 (gs_qr when rank-deficient)
//   tall_mm_dmma      Y <- Y M  (row tiles in shared memory, FP64 tensor cores; fp64 or fp32 out)
//   jacobi_svd_f64    one-sided Jacobi (round-robin pairs, one CTA)
// Graphs with min_dim <= 600 take the reference's exact path (l = min_dim,
// no power iterations), which is the exact truncated SVD of A: a dense
// one-sided Jacobi SVD of A directly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "common.cuh"
#include "tsvd.cuh"

namespace dgpu {

namespace {

constexpr int TT = 256;

// y[u] = sum_p w_p x[ids_p]: warp per row, NV column values per lane (one
// pass over the row for l <= 32 NV), 4 neighbour rows in flight.
// Rows above kSpmmHeavy arcs are left at zero here and accumulated by
// spmm_heavy_f64 (one warp walking a 100 k-arc hub row set the length of the
// whole product on R-MAT graphs: 625 GB/s of DRAM traffic at scale 22).
constexpr int kSpmmHeavy = 256;    // rows above this many arcs go to spmm_heavy_f64
constexpr int kSpmmChunk = 2048;   // arcs one block of spmm_heavy_f64 takes (8 warps x 256)
template <int NV>
__global__ void spmm_gather_f64(const int64_t* off, const int32_t* ids, const double* wts,
                                int64_t n, const double* __restrict__ x, double* __restrict__ y,
                                int l) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = warp; u < n; u += nw) {
    const int64_t b = off[u], e = off[u + 1] - off[u] > kSpmmHeavy ? off[u] : off[u + 1];
    double acc[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) acc[t] = 0.0;
    for (int64_t p0 = b; p0 < e; p0 += 32) {
      const int64_t p = p0 + lane;
      int v = 0;
      double w = 0.0;
      if (p < e) {
        v = ids[p];
        w = wts ? wts[p] : 1.0;
      }
      const int cnt = (int)(e - p0 < 32 ? e - p0 : 32);
      for (int s0 = 0; s0 < cnt; s0 += 4) {
        double xv[4][NV];
        double ww[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int src = s0 + h < cnt ? s0 + h : 0;
          const int vv = __shfl_sync(0xffffffffu, v, src);
          ww[h] = s0 + h < cnt ? __shfl_sync(0xffffffffu, w, src) : 0.0;
          const double* xr = x + (int64_t)vv * l;
#pragma unroll
          for (int t = 0; t < NV; ++t) {
            const int c = lane + 32 * t;
            xv[h][t] = c < l ? xr[c] : 0.0;
          }
        }
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
          for (int t = 0; t < NV; ++t) acc[t] = fma(ww[h], xv[h][t], acc[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      const int c = lane + 32 * t;
      if (c < l) y[u * l + c] = acc[t];
    }
  }
}

// heavy[0 .. *count): rows with more than kSpmmHeavy arcs; *maxdeg = the largest of them
__global__ void collect_heavy(const int64_t* off, int64_t n, int* heavy, int* count, int cap, int* maxdeg) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = off[u + 1] - off[u];
    if (c > kSpmmHeavy) {
      const int at = atomicAdd(count, 1);
      if (at < cap) heavy[at] = (int)u;
      atomicMax(maxdeg, (int)(c > 0x7fffffff ? 0x7fffffff : c));
    }
  }
}
// y[u] += sum over chunk blockIdx.x (kSpmmChunk arcs) of heavy row u = heavy[blockIdx.y]:
// 8 warps x 256 arcs, four neighbour rows in flight per warp, block-reduced
// in shared memory, one fp64 atomic per column (y[u] was left at zero).
template <int NV>
__global__ void __launch_bounds__(TT) spmm_heavy_f64(const int64_t* off, const int32_t* ids, const double* wts,
                                                     const int* heavy, const double* __restrict__ x,
                                                     double* __restrict__ y, int l) {
  extern __shared__ double red[];  // 8 x l
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t u = heavy[blockIdx.y];
  const int64_t rb = off[u], re = off[u + 1];
  const int64_t cb = rb + (int64_t)blockIdx.x * kSpmmChunk;
  if (cb >= re) return;
  const int64_t ce = cb + kSpmmChunk < re ? cb + kSpmmChunk : re;
  const int64_t b = cb + (int64_t)warp * (kSpmmChunk / 8);
  const int64_t e = b + kSpmmChunk / 8 < ce ? b + kSpmmChunk / 8 : ce;
  double acc[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) acc[t] = 0.0;
  for (int64_t p0 = b; p0 < e; p0 += 32) {
    const int64_t p = p0 + lane;
    int v = 0;
    double w = 0.0;
    if (p < e) {
      v = ids[p];
      w = wts ? wts[p] : 1.0;
    }
    const int cnt = (int)(e - p0 < 32 ? e - p0 : 32);
    for (int s0 = 0; s0 < cnt; s0 += 4) {
      double xv[4][NV];
      double ww[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int src = s0 + h < cnt ? s0 + h : 0;
        const int vv = __shfl_sync(0xffffffffu, v, src);
        ww[h] = s0 + h < cnt ? __shfl_sync(0xffffffffu, w, src) : 0.0;
        const double* xr = x + (int64_t)vv * l;
#pragma unroll
        for (int t = 0; t < NV; ++t) {
          const int c = lane + 32 * t;
          xv[h][t] = c < l ? xr[c] : 0.0;
        }
      }
#pragma unroll
      for (int h = 0; h < 4; ++h)
#pragma unroll
        for (int t = 0; t < NV; ++t) acc[t] = fma(ww[h], xv[h][t], acc[t]);
    }
  }
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = lane + 32 * t;
    if (c < l) red[warp * l + c] = acc[t];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < l; c += TT) {
    double sum = 0.0;
#pragma unroll
    for (int w8 = 0; w8 < 8; ++w8) sum += red[w8 * l + c];
    if (sum != 0.0) atomicAdd(&y[u * l + c], sum);
  }
}

// ---- FP64 tensor-core forms (mma.sync m8n8k4 .f64: a = A[lane>>2][lane&3],
// b = B[lane&3][lane>>2], d{0,1} = D[lane>>2][2 (lane&3) + {0,1}]). SIMT fp64
// FMAs run at ~6 TFLOP/s on this chip (the SIMT forms of both kernels below
// were bound by them: 384 / 290 ms at scale 21 against 147 / 89 ms);
// the DMMA pipe does 55 FMA/clk/SM (tools/micro_dmma.cu).
DAMF_D void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
// padded row strides that keep the fragment loads at two wavefronts
inline int gram_lp(int l) {  // == 8 or 24 mod 32, >= 8 ceil(l / 8)
  int lp = 8 * ((l + 7) / 8);
  while (lp % 32 != 8 && lp % 32 != 24) lp += 8;
  return lp;
}
inline int mm_lp(int l) {  // == 4 mod 8 (odd multiple of 4), >= l rounded up to 4
  int lp = (l + 3) & ~3;
  if (lp % 8 == 0) lp += 4;
  return lp;
}
// Upper triangle of G += Y^T Y in 8 x 8 tiles, tile q of the flat list to warp
// q % 8; up to GT tiles per warp per launch (pass p covers tiles [p 8 GT, +8 GT)).
constexpr int GT = 22;
__global__ void __launch_bounds__(TT) gram_dmma(const double* __restrict__ Y, int64_t n, int l, int lp,
                                                double* G, int pass) {
  extern __shared__ double sy[];  // RT x lp
  constexpr int RT = 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nt = (l + 7) / 8, T = nt * (nt + 1) / 2;
  const int fr = lane >> 2, fk = lane & 3;
  // this warp's tiles: (it, jt), jt >= it, from the flat index
  int ti[GT], tj[GT];
#pragma unroll
  for (int q = 0; q < GT; ++q) {
    int t = pass * 8 * GT + q * 8 + warp;
    int it = 0;
    if (t < T) {
      while (t >= nt - it) {
        t -= nt - it;
        ++it;
      }
      ti[q] = it;
      tj[q] = it + t;
    } else {
      ti[q] = -1;
      tj[q] = -1;
    }
  }
  double d0[GT], d1[GT];
#pragma unroll
  for (int q = 0; q < GT; ++q) d0[q] = d1[q] = 0.0;
  for (int64_t r0 = (int64_t)blockIdx.x * RT; r0 < n; r0 += (int64_t)gridDim.x * RT) {
    const int rows = (int)(n - r0 < RT ? n - r0 : RT);
    __syncthreads();
    for (int x = threadIdx.x; x < RT * lp; x += TT) {
      const int r = x / lp, c = x % lp;
      sy[x] = (r < rows && c < l) ? Y[(r0 + r) * l + c] : 0.0;
    }
    __syncthreads();
    for (int k0 = 0; k0 < RT; k0 += 4) {
      const double* row = sy + (k0 + fk) * lp + fr;
#pragma unroll
      for (int q = 0; q < GT; ++q)
        if (ti[q] >= 0) dmma884(d0[q], d1[q], row[8 * ti[q]], row[8 * tj[q]]);
    }
  }
#pragma unroll
  for (int q = 0; q < GT; ++q) {
    if (ti[q] < 0) continue;
    const int gi = 8 * ti[q] + fr, gj = 8 * tj[q] + 2 * fk;
    if (gi < l && gj < l && d0[q] != 0.0) atomicAdd(&G[gi * l + gj], d0[q]);
    if (gi < l && gj + 1 < l && d1[q] != 0.0) atomicAdd(&G[gi * l + gj + 1], d1[q]);
  }
}
// out[r][c] = sum_m Y[r][m] M[m][c] for c < mc (M: l x mc row-major), row tiles
// of 64 staged in shared memory (in place when out == Y and mc <= l): warp w
// owns rows 8 w .. 8 w + 7 of the tile and walks the columns in groups of MT8
// 8-column tiles.
constexpr int MT8 = 18;
template <typename TO>
__global__ void __launch_bounds__(TT) tall_mm_dmma(const double* Y, int64_t n, int l, int lp,
                                                   const double* __restrict__ M, int mc, TO* out, int ldo) {
  extern __shared__ double st[];  // 64 x lp
  constexpr int RT = 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int l4 = (l + 3) & ~3;
  for (int64_t r0 = (int64_t)blockIdx.x * RT; r0 < n; r0 += (int64_t)gridDim.x * RT) {
    const int rows = (int)(n - r0 < RT ? n - r0 : RT);
    __syncthreads();
    for (int x = threadIdx.x; x < RT * lp; x += TT) {
      const int r = x / lp, c = x % lp;
      st[x] = (r < rows && c < l) ? Y[(r0 + r) * l + c] : 0.0;
    }
    __syncthreads();
    for (int c0 = 0; c0 < mc; c0 += 8 * MT8) {
      double d0[MT8], d1[MT8];
#pragma unroll
      for (int t = 0; t < MT8; ++t) d0[t] = d1[t] = 0.0;
      for (int k0 = 0; k0 < l4; k0 += 4) {
        const double a = st[(8 * warp + fr) * lp + k0 + fk];
        const int km = k0 + fk;
        const double* mrow = M + (int64_t)km * mc + c0 + fr;
#pragma unroll
        for (int t = 0; t < MT8; ++t) {
          const double b = (km < l && c0 + 8 * t + fr < mc) ? __ldg(mrow + 8 * t) : 0.0;
          dmma884(d0[t], d1[t], a, b);
        }
      }
      const int r = 8 * warp + fr;
      if (r < rows) {
#pragma unroll
        for (int t = 0; t < MT8; ++t) {
          const int c = c0 + 8 * t + 2 * fk;
          if (c < mc) out[(r0 + r) * ldo + c] = (TO)d0[t];
          if (c + 1 < mc) out[(r0 + r) * ldo + c + 1] = (TO)d1[t];
        }
      }
    }
  }
}

// G = R^T R (R upper, row-major l x l, written in place of R), Rinv = R^-1.
// One CTA. fail = 1 when a pivot is not positive (rank-deficient sketch).
__global__ void chol_f64(const double* G, int l, double* R, double* Rinv, int* fail) {
  __shared__ double dj;
  __shared__ int bad;
  for (int x = threadIdx.x; x < l * l; x += blockDim.x) R[x] = 0.0;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  double gmax = 0.0;
  for (int i = 0; i < l; ++i) gmax = fmax(gmax, G[i * l + i]);
  for (int j = 0; j < l; ++j) {
    if (threadIdx.x == 0) {
      double s = G[j * l + j];
      for (int i = 0; i < j; ++i) s -= R[i * l + j] * R[i * l + j];
      // a residual below 1e-6 of the column's own norm (1e-12 in the Gram
      // entries, which carry ~1e-16 of cancellation error) is a numerically
      // dependent column: CholeskyQR cannot orthogonalise it; the caller
      // switches to the Gram-Schmidt path (gs_qr)
      if (!(s > 1e-12 * G[j * l + j]) || !(s > 1e-28 * gmax)) {
        bad = 1;
        s = 1.0;
      }
      dj = sqrt(s);
      R[j * l + j] = dj;
    }
    __syncthreads();
    for (int c = j + 1 + threadIdx.x; c < l; c += blockDim.x) {
      double s = G[j * l + c];
      for (int i = 0; i < j; ++i) s -= R[i * l + j] * R[i * l + c];
      R[j * l + c] = s / dj;
    }
    __syncthreads();
  }
  // R^-1 (upper): column c by back substitution, one thread per column
  for (int c = threadIdx.x; c < l; c += blockDim.x) {
    for (int i = l - 1; i >= 0; --i) {
      if (i > c) {
        Rinv[i * l + c] = 0.0;
        continue;
      }
      double s = i == c ? 1.0 : 0.0;
      for (int m = i + 1; m <= c; ++m) s -= R[i * l + m] * Rinv[m * l + c];
      Rinv[i * l + c] = s / R[i * l + i];
    }
  }
  if (threadIdx.x == 0 && bad) *fail = 1;
}

// ---- rank-deficient sketches: classical Gram-Schmidt, twice, column by column
// (the reference's Householder QR, svd.cpp:75-95 via qr_orthonormalize,
// orthogonalises any sketch and completes the basis; CholeskyQR2 needs full
// numerical rank). Used only after chol_f64 reports a dependent column.
// c[t] (t <= j, zeroed) += sum_r M[r][t] M[r][j]
__global__ void gs_dots(const double* __restrict__ M, int64_t n, int l, int j, double* c) {
  const int t = threadIdx.x;
  double acc = 0.0;
  for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
    const double mj = M[r * l + j];
    if (t <= j) acc = fma(M[r * l + t], mj, acc);
  }
  if (t <= j && acc != 0.0) atomicAdd(c + t, acc);
}
// M[r][j] -= sum_{t<j} M[r][t] c[t]   (one warp per row)
__global__ void gs_update(double* M, int64_t n, int l, int j, const double* __restrict__ c) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = w; r < n; r += nw) {
    double s = 0.0;
    for (int t = lane; t < j; t += 32) s = fma(M[r * l + t], c[t], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) M[r * l + j] -= s;
  }
}
// M[r][j] *= scale, or (fill) a fixed pseudo-random completion vector
__global__ void gs_col(double* M, int64_t n, int l, int j, double scale, int fill) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    if (fill) {
      unsigned long long x = (unsigned long long)r * 0x9E3779B97F4A7C15ull + (unsigned long long)(j + 1) * 0xBF58476D1CE4E5B9ull;
      x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
      M[r * l + j] = (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    } else {
      M[r * l + j] *= scale;
    }
  }
}

__global__ void scale_cols(double* M, int rows, int cols, const double* s) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < rows * cols; x += gridDim.x * blockDim.x)
    M[x] *= s[x % cols];
}

__global__ void norm2_f64(const double* x, int64_t m, double* out) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    s += x[i] * x[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

__global__ void dense_from_csr(const int64_t* off, const int32_t* ids, const double* wts, int n,
                               double* A /* column-major n x n */) {
  for (int u = blockIdx.x; u < n; u += gridDim.x)
    for (int64_t p = off[u] + threadIdx.x; p < off[u + 1]; p += blockDim.x)
      atomicAdd(&A[(int64_t)ids[p] * n + u], wts ? wts[p] : 1.0);  // A[u][v], column v
}

// One-sided Jacobi SVD of A (m x l, column-major): A V = U S. On exit the
// columns of A hold U S (unsorted), V (l x l column-major) the right vectors.
// Round-robin pairings; one warp per column pair.
__global__ void jacobi_svd_f64(double* A, int m, int l, double* V, int* sweeps_out) {
  __shared__ int perm[1024];
  __shared__ double smax[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int L = (l + 1) & ~1;  // even count; index l is a dummy when l is odd
  for (int x = threadIdx.x; x < l * l; x += blockDim.x) V[x] = (x / l == x % l) ? 1.0 : 0.0;
  for (int i = threadIdx.x; i < L; i += blockDim.x) perm[i] = i;
  __syncthreads();
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    double off = 0.0;
    for (int step = 0; step < L - 1; ++step) {
      for (int pr = warp; pr < L / 2; pr += nw) {
        int i = perm[pr], j = perm[L - 1 - pr];
        if (i >= l || j >= l) continue;
        if (i > j) {
          const int t = i;
          i = j;
          j = t;
        }
        double* ai = A + (int64_t)i * m;
        double* aj = A + (int64_t)j * m;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int r = lane; r < m; r += 32) {
          const double x = ai[r], y = aj[r];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (ga == 0.0 || fabs(ga) <= 1e-15 * sqrt(al * be)) continue;
        off = fmax(off, fabs(ga) / sqrt(al * be));
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int r = lane; r < m; r += 32) {
          const double x = ai[r], y = aj[r];
          ai[r] = c * x - s * y;
          aj[r] = s * x + c * y;
        }
        double* vi = V + (int64_t)i * l;
        double* vj = V + (int64_t)j * l;
        for (int r = lane; r < l; r += 32) {
          const double x = vi[r], y = vj[r];
          vi[r] = c * x - s * y;
          vj[r] = s * x + c * y;
        }
      }
      __syncthreads();
      // rotate the tournament (position 0 fixed)
      if (threadIdx.x == 0) {
        const int last = perm[L - 1];
        for (int q = L - 1; q > 1; --q) perm[q] = perm[q - 1];
        perm[1] = last;
      }
      __syncthreads();
    }
    if (lane == 0) smax[warp] = off;
    __syncthreads();
    double mx = 0.0;
    for (int w = 0; w < nw; ++w) mx = fmax(mx, smax[w]);
    __syncthreads();
    if (mx <= 1e-15) break;
  }
  if (threadIdx.x == 0) *sweeps_out = sweep;
}

__global__ void col_norms(const double* A, int m, int l, double* s) {
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int c = warp; c < l; c += nw) {
    double v = 0.0;
    for (int r = lane; r < m; r += 32) v = fma(A[(int64_t)c * m + r], A[(int64_t)c * m + r], v);
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s[c] = sqrt(v);
  }
}

// Counter-based Gaussians for large sketches (Philox-4x32-10 + Box-Muller):
// same distribution as the reference stream, not the same bits.
__device__ __forceinline__ void philox(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0, h1 = (uint32_t)(p1 >> 32),
                   l1 = (uint32_t)p1;
    c[0] = h1 ^ c[1] ^ k0;
    c[1] = l1;
    c[2] = h0 ^ c[3] ^ k1;
    c[3] = l0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}
__global__ void gaussian_fill(double* out, int64_t count, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c[4] = {(uint32_t)i, (uint32_t)(i >> 32), 0x5bd1e995u, 0u};
    philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t a = ((uint64_t)c[0] << 32) | c[1], b = ((uint64_t)c[2] << 32) | c[3];
    const double u1 = ((double)(a >> 11) + 0.5) * 0x1.0p-53, u2 = (double)(b >> 11) * 0x1.0p-53;
    out[i] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

}  // namespace

// reference rng.hpp: mt19937_64, rand_unit = (x >> 11) * 2^-53, Box-Muller
// with u1 > 0 rejection, one cosine sample per pair of draws
static void reference_gaussians(uint64_t seed, int64_t count, double* out) {
  std::mt19937_64 rng(seed);
  for (int64_t i = 0; i < count; ++i) {
    double u1;
    do {
      u1 = (double)(rng() >> 11) * 0x1.0p-53;
    } while (u1 <= 0.0);
    const double u2 = (double)(rng() >> 11) * 0x1.0p-53;
    out[i] = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
}

#define TCK(x)                           \
  do {                                   \
    cudaError_t _e = (x);                \
    if (_e != cudaSuccess) return _e;    \
  } while (0)

cudaError_t tsvd_init(const TsvdGraph& g, int d, uint64_t seed, cudaStream_t st, int nsm,
                      TsvdResult* res, bool exact_stream) {
  // sketches up to 2^26 Gaussians take the reference's stream (a few seconds on
  // one host core); larger ones a device counter-based generator
  constexpr int64_t kHostStreamMax = int64_t(1) << 26;
  const int64_t n = g.n;
  res->k = 0;
  res->status = 0;
  if (n <= 0 || g.arcs <= 0) {
    res->status = 6;  // ZeroMatrix: init_from_graph: graph has no edges
    return cudaSuccess;
  }
  const int64_t min_dim = n;
  const int l = (int)(min_dim <= 600 ? min_dim : std::min<int64_t>(min_dim, d + 10));
  std::vector<double*> tmp;
  auto alloc = [&](double** p, size_t count) -> cudaError_t {
    cudaError_t e = cudaMalloc(p, std::max<size_t>(count, 1) * sizeof(double));
    if (e == cudaSuccess) tmp.push_back(*p);
    return e;
  };
  auto free_all = [&]() {
    for (double* p : tmp) cudaFree(p);
  };
  int* dflag = nullptr;
  TCK(cudaMalloc(&dflag, 2 * sizeof(int)));
  cudaError_t err = cudaSuccess;
  double *U = nullptr, *V = nullptr, *S = nullptr;  // device: U (n x k, row-major), V, sigma
  int k = 0;
  std::vector<double> hs;
  do {
    if (min_dim <= 600) {
      // exact path: dense A, one-sided Jacobi: A V = U S
      double *A = nullptr, *Vd = nullptr, *s = nullptr;
      if ((err = alloc(&A, (size_t)n * n)) || (err = alloc(&Vd, (size_t)n * n)) ||
          (err = alloc(&s, (size_t)n)))
        break;
      cudaMemsetAsync(A, 0, (size_t)n * n * 8, st);
      dense_from_csr<<<(int)std::min<int64_t>(n, 4096), 128, 0, st>>>(g.off, g.ids, g.wts, (int)n, A);
      jacobi_svd_f64<<<1, 512, 0, st>>>(A, (int)n, (int)n, Vd, dflag);
      col_norms<<<32, 256, 0, st>>>(A, (int)n, (int)n, s);
      if ((err = cudaGetLastError())) break;
      // order by sigma on the host (n <= 600)
      hs.resize(n);
      std::vector<double> ha((size_t)n * n), hv((size_t)n * n);
      cudaMemcpyAsync(hs.data(), s, n * 8, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(ha.data(), A, (size_t)n * n * 8, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(hv.data(), Vd, (size_t)n * n * 8, cudaMemcpyDeviceToHost, st);
      if ((err = cudaStreamSynchronize(st))) break;
      std::vector<int> ord(n);
      for (int i = 0; i < n; ++i) ord[i] = i;
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return hs[a] > hs[b]; });
      int rank = 0;
      while (rank < n && hs[ord[rank]] > 0.0) ++rank;
      k = std::min(d, rank);
      const double floor_ = 1e-12 * (rank > 0 ? hs[ord[0]] : 0.0);
      while (k > 0 && hs[ord[k - 1]] <= floor_) --k;
      if (k == 0) {
        res->status = 6;
        break;
      }
      // X_b = U sqrt(S) = A_col / sigma * sqrt(sigma), Y_b = V sqrt(S); row-major n x k
      std::vector<float> xb((size_t)n * k), yb((size_t)n * k);
      res->sigma.assign(k, 0.0);
      for (int c = 0; c < k; ++c) {
        const int j = ord[c];
        const double sg = hs[j], r = std::sqrt(sg);
        res->sigma[c] = sg;
        for (int64_t r0 = 0; r0 < n; ++r0) {
          xb[r0 * k + c] = (float)(ha[(size_t)j * n + r0] / sg * r);
          yb[r0 * k + c] = (float)(hv[(size_t)j * n + r0] * r);
        }
      }
      res->xb_host.swap(xb);
      res->yb_host.swap(yb);
      res->k = k;
      break;
    }
    // ---- randomized path (l < min_dim)
    double *Y = nullptr, *Q = nullptr, *G = nullptr, *R = nullptr, *Ri = nullptr, *Racc = nullptr,
           *Rt = nullptr, *nrm = nullptr;
    if ((err = alloc(&Y, (size_t)n * l)) || (err = alloc(&Q, (size_t)n * l)) ||
        (err = alloc(&G, (size_t)l * l)) || (err = alloc(&R, (size_t)l * l)) ||
        (err = alloc(&Ri, (size_t)l * l)) || (err = alloc(&Racc, (size_t)l * l)) ||
        (err = alloc(&Rt, (size_t)l * l)) || (err = alloc(&nrm, 1)))
      break;
    if (exact_stream || (int64_t)n * l <= kHostStreamMax) {
      // the reference's own Gaussian stream (rng.hpp), sequential on the host
      std::vector<double> om((size_t)n * l);
      reference_gaussians(seed, (int64_t)n * l, om.data());
      if ((err = cudaMemcpyAsync(Q, om.data(), (size_t)n * l * 8, cudaMemcpyHostToDevice, st))) break;
      if ((err = cudaStreamSynchronize(st))) break;
      res->omega = 0;
    } else {
      gaussian_fill<<<nsm * 16, 256, 0, st>>>(Q, (int64_t)n * l, seed);
      res->omega = 1;
    }
    const int gs = nsm * 8;
    const int glp = gram_lp(l), mlp = mm_lp(l);
    const size_t gram_smem = (size_t)32 * glp * 8, mm_smem = (size_t)64 * mlp * 8;
    cudaFuncSetAttribute(tall_mm_dmma<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mm_smem);
    cudaFuncSetAttribute(gram_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_smem);
    cudaFuncSetAttribute(tall_mm_dmma<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mm_smem);
    const int gram_tiles = ((l + 7) / 8) * ((l + 7) / 8 + 1) / 2;
    const int gram_passes = (gram_tiles + 8 * GT - 1) / (8 * GT);
    // heavy rows of A and of A^T (collected once; order is irrelevant)
    const int kHeavyCap = (int)std::min<int64_t>(n, 0x7fffffff);  // every row could be heavy
    int* hvy[2] = {nullptr, nullptr};
    int hcount[2] = {0, 0}, hmax[2] = {0, 0};
    {
      double* raw = nullptr;  // (freed with the other temporaries)
      if ((err = alloc(&raw, (size_t)kHeavyCap + 8))) break;  // 2 lists of n ints + 4 counters
      hvy[0] = reinterpret_cast<int*>(raw);
      hvy[1] = hvy[0] + kHeavyCap;
      int* meta = hvy[1] + kHeavyCap;  // [count, maxdeg] x 2
      cudaMemsetAsync(meta, 0, 4 * sizeof(int), st);
      for (int tr = 0; tr < 2; ++tr)
        collect_heavy<<<nsm * 8, 256, 0, st>>>(tr ? g.toff : g.off, n, hvy[tr], meta + 2 * tr, kHeavyCap,
                                               meta + 2 * tr + 1);
      int hm[4] = {0, 0, 0, 0};
      cudaMemcpyAsync(hm, meta, sizeof(hm), cudaMemcpyDeviceToHost, st);
      if ((err = cudaStreamSynchronize(st))) break;
      for (int tr = 0; tr < 2; ++tr) {
        hcount[tr] = std::min(hm[2 * tr], kHeavyCap);
        hmax[tr] = hm[2 * tr + 1];
      }
    }
    cudaFuncSetAttribute(spmm_heavy_f64<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 288 * 8);
    cudaFuncSetAttribute(spmm_heavy_f64<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 288 * 8);
    auto apply = [&](const double* x, double* y, bool transposed) {
      const int64_t* o = transposed ? g.toff : g.off;
      const int32_t* i = transposed ? g.tids : g.ids;
      const double* w = transposed ? g.twts : g.wts;
      const int tr = transposed ? 1 : 0;
      if (l <= 160)
        spmm_gather_f64<5><<<gs, 256, 0, st>>>(o, i, w, n, x, y, l);
      else
        spmm_gather_f64<9><<<gs, 256, 0, st>>>(o, i, w, n, x, y, l);
      for (int h0 = 0; h0 < hcount[tr]; h0 += 32768) {
        const dim3 hg((unsigned)((hmax[tr] + kSpmmChunk - 1) / kSpmmChunk),
                      (unsigned)std::min(32768, hcount[tr] - h0));
        if (l <= 160)
          spmm_heavy_f64<5><<<hg, TT, (size_t)8 * l * 8, st>>>(o, i, w, hvy[tr] + h0, x, y, l);
        else
          spmm_heavy_f64<9><<<hg, TT, (size_t)8 * l * 8, st>>>(o, i, w, hvy[tr] + h0, x, y, l);
      }
    };
    // Gram-Schmidt QR in place on Ym (n x l), any rank: Q gets an orthonormal
    // basis whose leading columns span Ym's (dependent columns are replaced by
    // completion vectors, as a Householder Q would hold), Rgs (host, l x l
    // row-major, upper) = Q^T Ym with a zero diagonal entry per dependent column
    double* gc = nullptr;
    if ((err = alloc(&gc, (size_t)l + 1))) break;
    auto gs_qr = [&](double* Ym, std::vector<double>& Rgs) -> cudaError_t {
      Rgs.assign((size_t)l * l, 0.0);
      std::vector<double> hc(l + 1);
      cudaError_t e2 = cudaSuccess;
      for (int j = 0; j < l; ++j) {
        double orig2 = 0.0, fin2 = 0.0;
        for (int attempt = 0; attempt < 2; ++attempt) {  // attempt 1: the completion vector
          for (int pass = 0; pass < 3; ++pass) {         // two projections, then the final norm
            cudaMemsetAsync(gc, 0, (size_t)(l + 1) * 8, st);
            gs_dots<<<gs, 288, 0, st>>>(Ym, n, l, j, gc);
            cudaMemcpyAsync(hc.data(), gc, (size_t)(j + 1) * 8, cudaMemcpyDeviceToHost, st);
            if ((e2 = cudaStreamSynchronize(st))) return e2;
            if (pass == 0) orig2 = hc[j];
            if (pass == 2) {
              fin2 = hc[j];
              break;
            }
            if (attempt == 0)
              for (int t = 0; t < j; ++t) Rgs[(size_t)t * l + j] += hc[t];
            if (j > 0) gs_update<<<gs, 256, 0, st>>>(Ym, n, l, j, gc);
          }
          // dependent: what is left is rounding noise of the projections
          const bool dep = !(fin2 > 1e-20 * orig2) || !(orig2 > 0.0);
          if (!dep) {
            if (attempt == 0) Rgs[(size_t)j * l + j] = std::sqrt(fin2);
            gs_col<<<gs, 256, 0, st>>>(Ym, n, l, j, 1.0 / std::sqrt(fin2), 0);
            break;
          }
          if (attempt == 1) return cudaErrorUnknown;  // (a fixed vector inside the span: not expected)
          gs_col<<<gs, 256, 0, st>>>(Ym, n, l, j, 0.0, 1);
        }
      }
      return cudaGetLastError();
    };
    // CholeskyQR2 in place on Y (n x l); R of the factorisation into Rout.
    // A numerically dependent column (chol_f64's flag, read before the in-place
    // product so that Ym is intact) sends the matrix through gs_qr instead.
    std::vector<double> Rgs;
    auto cholqr2 = [&](double* Ym, double* Rout) -> int {
      int hf = 0;
      for (int pass = 0; pass < 2; ++pass) {
        cudaMemsetAsync(G, 0, (size_t)l * l * 8, st);
        cudaMemsetAsync(dflag, 0, sizeof(int), st);
        // upper triangle only (chol_f64 reads nothing else); one pass over Y per 176 tiles
        for (int ps = 0; ps < gram_passes; ++ps)
          gram_dmma<<<gs, TT, gram_smem, st>>>(Ym, n, l, glp, G, ps);
        chol_f64<<<1, 256, 0, st>>>(G, l, pass == 0 ? Racc : R, Ri, dflag);
        cudaMemcpyAsync(&hf, dflag, sizeof(int), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        if (hf) {
          if (gs_qr(Ym, Rgs) != cudaSuccess) return 1;
          res->gs_fallbacks += 1;
          if (Rout) {
            // R = R_gs (pass 0) or R_gs * R_pass1 (Ym was Y R_pass1^-1 already)
            cudaMemcpyAsync(R, Rgs.data(), (size_t)l * l * 8, cudaMemcpyHostToDevice, st);
            if (pass == 0)
              cudaMemcpyAsync(Rout, R, (size_t)l * l * 8, cudaMemcpyDeviceToDevice, st);
            else
              tall_mm_dmma<double><<<1, TT, mm_smem, st>>>(R, l, l, mlp, Racc, l, Rout, l);
            cudaStreamSynchronize(st);
          }
          return 0;
        }
        tall_mm_dmma<double><<<gs, TT, mm_smem, st>>>(Ym, n, l, mlp, Ri, l, Ym, l);
      }
      if (Rout) {
        // R = R_pass2 * R_pass1 (upper l x l), on the device via tall_mm
        tall_mm_dmma<double><<<1, TT, mm_smem, st>>>(R, l, l, mlp, Racc, l, Rout, l);
      }
      return 0;
    };
    apply(Q, Y, false);  // Y = A Omega
    cudaMemsetAsync(nrm, 0, 8, st);
    norm2_f64<<<gs, 256, 0, st>>>(Y, (int64_t)n * l, nrm);
    double hn = 0;
    cudaMemcpyAsync(&hn, nrm, 8, cudaMemcpyDeviceToHost, st);
    if ((err = cudaStreamSynchronize(st))) break;
    if (hn == 0.0) {
      res->status = 6;  // randomized_tsvd: all-zero matrix
      break;
    }
    if (cholqr2(Y, nullptr)) {
      res->status = 101;  // rank-deficient sketch: not supported on the device path
      break;
    }
    bool bad = false;
    for (int it = 0; it < 4 && !bad; ++it) {
      apply(Y, Q, true);  // Q = A^T Y
      if (cholqr2(Q, nullptr)) bad = true;
      if (!bad) {
        apply(Q, Y, false);  // Y = A Q
        if (cholqr2(Y, nullptr)) bad = true;
      }
    }
    if (bad) {
      res->status = 101;
      break;
    }
    // B^T = A^T Q -> Q2 R2 (Q2 in place in Q)
    apply(Y, Q, true);
    if (cholqr2(Q, Rt)) {
      res->status = 101;
      break;
    }
    // R2^T (l x l) column-major == R2 row-major: Jacobi on it directly
    double *Vc = nullptr, *s = nullptr;
    if ((err = alloc(&Vc, (size_t)l * l)) || (err = alloc(&s, (size_t)l))) break;
    // column-major copy of R2^T: element (r, c) of R2^T = R2[c][r] -> stored at c*l + r,
    // i.e. exactly R2's row-major layout
    jacobi_svd_f64<<<1, 512, 0, st>>>(Rt, l, l, Vc, dflag);
    col_norms<<<32, 256, 0, st>>>(Rt, l, l, s);
    if ((err = cudaGetLastError())) break;
    hs.resize(l);
    std::vector<double> ha((size_t)l * l), hv((size_t)l * l);
    cudaMemcpyAsync(hs.data(), s, l * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(ha.data(), Rt, (size_t)l * l * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(hv.data(), Vc, (size_t)l * l * 8, cudaMemcpyDeviceToHost, st);
    if ((err = cudaStreamSynchronize(st))) break;
    std::vector<int> ord(l);
    for (int i = 0; i < l; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return hs[a] > hs[b]; });
    int rank = 0;
    while (rank < l && hs[ord[rank]] > 0.0) ++rank;
    k = std::min(d, rank);
    const double floor_ = 1e-12 * (rank > 0 ? hs[ord[0]] : 0.0);
    while (k > 0 && hs[ord[k - 1]] <= floor_) --k;
    if (k == 0) {
      res->status = 6;
      break;
    }
    // Uc (l x k) = left vectors of R2^T = columns of (A V)/s; Vc (l x k)
    // X_b = Y Uc sqrt(S) (Y holds Q), Y_b = Q2 Vc sqrt(S) (Q holds Q2)
    std::vector<double> fu((size_t)l * k), fv((size_t)l * k);
    res->sigma.assign(k, 0.0);
    for (int c = 0; c < k; ++c) {
      const int j = ord[c];
      const double sg = hs[j], r = std::sqrt(sg);
      res->sigma[c] = sg;
      for (int m = 0; m < l; ++m) {
        fu[(size_t)m * k + c] = ha[(size_t)j * l + m] / sg * r;
        fv[(size_t)m * k + c] = hv[(size_t)j * l + m] * r;
      }
    }
    double *Fu = nullptr, *Fv = nullptr;
    if ((err = alloc(&Fu, (size_t)l * k)) || (err = alloc(&Fv, (size_t)l * k))) break;
    cudaMemcpyAsync(Fu, fu.data(), (size_t)l * k * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(Fv, fv.data(), (size_t)l * k * 8, cudaMemcpyHostToDevice, st);
    float *xb = nullptr, *yb = nullptr;
    if ((err = cudaMalloc(&xb, (size_t)n * k * 4))) break;
    if ((err = cudaMalloc(&yb, (size_t)n * k * 4))) {
      cudaFree(xb);
      break;
    }
    tall_mm_dmma<float><<<gs, TT, mm_smem, st>>>(Y, n, l, mlp, Fu, k, xb, k);
    tall_mm_dmma<float><<<gs, TT, mm_smem, st>>>(Q, n, l, mlp, Fv, k, yb, k);
    if ((err = cudaStreamSynchronize(st))) {
      cudaFree(xb);
      cudaFree(yb);
      break;
    }
    res->xb_dev = xb;
    res->yb_dev = yb;
    res->k = k;
  } while (0);
  (void)U;
  (void)V;
  (void)S;
  free_all();
  cudaFree(dflag);
  return err;
}

}  // namespace dgpu
