// K5: full-embedding materialisation Z = X * F (factor_state.cpp:120-123
// query_all, :215-222 rebase, enhancer.cpp:196-206 apply_transform).
// Tall-skinny n x k by k x k2 product, HBM-bound at 8 n k bytes.
//
// materialize_simt: persistent FP32 SIMT kernel. F (fp64 on the host side
// of the state) is converted once per CTA into a shared-memory fp32 tile;
// row tiles of X stream through registers with 128-bit loads; each thread
// owns a 4-row x 4-column register block. Safe in place (out == in): a CTA
// reads its whole row tile into shared memory before writing it.
#include <cuda_bf16.h>

#include "common.cuh"
#include "materialize.cuh"

namespace dgpu {

namespace {

constexpr int MT = 256;       // threads
constexpr int RT = 32;        // rows per tile
constexpr int CB = 128;       // output columns per pass

// F block: Fs[m][c] for m < k, c < cb (fp32), X tile Xs[r][m].
__global__ void __launch_bounds__(MT, 1)
    materialize_simt(const float* __restrict__ X, int64_t n, int k, int ldx,
                     const double* __restrict__ FT, int ldf, int k2, float* Z, int ldz,
                     int c0, int cb) {
  extern __shared__ __align__(16) float sm[];
  const int kp = (k + 3) & ~3;
  float* Fs = sm;                 // k x CB
  float* Xs = sm + (size_t)k * CB;  // RT x kp
  // F[m][c] = FT[c][m] (FT rows = output columns)
  for (int x = threadIdx.x; x < k * cb; x += MT) {
    const int c = x / k, m = x % k;
    Fs[m * CB + c] = (float)FT[(int64_t)(c0 + c) * ldf + m];
  }
  for (int x = threadIdx.x; x < k * CB; x += MT) {
    const int m = x / CB, c = x % CB;
    if (c >= cb) Fs[m * CB + c] = 0.0f;
  }
  __syncthreads();
  const int cq = threadIdx.x % 32;  // column quad -> columns 4cq..4cq+3
  const int rg = threadIdx.x / 32;  // row group -> rows 4rg..4rg+3
  const int64_t ntiles = (n + RT - 1) / RT;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * RT;
    const int rows = (int)(n - r0 < RT ? n - r0 : RT);
    // stage the X tile (k columns, 128-bit loads when aligned)
    if ((k & 3) == 0 && (ldx & 3) == 0) {
      const int q = k / 4;
      for (int x = threadIdx.x; x < rows * q; x += MT) {
        const int r = x / q, m4 = x % q;
        const float4 v = __ldcs(reinterpret_cast<const float4*>(X + (r0 + r) * (int64_t)ldx) + m4);
        *reinterpret_cast<float4*>(Xs + r * kp + 4 * m4) = v;
      }
    } else {
      for (int x = threadIdx.x; x < rows * k; x += MT) {
        const int r = x / k, m = x % k;
        Xs[r * kp + m] = X[(r0 + r) * (int64_t)ldx + m];
      }
    }
    __syncthreads();
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0f;
#pragma unroll 4
    for (int m = 0; m < k; ++m) {
      const float4 f = *reinterpret_cast<const float4*>(Fs + m * CB + 4 * cq);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const float xv = Xs[(4 * rg + a) * kp + m];
        acc[a][0] = fmaf(xv, f.x, acc[a][0]);
        acc[a][1] = fmaf(xv, f.y, acc[a][1]);
        acc[a][2] = fmaf(xv, f.z, acc[a][2]);
        acc[a][3] = fmaf(xv, f.w, acc[a][3]);
      }
    }
    __syncthreads();  // in-place safety: all reads of this tile are done
    const int c = c0 + 4 * cq;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int r = 4 * rg + a;
      if (r < rows && 4 * cq < cb) {
        float* zp = Z + (r0 + r) * (int64_t)ldz + c;
        if (4 * cq + 3 < cb && (ldz & 3) == 0 && (c & 3) == 0) {
          __stcs(reinterpret_cast<float4*>(zp), make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]));
        } else {
          for (int b = 0; b < 4 && 4 * cq + b < cb; ++b) zp[b] = acc[a][b];
        }
      }
    }
  }
}

// Precise variant (fp64 products and accumulation, fp32 in/out) for folds of
// ill-conditioned projections (rebase at cond(P) up to 1e8, query_all after
// many lazy updates): the 3xTF32 / fp32 paths lose log10(cond) digits to
// cancellation there, fp64 accumulation keeps the result at fp32 storage
// accuracy. Same tiling as materialize_simt, CBD output columns per pass.
template <int CBD>
__global__ void __launch_bounds__(MT, 1)
    materialize_f64(const float* __restrict__ X, int64_t n, int k, int ldx,
                    const double* __restrict__ FT, int ldf, int k2, float* Z, int ldz, int c0,
                    int cb) {
  extern __shared__ __align__(16) double smd[];
  double* Fs = smd;                  // k x CBD
  double* Xs = smd + (size_t)k * CBD;  // RT x k
  for (int x = threadIdx.x; x < k * CBD; x += MT) {
    const int m = x / CBD, c = x % CBD;
    Fs[m * CBD + c] = c < cb ? FT[(int64_t)(c0 + c) * ldf + m] : 0.0;
  }
  __syncthreads();
  constexpr int CPT = CBD / 32;       // columns per thread (lane-strided)
  const int lane = threadIdx.x % 32;  // columns lane + 32 j
  const int rg = threadIdx.x / 32;    // rows 4 rg .. 4 rg + 3
  const int64_t ntiles = (n + RT - 1) / RT;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * RT;
    const int rows = (int)(n - r0 < RT ? n - r0 : RT);
    for (int x = threadIdx.x; x < rows * k; x += MT) {
      const int r = x / k, m = x % k;
      Xs[r * k + m] = (double)X[(r0 + r) * (int64_t)ldx + m];
    }
    __syncthreads();
    double acc[4][CPT];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < CPT; ++b) acc[a][b] = 0.0;
    for (int m = 0; m < k; ++m) {
      double f[CPT];
#pragma unroll
      for (int b = 0; b < CPT; ++b) f[b] = Fs[m * CBD + lane + 32 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double xv = Xs[(4 * rg + a) * k + m];
#pragma unroll
        for (int b = 0; b < CPT; ++b) acc[a][b] = fma(xv, f[b], acc[a][b]);
      }
    }
    __syncthreads();  // in-place safety
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int r = 4 * rg + a;
      if (r >= rows) continue;
#pragma unroll
      for (int b = 0; b < CPT; ++b) {
        const int c = lane + 32 * b;
        if (c < cb) Z[(r0 + r) * (int64_t)ldz + c0 + c] = (float)acc[a][b];
      }
    }
  }
}

// Precise fold on the FP64 tensor cores (mma.sync.m8n8k4.f64): the same
// fp64 products and accumulation as materialize_f64 at tensor-pipe rate.
// CTA = 8 warps over a 64-row tile; warp w owns rows 8w..8w+7 and NB n8
// column tiles (NB*8 output columns per pass); F (k x NB*8, fp64) stays in
// shared memory for the CTA's lifetime, the X tile is staged as fp32 and
// widened on fragment load. In place safe (tile fully staged before writes).
constexpr int DT = 64;  // rows per tile
__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
template <int NB>
__global__ void __launch_bounds__(MT, 1)
    materialize_dmma(const float* __restrict__ X, int64_t n, int k, int ldx,
                     const double* __restrict__ FT, int ldf, float* Z, int ldz, int c0, int cb) {
  extern __shared__ __align__(16) double smd[];
  constexpr int NC = NB * 8;
  constexpr int SP = NC + 8;  // padded F row (2-way bank pattern for 8-byte fragments)
  const int kp = (k + 3) & ~3;
  double* Fs = smd;                                  // kp x SP
  float* Xs = reinterpret_cast<float*>(smd + (size_t)kp * SP);  // DT x (kp + 4)
  const int xs = kp + 4;
  for (int x = threadIdx.x; x < kp * NC; x += MT) {
    const int m = x / NC, c = x % NC;
    Fs[m * SP + c] = (m < k && c < cb) ? FT[(int64_t)(c0 + c) * ldf + m] : 0.0;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  const int64_t ntiles = (n + DT - 1) / DT;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * DT;
    const int rows = (int)(n - r0 < DT ? n - r0 : DT);
    __syncthreads();  // previous tile's fragments consumed; F staged
    for (int x = threadIdx.x; x < DT * kp; x += MT) {
      const int r = x / kp, m = x % kp;
      Xs[r * xs + m] = (r < rows && m < k) ? X[(r0 + r) * (int64_t)ldx + m] : 0.0f;
    }
    __syncthreads();
    double d0[NB], d1[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) d0[j] = d1[j] = 0.0;
    const float* xrow = Xs + (8 * warp + ar) * xs;
    for (int k0 = 0; k0 < kp; k0 += 4) {
      const double a = (double)xrow[k0 + ac];
      const double* frow = Fs + (k0 + ac) * SP + ar;
#pragma unroll
      for (int j = 0; j < NB; ++j) dmma_f64(d0[j], d1[j], a, frow[8 * j]);
    }
    __syncthreads();  // in-place safety: every warp finished reading the tile
    const int r = 8 * warp + ar;
    if (r < rows) {
      float* zr = Z + (r0 + r) * (int64_t)ldz + c0;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int c = 8 * j + 2 * ac;
        if (c + 1 < cb) {
          *reinterpret_cast<float2*>(zr + c) = make_float2((float)d0[j], (float)d1[j]);
        } else if (c < cb) {
          zr[c] = (float)d0[j];
        }
      }
    }
  }
}

}  // namespace

// Z[:, :k2] = X[:, :k] * F with fp64 products/accumulation on the FP64
// tensor cores (materialize_dmma). In place (Z == X) needs k2 <= 128.
cudaError_t launch_materialize_precise_dmma(const float* X, int64_t n, int k, int ldx,
                                            const double* FT, int ldf, int k2, float* Z, int ldz,
                                            cudaStream_t s, int nsm) {
  if (n <= 0 || k2 <= 0) return cudaSuccess;
  const bool wide = k > 128;
  const int nc = wide ? 64 : 128;
  if (X == Z && k2 > nc) return cudaErrorInvalidValue;
  if ((ldz & 1) || (reinterpret_cast<uintptr_t>(Z) & 7)) return cudaErrorInvalidValue;
  const int kp = (k + 3) & ~3;
  const size_t smem = (size_t)kp * (nc + 8) * 8 + (size_t)DT * (kp + 4) * 4;
  static size_t configured[2] = {0, 0};
  if (smem > configured[wide]) {
    cudaError_t e = wide ? cudaFuncSetAttribute(materialize_dmma<8>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                         : cudaFuncSetAttribute(materialize_dmma<16>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured[wide] = smem;
  }
  const int64_t ntiles = (n + DT - 1) / DT;
  const int grid = (int)(ntiles < nsm ? ntiles : nsm);
  for (int c0 = 0; c0 < k2; c0 += nc) {
    const int cb = min(nc, k2 - c0);
    if (wide)
      materialize_dmma<8><<<grid, MT, smem, s>>>(X, n, k, ldx, FT, ldf, Z, ldz, c0, cb);
    else
      materialize_dmma<16><<<grid, MT, smem, s>>>(X, n, k, ldx, FT, ldf, Z, ldz, c0, cb);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Z[:, :k2] = X[:, :k] * F with fp64 products/accumulation (see
// materialize_f64). In place (Z == X) needs k2 <= 128 (one pass).
cudaError_t launch_materialize_precise(const float* X, int64_t n, int k, int ldx,
                                       const double* FT, int ldf, int k2, float* Z, int ldz,
                                       cudaStream_t s, int nsm) {
  if (n <= 0 || k2 <= 0) return cudaSuccess;
  if (!(ldz & 1) && !(reinterpret_cast<uintptr_t>(Z) & 7) && !(X == Z && k2 > (k > 128 ? 64 : 128)))
    return launch_materialize_precise_dmma(X, n, k, ldx, FT, ldf, k2, Z, ldz, s, nsm);
  const bool wide = k > 128;
  const int cbd = wide ? 64 : 128;
  if (X == Z && k2 > cbd) return cudaErrorInvalidValue;
  const size_t smem = ((size_t)k * cbd + (size_t)RT * k) * 8;
  static size_t configured[2] = {0, 0};
  if (smem > configured[wide]) {
    cudaError_t e = wide ? cudaFuncSetAttribute(materialize_f64<64>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                         : cudaFuncSetAttribute(materialize_f64<128>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured[wide] = smem;
  }
  const int64_t ntiles = (n + RT - 1) / RT;
  const int grid = (int)(ntiles < nsm ? ntiles : nsm);
  for (int c0 = 0; c0 < k2; c0 += cbd) {
    const int cb = min(cbd, k2 - c0);
    if (wide)
      materialize_f64<64><<<grid, MT, smem, s>>>(X, n, k, ldx, FT, ldf, k2, Z, ldz, c0, cb);
    else
      materialize_f64<128><<<grid, MT, smem, s>>>(X, n, k, ldx, FT, ldf, k2, Z, ldz, c0, cb);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

size_t materialize_smem(int k) { return ((size_t)k * CB + (size_t)RT * ((k + 3) & ~3)) * 4; }

namespace {
// F = P (fp64, given transposed) -> exact-TF32 hi part and fp32 lo part, both
// in the FT layout the tensor-core kernel stages (row j = output column j).
__global__ void split_f_kernel(const double* FT, int ldf, int k, float* hi, float* lo) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < k * k; x += gridDim.x * blockDim.x) {
    const int j = x / k, m = x % k;
    const double f = FT[(int64_t)j * ldf + m];
    const float h = __uint_as_float(__float_as_uint((float)f) & 0xFFFFE000u);
    hi[x] = h;
    lo[x] = (float)(f - (double)h);
  }
}
// bf16 hi/lo split for the d = 256 kind::f16 path (materialize_tc.cu)
__global__ void split_f_bf16_kernel(const double* FT, int ldf, int k, __nv_bfloat16* hi, __nv_bfloat16* lo) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < k * k; x += gridDim.x * blockDim.x) {
    const int j = x / k, m = x % k;
    const double f = FT[(int64_t)j * ldf + m];
    const __nv_bfloat16 h = __double2bfloat16(f);
    hi[x] = h;
    lo[x] = __double2bfloat16(f - (double)__bfloat162float(h));
  }
}
float* g_fsplit = nullptr;
}  // namespace

// Z[:, :k2] = X[:, :k] * F, F given transposed (FT[c][m] = F[m][c], fp64 on
// device). In-place (Z == X) requires k2 <= CB so one pass covers all
// output columns.
cudaError_t launch_materialize(const float* X, int64_t n, int k, int ldx, const double* FT,
                               int ldf, int k2, float* Z, int ldz, cudaStream_t s, int nsm) {
  if (n <= 0 || k2 <= 0) return cudaSuccess;
  if (k2 == k && materialize_tc_supported(k, ldx, ldz, X, Z)) {
    if (!g_fsplit) {
      cudaError_t e = cudaMalloc(&g_fsplit, 2 * kMaxD * kMaxD * sizeof(float));
      if (e != cudaSuccess) return e;
    }
    if (k == 256) {
      __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(g_fsplit);
      split_f_bf16_kernel<<<64, 256, 0, s>>>(FT, ldf, k, h, h + k * k);
      return launch_materialize_tc(X, n, k, ldx, g_fsplit, reinterpret_cast<float*>(h + k * k), Z, ldz,
                                   s, nsm);
    }
    split_f_kernel<<<64, 256, 0, s>>>(FT, ldf, k, g_fsplit, g_fsplit + k * k);
    return launch_materialize_tc(X, n, k, ldx, g_fsplit, g_fsplit + k * k, Z, ldz, s, nsm);
  }
  if (X == Z && k2 > CB) return cudaErrorInvalidValue;
  const size_t smem = materialize_smem(k);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(materialize_simt,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  const int64_t ntiles = (n + RT - 1) / RT;
  const int grid = (int)(ntiles < nsm ? ntiles : nsm);
  for (int c0 = 0; c0 < k2; c0 += CB) {
    const int cb = min(CB, k2 - c0);
    materialize_simt<<<grid, MT, smem, s>>>(X, n, k, ldx, FT, ldf, k2, Z, ldz, c0, cb);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace dgpu
