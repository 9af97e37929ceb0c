// K5: full-embedding materialisation Z = X * F (factor_state.cpp:120-123
// query_all, :215-222 rebase, enhancer.cpp:196-206 apply_transform).
// Tall-skinny n x k by k x k2 product, HBM-bound at 8 n k bytes.
//
// materialize_simt: persistent FP32 SIMT kernel. F (fp64 on the host side
// of the state) is converted once per CTA into a shared-memory fp32 tile;
// row tiles of X stream through registers with 128-bit loads; each thread
// owns a 4-row x 4-column register block. Safe in place (out == in): a CTA
// reads its whole row tile into shared memory before writing it.
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

}  // namespace

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
      cudaError_t e = cudaMalloc(&g_fsplit, 2 * 128 * 128 * sizeof(float));
      if (e != cudaSuccess) return e;
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
