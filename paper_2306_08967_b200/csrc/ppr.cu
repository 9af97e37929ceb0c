// K6-K8: the dynamic Personalized-PageRank enhancer (enhancer.cpp:26-206).
//
// State (base coordinates, sharing P_X with the factors): Z_b, r_b fp32
// n x d, plus key[u] = |r_b[u]|_inf / max(deg u, 1) (fp32), kept current by
// every kernel that writes r_b, which replaces the reference's FIFO + lazy
// max-heap (enhancer.cpp:108-157): the push scans keys against the
// threshold alpha*eps/s_max at every call.
//
// The push is frontier-synchronous (Jacobi rounds) instead of FIFO
// Gauss-Seidel, in PULL form so no floating-point atomics are needed:
//   F  = {u : key[u] * s_max > alpha*eps}                  (compaction)
//   P1 u in F : delta[u] = r[u]; Z[u] += r[u]; stamp[u] = R; mark in-nbrs
//   P2 L = {v : mark[v] == R}                               (compaction)
//   P3 v in L : r[v] = [v not in F] r[v]
//                      + (1-alpha)/max(deg v,1) sum_{u in out(v) cap F} w delta[u]
//   next F = {v in L : key[v] over threshold}               (compaction)
// One cooperative kernel runs all rounds with grid-wide barriers. All
// compactions are block-count / prefix / scatter (atomics-free, order
// preserving, deterministic).
#include <cooperative_groups.h>

#include "common.cuh"
#include "ppr.cuh"

namespace cg = cooperative_groups;

namespace dgpu {

namespace {
constexpr int PT_ = 256;  // threads per block
constexpr int PW = PT_ / 32;

// Block-exclusive scan of one flag per thread; returns the thread's offset
// and writes the block total to *total.
DAMF_D int block_scan(int flag, int* wsum, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned ball = __ballot_sync(0xffffffffu, flag);
  const int pre = __popc(ball & ((1u << lane) - 1u));
  if (lane == 0) wsum[w] = __popc(ball);
  __syncthreads();
  int off = 0, tot = 0;
  for (int i = 0; i < PW; ++i) {
    if (i < w) off += wsum[i];
    tot += wsum[i];
  }
  __syncthreads();
  *total = tot;
  return off + pre;
}

// Grid-wide, order-preserving compaction of items i in [0, count) with
// pred(i) -> (keep, value). Each block owns a contiguous chunk.
template <class Pred>
DAMF_D int grid_compact(cg::grid_group& g, int count, Pred pred, int* out, int* blk) {
  __shared__ int wsum[PW];
  const int G = gridDim.x;
  const int chunk = (count + G - 1) / G;
  const int lo = min(count, (int)blockIdx.x * chunk), hi = min(count, lo + chunk);
  int mine = 0;
  for (int base = lo; base < hi; base += PT_) {
    const int i = base + threadIdx.x;
    int v;
    const int f = (i < hi) && pred(i, v);
    int tot;
    block_scan(f, wsum, &tot);
    mine += tot;
  }
  if (threadIdx.x == 0) blk[blockIdx.x] = mine;
  g.sync();
  int off = 0, total = 0;
  for (int b = 0; b < G; ++b) {
    const int c = blk[b];
    if (b < (int)blockIdx.x) off += c;
    total += c;
  }
  for (int base = lo; base < hi; base += PT_) {
    const int i = base + threadIdx.x;
    int v = 0;
    const int f = (i < hi) && pred(i, v);
    int tot;
    const int pos = block_scan(f, wsum, &tot);
    if (f) out[off + pos] = v;
    off += tot;
  }
  g.sync();
  return total;
}

DAMF_D float row_key(const float* r, int k, double deg) {
  float m = 0.0f;
  for (int j = threadIdx.x & 31; j < k; j += 32) m = fmaxf(m, fabsf(r[j]));
  m = warp_max(m);
  return (float)((double)m / fmax(deg, 1.0));
}

__global__ void __launch_bounds__(PT_) ppr_push_kernel(PprArgs A) {
  cg::grid_group g = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * PT_ + threadIdx.x) >> 5;  // global warp id
  const int nwarps = gridDim.x * PW;
  const int k = A.ctl->k, d = A.d;
  const float thr = (float)(A.alpha_eps / *A.smax);
  const double om = 1.0 - A.alpha;
  int R = (int)A.stats[2];  // device-resident round stamp base (monotonic)
  // initial frontier
  int nF;
  if (A.ncand >= 0) {
    nF = grid_compact(
        g, A.ncand,
        [&](int i, int& v) {
          v = A.cand[i];
          return A.key[v] > thr;
        },
        A.listF, A.blk);
  } else {
    nF = grid_compact(
        g, (int)A.n,
        [&](int i, int& v) {
          v = i;
          return A.key[i] > thr;
        },
        A.listF, A.blk);
  }
  long long pushes = 0;
  int rounds = 0;
  while (nF > 0) {
    ++R;
    ++rounds;
    pushes += nF;
    if (pushes > A.push_guard || rounds > 1000000) {
      if (blockIdx.x == 0 && threadIdx.x == 0) A.ctl->err = 9;  // NonConvergence
      break;
    }
    // P1: move residual into Z, stamp, mark affected rows
    for (int q = gw; q < nF; q += nwarps) {
      const int u = A.listF[q];
      const float* ru = A.rb + (int64_t)u * d;
      float* zu = A.Zb + (int64_t)u * d;
      float* du = A.delta + (int64_t)u * d;
      for (int j = lane; j < k; j += 32) {
        const float r = ru[j];
        du[j] = r;
        zu[j] += r;
      }
      if (lane == 0) {
        A.stamp[u] = R;
        A.mark[u] = R;
      }
      const DevCSR& in = A.directed ? A.in : A.out;
      const int64_t base = in.off[u];
      const int c = in.cnt[u];
      for (int p = lane; p < c; p += 32) A.mark[in.ids[base + p]] = R;
    }
    g.sync();
    // P2: affected list
    const int nL = grid_compact(
        g, (int)A.n,
        [&](int i, int& v) {
          v = i;
          return A.mark[i] == R;
        },
        A.listL, A.blk);
    // P3: pull update of affected rows
    if (blockIdx.x == 0 && threadIdx.x == 0) A.stats[4] += nL;
    for (int q = gw; q < nL; q += nwarps) {
      const int v = A.listL[q];
      float acc[kMaxD / 32];
#pragma unroll
      for (int t = 0; t < kMaxD / 32; ++t) acc[t] = 0.0f;
      const int64_t base = A.out.off[v];
      const int c = A.out.cnt[v];
      int matched = 0;
      for (int p = 0; p < c; ++p) {
        const int u = A.out.ids[base + p];
        if (A.stamp[u] != R) continue;
        ++matched;
        const float w = A.out.wts ? (float)A.out.wts[base + p] : 1.0f;
        const float* du = A.delta + (int64_t)u * d;
#pragma unroll
        for (int t = 0; t < kMaxD / 32; ++t) {
          const int j = lane + 32 * t;
          if (j < k) acc[t] = fmaf(w, du[j], acc[t]);
        }
      }
      const double degv = A.deg[v];
      const float coef = (float)(om / fmax(degv, 1.0));
      float* rv = A.rb + (int64_t)v * d;
      const bool inF = A.stamp[v] == R;
      float m = 0.0f;
#pragma unroll
      for (int t = 0; t < kMaxD / 32; ++t) {
        const int j = lane + 32 * t;
        if (j < k) {
          const float nr = (inF ? 0.0f : rv[j]) + coef * acc[t];
          rv[j] = nr;
          m = fmaxf(m, fabsf(nr));
        }
      }
      m = warp_max(m);
      if (lane == 0) {
        A.key[v] = (float)((double)m / fmax(degv, 1.0));
        atomicAdd((unsigned long long*)&A.stats[5], (unsigned long long)c);        // stats only
        atomicAdd((unsigned long long*)&A.stats[6], (unsigned long long)matched);
      }
    }
    g.sync();
    // next frontier from the affected list
    nF = grid_compact(
        g, nL,
        [&](int i, int& v) {
          v = A.listL[i];
          return A.key[v] > thr;
        },
        A.listF, A.blk);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.stats[0] += pushes;
    A.stats[1] += rounds;
    A.stats[3] += pushes;
    A.stats[2] = R;  // next round base
    if (A.t_end) *A.t_end = globaltimer();
  }
}

// r_b[u] = alpha X_b[u] + (1-alpha)/deg(u) sum_{v in out(u)} w Z_b[v] - Z_b[u]
// for the touched rows (enhancer.cpp:77-96); one block per row, warps split
// the neighbour list, fixed-order smem reduction.
__global__ void __launch_bounds__(PT_) ppr_absorb_kernel(PprArgs A, const int64_t* rows, int nrows) {
  __shared__ float part[PW][kMaxD];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k = A.ctl->k, d = A.d;
  for (int q = blockIdx.x; q < nrows; q += gridDim.x) {
    const int64_t u = rows[q];
    float acc[kMaxD / 32];
#pragma unroll
    for (int t = 0; t < kMaxD / 32; ++t) acc[t] = 0.0f;
    const int64_t base = A.out.off[u];
    const int c = A.out.cnt[u];
    for (int p = w; p < c; p += PW) {
      const int v = A.out.ids[base + p];
      const float wt = A.out.wts ? (float)A.out.wts[base + p] : 1.0f;
      const float* zv = A.Zb + (int64_t)v * d;
#pragma unroll
      for (int t = 0; t < kMaxD / 32; ++t) {
        const int j = lane + 32 * t;
        if (j < k) acc[t] = fmaf(wt, zv[j], acc[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < kMaxD / 32; ++t) {
      const int j = lane + 32 * t;
      if (j < k) part[w][j] = acc[t];
    }
    __syncthreads();
    const double deg = A.deg[u];
    if (w == 0) {
      float m = 0.0f;
      for (int j = lane; j < k; j += 32) {
        float s = 0.0f;
        for (int x = 0; x < PW; ++x) s += part[x][j];
        const float xu = A.Xb[u * d + j];
        const float zu = A.Zb[u * d + j];
        float r = (float)A.alpha * xu - zu;
        if (deg > 0.0) r += (float)((1.0 - A.alpha) / deg) * s;
        A.rb[u * d + j] = r;
        m = fmaxf(m, fabsf(r));
      }
      m = warp_max(m);
      if (lane == 0) A.key[u] = (float)((double)m / fmax(deg, 1.0));
    }
    __syncthreads();
  }
}

// key[u] for all rows (after init / transform / rebase).
__global__ void ppr_keys_kernel(PprArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = gw; u < A.n; u += nw) {
    const float kk = row_key(A.rb + u * A.d, A.ctl->k, A.deg[u]);
    if (lane == 0) A.key[u] = kk;
  }
}

// init_propagate (enhancer.cpp:26-47): Z_b = 0, r_b = alpha X_b.
__global__ void ppr_init_kernel(PprArgs A) {
  const int64_t total = A.n * (int64_t)A.d;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    A.Zb[x] = 0.0f;
    A.rb[x] = (float)A.alpha * A.Xb[x];
  }
}

// proj_row_bound (factor_state.cpp:251-259) from PT (P transposed):
// col1 = max_j sum_i |P_ij| = max_j sum_i |PT[j][i]|; rowinf = max_i sum_j |P_ij|.
__global__ void smax_kernel(const double* PT0, const double* PT1, const DevCtl* ctl, int ld,
                            double* out) {
  __shared__ double cmax[PT_], rmax[PT_];
  const int k = ctl->k;
  const double* PT = ctl->pp[0] ? PT1 : PT0;
  double c1 = 0, ri = 0;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    double s = 0;
    for (int i = 0; i < k; ++i) s += fabs(PT[(int64_t)j * ld + i]);
    c1 = fmax(c1, s);
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    double s = 0;
    for (int j = 0; j < k; ++j) s += fabs(PT[(int64_t)j * ld + i]);
    ri = fmax(ri, s);
  }
  cmax[threadIdx.x] = c1;
  rmax[threadIdx.x] = ri;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      a = fmax(a, cmax[t]);
      b = fmax(b, rmax[t]);
    }
    *out = k == 0 ? 1.0 : fmax(a, sqrt(a * b));
  }
}

}  // namespace

cudaError_t launch_ppr_push(const PprArgs& a, int grid, cudaStream_t s) {
  void* args[] = {(void*)&a};
  return cudaLaunchCooperativeKernel((void*)ppr_push_kernel, dim3(grid), dim3(PT_), args, 0, s);
}

int ppr_push_max_grid(int nsm) {
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ppr_push_kernel, PT_, 0);
  return per * nsm;
}

cudaError_t launch_ppr_absorb(const PprArgs& a, const int64_t* rows, int nrows, cudaStream_t s) {
  if (nrows <= 0) return cudaSuccess;
  ppr_absorb_kernel<<<min(nrows, 1024), PT_, 0, s>>>(a, rows, nrows);
  return cudaGetLastError();
}

cudaError_t launch_ppr_keys(const PprArgs& a, int nsm, cudaStream_t s) {
  ppr_keys_kernel<<<nsm * 4, PT_, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_ppr_init(const PprArgs& a, int nsm, cudaStream_t s) {
  ppr_init_kernel<<<nsm * 8, PT_, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_smax(const double* PT0, const double* PT1, const DevCtl* ctl, int ld,
                        double* out, cudaStream_t s) {
  smax_kernel<<<1, PT_, 0, s>>>(PT0, PT1, ctl, ld, out);
  return cudaGetLastError();
}

}  // namespace dgpu
