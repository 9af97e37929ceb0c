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

constexpr int HEAVY = 2048;  // rows with more out-arcs are pulled in chunks
constexpr int CH = 1024;     // neighbours per chunk
constexpr int HB = 8;        // delta rows gathered per batch (loads in flight)

// Pull the stamped neighbours u in out(v)[beg, end) into acc (lane-parallel
// over 32 ids/stamps per step, ballot of hits, then the hit rows gathered HB
// at a time with all loads issued before the FMAs). Returns pulled arcs.
template <int KPL>
DAMF_D int pull_range(const PprArgs& A, int64_t base, int beg, int end, int R, int k,
                      float (&acc)[KPL]) {
  const int lane = threadIdx.x & 31;
  int matched = 0;
  for (int p0 = beg; p0 < end; p0 += 32) {
    const int p = p0 + lane;
    int u = -1;
    float w = 0.0f;
    if (p < end) {
      u = A.out.ids[base + p];
      w = A.out.wts ? (float)A.out.wts[base + p] : 1.0f;
    }
    const bool hit = u >= 0 && A.stamp[u] == R;
    unsigned mask = __ballot_sync(0xffffffffu, hit);
    matched += __popc(mask);
    while (mask) {
      int ub[HB];
      float wb[HB];
#pragma unroll
      for (int q = 0; q < HB; ++q) {
        if (mask) {
          const int s0 = __ffs(mask) - 1;
          mask &= mask - 1;
          ub[q] = __shfl_sync(0xffffffffu, u, s0);
          wb[q] = __shfl_sync(0xffffffffu, w, s0);
        } else {
          ub[q] = -1;
          wb[q] = 0.0f;
        }
      }
      float x[HB][KPL];
#pragma unroll
      for (int q = 0; q < HB; ++q) {
        const float* dq = A.delta + (int64_t)(ub[q] < 0 ? ub[0] : ub[q]) * A.d;
#pragma unroll
        for (int t = 0; t < KPL; ++t) {
          const int j = lane + 32 * t;
          x[q][t] = (j < k && ub[q] >= 0) ? dq[j] : 0.0f;
        }
      }
#pragma unroll
      for (int q = 0; q < HB; ++q)
#pragma unroll
        for (int t = 0; t < KPL; ++t) acc[t] = fmaf(wb[q], x[q][t], acc[t]);
    }
  }
  return matched;
}

// r[v] = [v not pushed] r[v] + (1-alpha)/max(deg v,1) * acc ; key[v]. Rows with
// no pulled contribution that were not pushed are unchanged (skipped).
template <int KPL>
DAMF_D void finish_row(const PprArgs& A, int v, int R, int k, double om, const float (&acc)[KPL],
                       bool any) {
  const int lane = threadIdx.x & 31;
  const bool inF = A.stamp[v] == R;
  if (!inF && !any) return;
  const double degv = A.deg[v];
  const float coef = (float)(om / fmax(degv, 1.0));
  float* rv = A.rb + (int64_t)v * A.d;
  float m = 0.0f;
#pragma unroll
  for (int t = 0; t < KPL; ++t) {
    const int j = lane + 32 * t;
    if (j < k) {
      const float nr = (inF ? 0.0f : rv[j]) + coef * acc[t];
      rv[j] = nr;
      m = fmaxf(m, fabsf(nr));
    }
  }
  m = warp_max(m);
  if (lane == 0) A.key[v] = (float)((double)m / fmax(degv, 1.0));
}

template <int KPL>
__global__ void __launch_bounds__(PT_, 3) ppr_push_kernel(PprArgs A) {
  cg::grid_group g = cg::this_grid();
  __shared__ long long red64[PW];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = (blockIdx.x * PT_ + threadIdx.x) >> 5;  // global warp id
  const int nwarps = gridDim.x * PW;
  const int k = A.ctl->k, d = A.d;
  const int n = (int)A.n;
  const float thr = (float)(A.alpha_eps / *A.smax);
  const double om = 1.0 - A.alpha;
  int R = (int)A.stats[2];  // device-resident round stamp base (monotonic)
  // ---- heavy rows (out-degree > HEAVY): list, chunk prefix, row -> index
  const int nH = grid_compact(
      g, n,
      [&](int i, int& v) {
        v = i;
        return A.out.cnt[i] > HEAVY;
      },
      A.heavy, A.blk);
  if (blockIdx.x == 0) {
    // exclusive prefix of chunk counts (block 0, fixed order)
    __shared__ int wsum[PW];
    int carry = 0;
    for (int b0 = 0; b0 < nH; b0 += PT_) {
      const int i = b0 + threadIdx.x;
      const int c = i < nH ? (A.out.cnt[A.heavy[i]] + CH - 1) / CH : 0;
      int x = c;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[wib] = x;
      __syncthreads();
      int pre = 0, tot = 0;
      for (int w = 0; w < PW; ++w) {
        if (w < wib) pre += wsum[w];
        tot += wsum[w];
      }
      if (i < nH) A.hoff[i] = carry + pre + x - c;
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) A.hoff[nH] = carry;
  }
  for (int i = blockIdx.x * PT_ + threadIdx.x; i < nH; i += gridDim.x * PT_) A.hidx[A.heavy[i]] = i;
  g.sync();
  const int nchunks = A.hoff[nH];
  // ---- rounds
  const bool init_all = A.ncand < 0;
  int ncand = init_all ? n : A.ncand;
  const int* candL = init_all ? nullptr : A.cand;
  bool cand_all = init_all;
  bool mark_mode = true;
  long long pushes = 0, pulled = 0, affected = 0, aff_arcs = 0;
  int rounds = 0;
  for (;;) {
    ++R;
    // P1: push candidates over threshold (delta, Z, stamp, in-neighbour marks)
    long long mine = 0;
    for (int base = gw * 32; base < ncand; base += nwarps * 32) {
      const int i = base + lane;
      int v = -1;
      if (i < ncand) v = cand_all ? i : candL[i];
      const bool hit = v >= 0 && A.key[v] > thr;
      unsigned mask = __ballot_sync(0xffffffffu, hit);
      mine += __popc(mask);
      while (mask) {
        const int s0 = __ffs(mask) - 1;
        mask &= mask - 1;
        const int u = __shfl_sync(0xffffffffu, v, s0);
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
          if (mark_mode) A.mark[u] = R;
        }
        if (mark_mode) {
          const DevCSR& in = A.directed ? A.in : A.out;
          const int64_t ib = in.off[u];
          const int c = in.cnt[u];
          for (int p = lane; p < c; p += 32) A.mark[in.ids[ib + p]] = R;
        }
      }
    }
    // grid-wide push count
    mine = (lane == 0) ? mine : 0;
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if (lane == 0) red64[wib] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t = 0;
      for (int w = 0; w < PW; ++w) t += red64[w];
      A.blk64[blockIdx.x] = t;
    }
    g.sync();
    long long nF = 0;
    for (int b = 0; b < (int)gridDim.x; ++b) nF += A.blk64[b];
    if (nF == 0) break;
    ++rounds;
    pushes += nF;
    if (pushes > A.push_guard || rounds > 1000000) {
      if (blockIdx.x == 0 && threadIdx.x == 0) A.ctl->err = 9;  // NonConvergence
      break;
    }
    const bool dense = !mark_mode || nF * 32 > (long long)n;
    int nL = n;
    if (!dense) {
      // P2: affected rows (marked this round); heavy ones flagged active
      nL = grid_compact(
          g, n,
          [&](int i, int& v) {
            v = i;
            const bool m = A.mark[i] == R;
            if (m && A.hidx[i] >= 0) A.hact[A.hidx[i]] = R;
            return m;
          },
          A.listL, A.blk);
    }
    affected += nL;
    // P3a: light rows, one warp per row; P3b: heavy chunks, one warp per chunk
    long long my_pulled = 0, my_arcs = 0;
    for (int q = gw; q < nL; q += nwarps) {
      const int v = dense ? q : A.listL[q];
      if (A.hidx[v] >= 0) continue;
      float acc[KPL];
#pragma unroll
      for (int t = 0; t < KPL; ++t) acc[t] = 0.0f;
      const int c = A.out.cnt[v];
      const int got = pull_range<KPL>(A, A.out.off[v], 0, c, R, k, acc);
      my_pulled += got;
      my_arcs += c;
      finish_row<KPL>(A, v, R, k, om, acc, got > 0);
    }
    for (int c = gw; c < nchunks; c += nwarps) {
      int lo = 0, hi = nH;  // hub h with hoff[h] <= c < hoff[h+1]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (A.hoff[mid] <= c) lo = mid; else hi = mid;
      }
      const int h = lo;
      if (!dense && A.hact[h] != R) continue;
      const int v = A.heavy[h];
      const int beg = (c - A.hoff[h]) * CH;
      const int end = min(beg + CH, A.out.cnt[v]);
      float acc[KPL];
#pragma unroll
      for (int t = 0; t < KPL; ++t) acc[t] = 0.0f;
      my_pulled += pull_range<KPL>(A, A.out.off[v], beg, end, R, k, acc);
      my_arcs += end - beg;
      float* part = A.hpart + (int64_t)c * d;
#pragma unroll
      for (int t = 0; t < KPL; ++t) {
        const int j = lane + 32 * t;
        if (j < k) part[j] = acc[t];
      }
    }
    g.sync();
    // P3c: heavy rows reduce their chunk partials in order
    for (int h = gw; h < nH; h += nwarps) {
      if (!dense && A.hact[h] != R) continue;
      float acc[KPL];
#pragma unroll
      for (int t = 0; t < KPL; ++t) acc[t] = 0.0f;
      for (int c = A.hoff[h]; c < A.hoff[h + 1]; ++c) {
        const float* part = A.hpart + (int64_t)c * d;
#pragma unroll
        for (int t = 0; t < KPL; ++t) {
          const int j = lane + 32 * t;
          if (j < k) acc[t] += part[j];
        }
      }
      finish_row<KPL>(A, A.heavy[h], R, k, om, acc, true);
    }
    if (lane == 0) {
      atomicAdd((unsigned long long*)&A.stats[5], (unsigned long long)my_arcs);   // accounting only
      atomicAdd((unsigned long long*)&A.stats[6], (unsigned long long)my_pulled);
    }
    g.sync();
    // next candidates: every row (dense) or the affected list (sparse)
    cand_all = dense;
    ncand = dense ? n : nL;
    candL = A.listL;
    mark_mode = nF * 32 <= (long long)n;
  }
  for (int i = blockIdx.x * PT_ + threadIdx.x; i < nH; i += gridDim.x * PT_) A.hidx[A.heavy[i]] = -1;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.stats[0] += pushes;
    A.stats[1] += rounds;
    A.stats[2] = R;  // next round base
    A.stats[3] += pushes;
    A.stats[4] += affected;
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
  if (a.d <= 128)
    return cudaLaunchCooperativeKernel((void*)ppr_push_kernel<4>, dim3(grid), dim3(PT_), args, 0, s);
  return cudaLaunchCooperativeKernel((void*)ppr_push_kernel<8>, dim3(grid), dim3(PT_), args, 0, s);
}

int ppr_push_max_grid(int nsm, int d) {
  int per = 0;
  if (d <= 128)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ppr_push_kernel<4>, PT_, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ppr_push_kernel<8>, PT_, 0);
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
