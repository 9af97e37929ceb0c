// K6-K8: the dynamic Personalized-PageRank enhancer (enhancer.cpp:26-206).
//
// State (base coordinates, sharing P_X with the factors): Z_b, r_b fp32
// n x d, plus key[u] >= |r_b[u]|_inf / max(deg u, 1) (fp32): exact after an
// absorb, a pull round or an evaluation of the row, an upper bound after
// scatter contributions (each adds its largest possible effect). It replaces
// the reference's FIFO + lazy max-heap (enhancer.cpp:108-157): a row under
// the threshold alpha*eps/s_max by its bound needs no look at r.
//
// The push is frontier-synchronous (Jacobi rounds) instead of FIFO
// Gauss-Seidel. Each round chooses its direction from the frontier's
// in-arc count:
//   pull (dense rounds):    every affected row v gathers
//       r[v] += (1-alpha)/max(deg v,1) sum_{u in out(v), stamp[u] == R} w delta[u]
//     with plain stores; only chunked heavy rows combine their partial sums
//     with vector float reductions (red.global.add.v4.f32).
//   scatter (sparse rounds): r[v] += (1-alpha) w / deg(v) * delta[u] for
//     v in in(u) with float reductions; a target whose key bound crosses the
//     threshold is appended to the next candidate list by its first toucher
//     (atomicExch on mark[v]).
// Work is handed out through per-warp static batches plus 32 atomic queue
// heads. Floating-point reductions make the fp32 summation order, and with it
// the last bits of r / Z and the push count, vary from run to run; the
// reference's contract -- every row's defect under alpha*eps*max(deg,1)
// after the push (enhancer.cpp:125-155, eval.cpp:591-610) -- holds for every
// order, and tests/test_gpu_ppr_materialize.py checks it (plus the distance
// to the exact fixed point) rather than bitwise equality with the FIFO push.
#include <cooperative_groups.h>

#include <algorithm>

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
// pred(i) -> (keep, value). Each block owns a contiguous, tile-aligned range;
// each thread evaluates IPT consecutive items per tile (independent loads in
// flight), then a block scan of the per-thread counts places them in order.
template <class Pred>
DAMF_D int grid_compact(cg::grid_group& g, int count, Pred pred, int* out, int* blk);

DAMF_D float row_key(const float* r, int k, double deg) {
  float m = 0.0f;
  for (int j = threadIdx.x & 31; j < k; j += 32) m = fmaxf(m, fabsf(r[j]));
  m = warp_max(m);
  return (float)((double)m / fmax(deg, 1.0));
}

constexpr int HEAVY = PPR_HEAVY;
constexpr int CH = PPR_CH;
#ifndef DAMF_PROF
#define DAMF_PROF 0  // phase timers (tools/prof_ppr.py builds with make EXTRA=-DDAMF_PROF=1)
#endif
#ifndef PPR_G
#define PPR_G 16
#endif
constexpr int G = PPR_G;      // lanes per row group
constexpr int NG = 32 / G;    // row groups per warp
constexpr unsigned GMASK = (1u << G) - 1u;
constexpr unsigned GLEADS = G == 8 ? 0x01010101u : 0x00010001u;
constexpr int SMALL = 32;     // rows with <= SMALL arcs are pulled by one group
constexpr int BIGMARK = 1024; // pushers with more in-arcs are marked grid-wide

// Block-exclusive scan of one int per thread; block total in *total.
DAMF_D int block_scan_val(int x, int* wsum, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = x;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  int off = 0, tot = 0;
  for (int i = 0; i < PW; ++i) {
    if (i < w) off += wsum[i];
    tot += wsum[i];
  }
  __syncthreads();
  *total = tot;
  return off + inc - x;
}

// Grid-wide exclusive scan out[i] = sum_{j<i} val(j), out[count] = total.
template <class Val>
DAMF_D int grid_scan(cg::grid_group& g, int count, Val val, int* out, int* blk) {
  __shared__ int wsum[PW];
  const int GB = gridDim.x;
  const int chunk = (count + GB - 1) / GB;
  const int lo = min(count, (int)blockIdx.x * chunk), hi = min(count, lo + chunk);
  int mine = 0;
  for (int base = lo; base < hi; base += PT_) {
    const int i = base + threadIdx.x;
    int tot;
    block_scan_val(i < hi ? val(i) : 0, wsum, &tot);
    mine += tot;
  }
  if (threadIdx.x == 0) blk[blockIdx.x] = mine;
  g.sync();
  int off = 0, total = 0;
  for (int b = 0; b < GB; ++b) {
    const int c = blk[b];
    if (b < (int)blockIdx.x) off += c;
    total += c;
  }
  for (int base = lo; base < hi; base += PT_) {
    const int i = base + threadIdx.x;
    int tot;
    const int pos = block_scan_val(i < hi ? val(i) : 0, wsum, &tot);
    if (i < hi) out[i] = off + pos;
    off += tot;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[count] = total;
  g.sync();
  return total;
}

template <class Pred>
DAMF_D int grid_compact(cg::grid_group& g, int count, Pred pred, int* out, int* blk) {
  constexpr int IPT = 8, TILE = PT_ * IPT;
  __shared__ int wsum[PW];
  const int GB = gridDim.x;
  const long long per = ((long long)(count + GB - 1) / GB + TILE - 1) / TILE * TILE;
  const int lo = (int)min((long long)count, (long long)blockIdx.x * per);
  const int hi = (int)min((long long)count, (long long)lo + per);
  int mine = 0;
  for (int base = lo; base < hi; base += TILE) {
    int c = 0;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const int i = base + threadIdx.x * IPT + j;
      int v;
      c += (i < hi) && pred(i, v);
    }
    int tot;
    block_scan_val(c, wsum, &tot);
    mine += tot;
  }
  if (threadIdx.x == 0) blk[blockIdx.x] = mine;
  g.sync();
  int off = 0, total = 0;
  for (int b = 0; b < GB; ++b) {
    const int c = blk[b];
    if (b < (int)blockIdx.x) off += c;
    total += c;
  }
  for (int base = lo; base < hi; base += TILE) {
    int vals[IPT];
    unsigned f = 0;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const int i = base + threadIdx.x * IPT + j;
      if ((i < hi) && pred(i, vals[j])) f |= 1u << j;
    }
    int tot;
    int pos = off + block_scan_val(__popc(f), wsum, &tot);
#pragma unroll
    for (int j = 0; j < IPT; ++j)
      if (f >> j & 1u) out[pos++] = vals[j];
    off += tot;
  }
  g.sync();
  return total;
}

// Per-lane column slice of a row: VEC -> PER float4 at 4*gl + 32*t,
// scalar -> PER floats at gl + 8*t. NE = elements per lane. Within a warp,
// group q "owns" slice elements with (VEC ? t : e) % 4 == q for warp-wide
// write-back after the cross-group reduction.
template <int PER, bool VEC>
struct Cols {
  static constexpr int NE = VEC ? 4 * PER : PER;
  DAMF_D static int col(int gl, int e) { return VEC ? 4 * gl + 4 * G * (e >> 2) + (e & 3) : gl + G * e; }
  DAMF_D static bool owns(int grp, int e) { return (VEC ? (e >> 2) : e) % NG == grp; }
  template <bool CG = false>
  DAMF_D static void load(const float* row, int gl, int k, float (&x)[NE]) {
    if (VEC) {
#pragma unroll
      for (int t = 0; t < PER; ++t) {
        const int j = 4 * gl + 4 * G * t;
        const float4* p = reinterpret_cast<const float4*>(row + j);
        float4 v = j < k ? (CG ? __ldcg(p) : *p) : make_float4(0.f, 0.f, 0.f, 0.f);
        x[4 * t] = v.x;
        x[4 * t + 1] = v.y;
        x[4 * t + 2] = v.z;
        x[4 * t + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int j = gl + G * e;
        x[e] = j < k ? (CG ? __ldcg(row + j) : row[j]) : 0.0f;
      }
    }
  }
  DAMF_D static void store(float* row, int gl, int k, const float (&x)[NE]) {
    if (VEC) {
#pragma unroll
      for (int t = 0; t < PER; ++t) {
        const int j = 4 * gl + 4 * G * t;
        if (j < k)
          *reinterpret_cast<float4*>(row + j) = make_float4(x[4 * t], x[4 * t + 1], x[4 * t + 2], x[4 * t + 3]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int j = gl + G * e;
        if (j < k) row[j] = x[e];
      }
    }
  }
};

// Group (8 lanes) pull of the stamped neighbours u in out(v)[beg, end) into
// acc: 8 ids/stamps per step, group ballot, hit rows gathered two at a time.
template <int PER, bool VEC>
DAMF_D int pull_group(const PprArgs& A, int64_t base, int beg, int end, int R, int k, int gl,
                      unsigned gm, float (&acc)[Cols<PER, VEC>::NE]) {
  using CL = Cols<PER, VEC>;
  int matched = 0;
  const int shift = (threadIdx.x & 31) & ~(G - 1);
  for (int p0 = beg; p0 < end; p0 += G) {
    const int p = p0 + gl;
    int u = -1;
    float w = 0.0f;
    if (p < end) {
      u = A.out.ids[base + p];
      w = A.out.wts ? (float)A.out.wts[base + p] : 1.0f;
    }
    const bool hit = u >= 0 && A.stamp[u] == R;
    unsigned mask = (__ballot_sync(gm, hit) >> shift) & GMASK;
    matched += __popc(mask);
    while (mask) {
      const int s0 = __ffs(mask) - 1;
      mask &= mask - 1;
      int s1 = s0;
      const bool two = mask != 0;
      if (two) {
        s1 = __ffs(mask) - 1;
        mask &= mask - 1;
      }
      const int u0 = __shfl_sync(gm, u, s0, G);
      const float w0 = __shfl_sync(gm, w, s0, G);
      const int u1 = __shfl_sync(gm, u, s1, G);
      const float w1 = two ? __shfl_sync(gm, w, s1, G) : 0.0f;
      float x0[CL::NE], x1[CL::NE];
      CL::load(A.delta + (int64_t)u0 * A.d, gl, k, x0);
      CL::load(A.delta + (int64_t)u1 * A.d, gl, k, x1);
#pragma unroll
      for (int e = 0; e < CL::NE; ++e) acc[e] = fmaf(w1, x1[e], fmaf(w0, x0[e], acc[e]));
    }
  }
  return matched;
}

// Warp pull of out(v)[beg, end): 32 ids/stamps per step, hits compacted in
// shared memory, each group gathers two hit rows per step (8 rows in flight
// per warp). acc holds the group's partial (reduce across groups after).
template <int PER, bool VEC>
DAMF_D int pull_warp(const PprArgs& A, int64_t base, int beg, int end, int R, int k, int lane,
                     int* sid, float* sw, float (&acc)[Cols<PER, VEC>::NE]) {
  using CL = Cols<PER, VEC>;
  const int grp = lane / G, gl = lane & (G - 1);
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
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    const int nh = __popc(m);
    if (hit) {
      const int pos = __popc(m & ((1u << lane) - 1u));
      sid[pos] = u;
      sw[pos] = w;
    }
    __syncwarp();
    for (int q = 2 * grp; q < nh; q += 2 * NG) {
      const bool two = q + 1 < nh;
      const int u0 = sid[q], u1 = two ? sid[q + 1] : u0;
      const float w0 = sw[q], w1 = two ? sw[q + 1] : 0.0f;
      float x0[CL::NE], x1[CL::NE];
      CL::load(A.delta + (int64_t)u0 * A.d, gl, k, x0);
      CL::load(A.delta + (int64_t)u1 * A.d, gl, k, x1);
#pragma unroll
      for (int e = 0; e < CL::NE; ++e) acc[e] = fmaf(w1, x1[e], fmaf(w0, x0[e], acc[e]));
    }
    __syncwarp();
    matched += nh;
  }
  return matched;
}

// r[v] = [v pushed this round ? 0 : r[v]] + (1-alpha)/max(deg v,1) acc ; key[v].
// Rows with no pulled arc that were not pushed are unchanged (skipped).
template <int PER, bool VEC>
DAMF_D void finish_group(const PprArgs& A, int v, int R, int k, double om, int gl, unsigned gm,
                         const float (&acc)[Cols<PER, VEC>::NE], bool any) {
  using CL = Cols<PER, VEC>;
  const bool inF = A.stamp[v] == R;
  if (!inF && !any) return;
  const double degv = A.deg[v];
  const float coef = (float)(om / fmax(degv, 1.0));
  float* rv = A.rb + (int64_t)v * A.d;
  float r[CL::NE];
  if (inF) {
#pragma unroll
    for (int e = 0; e < CL::NE; ++e) r[e] = 0.0f;
  } else {
    CL::load(rv, gl, k, r);
  }
  float m = 0.0f;
#pragma unroll
  for (int e = 0; e < CL::NE; ++e) {
    r[e] = fmaf(coef, acc[e], r[e]);
    if (CL::col(gl, e) < k) m = fmaxf(m, fabsf(r[e]));
  }
  CL::store(rv, gl, k, r);
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(gm, m, o, G));
  if (gl == 0) A.key[v] = (float)((double)m / fmax(degv, 1.0));
}

// Warp-wide finish after the cross-group reduction (every group holds the
// full sum; group q reads/writes the slice elements it owns).
template <int PER, bool VEC>
DAMF_D void finish_warp(const PprArgs& A, int v, int R, int k, double om, int lane,
                        const float (&acc)[Cols<PER, VEC>::NE], bool any) {
  using CL = Cols<PER, VEC>;
  const int grp = lane / G, gl = lane & (G - 1);
  const bool inF = A.stamp[v] == R;
  if (!inF && !any) return;
  const double degv = A.deg[v];
  const float coef = (float)(om / fmax(degv, 1.0));
  float* rv = A.rb + (int64_t)v * A.d;
  float m = 0.0f;
  if (VEC) {
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int j = 4 * gl + 4 * G * t;
      if (t % NG != grp || j >= k) continue;
      float4 r = inF ? make_float4(0.f, 0.f, 0.f, 0.f) : *reinterpret_cast<const float4*>(rv + j);
      r.x = fmaf(coef, acc[4 * t], r.x);
      r.y = fmaf(coef, acc[4 * t + 1], r.y);
      r.z = fmaf(coef, acc[4 * t + 2], r.z);
      r.w = fmaf(coef, acc[4 * t + 3], r.w);
      *reinterpret_cast<float4*>(rv + j) = r;
      m = fmaxf(m, fmaxf(fmaxf(fabsf(r.x), fabsf(r.y)), fmaxf(fabsf(r.z), fabsf(r.w))));
    }
  } else {
#pragma unroll
    for (int e = 0; e < CL::NE; ++e) {
      const int j = gl + G * e;
      if (e % NG != grp || j >= k) continue;
      const float r = fmaf(coef, acc[e], inF ? 0.0f : rv[j]);
      rv[j] = r;
      m = fmaxf(m, fabsf(r));
    }
  }
  m = warp_max(m);
  if (lane == 0) A.key[v] = (float)((double)m / fmax(degv, 1.0));
}

template <int PER, bool VEC>
DAMF_D void reduce_groups(float (&acc)[Cols<PER, VEC>::NE]) {
#pragma unroll
  for (int e = 0; e < Cols<PER, VEC>::NE; ++e) {
#pragma unroll
    for (int o = G; o < 32; o <<= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
  }
}

// Heavy-row chunk partial -> hacc[h] (vector reductions, owned slice only).
template <int PER, bool VEC>
DAMF_D void chunk_accumulate(float* hrow, int k, int lane, const float (&acc)[Cols<PER, VEC>::NE]) {
  const int grp = lane / G, gl = lane & (G - 1);
  if (VEC) {
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int j = 4 * gl + 4 * G * t;
      if (t % NG != grp || j >= k) continue;
      atomicAdd(reinterpret_cast<float4*>(hrow + j),
                make_float4(acc[4 * t], acc[4 * t + 1], acc[4 * t + 2], acc[4 * t + 3]));
    }
  } else {
#pragma unroll
    for (int e = 0; e < Cols<PER, VEC>::NE; ++e) {
      const int j = gl + G * e;
      if (e % NG != grp || j >= k) continue;
      atomicAdd(hrow + j, acc[e]);
    }
  }
}

// ---- work distribution: NQ counters per phase, each on its own 128-byte
// line, each owning a contiguous slice of the item space. A warp starts at
// queue (warp id mod NQ), grabs batches there until the slice is drained
// (checked with a plain load first, so drained queues cost no atomics), then
// moves on. Same-address atomics serialise in L2; spreading them over NQ
// lines and sizing batches to the remaining work keeps grabs cheap.
constexpr int NQ = 32, QS = 16;  // queues per phase, u64 stride between counters
constexpr int WQ_P1 = 0, WQ_P3 = NQ * QS, WQ_MK = 2 * NQ * QS, WQ_SC = 3 * NQ * QS;
// scalar counters at WQ_SC + QS * i
// (item counters alternate by round parity: reset after a round's last sync
// while the next round may already append)
constexpr int SC_MITEMS = 0 /* 0..1 */, SC_PUSH = 2 /* 2..4 */, SC_ITEMS = 5 /* 5..6 */,
              SC_S = 7 /* 7..9 */, SC_ARCS = 10;

struct Grabber {
  unsigned long long* q;
  int total, SB, dlo, len, q0, wpq, gw, nw, i;
  // The first half of the items is dealt statically in SB-item batches
  // strided over the warps (batch i of warp w = items [(i*nw + w)*SB, +SB)),
  // which mixes expensive and cheap items evenly; the rest goes through NQ
  // queues (dynamic, absorbs the imbalance).
  DAMF_D Grabber(unsigned long long* qbase, int total_, int gw_, int nw_, int SB_)
      : q(qbase), total(total_), SB(SB_), q0(gw_ % NQ), wpq(max(1, nw_ / NQ)), gw(gw_), nw(nw_),
        i(0) {
    const long long per = (long long)nw * SB;
    dlo = (int)(total / (2 * per) * per);
    if (total <= 4 * per) dlo = total;  // small: all static (a few strided batches per warp, no grabs)
    len = (total - dlo + NQ - 1) / NQ;
  }
  // warp-uniform; returns false when every item is taken
  DAMF_D bool next(int lane, int minB, int maxB, int& start, int& cnt) {
    const long long s0 = ((long long)i * nw + gw) * SB;
    if (s0 < dlo) {
      ++i;
      start = (int)s0;
      cnt = (int)min((long long)SB, dlo - s0);
      return true;
    }
    if (len == 0) return false;
    for (;;) {
      // lane l inspects queue (q0 + l) % NQ: one round trip for all queues
      const int sl = (q0 + lane) % NQ;
      const int lo = dlo + sl * len, hi = min(total, lo + len);
      const int cur = (int)min((unsigned long long)len, *(volatile unsigned long long*)(q + sl * QS));
      const unsigned m = __ballot_sync(0xffffffffu, lo + cur < hi);
      if (!m) return false;
      const int j = __ffs(m) - 1;
      const int qs = __shfl_sync(0xffffffffu, sl, j);
      const int qlo = __shfl_sync(0xffffffffu, lo, j), qhi = __shfl_sync(0xffffffffu, hi, j);
      const int rem = __shfl_sync(0xffffffffu, hi - lo - cur, j);
      const int B = (min(maxB, max(minB, rem / (2 * wpq))) + 3) & ~3;
      int got = 0;
      if (lane == 0) got = (int)min((unsigned long long)len, atomicAdd(q + qs * QS, (unsigned long long)B));
      got = __shfl_sync(0xffffffffu, got, 0);
      if (qlo + got >= qhi) continue;
      start = qlo + got;
      cnt = min(B, qhi - start);
      return true;
    }
  }
};

// One dense PULL round over every item (heavy-row chunks encoded -(c+1)
// first, then light rows), used both inside the cooperative kernel and by
// the lean standalone pull kernel. Items come from the grabber; small rows
// go to 8-lane groups, long rows and chunks to whole warps.
template <int PER, bool VEC>
DAMF_D void dense_pull(const PprArgs& A, unsigned long long* wq, int R, int nchunks, int n, int k,
                       double om, int lane, int grp, int gl, unsigned gm, int gw, int nw, int* sid,
                       float* sw, long long& c_aff, long long& c_arcs, long long& c_pulled) {
  using CL = Cols<PER, VEC>;
  const int d = A.d;
    // ---------------- PULL: items = heavy chunks (-(c+1)) then light rows
    const int nitems = nchunks + n;
    Grabber gb(wq + WQ_P3, nitems, gw, nw, NG);
    int start, cnt;
    while (gb.next(lane, NG, 32, start, cnt)) {
      const int stop = start + cnt;
      for (int base = start; base < stop; base += NG) {
        const int ii = base + grp;
        int v = -1, h = -1, beg = 0, end = 0;
        bool valid = ii < stop;
        if (valid) {
          if (ii < nchunks) {
            const int c = ii;
            h = A.cidx[c];
            v = A.heavy[h];
            beg = (c - A.hoff[h]) * CH;
            end = min(beg + CH, A.out.cnt[v]);
          } else {
            v = ii - nchunks;
            if (A.hidx[v] >= 0) valid = false;
            else end = A.out.cnt[v];
          }
        }
        const bool big = valid && (h >= 0 || end > SMALL);
        if (valid && !big) {
          float acc[CL::NE];
#pragma unroll
          for (int e = 0; e < CL::NE; ++e) acc[e] = 0.0f;
          const int got = end ? pull_group<PER, VEC>(A, A.out.off[v], 0, end, R, k, gl, gm, acc) : 0;
          if (gl == 0) {
            c_aff += 1;
            c_arcs += end;
            c_pulled += got;
          }
          finish_group<PER, VEC>(A, v, R, k, om, gl, gm, acc, got > 0);
        }
        unsigned bm = __ballot_sync(0xffffffffu, big) & GLEADS;
        while (bm) {
          const int src = __ffs(bm) - 1;
          bm &= bm - 1;
          const int bv = __shfl_sync(0xffffffffu, v, src);
          const int bh = __shfl_sync(0xffffffffu, h, src);
          const int bb = __shfl_sync(0xffffffffu, beg, src);
          const int be = __shfl_sync(0xffffffffu, end, src);
          float acc[CL::NE];
#pragma unroll
          for (int e = 0; e < CL::NE; ++e) acc[e] = 0.0f;
          const int got = pull_warp<PER, VEC>(A, A.out.off[bv], bb, be, R, k, lane, sid, sw, acc);
          if (lane == 0) {
            c_aff += bh < 0;
            c_arcs += be - bb;
            c_pulled += got;
          }
          if (bh >= 0) {
            // chunk partial -> hacc[bh]; the warp completing the row's last
            // chunk finishes the row (threadfence-reduction pattern)
            if (got) {
              reduce_groups<PER, VEC>(acc);
              chunk_accumulate<PER, VEC>(A.hacc + (int64_t)bh * d, k, lane, acc);
            }
            __threadfence();
            __syncwarp();
            int old = 0;
            if (lane == 0) old = atomicAdd(&A.hdone[bh], 1);
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old == A.hoff[bh + 1] - A.hoff[bh] - 1) {
              __threadfence();
              float* hrow = A.hacc + (int64_t)bh * d;
              CL::template load<true>(hrow, gl, k, acc);
              __syncwarp();
              if (grp == 0) {
                float zero[CL::NE];
#pragma unroll
                for (int e = 0; e < CL::NE; ++e) zero[e] = 0.0f;
                CL::store(hrow, gl, k, zero);
              }
              if (lane == 0) {
                A.hdone[bh] = 0;
                c_aff += 1;
              }
              finish_warp<PER, VEC>(A, bv, R, k, om, lane, acc, true);
            }
          } else {
            reduce_groups<PER, VEC>(acc);
            finish_warp<PER, VEC>(A, bv, R, k, om, lane, acc, got > 0);
          }
        }
      }
    }
}

constexpr int MCH = PPR_MCH;  // in-arcs per scatter item (ppr.cuh)

// One cooperative kernel runs every round of the push with grid barriers.
// Each round:
//   P1  candidates (all rows after a pull round; the rows the previous
//       scatter touched, with their key recomputed here from r, otherwise):
//       key * s_max > alpha eps  ->  delta = r, Z += r, r = 0, key = 0,
//       stamp = R; pushers append their in-arc chunks as scatter items and
//       count S = sum of their in-degrees.
//   --- barrier ---
//   If S is large (S * 64 > arcs): PULL round (no atomics): every row v
//       r[v] += (1-alpha)/max(deg v,1) sum_{u in out(v), stamp u = R} w delta[u],
//       heavy rows (> HEAVY arcs) split into CH-arc chunks accumulated in
//       hacc[h] and finished by the warp completing the last chunk.
//   Else SCATTER round: for every pushed u and v in in(u):
//       r[v] += (1-alpha) w / max(deg v,1) delta[u]   (red.global.add.v4.f32),
//       the first toucher of v appends it to the next candidate list.
//   --- barrier ---
// The scatter makes the fp32 summation order of touched rows
// nondeterministic (as in the fused per-event push); the defect bound, the
// reference's contract (enhancer.cpp:98-157), is unaffected.
template <int PER, bool VEC>
__global__ void __launch_bounds__(PT_, ((VEC ? 4 * PER : PER) >= 16) ? 2 : 3) ppr_push_kernel(PprArgs A) {
  using CL = Cols<PER, VEC>;
  cg::grid_group g = cg::this_grid();
  __shared__ int s_id[PW][32];
  __shared__ int s_pair[PW][32];
  __shared__ float s_w[PW][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int grp = lane / G, gl = lane & (G - 1);
  const unsigned gm = GMASK << (grp * G);
  const unsigned lt = (1u << lane) - 1u;
  const int gw = blockIdx.x * PW + wib, nw = gridDim.x * PW;
  int* sid = s_id[wib];
  int* spair = s_pair[wib];
  float* sw = s_w[wib];
  unsigned long long* wq = A.wq;
  unsigned long long* sc = wq + WQ_SC;
  const int k = A.ctl->k, d = A.d;
  const int n = (int)A.n;
  const float thr = (float)(A.alpha_eps / *A.smax);
  const double om = 1.0 - A.alpha;
  const DevCSR& inC = A.directed ? A.in : A.out;
  // Isolated edges (u - v, both of degree 1, undirected): their residual
  // bounces between the two rows, shrinking by (1-alpha)^2 per two pushes,
  // which on R-MAT graphs (many such components) keeps ~50 extra rounds
  // alive with a few hundred rows each. A pushed paired row instead takes
  // the pair to its fixed point in one step: with c_uv = (1-alpha) w / deg v
  // (what pushing u adds to r[v]) the infinite alternating sequence pushes
  //   S_u = (r_u + c_vu r_v) / (1 - c_uv c_vu),  S_v = (r_v + c_uv r_u) / (...)
  // out of u and v; Z[u] += S_u, Z[v] += S_v, r[u] = r[v] = 0 (zero residual,
  // inside the defect bound enhancer.cpp:98-157 asks for). Both rows of a
  // pair may be closed concurrently in one round: the residuals are taken
  // with atomicExch and the Z updates are atomic, so each part is counted once.
  auto pair_of = [&](int u) -> int {
    if (A.directed || inC.cnt[u] != 1) return -1;
    const int v = inC.ids[inC.off[u]];
    if (v == u || inC.cnt[v] != 1 || inC.ids[inC.off[v]] != u) return -1;
    return v;
  };
  auto close_pair = [&](int u, int v) {
    const double wu = inC.wts ? inC.wts[inC.off[u]] : 1.0;
    const double wv = inC.wts ? inC.wts[inC.off[v]] : 1.0;
    const float cuv = (float)(om * wu / fmax(A.deg[v], 1.0));
    const float cvu = (float)(om * wv / fmax(A.deg[u], 1.0));
    const float inv = (float)(1.0 / (1.0 - (double)cuv * (double)cvu));
    float* ru = A.rb + (int64_t)u * d;
    float* rv = A.rb + (int64_t)v * d;
    float* zu = A.Zb + (int64_t)u * d;
    float* zv = A.Zb + (int64_t)v * d;
#pragma unroll
    for (int e = 0; e < CL::NE; ++e) {
      const int j = CL::col(gl, e);
      if (j < k) {
        const float a = atomicExch(ru + j, 0.0f), b = atomicExch(rv + j, 0.0f);
        atomicAdd(zu + j, (a + cvu * b) * inv);
        atomicAdd(zv + j, (b + cuv * a) * inv);
      }
    }
    if (gl == 0) {
      A.key[u] = 0.0f;
      A.key[v] = 0.0f;
    }
  };
  const bool resume = A.split && A.pst->phase == 1;
  int R = resume ? A.pst->R : (int)A.stats[2];  // device-resident round stamp base (monotonic)
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < WQ_SC + 16 * QS; i += PT_) wq[i] = 0;
  // The heavy-row lists (rows above HEAVY out-arcs: list, chunk prefix, chunk
  // -> row) and the exact arc count serve dense pull rounds only; a push that
  // starts from a candidate list builds them the first time a round turns
  // dense (three passes over every row's arc count, ~0.3 ms at 8.4 M rows --
  // a fifth of the push after 1,000 insertions, which never pulls).
  int nH = 0, nchunks = 0;
  long long narcs = A.narcs_hint;
  bool have_heavy = resume;
  auto build_heavy = [&]() {
    nH = grid_compact(
        g, n,
        [&](int i, int& v) {
          v = i;
          return A.out.cnt[i] > HEAVY;
        },
        A.heavy, A.blk);
    nchunks = grid_scan(
        g, nH, [&](int h) { return (A.out.cnt[A.heavy[h]] + CH - 1) / CH; }, A.hoff, A.blk);
    for (int h = blockIdx.x * PT_ + threadIdx.x; h < nH; h += gridDim.x * PT_) {
      A.hidx[A.heavy[h]] = h;
      for (int c = A.hoff[h]; c < A.hoff[h + 1]; ++c) A.cidx[c] = h;
    }
    unsigned long long arcs = 0;
    for (int i = blockIdx.x * PT_ + threadIdx.x; i < n; i += gridDim.x * PT_) arcs += A.out.cnt[i];
    for (int o = 16; o > 0; o >>= 1) arcs += __shfl_xor_sync(0xffffffffu, arcs, o);
    if (lane == 0 && arcs) atomicAdd(&sc[SC_ARCS * QS], arcs);
    g.sync();
    narcs = (long long)*(volatile unsigned long long*)&sc[SC_ARCS * QS];
    have_heavy = true;
  };
  if (resume) {
    nH = A.pst->nH;
    nchunks = A.pst->nchunks;
    narcs = A.pst->narcs;
  }
  g.sync();  // counters zeroed
  if (!resume && A.ncand < 0) build_heavy();  // whole-graph scan: dense rounds are the rule
  // ---- rounds
  bool cand_all = resume || A.ncand < 0;
  int ncand = cand_all ? n : A.ncand;
  const int* candL = cand_all ? nullptr : A.cand;
  // candidates' keys must be recomputed from r: after a scatter round, and for
  // a caller's candidate list (one group per candidate spreads a short list
  // over the whole grid; the key scan hands a warp 32 of them)
  bool fresh = !cand_all;
  long long pushes = resume ? A.pst->pushes : 0;
  long long c_aff = 0, c_arcs = 0, c_pulled = 0;  // lane-0 accounting
  int rounds = resume ? A.pst->rounds : 0;
  int cur = resume ? A.pst->cur : 0;  // items[cur]: rows touched by this round's scatter
  bool split_exit = false;
  // per-phase wall time (block 0 thread 0, %globaltimer ns) -> ctl->prof[24..28],
  // only in DAMF_PROF builds: the global read-modify-write would otherwise sit
  // on block 0's path into every phase
  const bool tl = blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long tp = (DAMF_PROF && tl) ? globaltimer() : 0;
  auto tmark = [&](int slot) {
    if (DAMF_PROF && tl) {
      const unsigned long long t = globaltimer();
      A.ctl->prof[slot] += t - tp;
      tp = t;
    }
  };
  unsigned long long tr0 = 0;  // DAMF_PROF: round start (block 0 thread 0)
  for (;;) {
    if (DAMF_PROF && tl) tr0 = globaltimer();
    ++R;
    const int par = R & 1;
    unsigned long long* pushc = &sc[(SC_PUSH + R % 3) * QS];
    unsigned long long* sumS = &sc[(SC_S + R % 3) * QS];
    // ---------------- P1: push
    long long mine = 0, myS = 0;  // mine: warp-uniform; myS: per lane
    // pushed row u (whole group): delta = r, Z += r, r = 0, key = 0, stamp;
    // x = r slice already in registers
    auto push_row = [&](int u, const float (&x)[CL::NE]) {
      float z[CL::NE], zero[CL::NE];
      CL::load(A.Zb + (int64_t)u * d, gl, k, z);
      CL::store(A.delta + (int64_t)u * d, gl, k, x);
#pragma unroll
      for (int e = 0; e < CL::NE; ++e) {
        z[e] += x[e];
        zero[e] = 0.0f;
      }
      CL::store(A.Zb + (int64_t)u * d, gl, k, z);
      CL::store(A.rb + (int64_t)u * d, gl, k, zero);
      if (gl == 0) {
        A.stamp[u] = R;
        A.key[u] = 0.0f;
      }
    };
    // scatter items of the pushed rows (uniform within the calling group set)
    auto add_items = [&](int u, bool pushed) {
      const int c = pushed ? inC.cnt[u] : 0;
      const int nit = (c + MCH - 1) / MCH;
      int tot = nit;  // warp-aggregate the reservations (one atomic per warp)
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, tot, o);
        if (lane >= o) tot += y;
      }
      const int all = __shfl_sync(0xffffffffu, tot, 31);
      if (all == 0) return 0;
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(&sc[(SC_MITEMS + par) * QS], (unsigned long long)all);
      base = __shfl_sync(0xffffffffu, base, 0);
      // the whole warp writes the items (a hub's in-list is thousands of
      // items: one lane alone would hold its round up); item idx belongs to
      // the last lane whose exclusive offset is <= idx
      const int excl = tot - nit;
      for (int b = 0; b < all; b += 32) {
        const int idx = b + lane;
        int l = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const int e = __shfl_sync(0xffffffffu, excl, (l + step) & 31);
          if (l + step < 32 && e <= idx) l += step;
        }
        const int uo = __shfl_sync(0xffffffffu, u, l);
        const int eo = __shfl_sync(0xffffffffu, excl, l);
        if (idx < all) {
          A.mitems[2 * (base + idx)] = uo;
          A.mitems[2 * (base + idx) + 1] = idx - eo;
        }
      }
      return c;
    };
    if (!fresh) {
      // keys are current: lane-per-candidate check, groups copy the pushers
      Grabber gb(wq + WQ_P1, ncand, gw, nw, 32);
      int start, cnt;
      while (gb.next(lane, 32, 128, start, cnt)) {
        for (int s0 = start; s0 < start + cnt; s0 += 32) {
          const int q = s0 + lane;
          int v = -1;
          if (q < start + cnt) v = cand_all ? q : candL[q];
          const bool push = v >= 0 && A.key[v] > thr;
          const unsigned pm = __ballot_sync(0xffffffffu, push);
          if (!pm) continue;
          const int np = __popc(pm);
          mine += np;
          const int pv = push ? pair_of(v) : -1;
          if (push) {
            sid[__popc(pm & lt)] = v;
            spair[__popc(pm & lt)] = pv;
          }
          myS += add_items(v, push && pv < 0);
          __syncwarp();
          for (int j = grp; j < np; j += NG) {
            const int u = sid[j], pu = spair[j];
            if (pu >= 0) {
              close_pair(u, pu);
              continue;
            }
            float x[CL::NE];
            CL::load(A.rb + (int64_t)u * d, gl, k, x);
            push_row(u, x);
          }
          __syncwarp();
        }
      }
    } else {
      // after a scatter: group per candidate, key from r, push if over
      Grabber gb(wq + WQ_P1, ncand, gw, nw, NG);
      int start, cnt;
      while (gb.next(lane, NG, 32, start, cnt)) {
        for (int base = start; base < start + cnt; base += NG) {
          const int q = base + grp;
          const int v = q < start + cnt ? candL[q] : -1;
          bool push = false;
          int pv = -1;
          float x[CL::NE];
          if (v >= 0) {
            CL::load(A.rb + (int64_t)v * d, gl, k, x);
            float m = 0.0f;
#pragma unroll
            for (int e = 0; e < CL::NE; ++e)
              if (CL::col(gl, e) < k) m = fmaxf(m, fabsf(x[e]));
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(gm, m, o, G));
            const float key = (float)((double)m / fmax(A.deg[v], 1.0));
            push = key > thr;
            if (push) {
              pv = pair_of(v);
              if (pv >= 0) close_pair(v, pv);
              else push_row(v, x);
            } else if (gl == 0) {
              A.key[v] = key;
            }
          }
          const unsigned pm = __ballot_sync(0xffffffffu, push && gl == 0);
          mine += __popc(pm);
          myS += add_items(v, push && gl == 0 && pv < 0);
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) myS += __shfl_xor_sync(0xffffffffu, myS, o);
    if (lane == 0 && mine) {
      atomicAdd(pushc, (unsigned long long)mine);
      atomicAdd(sumS, (unsigned long long)myS);
    }
    g.sync();
    tmark(24);
    const long long nF = (long long)*(volatile unsigned long long*)pushc;
    const long long S = (long long)*(volatile unsigned long long*)sumS;
    const int nmi = (int)*(volatile unsigned long long*)&sc[(SC_MITEMS + par) * QS];
    if (blockIdx.x == 0) {
      if (threadIdx.x < NQ) wq[WQ_P1 + threadIdx.x * QS] = 0;
      if (threadIdx.x == 0) {
        sc[(SC_PUSH + (R + 1) % 3) * QS] = 0;
        sc[(SC_S + (R + 1) % 3) * QS] = 0;
        // the previous round's touched count: read by every thread before
        // this round's P1 barrier, next appended in round R + 1
        sc[(SC_ITEMS + (par ^ 1)) * QS] = 0;
      }
    }
    if (nF == 0) break;
    ++rounds;
    pushes += nF;
    if (pushes > A.push_guard || rounds > 1000000) {
      if (blockIdx.x == 0 && threadIdx.x == 0) A.ctl->err = 9;  // NonConvergence
      break;
    }
    // (force_pull: diagnostic switch, every round in the atomics-free pull form)
    bool dense = S * 64 > narcs || A.force_pull;
    if (dense && !have_heavy) {  // (grid-uniform: S and narcs are)
      build_heavy();
      dense = S * 64 > narcs || A.force_pull;
    }
    if (tl && A.trace && rounds <= 1024) {
      long long* t = A.trace + 4 * (rounds - 1);
      t[0] = nF;
      t[1] = dense;
      t[2] = S;
      t[3] = nmi;
      // DAMF_PROF builds: push-phase ns in the high half of t[3], round ns
      // in t[1] >> 1 (added at the end of the round)
      if (DAMF_PROF) t[3] |= (long long)((globaltimer() - tr0) << 32);
    }
    if (dense && A.split) {
      // hand the round to the lean pull kernel (more warps per SM than this
      // cooperative kernel's register budget allows) and resume after it
      if (tl) {
        A.pst->R = R;
        A.pst->rounds = rounds;
        A.pst->pushes = pushes;
        A.pst->nH = nH;
        A.pst->nchunks = nchunks;
        A.pst->narcs = narcs;
        A.pst->cur = cur ^ 1;
        A.pst->phase = 1;
        A.pst->pull_pending = 1;
      }
      split_exit = true;
      break;
    }
    if (dense) {
      dense_pull<PER, VEC>(A, wq, R, nchunks, n, k, om, lane, grp, gl, gm, gw, nw, sid, sw, c_aff,
                           c_arcs, c_pulled);
    } else {
      // ---------------- SCATTER over the pushed rows' in-arc chunks
      int* L = A.items[cur];
      Grabber gb(wq + WQ_MK, nmi, gw, nw, 1);
      int start, cnt;
      while (gb.next(lane, 1, 4, start, cnt)) {
        for (int it = start; it < start + cnt; ++it) {
          const int u = A.mitems[2 * it], ci = A.mitems[2 * it + 1];
          const int64_t ib = inC.off[u];
          const int beg = ci * MCH, end = min(beg + MCH, inC.cnt[u]);
          // Random-row reductions that miss L2 run at ~80 GB/s (each one waits
          // for its line from DRAM inside the atomic unit): first pull this
          // item's target rows into L2 with bulk prefetches (all in flight at
          // once), then reduce into L2-resident lines.
          // (bulk prefetches need 16-byte aligned rows: d % 4 == 0)
          for (int p0 = beg; (d & 3) == 0 && p0 < end; p0 += 32) {
            const int p = p0 + lane;
            if (p < end) {
              const float* row = A.rb + (int64_t)inC.ids[ib + p] * d;
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row), "r"((unsigned)(k * 4 + 15) & ~15u)
                           : "memory");
            }
          }
          float x[CL::NE];
          CL::load(A.delta + (int64_t)u * d, gl, k, x);
          if (lane == 0) c_arcs += end - beg;
          // |delta_u|_inf: what this push can add to a target's key (below)
          float dmax = 0.0f;
#pragma unroll
          for (int e = 0; e < CL::NE; ++e)
            if (CL::col(gl, e) < k) dmax = fmaxf(dmax, fabsf(x[e]));
#pragma unroll
          for (int o = G / 2; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(gm, dmax, o, G));
          for (int p0 = beg; p0 < end; p0 += 32) {
            const int p = p0 + lane;
            const bool ok = p < end;
            int v = 0;
            float coef = 0.0f;
            bool t = false;
            if (ok) {
              v = inC.ids[ib + p];
              const double w = inC.wts ? inC.wts[ib + p] : 1.0;
              const double dg = fmax(A.deg[v], 1.0);
              coef = (float)(om * w / dg);
              // key[v] is kept as an upper bound of |r_v|_inf / max(deg v, 1):
              // this contribution raises it by at most |coef| |delta|_inf / dg.
              // Only a target whose bound crosses the threshold is a candidate
              // of the next round (a target under it cannot be over it), and
              // its first toucher appends it. The candidate threshold sits 1 %
              // lower: fp32 rounding of many small increments stays inside it.
              const float inc = (float)(fabs(om * w) / (dg * dg) * (double)dmax * (1.0 + 1e-4));
              const float kb = atomicAdd(&A.key[v], inc) + inc;
              t = kb > 0.99f * thr && __ldcg(&A.mark[v]) != R && atomicExch(&A.mark[v], R) != R;
            }
            const unsigned tm = __ballot_sync(0xffffffffu, t);
            if (tm) {
              unsigned long long b0 = 0;
              const int leader = __ffs(tm) - 1;
              if (lane == leader)
                b0 = atomicAdd(&sc[(SC_ITEMS + par) * QS], (unsigned long long)__popc(tm));
              b0 = __shfl_sync(0xffffffffu, b0, leader);
              if (t) L[b0 + __popc(tm & lt)] = v;
              if (lane == 0) c_aff += __popc(tm);
            }
            const int na = min(32, end - p0);
            for (int a0 = 0; a0 < na; a0 += NG) {
              const int a = a0 + grp;
              const int va = __shfl_sync(0xffffffffu, v, a);
              const float ca = __shfl_sync(0xffffffffu, coef, a);
              if (a >= na) continue;
              float* rv = A.rb + (int64_t)va * d;
              if (VEC) {
#pragma unroll
                for (int t4 = 0; t4 < PER; ++t4) {
                  const int j = 4 * gl + 4 * G * t4;
                  if (j < k)
                    atomicAdd(reinterpret_cast<float4*>(rv + j),
                              make_float4(ca * x[4 * t4], ca * x[4 * t4 + 1], ca * x[4 * t4 + 2],
                                          ca * x[4 * t4 + 3]));
                }
              } else {
#pragma unroll
                for (int e = 0; e < CL::NE; ++e) {
                  const int j = gl + G * e;
                  if (j < k) atomicAdd(rv + j, ca * x[e]);
                }
              }
            }
          }
        }
      }
    }
    g.sync();
    tmark(dense ? 26 : 27);
    if (DAMF_PROF && tl && A.trace && rounds <= 1024)
      A.trace[4 * (rounds - 1) + 1] |= (long long)((globaltimer() - tr0) << 1);
    const int ntouched = dense ? 0 : (int)*(volatile unsigned long long*)&sc[(SC_ITEMS + par) * QS];
    if (blockIdx.x == 0) {
      if (threadIdx.x < NQ) {
        wq[WQ_P3 + threadIdx.x * QS] = 0;
        wq[WQ_MK + threadIdx.x * QS] = 0;
      }
      if (threadIdx.x == 0) {
        sc[(SC_MITEMS + par) * QS] = 0;
      }
    }
    cand_all = dense;
    fresh = !dense;
    ncand = dense ? n : ntouched;
    candL = A.items[cur];
    cur ^= 1;
  }
  if (!split_exit && have_heavy)
    for (int h = blockIdx.x * PT_ + threadIdx.x; h < nH; h += gridDim.x * PT_) A.hidx[A.heavy[h]] = -1;
  // accounting (bench algorithmic bytes): lane-0 counters of groups/warps
  for (int o = 16; o > 0; o >>= 1) {
    c_aff += __shfl_xor_sync(0xffffffffu, c_aff, o);
    c_arcs += __shfl_xor_sync(0xffffffffu, c_arcs, o);
    c_pulled += __shfl_xor_sync(0xffffffffu, c_pulled, o);
  }
  if (lane == 0 && (c_aff | c_arcs | c_pulled)) {
    atomicAdd((unsigned long long*)&A.stats[4], (unsigned long long)c_aff);
    atomicAdd((unsigned long long*)&A.stats[5], (unsigned long long)c_arcs);
    atomicAdd((unsigned long long*)&A.stats[6], (unsigned long long)c_pulled);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && !split_exit) {
    if (A.trace) A.trace[4 * 1024] = rounds;
    A.stats[0] += pushes;
    A.stats[1] += rounds;
    A.stats[2] = R;  // next round base
    A.stats[3] += pushes;
    if (A.split) {
      A.pst->phase = 0;
      A.pst->pull_pending = 0;
    }
    if (A.t_end) *A.t_end = globaltimer();
  }
}

// Dense PULL round as a standalone (non-cooperative) kernel: same work as the
// in-kernel round, but with a register budget that fits 4 CTAs (32 warps)
// per SM — random 512-byte gathers need ~24-32 warps per SM to approach HBM
// peak (tools/micro_gather.cu). Round state comes from PprState.
template <int PER, bool VEC>
#ifndef PPR_PULL_MINB
#define PPR_PULL_MINB 8
#endif
__global__ void __launch_bounds__(PT_, PPR_PULL_MINB) ppr_pull_kernel(PprArgs A) {
  __shared__ int s_id[PW][32];
  __shared__ float s_w[PW][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int grp = lane / G, gl = lane & (G - 1);
  const unsigned gm = GMASK << (grp * G);
  const int gw = blockIdx.x * PW + wib, nw = gridDim.x * PW;
  long long c_aff = 0, c_arcs = 0, c_pulled = 0;
  dense_pull<PER, VEC>(A, A.wq, A.pst->R, A.pst->nchunks, (int)A.n, A.ctl->k, 1.0 - A.alpha, lane,
                       grp, gl, gm, gw, nw, s_id[wib], s_w[wib], c_aff, c_arcs, c_pulled);
  for (int o = 16; o > 0; o >>= 1) {
    c_aff += __shfl_xor_sync(0xffffffffu, c_aff, o);
    c_arcs += __shfl_xor_sync(0xffffffffu, c_arcs, o);
    c_pulled += __shfl_xor_sync(0xffffffffu, c_pulled, o);
  }
  if (lane == 0 && (c_aff | c_arcs | c_pulled)) {
    atomicAdd((unsigned long long*)&A.stats[4], (unsigned long long)c_aff);
    atomicAdd((unsigned long long*)&A.stats[5], (unsigned long long)c_arcs);
    atomicAdd((unsigned long long*)&A.stats[6], (unsigned long long)c_pulled);
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
__global__ void __launch_bounds__(1024) smax_kernel(const double* PT0, const double* PT1,
                                                    const DevCtl* ctl, int ld, double* out) {
  // one CTA of 32 warps: row sums by warps (coalesced, 4-8 rows per warp),
  // column sums by threads over a quarter of the rows each; fixed orders
  __shared__ double cmax[32], part[4][kMaxD], rmax[kMaxD];
  const int k = ctl->k;
  const double* PT = ctl->pp[0] ? PT1 : PT0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double c1 = 0;
  for (int j = warp; j < k; j += 32) {
    double s = 0;
    for (int i = lane; i < k; i += 32) s += fabs(PT[(int64_t)j * ld + i]);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    c1 = fmax(c1, s);
  }
  if (lane == 0) cmax[warp] = c1;
  {
    const int i = threadIdx.x % kMaxD, q = threadIdx.x / kMaxD;  // kMaxD = 256: q in [0, 4)
    const int per = (k + 3) / 4, j0 = q * per, j1 = min(k, j0 + per);
    double s = 0;
    if (i < k)
      for (int j = j0; j < j1; ++j) s += fabs(PT[(int64_t)j * ld + i]);
    part[q][i] = s;
  }
  __syncthreads();
  if (threadIdx.x < kMaxD) {
    const int i = threadIdx.x;
    rmax[i] = i < k ? ((part[0][i] + part[1][i]) + (part[2][i] + part[3][i])) : 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int t = 0; t < 32; ++t) a = fmax(a, cmax[t]);
    for (int t = 0; t < k; ++t) b = fmax(b, rmax[t]);
    *out = k == 0 ? 1.0 : fmax(a, sqrt(a * b));
  }
}

}  // namespace

namespace {
template <int PER, bool VEC>
cudaError_t launch_push_t(const PprArgs& a, int grid, cudaStream_t s) {
  void* args[] = {(void*)&a};
  return cudaLaunchCooperativeKernel((void*)ppr_push_kernel<PER, VEC>, dim3(grid), dim3(PT_), args, 0, s);
}
template <int PER, bool VEC>
int max_grid_t(int nsm) {
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ppr_push_kernel<PER, VEC>, PT_, 0);
  return per * nsm;
}
}  // namespace

// Vectorised kernels when rows are 16-byte aligned (d % 4 == 0), otherwise a
// scalar column slice; PER sized to the row width d.
cudaError_t launch_ppr_push(const PprArgs& a, int grid, cudaStream_t s) {
  const int d = a.d;
  if (d % 4 == 0) {
    const int per = (d + 4 * G - 1) / (4 * G);
    if (per <= 1) return launch_push_t<1, true>(a, grid, s);
    if (per <= 2) return launch_push_t<2, true>(a, grid, s);
    if (per <= 4) return launch_push_t<4, true>(a, grid, s);
    return launch_push_t<8, true>(a, grid, s);
  }
  if (d <= 4 * G) return launch_push_t<4, false>(a, grid, s);
  return launch_push_t<32, false>(a, grid, s);
}

namespace {
template <int PER, bool VEC>
cudaError_t launch_pull_t(const PprArgs& a, int nsm, cudaStream_t s) {
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ppr_pull_kernel<PER, VEC>, PT_, 0);
  ppr_pull_kernel<PER, VEC><<<std::max(per, 1) * nsm, PT_, 0, s>>>(a);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_ppr_pull(const PprArgs& a, int nsm, cudaStream_t s) {
  const int d = a.d;
  if (d % 4 == 0) {
    const int per = (d + 4 * G - 1) / (4 * G);
    if (per <= 1) return launch_pull_t<1, true>(a, nsm, s);
    if (per <= 2) return launch_pull_t<2, true>(a, nsm, s);
    if (per <= 4) return launch_pull_t<4, true>(a, nsm, s);
    return launch_pull_t<8, true>(a, nsm, s);
  }
  if (d <= 4 * G) return launch_pull_t<4, false>(a, nsm, s);
  return launch_pull_t<32, false>(a, nsm, s);
}

int ppr_push_max_grid(int nsm, int d) {
  if (d % 4 == 0) {
    const int per = (d + 4 * G - 1) / (4 * G);
    if (per <= 1) return max_grid_t<1, true>(nsm);
    if (per <= 2) return max_grid_t<2, true>(nsm);
    if (per <= 4) return max_grid_t<4, true>(nsm);
    return max_grid_t<8, true>(nsm);
  }
  if (d <= 4 * G) return max_grid_t<4, false>(nsm);
  return max_grid_t<32, false>(nsm);
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
  smax_kernel<<<1, 1024, 0, s>>>(PT0, PT1, ctl, ld, out);
  return cudaGetLastError();
}

}  // namespace dgpu
