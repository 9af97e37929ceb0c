// Per-event kernel (K1-K4 + K9): graph mutation and the space-projection
// update of DAMF (update_engine.cpp:56-226, factor_state.cpp:129-213) for a
// range of events, run by ONE thread-block cluster of C CTAs that stays
// resident for the whole range (no host round trip between events).
//
// Per rank-1 step (Appendix B of SURVEY.md):
//   1. gather the touched base rows (fp32 -> fp64), w = S^-1/2 (g P)      K1
//   2. singular system of the bordered (k+1)^2 matrix M = D + a b^T via the
//      eigen-decomposition of M M^T: node steps are one symmetric rank-1
//      modification of D^2; edge steps are a rank-1 update followed by a
//      rank-1 downdate (the 2x2 core [[|b|^2,1],[1,0]] split by sign). Each
//      is a secular equation solved root-parallel (one warp per root) with
//      Gu-Eisenstat z-hat recomputation and LAPACK-style deflation.       K2
//   3. closed forms F = S1^1/2 H S2^-1/2, G = S1^1/2 E S2^-1/2 (edge), the
//      inverses from the orthonormal-column identity
//      A^-1 = A^T + d (A d)^T / (1 - |d|^2), P <- P F and P^-1 <- F^-1 P^-1
//      as cluster-split fp64 GEMMs, and the row fixes X_b[u] += ex P^-1.    K3
//   4. conditioning bookkeeping for the rebase policy.                     K4
// Rank growth, shrinkage or an ill-conditioned F fold eagerly (X_b <- X_b P F)
// exactly like factor_state.cpp:168-192.
//
// Matrices exchanged between CTAs are stored "one owned vector per row":
// P is kept TRANSPOSED (PT[j][i] = P[i][j]) and Q = P^-1 row-major, so every
// GEMM is Out[t][:] = sum_m Coef[t][m] In[m][:] with Coef row t owned locally
// and In streamed with coalesced loads.
#include <cooperative_groups.h>

#include <cfloat>

#include "common.cuh"
#include "event_kernel.cuh"

namespace cg = cooperative_groups;

namespace dgpu {

namespace {

constexpr int NT = kEventThreads;  // 256 threads per CTA
constexpr int NW = NT / 32;
constexpr int NMAX = kMaxD + 1;    // k + 1 <= 257
constexpr int NPAD = kMaxD + 4;
constexpr double EPS = DBL_EPSILON;
constexpr int TCH = 9;  // GEMM output rows per chunk (registers)

template <int C>
struct Smem {
  static constexpr int PER = (NMAX + C - 1) / C;  // owned block size (max)
  // small vectors (fp64)
  double sig[NPAD], gA[NPAD], gB[NPAD], wA[NPAD], wB[NPAD];
  double av[NPAD], bv[NPAD], Dg[NPAD], dd[NPAD], zz[NPAD], um[NPAD];
  double sd[NPAD], sz[NPAD], kd[NPAD], kz[NPAD], kz2[NPAD];
  int kidx[NPAD], defl[NPAD], src[NPAD], org[NPAD];
  double tau[NPAD], zhat[NPAD], lamA[NPAD], lamB[NPAD];
  double s2[NPAD], exv[NPAD], eyv[NPAD], dH[NPAD], dE[NPAD], AHdH[NPAD], AEdE[NPAD];
  int rot_p[NPAD], rot_q[NPAD];
  double rot_c[NPAD], rot_s[NPAD];
  double partH[C][kMaxD], partE[C][kMaxD];
  double pnorm[C][4];
  double coef[TCH * NPAD];        // staged GEMM coefficient rows
  double red[NT * TCH];           // GEMM split-K reduction
  double vscr[NW][NPAD];          // per-warp eigenvector scratch
  double bred[NW];
  long long found[C][2];          // graph row-scan results
  int K, nrot, need;
  int k, pp[2];
  double rhoN, sumkz2;
  int err;
};

// ----------------------------------------------------------------- reductions
template <int C>
DAMF_D double block_sum(Smem<C>& S, double v) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) S.bred[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) t += S.bred[w];  // fixed order: identical in every CTA
  return t;
}

template <int C>
DAMF_D int block_or(Smem<C>& S, int v) {
  return __syncthreads_or(v);
}

template <int C>
DAMF_D void bcast(cg::cluster_group& cl, double* local, int idx, double val) {
#pragma unroll 1
  for (int r = 0; r < C; ++r) *cl.map_shared_rank(local + idx, r) = val;
}
template <int C>
DAMF_D void bcast_i(cg::cluster_group& cl, int* local, int idx, int val) {
#pragma unroll 1
  for (int r = 0; r < C; ++r) *cl.map_shared_rank(local + idx, r) = val;
}

DAMF_D void block_range(int total, int C, int rank, int& lo, int& hi) {
  const int per = (total + C - 1) / C;
  lo = min(total, rank * per);
  hi = min(total, lo + per);
}

// ------------------------------------------------------------- row GEMM
// Out[t][j] = sum_m Coef[t][m] In[m][j], t in [t0,t1), j < J, m < M.
// Coef/In/Out global fp64 with leading dims. Coef rows are staged in smem;
// In is streamed once per CTA with coalesced loads (split-K over thread
// groups, reduced through smem in a fixed order). Optionally accumulates
// the Frobenius norm^2 of the written block into *fro (thread 0 result).
template <int C>
DAMF_D void rows_gemm(Smem<C>& S, double* Out, int ldo, const double* Coef, int ldc,
                      const double* __restrict__ In, int ldi, int t0, int t1, int M, int J,
                      double* fro) {
  double frob = 0.0;
  int jt = 32;
  while (jt < J) jt <<= 1;
  if (jt > NT) jt = NT;
  const int G = NT / jt;
  const int j = threadIdx.x % jt, g = threadIdx.x / jt;
  for (int c0 = t0; c0 < t1; c0 += TCH) {
    const int nt = min(TCH, t1 - c0);
    __syncthreads();
    for (int x = threadIdx.x; x < nt * M; x += NT) {
      const int t = x / M, m = x % M;
      S.coef[t * NPAD + m] = Coef[(int64_t)(c0 + t) * ldc + m];
    }
    __syncthreads();
    for (int jb = 0; jb < J; jb += jt) {
      const int jj = jb + j;
      double acc[TCH];
#pragma unroll
      for (int t = 0; t < TCH; ++t) acc[t] = 0.0;
      if (jj < J) {
        for (int m = g; m < M; m += G) {
          const double x = In[(int64_t)m * ldi + jj];
#pragma unroll
          for (int t = 0; t < TCH; ++t)
            if (t < nt) acc[t] = fma(S.coef[t * NPAD + m], x, acc[t]);
        }
      }
      if (G > 1) {
#pragma unroll
        for (int t = 0; t < TCH; ++t)
          if (t < nt) S.red[(t * G + g) * jt + j] = acc[t];
        __syncthreads();
        if (g == 0 && jj < J) {
          for (int t = 0; t < nt; ++t) {
            double s = 0;
            for (int q = 0; q < G; ++q) s += S.red[(t * G + q) * jt + j];
            Out[(int64_t)(c0 + t) * ldo + jj] = s;
            frob += s * s;
          }
        }
        __syncthreads();
      } else if (jj < J) {
        for (int t = 0; t < nt; ++t) {
          Out[(int64_t)(c0 + t) * ldo + jj] = acc[t];
          frob += acc[t] * acc[t];
        }
      }
    }
  }
  if (fro) *fro = block_sum(S, frob);
  __syncthreads();
}

// ------------------------------------------------------------ secular solver
// Root j of 1 + rho * sum_i kz2[i] / (kd[i] - lambda) = 0 (kd ascending,
// rho > 0, sum kz2 <= 1), one warp. Returns tau and the origin pole o with
// lambda = kd[o] + tau, so lambda - kd[i] is formed as tau - (kd[i]-kd[o]).
DAMF_D void secular_root(const double* kd, const double* kz2, int K, double rho, double sumz2,
                         int j, double& tau_out, int& org_out) {
  const int lane = threadIdx.x & 31;
  int o;
  double lo, hi;
  if (j < K - 1) {
    const double mid = 0.5 * (kd[j + 1] - kd[j]);
    double s = 0;
    for (int i = lane; i < K; i += 32) s += kz2[i] / ((kd[i] - kd[j]) - mid);
    s = warp_sum(s);
    if (1.0 + rho * s >= 0.0) {
      o = j;
      lo = 0.0;
      hi = mid;
    } else {
      o = j + 1;
      lo = -mid;
      hi = 0.0;
    }
  } else {
    o = j;
    lo = 0.0;
    hi = rho * sumz2 * (1.0 + 4.0 * EPS);
  }
  const double dorg = kd[o];
  double tau = 0.5 * (lo + hi);
  for (int it = 0; it < 120; ++it) {
    double psi = 0, phi = 0, dpsi = 0, dphi = 0, aerr = 0;
    for (int i = lane; i < K; i += 32) {
      const double del = (kd[i] - dorg) - tau;
      const double t = kz2[i] / del;
      const double dt = t / del;
      if (i <= j) {
        psi += t;
        dpsi += dt;
      } else {
        phi += t;
        dphi += dt;
      }
      aerr += fabs(t);
    }
    psi = rho * warp_sum(psi);
    phi = rho * warp_sum(phi);
    dpsi = rho * warp_sum(dpsi);
    dphi = rho * warp_sum(dphi);
    aerr = rho * warp_sum(aerr);
    const double f = 1.0 + psi + phi;
    if (f < 0.0)
      lo = fmax(lo, tau);
    else
      hi = fmin(hi, tau);
    if (fabs(f) <= 4.0 * EPS * K * (1.0 + aerr)) break;
    const double D1 = (kd[j] - dorg) - tau;
    double nt;
    bool ok = false;
    if (j < K - 1) {
      const double D2 = (kd[j + 1] - dorg) - tau;
      const double q1 = dpsi * D1 * D1, q2 = dphi * D2 * D2;
      const double c = 1.0 + psi - dpsi * D1 + phi - dphi * D2;
      const double Bq = c * (D1 + D2) + q1 + q2;
      const double Cq = D1 * D2 * f;
      const double disc = Bq * Bq - 4.0 * c * Cq;
      if (disc >= 0.0) {
        const double sq = sqrt(disc);
        const double den = Bq + (Bq >= 0.0 ? sq : -sq);
        if (den != 0.0) {
          nt = tau + 2.0 * Cq / den;
          ok = true;
        }
      }
    } else {
      const double q1 = dpsi * D1 * D1;
      const double c = 1.0 + psi - dpsi * D1 + phi;
      if (c > 0.0) {
        nt = tau + D1 + q1 / c;
        ok = true;
      }
    }
    if (!ok || !(nt > lo && nt < hi)) nt = 0.5 * (lo + hi);
    if (nt == tau || hi - lo <= 2.0 * EPS * fmax(fabs(lo), fabs(hi))) {
      tau = nt;
      break;
    }
    tau = nt;
  }
  tau_out = tau;
  org_out = o;
}

// Eigen-decomposition of diag(dd) + rho z z^T over n entries, cluster-wide.
// dd must be descending when rho > 0 and ascending when rho < 0; both map to
// the canonical ascending problem by index reversal (c = n-1-i) and, for
// rho < 0, negation. Outputs the actual eigenvalues in canonical output order
// (lamOut, all CTAs) and eigenvector e as row e of QT (global, ld ldq), for e
// in this CTA's block. Ends WITHOUT a cluster barrier.
template <int C>
DAMF_D void eig_rank1(Smem<C>& S, cg::cluster_group& cl, const double* dd, const double* z,
                      double rho, int n, double* QT, int ldq, double* lamOut) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)cl.block_rank();
  const bool neg = rho < 0.0;
  for (int c = tid; c < n; c += NT) {
    const int i = n - 1 - c;
    S.sd[c] = neg ? -dd[i] : dd[i];
    S.sz[c] = z[i];
  }
  __syncthreads();
  double zn2 = 0;
  for (int c = tid; c < n; c += NT) zn2 += S.sz[c] * S.sz[c];
  zn2 = block_sum(S, zn2);
  const double rhoN = fabs(rho) * zn2;
  const double zinv = zn2 > 0.0 ? 1.0 / sqrt(zn2) : 0.0;
  for (int c = tid; c < n; c += NT) S.sz[c] *= zinv;
  __syncthreads();
  const double tol = 8.0 * EPS * fmax(fmax(fabs(S.sd[0]), fabs(S.sd[n - 1])), rhoN);
  int need = 0;
  for (int c = tid; c < n; c += NT) {
    if (rhoN * fabs(S.sz[c]) <= tol) need = 1;
    if (c + 1 < n) {
      const double a = S.sz[c], b = S.sz[c + 1];
      const double tt = hypot(a, b);
      const double cs = (b / tt) * (-a / tt);
      if (fabs((S.sd[c + 1] - S.sd[c]) * cs) <= tol) need = 1;
    }
  }
  need = block_or(S, need);
  if (!need) {
    for (int c = tid; c < n; c += NT) {
      S.kd[c] = S.sd[c];
      S.kz[c] = S.sz[c];
      S.kz2[c] = S.sz[c] * S.sz[c];
      S.kidx[c] = c;
      S.defl[c] = 0;
    }
    if (tid == 0) {
      S.K = n;
      S.nrot = 0;
    }
  } else if (tid == 0) {
    // LAPACK dlaed2-style deflation, sequential (rare path).
    int nrot = 0;
    for (int c = 0; c < n; ++c) S.defl[c] = rhoN * fabs(S.sz[c]) <= tol;
    int pj = -1;
    for (int nj = 0; nj < n; ++nj) {
      if (S.defl[nj]) continue;
      if (pj < 0) {
        pj = nj;
        continue;
      }
      double s = S.sz[pj], c = S.sz[nj];
      const double tt = hypot(c, s);
      const double t = S.sd[nj] - S.sd[pj];
      c /= tt;
      s = -s / tt;
      if (fabs(t * c * s) <= tol) {
        S.sz[nj] = tt;
        S.sz[pj] = 0.0;
        const double dp = S.sd[pj], dn = S.sd[nj];
        S.sd[pj] = c * c * dp + s * s * dn;
        S.sd[nj] = s * s * dp + c * c * dn;
        S.rot_p[nrot] = pj;
        S.rot_q[nrot] = nj;
        S.rot_c[nrot] = c;
        S.rot_s[nrot] = s;
        ++nrot;
        S.defl[pj] = 1;
      }
      pj = nj;
    }
    int K = 0;
    for (int c = 0; c < n; ++c)
      if (!S.defl[c]) {
        S.kd[K] = S.sd[c];
        S.kz[K] = S.sz[c];
        S.kz2[K] = S.sz[c] * S.sz[c];
        S.kidx[K] = c;
        ++K;
      }
    S.K = K;
    S.nrot = nrot;
  }
  __syncthreads();
  const int K = S.K;
  double sz2 = 0;
  for (int j = tid; j < K; j += NT) sz2 += S.kz2[j];
  sz2 = block_sum(S, sz2);
  // --- roots (this CTA's block of K)
  int lo, hi;
  block_range(K, C, rank, lo, hi);
  for (int j = lo + warp; j < hi; j += NW) {
    double t;
    int o;
    secular_root(S.kd, S.kz2, K, rhoN, sz2, j, t, o);
    if (lane < C) {
      *cl.map_shared_rank(S.tau + j, lane) = t;
      *cl.map_shared_rank(S.org + j, lane) = o;
    }
  }
  cl.sync();
  // --- Gu-Eisenstat z-hat: zhat_i^2 = prod_j (lam_j - d_i) / prod_{j!=i} (d_j - d_i) / rho
  for (int i = lo + warp; i < hi; i += NW) {
    const double di = S.kd[i];
    double p = 1.0;
    for (int j = lane; j < K; j += 32) {
      const double lmd = S.tau[j] - (di - S.kd[S.org[j]]);  // lambda_j - d_i
      p *= (j == i) ? lmd / rhoN : lmd / (S.kd[j] - di);
    }
    p = warp_prod(p);
    const double zh = copysign(sqrt(fmax(p, 0.0)), S.kz[i]);
    if (lane < C) *cl.map_shared_rank(S.zhat + i, lane) = zh;
  }
  cl.sync();
  // --- output order (ascending canonical eigenvalues)
  if (!need) {
    for (int e = tid; e < n; e += NT) {
      S.src[e] = e;
      const double l = S.kd[S.org[e]] + S.tau[e];
      lamOut[e] = neg ? -l : l;
    }
  } else {
    // items: roots 0..K-1, then deflated canonical entries; rank by counting.
    for (int it = tid; it < n; it += NT) {
      double v;
      int item = it;
      if (it < K) {
        v = S.kd[S.org[it]] + S.tau[it];
      } else {
        int cnt = it - K, c = 0;
        for (c = 0; c < n; ++c)
          if (S.defl[c] && cnt-- == 0) break;
        v = S.sd[c];
        item = K + c;  // encode deflated canonical index c
      }
      int r = 0;
      for (int o2 = 0; o2 < n; ++o2) {
        double w;
        if (o2 < K) {
          w = S.kd[S.org[o2]] + S.tau[o2];
        } else {
          int cnt = o2 - K, c = 0;
          for (c = 0; c < n; ++c)
            if (S.defl[c] && cnt-- == 0) break;
          w = S.sd[c];
        }
        if (w < v || (w == v && o2 < it)) ++r;
      }
      S.src[r] = item;
      lamOut[r] = neg ? -v : v;
    }
  }
  __syncthreads();
  // --- eigenvectors for this CTA's block of output columns
  int elo, ehi;
  block_range(n, C, rank, elo, ehi);
  double* v = S.vscr[warp];
  for (int e = elo + warp; e < ehi; e += NW) {
    const int item = S.src[e];
    for (int c = lane; c < n; c += 32) v[c] = 0.0;
    __syncwarp();
    if (item < K) {
      const double dj = S.kd[S.org[item]], tj = S.tau[item];
      double nn = 0;
      for (int t = lane; t < K; t += 32) {
        const double y = S.zhat[t] / ((S.kd[t] - dj) - tj);
        v[S.kidx[t]] = y;
        nn += y * y;
      }
      nn = warp_sum(nn);
      const double inv = 1.0 / sqrt(nn);
      __syncwarp();
      for (int c = lane; c < n; c += 32) v[c] *= inv;
    } else if (lane == 0) {
      v[item - K] = 1.0;
    }
    __syncwarp();
    if (lane == 0)
      for (int r = S.nrot - 1; r >= 0; --r) {
        const int p = S.rot_p[r], q = S.rot_q[r];
        const double cc = S.rot_c[r], ss = S.rot_s[r];
        const double yp = v[p], yq = v[q];
        v[p] = cc * yp - ss * yq;
        v[q] = ss * yp + cc * yq;
      }
    __syncwarp();
    for (int i = lane; i < n; i += 32) QT[(int64_t)e * ldq + i] = v[n - 1 - i];
    __syncwarp();
  }
  __syncthreads();
}

// --------------------------------------------------------- graph mutation K9
// Cluster-wide scan of row u for target v: returns the position or -1.
template <int C>
DAMF_D long long find_arc(Smem<C>& S, cg::cluster_group& cl, const DevCSR& g, int64_t u,
                          int64_t v, int slot) {
  const int rank = (int)cl.block_rank();
  const long long cnt = g.cnt[u];
  const int64_t base = g.off[u];
  const long long per = (cnt + C - 1) / C;
  const long long lo = min(cnt, (long long)rank * per), hi = min(cnt, lo + per);
  long long pos = -1;
  for (long long p = lo + threadIdx.x; p < hi; p += NT)
    if (g.ids[base + p] == (int32_t)v) pos = p;
  // block max
  __shared__ long long bmax[NW];
  long long m = pos;
  for (int o = 16; o > 0; o >>= 1) {
    long long x = __shfl_xor_sync(0xffffffffu, m, o);
    m = x > m ? x : m;
  }
  if ((threadIdx.x & 31) == 0) bmax[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < C) {
    long long mm = -1;
    for (int w = 0; w < NW; ++w) mm = bmax[w] > mm ? bmax[w] : mm;
    *cl.map_shared_rank(&S.found[rank][slot], threadIdx.x) = mm;
  }
  cl.sync();
  long long res = -1;
  for (int r = 0; r < C; ++r) res = S.found[r][slot] > res ? S.found[r][slot] : res;
  __syncthreads();
  return res;
}

// Append arc u->v (CTA-uniform call; relocates a full row to the pool top).
template <int C>
DAMF_D bool insert_arc(Smem<C>& S, const DevCSR& g, int64_t u, int32_t v, double w) {
  __syncthreads();
  const int c = g.cnt[u];
  if (c == g.cap[u]) {
    const int ncap = c < 4 ? 8 : 2 * c;
    const int64_t noff = *g.pool_top;
    if (noff + ncap > g.pool_size) return false;
    const int64_t ooff = g.off[u];
    for (int p = threadIdx.x; p < c; p += NT) {
      g.ids[noff + p] = g.ids[ooff + p];
      if (g.wts) g.wts[noff + p] = g.wts[ooff + p];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      g.off[u] = noff;
      g.cap[u] = ncap;
      *g.pool_top = noff + ncap;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int64_t at = g.off[u] + c;
    g.ids[at] = v;
    if (g.wts) g.wts[at] = w;
    g.cnt[u] = c + 1;
  }
  __syncthreads();
  return true;
}

DAMF_D void erase_at(const DevCSR& g, int64_t u, long long pos) {
  const int64_t base = g.off[u];
  const int last = g.cnt[u] - 1;
  g.ids[base + pos] = g.ids[base + last];
  if (g.wts) g.wts[base + pos] = g.wts[base + last];
  g.cnt[u] = last;
}

// ------------------------------------------------------------ rank-1 step
template <int C>
DAMF_D void rank1_step(const EventKernelArgs& A, Smem<C>& S, cg::cluster_group& cl,
                       const StepDesc& st) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)cl.block_rank();
  const int d = A.d;
  const int k = S.k;
  const int n = k + 1;
  const bool edge = st.kind == kStepEdge;
  const int sA = st.kind == kStepNodeRow ? 1 : 0;
  const int sB = 1 - sA;
  float* baseA = sA ? A.Yb : A.Xb;
  float* baseB = sB ? A.Yb : A.Xb;
  const double* PTA = A.PT[sA][S.pp[sA]];
  const double* PTB = A.PT[sB][S.pp[sB]];
  const double* QA = A.Q[sA][S.pp[sA]];
  const double* QB = A.Q[sB][S.pp[sB]];
  const int ld = A.ld;

  // ---- 1. gather (fp64) -------------------------------------------------
  for (int j = tid; j < k; j += NT) {
    double s = 0;
    for (int t = 0; t < st.nb; ++t)
      s += A.sp_vals[st.b_off + t] * (double)baseA[A.sp_rows[st.b_off + t] * (int64_t)d + j];
    S.gA[j] = s;
    S.gB[j] = edge ? st.c_val * (double)baseB[st.c_row * (int64_t)d + j] : 0.0;
    S.sig[j] = A.sigma[j];
  }
  __syncthreads();
  // ---- w = S^-1/2 (g P), this CTA's block of columns --------------------
  {
    int lo, hi;
    block_range(k, C, rank, lo, hi);
    for (int j = lo + warp; j < hi; j += NW) {
      double sa = 0, sb = 0;
      for (int i = lane; i < k; i += 32) {
        sa += S.gA[i] * PTA[(int64_t)j * ld + i];
        if (edge) sb += S.gB[i] * PTB[(int64_t)j * ld + i];
      }
      sa = warp_sum(sa) / sqrt(S.sig[j]);
      sb = warp_sum(sb) / sqrt(S.sig[j]);
      if (lane < C) {
        *cl.map_shared_rank(S.wA + j, lane) = sa;
        *cl.map_shared_rank(S.wB + j, lane) = sb;
      }
    }
  }
  cl.sync();
  // ---- 2. bordered system (redundant per CTA) -----------------------------
  double wa2 = 0, wb2 = 0;
  for (int j = tid; j < k; j += NT) {
    wa2 += S.wA[j] * S.wA[j];
    wb2 += S.wB[j] * S.wB[j];
  }
  wa2 = block_sum(S, wa2);
  wb2 = block_sum(S, wb2);
  const double bnorm = sqrt(st.bnorm2);
  const double RA = sqrt(fmax(0.0, st.bnorm2 - wa2));
  const double rA = fmax(RA, 1e-12 * fmax(1.0, bnorm));  // update_engine.cpp:69-70,154
  const double cnorm2 = st.c_val * st.c_val;
  const double RB = edge ? sqrt(fmax(0.0, cnorm2 - wb2)) : 0.0;
  const double rB = fmax(RB, 1e-12 * fmax(1.0, fabs(st.c_val)));
  bool allow_grow;
  if (edge)  // update_engine.cpp:167-170
    allow_grow = k < d && k < min(A.ctl->rows_x, A.ctl->rows_y) &&
                 RA >= 1e-6 * fmax(1.0, bnorm) && RB >= 1e-6 * fmax(1.0, fabs(st.c_val));
  else  // update_engine.cpp:79-81
    allow_grow = k < d && (long long)k < min(st.n_a, st.n_b + 1) && RA >= 1e-6 * fmax(1.0, bnorm);
  double lp = 1.0, lm = 0.0;
  if (edge) {
    double beta = 0;
    for (int j = tid; j < k; j += NT) beta += S.wB[j] * S.wB[j];
    beta = block_sum(S, beta) + rB * rB;
    const double sq = sqrt(beta * beta + 4.0);
    lp = 0.5 * (beta + sq);
    lm = -2.0 / (beta + sq);
  }
  const double np_ = 1.0 / sqrt(lp * lp + 1.0), nm_ = 1.0 / sqrt(lm * lm + 1.0);
  for (int i = tid; i < n; i += NT) {
    const double Di = i < k ? S.sig[i] : 0.0;
    const double ai = i < k ? S.wA[i] : rA;
    const double bi = i < k ? S.wB[i] : rB;
    S.Dg[i] = Di;
    S.av[i] = ai;
    S.bv[i] = edge ? bi : (i == k ? 1.0 : 0.0);
    S.dd[i] = Di * Di;
    if (edge) {
      S.zz[i] = (lp * ai + Di * bi) * np_;
      S.um[i] = (lm * ai + Di * bi) * nm_;
    } else {
      S.zz[i] = ai;
    }
  }
  __syncthreads();
  // ---- 3. eigen step A: D^2 + rho z z^T -----------------------------------
  eig_rank1<C>(S, cl, S.dd, S.zz, edge ? lp : 1.0, n, A.ws_Q1T, ld, S.lamA);
  if (!edge) cl.sync();  // node steps read other CTAs' Q1T rows (t -> n-1-t)
  int tlo, thi;
  block_range(n, C, rank, tlo, thi);
  if (edge) {
    // z2 = Q1^T u_minus for this CTA's columns, broadcast
    for (int e = tlo + warp; e < thi; e += NW) {
      double s = 0;
      for (int i = lane; i < n; i += 32) s += A.ws_Q1T[(int64_t)e * ld + i] * S.um[i];
      s = warp_sum(s);
      if (lane < C) *cl.map_shared_rank(S.zz + e, lane) = s;
    }
    cl.sync();
    // ---- eigen step B: Lambda1 + lm z2 z2^T (downdate) ----------------------
    eig_rank1<C>(S, cl, S.lamA, S.zz, lm, n, A.ws_Q2T, ld, S.lamB);
    // E columns (rows of ET) t in block: ET[t] = sum_e Q2T[t][e] Q1T[e]
    rows_gemm<C>(S, A.ws_ET, ld, A.ws_Q2T, ld, A.ws_Q1T, ld, tlo, thi, n, n, nullptr);
  }
  const double* lamF = edge ? S.lamB : S.lamA;
  // final order t (descending): edge t = e; node t = n-1-e
  auto lam_t = [&](int t) { return edge ? lamF[t] : lamF[n - 1 - t]; };
  auto Erow = [&](int t) -> const double* {
    return edge ? A.ws_ET + (int64_t)t * ld : A.ws_Q1T + (int64_t)(n - 1 - t) * ld;
  };
  // ---- truncation (update_engine.cpp:39-52, svd.cpp:37-38) ----------------
  for (int t = tid; t < n; t += NT) S.s2[t] = sqrt(fmax(lam_t(t), 0.0));
  __syncthreads();
  int k2 = allow_grow ? n : k;
  while (k2 > 0 && S.s2[k2 - 1] <= 0.0) --k2;
  const double floor_ = k2 > 0 ? 1e-12 * S.s2[0] : 0.0;
  while (k2 > 0 && S.s2[k2 - 1] < floor_) --k2;
  // ---- 4. per-column H, F, G, ex, ey, partial sums --------------------------
  {
    double* pH = S.vscr[0];  // reuse as accumulators (NW*NPAD doubles, need 2*k)
    for (int i = tid; i < 2 * NPAD; i += NT) pH[i] = 0.0;
    __syncthreads();
    // warp per column t of this CTA (t < k2)
    for (int t = tlo; t < min(thi, k2); ++t) {
      const double* Et = Erow(t);
      const double st_ = S.s2[t], rst = sqrt(st_);
      // aE = a . E_t, bH = b . H_t computed by warp 0..1 then shared
      double aE = 0;
      for (int i = tid; i < n; i += NT) aE += S.av[i] * Et[i];
      aE = block_sum(S, aE);
      double bH = 0;
      for (int i = tid; i < n; i += NT) {
        const double Hi = (S.Dg[i] * Et[i] + S.bv[i] * aE) / st_;
        A.ws_HT[(int64_t)t * ld + i] = Hi;
        bH += S.bv[i] * Hi;
        if (i < k) {
          // F column t (A side): sqrt(sig_i) H_it / sqrt(s_t)
          A.ws_FT[(int64_t)t * ld + i] = sqrt(S.sig[i]) * Hi / rst;
          // G column t (B side)
          A.ws_GT[(int64_t)t * ld + i] =
              edge ? sqrt(S.sig[i]) * Et[i] / rst : Hi * rst / sqrt(S.sig[i]);
        }
      }
      bH = block_sum(S, bH);
      const double dHt = (S.Dg[k] * Et[k] + S.bv[k] * aE) / st_;  // H[k][t]
      const double dEt = Et[k];
      double exv, eyv;
      if (edge) {
        exv = bH / rst;  // (b^T H_t)/sqrt(s_t)
        eyv = aE / rst;  // (a^T E_t)/sqrt(s_t)
      } else {
        exv = dHt / rst;  // H[k][t]/sqrt(s_t)
        eyv = dHt * rst;  // appended row value
      }
      if (tid < C) {
        *cl.map_shared_rank(S.exv + t, tid) = exv;
        *cl.map_shared_rank(S.eyv + t, tid) = eyv;
        *cl.map_shared_rank(S.dH + t, tid) = dHt;
        *cl.map_shared_rank(S.dE + t, tid) = dEt;
      }
      for (int i = tid; i < k; i += NT) {
        pH[i] += A.ws_HT[(int64_t)t * ld + i] * dHt;
        pH[NPAD + i] += Et[i] * dEt;
      }
      __syncthreads();
    }
    // partial sums to every CTA
    for (int x = tid; x < C * k; x += NT) {
      const int r = x / k, i = x % k;
      *cl.map_shared_rank(&S.partH[rank][i], r) = pH[i];
      *cl.map_shared_rank(&S.partE[rank][i], r) = pH[NPAD + i];
    }
  }
  cl.sync();
  double nH = 0, nE = 0;
  for (int t = tid; t < min(k2, k); t += NT) {
    nH += S.dH[t] * S.dH[t];
    nE += S.dE[t] * S.dE[t];
  }
  nH = block_sum(S, nH);
  nE = block_sum(S, nE);
  for (int i = tid; i < k; i += NT) {
    double a = 0, b = 0;
    for (int r = 0; r < C; ++r) {
      a += S.partH[r][i];
      b += S.partE[r][i];
    }
    S.AHdH[i] = a;
    S.AEdE[i] = b;
  }
  __syncthreads();
  const double gH = 1.0 - nH, gE = 1.0 - nE;
  const bool lazy = k2 == k && gH > 1e-10 && (!edge || gE > 1e-10);
  const int npp = 1 - S.pp[sA], nppB = 1 - S.pp[sB];
  double* PTA_n = A.PT[sA][npp];
  double* PTB_n = A.PT[sB][nppB];
  double* QA_n = A.Q[sA][npp];
  double* QB_n = A.Q[sB][nppB];
  if (lazy) {
    // ---- 5. inverse rows and the four GEMMs (this CTA's rows t) -----------
    for (int t = tlo; t < min(thi, k); ++t) {
      const double rst = sqrt(S.s2[t]);
      for (int j = tid; j < k; j += NT) {
        const double ahinv = A.ws_HT[(int64_t)t * ld + j] + S.dH[t] * S.AHdH[j] / gH;
        A.ws_Fi[(int64_t)t * ld + j] = rst * ahinv / sqrt(S.sig[j]);
        if (edge) {
          const double aeinv = Erow(t)[j] + S.dE[t] * S.AEdE[j] / gE;
          A.ws_Gi[(int64_t)t * ld + j] = rst * aeinv / sqrt(S.sig[j]);
        } else {
          A.ws_Gi[(int64_t)t * ld + j] = ahinv * sqrt(S.sig[j]) / rst;
        }
      }
    }
    __syncthreads();
    const int t1 = min(thi, k);
    double fro[4];
    rows_gemm<C>(S, PTA_n, ld, A.ws_FT, ld, PTA, ld, tlo, t1, k, k, &fro[0]);
    rows_gemm<C>(S, QA_n, ld, A.ws_Fi, ld, QA, ld, tlo, t1, k, k, &fro[1]);
    rows_gemm<C>(S, PTB_n, ld, A.ws_GT, ld, PTB, ld, tlo, t1, k, k, &fro[2]);
    rows_gemm<C>(S, QB_n, ld, A.ws_Gi, ld, QB, ld, tlo, t1, k, k, &fro[3]);
    if (tid < C)
      for (int q = 0; q < 4; ++q) *cl.map_shared_rank(&S.pnorm[rank][q], tid) = fro[q];
    cl.sync();
    // ---- 6. row fixes: base[row] += val * (ex Q_new), this CTA's columns ----
    int jlo, jhi;
    block_range(k, C, rank, jlo, jhi);
    for (int j = jlo + tid; j < jhi; j += NT) {
      double ya = 0, yb = 0;
      for (int t = 0; t < k; ++t) {
        ya += S.exv[t] * QA_n[(int64_t)t * ld + j];
        yb += S.eyv[t] * QB_n[(int64_t)t * ld + j];
      }
      for (int q = 0; q < st.nb; ++q) {
        float* r = baseA + A.sp_rows[st.b_off + q] * (int64_t)d + j;
        *r = (float)((double)*r + A.sp_vals[st.b_off + q] * ya);
      }
      if (edge) {
        float* r = baseB + st.c_row * (int64_t)d + j;
        *r = (float)((double)*r + st.c_val * yb);
      } else {
        baseB[st.c_row * (int64_t)d + j] = (float)yb;  // appended row
      }
    }
    if (rank == 0 && tid == 0) {
      // cond(P_X) <= |P_X|_F |P_X^-1|_F (query-transparent rebase policy)
      const int xA = sA == 0;
      double p2 = 0, q2 = 0;
      for (int r = 0; r < C; ++r) {
        p2 += S.pnorm[r][xA ? 0 : 2];
        q2 += S.pnorm[r][xA ? 1 : 3];
      }
      A.ctl->cond_est = sqrt(p2) * sqrt(q2);
      if (A.ctl->cond_est > A.rebase_cond) A.ctl->need_rebase = 1;
    }
    if (rank == 0)
      for (int t = tid; t < k; t += NT) A.sigma[t] = S.s2[t];
    S.pp[sA] = npp;
    S.pp[sB] = nppB;
    if (rank == 0 && tid == 0) {
      A.ctl->pp[sA] = npp;
      A.ctl->pp[sB] = nppB;
      A.ctl->rank1 += 1;
    }
  } else {
    // ---- eager fold (rank change or ill-conditioned step) ------------------
    // T_A = P_A F_top (k x k2), T_B = P_B G_top; stored transposed in the new
    // PT buffers: TT[t][i] = sum_m F[m][t] PT[i][m]... computed as rows of
    // (F^T P^T): TT[t][:] = sum_m FT[t][m] PT[m][:].
    rows_gemm<C>(S, PTA_n, ld, A.ws_FT, ld, PTA, ld, tlo, min(thi, k2), k, k, nullptr);
    rows_gemm<C>(S, PTB_n, ld, A.ws_GT, ld, PTB, ld, tlo, min(thi, k2), k, k, nullptr);
    cl.sync();
    // fold every row of both sides (and Z_b, r_b with the X-side transform)
    const int nmat = A.alpha_is_one ? 2 : 4;
    for (int mat = 0; mat < nmat; ++mat) {
      float* base;
      const double* TT;
      long long rows;
      if (mat == 0) {
        base = baseA;
        TT = PTA_n;
        rows = sA ? A.ctl->rows_y : A.ctl->rows_x;
      } else if (mat == 1) {
        base = baseB;
        TT = PTB_n;
        rows = sB ? A.ctl->rows_y : A.ctl->rows_x;
      } else {
        base = mat == 2 ? A.Zb : A.rb;
        TT = sA == 0 ? PTA_n : PTB_n;
        rows = A.ctl->rows_x;
      }
      double* rowv = S.vscr[warp];
      for (long long r = (long long)rank * NW + warp; r < rows; r += (long long)C * NW) {
        for (int i = lane; i < k; i += 32) rowv[i] = base[r * d + i];
        __syncwarp();
        for (int t = lane; t < k2; t += 32) {
          double s = 0;
          for (int i = 0; i < k; ++i) s += rowv[i] * TT[(int64_t)t * ld + i];
          base[r * d + t] = (float)s;
        }
        for (int t = k2 + lane; t < k; t += 32) base[r * d + t] = 0.0f;
        __syncwarp();
      }
    }
    cl.sync();
    // residual keys of the folded r_b rows (enhancer.cpp:196-206 re-keying)
    if (!A.alpha_is_one) {
      const long long rows = A.ctl->rows_x;
      for (long long r = (long long)rank * NW + warp; r < rows; r += (long long)C * NW) {
        float m = 0.0f;
        for (int t = lane; t < k2; t += 32) m = fmaxf(m, fabsf(A.rb[r * d + t]));
        m = warp_max(m);
        if (lane == 0) A.key[r] = (float)((double)m / fmax(A.deg[r], 1.0));
      }
    }
    // current-coordinate row deltas (types.hpp:101-116 outer products)
    int jlo, jhi;
    block_range(k2, C, rank, jlo, jhi);
    for (int j = jlo + tid; j < jhi; j += NT) {
      for (int q = 0; q < st.nb; ++q) {
        float* r = baseA + A.sp_rows[st.b_off + q] * (int64_t)d + j;
        *r = (float)((double)*r + A.sp_vals[st.b_off + q] * S.exv[j]);
      }
      if (edge) {
        float* r = baseB + st.c_row * (int64_t)d + j;
        *r = (float)((double)*r + st.c_val * S.eyv[j]);
      } else {
        baseB[st.c_row * (int64_t)d + j] = (float)S.eyv[j];
      }
    }
    // P = Q = I (k2 x k2) in the new buffers
    for (int x = rank * NT + tid; x < k2 * k2; x += C * NT) {
      const int i = x / k2, j = x % k2;
      const double v = i == j ? 1.0 : 0.0;
      PTA_n[(int64_t)i * ld + j] = v;
      PTB_n[(int64_t)i * ld + j] = v;
      QA_n[(int64_t)i * ld + j] = v;
      QB_n[(int64_t)i * ld + j] = v;
    }
    if (rank == 0)
      for (int t = tid; t < k2; t += NT) A.sigma[t] = S.s2[t];
    S.pp[sA] = npp;
    S.pp[sB] = nppB;
    S.k = k2;
    if (rank == 0 && tid == 0) {
      A.ctl->pp[sA] = npp;
      A.ctl->pp[sB] = nppB;
      A.ctl->k = k2;
      A.ctl->rank1 += 1;
      A.ctl->folds += 1;
      A.ctl->cond_est = 1.0;
    }
  }
  // appended rows (node steps)
  if (!edge && rank == 0 && tid == 0) {
    if (sB == 0)
      A.ctl->rows_x += 1;
    else
      A.ctl->rows_y += 1;
  }
  cl.sync();
}

}  // namespace

// ------------------------------------------------------------------ kernel
template <int C>
__global__ void __launch_bounds__(NT, 1) damf_event_kernel(EventKernelArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<C>& S = *reinterpret_cast<Smem<C>*>(smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  if (threadIdx.x == 0) {
    S.k = A.ctl->k;
    S.pp[0] = A.ctl->pp[0];
    S.pp[1] = A.ctl->pp[1];
  }
  __syncthreads();
  for (int64_t e = A.e_begin; e < A.e_end; ++e) {
    if (*(volatile int*)&A.ctl->err) break;
    const EventDesc ev = A.ev[e];
    if (A.t_begin && rank == 0 && threadIdx.x == 0) A.t_begin[e] = globaltimer();
    int err = 0;
    // ---- graph mutation (graph.cpp:83-185) -----------------------------
    if (ev.kind == 1) {  // AddEdge
      const bool two = A.undirected && ev.u != ev.v;
      const long long p1 = find_arc<C>(S, cl, A.out, ev.u, ev.v, 0);
      const long long p2 = two ? find_arc<C>(S, cl, A.out, ev.v, ev.u, 1) : -1;
      if (p1 >= 0 || p2 >= 0) {
        err = 3;  // DuplicateEdge
      } else if (rank == 0) {
        bool ok = insert_arc<C>(S, A.out, ev.u, (int32_t)ev.v, ev.w);
        if (A.directed) ok = ok && insert_arc<C>(S, A.in, ev.v, (int32_t)ev.u, ev.w);
        if (two) ok = ok && insert_arc<C>(S, A.out, ev.v, (int32_t)ev.u, ev.w);
        if (!ok) err = 13;  // TooLarge
        if (threadIdx.x == 0) {
          A.deg[ev.u] += ev.w;
          if (two) A.deg[ev.v] += ev.w;
        }
      }
    } else if (ev.kind == 2) {  // RemoveEdge
      const bool two = A.undirected && ev.u != ev.v;
      const long long p1 = find_arc<C>(S, cl, A.out, ev.u, ev.v, 0);
      const long long p2 = two ? find_arc<C>(S, cl, A.out, ev.v, ev.u, 1) : -1;
      if (p1 < 0) {
        err = 4;  // MissingEdge
      } else {
        long long pi = -1;
        if (A.directed) pi = find_arc<C>(S, cl, A.in, ev.v, ev.u, 0);
        if (rank == 0 && threadIdx.x == 0) {
          const double w1 = A.out.wts ? A.out.wts[A.out.off[ev.u] + p1] : 1.0;
          erase_at(A.out, ev.u, p1);
          A.deg[ev.u] -= w1;
          if (A.directed && pi >= 0) erase_at(A.in, ev.v, pi);
          double w2 = w1;
          if (two && p2 >= 0) {
            w2 = A.out.wts ? A.out.wts[A.out.off[ev.v] + p2] : 1.0;
            erase_at(A.out, ev.v, p2);
            A.deg[ev.v] -= w2;
          }
          // patch the removal weights into the step descriptors (c = -w)
          if (ev.nsteps >= 1) A.steps[ev.step0].c_val = -w1;
          if (ev.nsteps >= 2) A.steps[ev.step0 + 1].c_val = -w2;
        }
      }
    } else if (ev.kind == 0 && rank == 0) {  // AddNode: new id = ev.u
      const int64_t nn = ev.u;
      if (threadIdx.x == 0) {
        const int cap0 = max(8, (int)(2 * (ev.in_cnt + ev.out_cnt)));
        const int64_t off0 = *A.out.pool_top;
        if (off0 + cap0 > A.out.pool_size) {
          err = 13;
        } else {
          A.out.off[nn] = off0;
          A.out.cap[nn] = cap0;
          A.out.cnt[nn] = 0;
          *A.out.pool_top = off0 + cap0;
          A.deg[nn] = 0.0;
          if (A.directed) {
            const int64_t off1 = *A.in.pool_top;
            A.in.off[nn] = off1;
            A.in.cap[nn] = cap0;
            A.in.cnt[nn] = 0;
            *A.in.pool_top = off1 + cap0;
          }
        }
        S.err = err;
      }
      __syncthreads();
      err = S.err;
      bool ok = err == 0;
      for (int64_t t = 0; ok && t < ev.in_cnt; ++t) {
        const int64_t s = A.nb_ids[ev.in_off + t];
        const double w = A.nb_w[ev.in_off + t];
        ok = insert_arc<C>(S, A.out, s, (int32_t)nn, w);
        if (ok && A.directed) ok = insert_arc<C>(S, A.in, nn, (int32_t)s, w);
        if (threadIdx.x == 0) A.deg[s] += w;
      }
      for (int64_t t = 0; ok && t < ev.out_cnt; ++t) {
        const int64_t tt = A.nb_ids[ev.out_off + t];
        const double w = A.nb_w[ev.out_off + t];
        ok = insert_arc<C>(S, A.out, nn, (int32_t)tt, w);
        if (ok && A.directed) ok = insert_arc<C>(S, A.in, tt, (int32_t)nn, w);
        if (threadIdx.x == 0) A.deg[nn] += w;
      }
      if (!ok && err == 0) err = 13;
    }
    // agree on the error across the cluster
    if (threadIdx.x == 0) S.err = err;
    cl.sync();
    if (rank == 0 && threadIdx.x == 0 && S.err) {
      A.ctl->err = S.err;
      A.ctl->err_event = e;
    }
    int any = 0;
    for (int r = 0; r < C; ++r) any |= *cl.map_shared_rank(&S.err, r);
    cl.sync();
    if (any) break;
    // ---- factor update (update_engine.cpp:206-226) ----------------------
    if (!(A.mode & 1)) {
      for (int s = 0; s < ev.nsteps; ++s) {
        const StepDesc st = A.steps[ev.step0 + s];
        rank1_step<C>(A, S, cl, st);
      }
    }
    if (A.t_end && rank == 0 && threadIdx.x == 0) A.t_end[e] = globaltimer();
  }
}

// ------------------------------------------------------------------ launch
template <int C>
static cudaError_t launch_c(const EventKernelArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(Smem<C>);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(damf_event_kernel<C>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (C > 8) {
      e = cudaFuncSetAttribute(damf_event_kernel<C>,
                               cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, damf_event_kernel<C>, a);
}

int event_cluster_size() {
  static int chosen = 0;
  if (chosen) return chosen;
  // Prefer 16 CTAs (non-portable) when the device can co-schedule it.
  int c16 = 0;
  {
    cudaFuncSetAttribute(damf_event_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(Smem<16>));
    cudaFuncSetAttribute(damf_event_kernel<16>,
                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16, 1, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = sizeof(Smem<16>);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&c16, damf_event_kernel<16>, &cfg) != cudaSuccess) c16 = 0;
    cudaGetLastError();
  }
  chosen = c16 > 0 ? 16 : 8;
  return chosen;
}

size_t event_kernel_smem(int C) { return C == 16 ? sizeof(Smem<16>) : sizeof(Smem<8>); }

cudaError_t launch_event_kernel(const EventKernelArgs& a, cudaStream_t s) {
  return event_cluster_size() == 16 ? launch_c<16>(a, s) : launch_c<8>(a, s);
}

}  // namespace dgpu
