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
//      is a secular equation solved root-parallel (one 16-lane group per
//      root) with Gu-Eisenstat z-hat recomputation and LAPACK-style
//      deflation.                                                          K2
//   3. closed forms F = S1^1/2 H S2^-1/2, G = S1^1/2 E S2^-1/2 (edge), the
//      inverses from the orthonormal-column identity
//      A^-1 = A^T + d (A d)^T / (1 - |d|^2), P <- P F and P^-1 <- F^-1 P^-1
//      on the FP64 tensor cores (DMMA m8n8k4), and the row fixes
//      X_b[u] += (ex F^-1) P_old^-1 computed before the new P^-1 exists.     K3
//   4. conditioning bookkeeping for the rebase policy.                     K4
// Rank growth, shrinkage or an ill-conditioned F fold eagerly (X_b <- X_b P F)
// exactly like factor_state.cpp:168-192.
//
// Data placement (what drives the latency): a cluster barrier costs ~400
// cycles but ~1800 when global stores are pending (the release drains them),
// so only the matrices every CTA needs (Q1^T, the new P^T and P^-1, touched
// rows) go through L2; each CTA's owned rows of Q2^T, E, H, F, G, F^-1, G^-1
// stay in its shared memory, and small vectors move over DSMEM.
// Ownership: CTA r owns output index t in [r*ceil(k/C), ...) of [0,k); the
// discarded (k+1)-th direction belongs to the last CTA.
#include <cooperative_groups.h>

#include <cfloat>

#include "common.cuh"
#include "event_kernel.cuh"
#ifndef DAMF_PROF_RANK
#define DAMF_PROF_RANK 0  // CTA whose clock feeds the phase counters (dev profiling)
#endif
// Phase counters are compiled in only with -DDAMF_PROF=1 (tools/prof_cfg5.py,
// tools/prof_events.py): they accumulate in shared memory (a global
// read-modify-write per phase would sit in front of every cluster barrier's
// release) and are flushed to ctl->prof when the kernel ends.
#ifndef DAMF_PROF
#define DAMF_PROF 0
#endif
#if DAMF_PROF
#define DAMF_PROF_PTR(S) (S).lprof
#define DAMF_PROF_ADD(S, slot, v) (S).lprof[slot] += (unsigned long long)(v)
#else
#define DAMF_PROF_PTR(S) nullptr
#define DAMF_PROF_ADD(S, slot, v) (void)0
#endif

namespace cg = cooperative_groups;

namespace dgpu {

namespace {

constexpr int NT = kEventThreads;  // 256 threads per CTA
constexpr int NW = NT / 32;
constexpr int NMAX = kMaxD + 1;    // k + 1 <= 257
constexpr int NPAD = kMaxD + 4;
constexpr double EPS = DBL_EPSILON;
constexpr int PLD = 132;           // private-matrix row stride (d <= 128 in smem)
#ifndef DAMF_GEMM_KU
#define DAMF_GEMM_KU 8
#endif
constexpr int PCAP = 2048;         // fused-PPR candidate list entries kept in shared memory
constexpr int GBUF_D = 4224;       // GEMM staging slot: 32 rows x 132 doubles (33 KB)

// One row GEMM of a staged call: Out[o0 + r][:] = Coef[r][:] In (see rows_gemm_staged).
struct GemmJob {
  double* Out;
  const double* Coef;
  const double* In;
  double* fro;
};

template <int C>
struct Smem {
  static constexpr int PROWS = (128 + C - 1) / C + 1;  // owned rows (+ the discarded one)
  // small vectors (fp64)
  double sig[NPAD], gA[NPAD], gB[NPAD], wA[NPAD], wB[NPAD];
  double av[NPAD], bv[NPAD], Dg[NPAD], dd[NPAD], zz[NPAD], um[NPAD];
  double sd[NPAD], sz[NPAD], kd[NPAD], kz[NPAD], kz2[NPAD];
  int kidx[NPAD], defl[NPAD], src[NPAD], org[NPAD];
  double tau[NPAD], zhat[NPAD], lamA[NPAD], lamB[NPAD];
  double s2[NPAD], exv[NPAD], eyv[NPAD], dH[NPAD], dE[NPAD];
  double cH[NPAD], cE[NPAD], yA1[NPAD], yB1[NPAD];  // dropped columns of H / E (top k)
  // sqrt(sigma_i), 1/sqrt(sigma_i) of the old spectrum and sqrt(s_t), 1/sqrt(s_t)
  // of the new one, computed once per step (every closed form scales by them;
  // an IEEE sqrt / division is ~100-130 dependent cycles on this chip)
  double rsig[NPAD], irsig[NPAD], rs2[NPAD], irs2[NPAD];
  int rot_p[NPAD], rot_q[NPAD];
  double rot_c[NPAD], rot_s[NPAD];
  double partL[2][kMaxD];         // this CTA's partial column sums
  double partS[4];                // this CTA's partial scalars
  double pnorm[C][4];
  double priv[4][PROWS * PLD];    // owned rows of Q2T/F, E/G^-1, H/F^-1, G
  double bred[NW];
  long long found[C][2];          // graph row-scan results
  int lcnt3[3];                   // fused PPR: rows in this CTA's candidate lists (round mod 3)
  // The fused-PPR candidate lists live only inside an event's push and the
  // GEMM staging ring only inside the factor update: one region serves both
  // (keeps the carve-out small enough to leave L1 for the push's row reads)
  union alignas(16) {
    int plist[3][PCAP];           // fused PPR: candidate lists (round mod 3); overflow in global
    double gbuf[2][GBUF_D];       // GEMM operand staging: two slots of chunk rows x ld doubles
    double vscr[NW][NPAD];        // per-warp row scratch (deflation rotations, eager folds)
  };
  int K, nrot, need, heavy;
  int pf_stage;                   // side-job request for the CTA without roots (prefetch_next_event)
  long long pf_e;                 // ... the event it looks ahead to
  int k, pp[2];
  int err;
  unsigned long long gbar[2];     // GEMM staging: bulk-copy completion per slot
  unsigned gq[2];                 // completed phases per slot
  GemmJob gjobs[4];               // the staged GEMM's job list (uniform reads from shared memory)
  double gfro[4];                 // ... and its Frobenius norms
  long long gprof[8];             // DAMF_PROF: staged-GEMM wait / DMMA / call / prologue / bar / issue / epilogue / tail
#if DAMF_PROF
  unsigned long long lprof[128];  // phase counters of this CTA (flushed at kernel end)
  unsigned long long tlog[64][4]; // %globaltimer: roots begin, group 0 done, CTA done (arrive), barrier release
  int tlog_n;
#endif
};
static_assert(sizeof(Smem<16>) <= 232448, "event kernel shared memory above the 227 KB opt-in limit");

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

// 16-lane group reductions (xor butterfly: bitwise identical in all lanes)
DAMF_D double gsum(double v, unsigned mask) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, 16);
  return v;
}
DAMF_D double gprod(double v, unsigned mask) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v *= __shfl_xor_sync(mask, v, o, 16);
  return v;
}

DAMF_D void block_range(int total, int C, int rank, int& lo, int& hi) {
  const int per = (total + C - 1) / C;
  lo = min(total, rank * per);
  hi = min(total, lo + per);
}

// Owned output indices: [r*ceil(k/C), ...) of [0,k); the last CTA also owns
// [k, n) (the (k+1)-th singular direction).
DAMF_D void own_range(int k, int n, int C, int rank, int& lo, int& hi) {
  block_range(k, C, rank, lo, hi);
  if (rank == C - 1) hi = n;
}

template <int C>
DAMF_D long long block_max_ll(Smem<C>& S, long long v) {
  for (int o = 16; o > 0; o >>= 1) {
    const long long x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x > v ? x : v;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) S.bred[threadIdx.x >> 5] = __longlong_as_double(v);
  __syncthreads();
  long long m = -1;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const long long x = __double_as_longlong(S.bred[w]);
    m = x > m ? x : m;
  }
  __syncthreads();
  return m;
}

// ------------------------------------------------------------- row GEMM
// FP64 tensor-core MMA (DMMA): D[8x8] += A[8x4] (row) * B[4x8] (col).
// Fragments (PTX ISA, mma.m8n8k4 .f64): a = A[lane>>2][lane&3],
// b = B[lane&3][lane>>2], d{0,1} = D[lane>>2][2*(lane&3) + {0,1}].
DAMF_D void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Out[o0 + r][j] = sum_m Coef[r][m] In[m][j] for r < nt (<= 16), j < J, m < M.
// Coef rows (local smem or global, stride ldc) feed the A fragments; In is
// streamed from L2 with TP*KU independent loads in flight per lane; each
// warp owns TP 8-column tiles. Returns the Frobenius norm^2 of the block
// (block-reduced) when fro != nullptr.
template <int C>
DAMF_D void rows_gemm16(Smem<C>& S, double* Out, int ldo, int o0, const double* Coef, int ldc,
                        int nt, const double* __restrict__ In, int ldi, int M, int J,
                        double* fro) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int MP = (M + 3) & ~3;
  double frob = 0.0;
  const int ntiles = (J + 7) >> 3;
  const int ar = lane >> 2, ac = lane & 3;
  const int mt = (nt + 7) >> 3;  // m8 tiles (1 or 2)
  constexpr int TP = 2;
  constexpr int KU = DAMF_GEMM_KU;
  for (int tb = warp * TP; tb < ntiles; tb += NW * TP) {
    double d0[TP][2], d1[TP][2];
    int bc[TP];
    bool bok[TP];
#pragma unroll
    for (int p = 0; p < TP; ++p) {
      bc[p] = ((tb + p) << 3) + (lane >> 2);
      bok[p] = (tb + p) < ntiles && bc[p] < J;
      d0[p][0] = d1[p][0] = d0[p][1] = d1[p][1] = 0.0;
    }
    for (int k0 = 0; k0 < MP; k0 += 4 * KU) {
      double b[TP][KU];
#pragma unroll
      for (int q = 0; q < KU; ++q)
#pragma unroll
        for (int p = 0; p < TP; ++p) {
          const int m = k0 + 4 * q + ac;
          b[p][q] = (bok[p] && m < M) ? In[(int64_t)m * ldi + bc[p]] : 0.0;
        }
#pragma unroll
      for (int q = 0; q < KU; ++q) {
        const int m = k0 + 4 * q + ac;
        if (k0 + 4 * q >= MP) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h >= mt) break;
          const int r = 8 * h + ar;
          const double a = (r < nt && m < M) ? Coef[(int64_t)r * ldc + m] : 0.0;
#pragma unroll
          for (int p = 0; p < TP; ++p) dmma(d0[p][h], d1[p][h], a, b[p][q]);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < TP; ++p) {
      const int col = ((tb + p) << 3) + 2 * ac;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 8 * h + ar;
        if (h < mt && r < nt && (tb + p) < ntiles) {
          if (col < J) {
            Out[(int64_t)(o0 + r) * ldo + col] = d0[p][h];
            frob += d0[p][h] * d0[p][h];
          }
          if (col + 1 < J) {
            Out[(int64_t)(o0 + r) * ldo + col + 1] = d1[p][h];
            frob += d1[p][h] * d1[p][h];
          }
        }
      }
    }
  }
  if (fro) *fro = block_sum(S, frob);
  __syncthreads();
}

template <int C>
DAMF_D void rows_gemm(Smem<C>& S, double* Out, int ldo, int o0, const double* Coef, int ldc,
                      int nt, const double* __restrict__ In, int ldi, int M, int J, double* fro) {
  double total = 0.0;
  for (int c = 0; c < nt; c += 16) {
    double f = 0.0;
    rows_gemm16<C>(S, Out, ldo, o0 + c, Coef + (int64_t)c * ldc, ldc, min(16, nt - c), In, ldi,
                   M, J, fro ? &f : nullptr);
    total += f;
  }
  if (fro) *fro = total;
}

// Several row GEMMs with the same shapes, Out_j[o0 + r][:] = Coef_j[r][:] In_j,
// with In_j streamed through shared memory instead of per-lane L2 loads:
// thread 0 bulk-copies chunks of CR rows (contiguous, rows x ldi doubles) of
// In_0, In_1, ... into a two-slot ring (cp.async.bulk + mbarrier), so the
// copy of the next chunk -- also across GEMMs -- overlaps the DMMAs of this
// one and each GEMM pays one L2 latency instead of one per K-chunk per warp.
// nt <= 8 * MT rows, J <= 64 * TPW columns (8 warps x TPW 8-column tiles).

DAMF_D unsigned ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
DAMF_D void mbar_wait_parity(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "GW_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra GW_WAIT;\n\t}" ::"r"((unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}
template <int C>
DAMF_D void stage_chunk(Smem<C>& S, int slot, const double* src, unsigned bytes) {
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&S.gbar[slot]);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (unsigned)__cvta_generic_to_shared(S.gbuf[slot])),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// KF > 0: shapes fixed at compile time (M = J = KF, ldi = ldc = KF + 4, the
// k = 128 update GEMMs), so the chunk loops unroll without predicates.
template <int C, int MT, int TPW, int KF>
__device__ __noinline__ void rows_gemm_staged(int nj, int ldo, int o0, int ldc_, int nt, int ldi_,
                                              int M_, int J_) {
  // the block's shared window, re-derived here so that its accesses compile to
  // LDS / STS (a reference parameter of a non-inlined function is generic)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<C>& S = *reinterpret_cast<Smem<C>*>(smem_raw);
  const GemmJob* jobs = S.gjobs;
  const int ldc = KF ? KF + 4 : ldc_, ldi = KF ? KF + 4 : ldi_, M = KF ? KF : M_, J = KF ? KF : J_;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  const int ntiles = (J + 7) >> 3;
  const int CR = min((GBUF_D / ldi) & ~3, (M + 3) & ~3);  // rows per chunk (multiple of 4)
  const int nch = (M + CR - 1) / CR;
  const int T = nj * nch;
  const unsigned q0 = S.gq[0], q1 = S.gq[1];
#if DAMF_PROF
  const long long _gs = clock64();
#endif
  auto issue = [&](int t) {
    const int j = t / nch, c = t % nch;
    const int rows = min(CR, M - c * CR);
    stage_chunk<C>(S, t & 1, jobs[j].In + (int64_t)c * CR * ldi, (unsigned)(rows * ldi * 8));
  };
  if (threadIdx.x == 0) {
    // In was written through the generic proxy (other CTAs, before a cluster
    // barrier): order it before the bulk copies. Once per call -- the fence
    // waits for this thread's outstanding stores, so not once per chunk.
    asm volatile("fence.proxy.async;" ::: "memory");
    issue(0);
    if (T > 1) issue(1);
  }
#if DAMF_PROF
  if (threadIdx.x == 0 && ctarank() == 0) S.gprof[3] += clock64() - _gs;
#endif
  int bc[TPW];
  bool bok[TPW];
#pragma unroll
  for (int p = 0; p < TPW; ++p) {
    const int tb = warp + NW * p;  // this warp's 8-column tiles
    bc[p] = (tb << 3) + (lane >> 2);
    bok[p] = tb < ntiles && bc[p] < J;
  }
  // two accumulator sets (even / odd k-steps): 2 * TPW * MT independent DMMA chains per warp
  double d0[2][TPW][MT], d1[2][TPW][MT];
  double frob = 0.0;
  for (int t = 0; t < T; ++t) {
    const int j = t / nch, c = t % nch;
    if (c == 0) {
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int p = 0; p < TPW; ++p)
#pragma unroll
          for (int h = 0; h < MT; ++h) d0[u][p][h] = d1[u][p][h] = 0.0;
      frob = 0.0;
    }
    const int slot = t & 1;
#if DAMF_PROF
    long long _g0 = clock64();
#endif
    mbar_wait_parity(&S.gbar[slot], ((slot ? q1 : q0) + (t >> 1)) & 1);
#if DAMF_PROF
    long long _g1 = clock64();
    if (threadIdx.x == 0 && ctarank() == 0) S.gprof[0] += _g1 - _g0;
#endif
    const double* sb = S.gbuf[slot];
    // KF: the coefficient rows are this CTA's private rows in shared memory
    const double* Coef = KF ? reinterpret_cast<const double*>(
                                  smem_raw + (reinterpret_cast<const unsigned char*>(jobs[j].Coef) -
                                              reinterpret_cast<const unsigned char*>(&S)))
                            : jobs[j].Coef;
    const int m0 = c * CR, rows = (KF && KF % CR == 0) ? CR : min(CR, M - m0);
    for (int mm = 0; mm < rows; mm += 16) {
      // operands of four k-steps loaded before their DMMAs
      double a[4][MT], b[4][TPW];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int mr = mm + 4 * u + ac;
        const bool mok = mr < rows;
#pragma unroll
        for (int h = 0; h < MT; ++h) {
          const int r = 8 * h + ar;
          a[u][h] = (r < nt && mok) ? Coef[(int64_t)r * ldc + m0 + mr] : 0.0;
        }
#pragma unroll
        for (int p = 0; p < TPW; ++p) b[u][p] = (bok[p] && mok) ? sb[mr * ldi + bc[p]] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int p = 0; p < TPW; ++p)
#pragma unroll
          for (int h = 0; h < MT; ++h) dmma(d0[u & 1][p][h], d1[u & 1][p][h], a[u][h], b[u][p]);
    }
#if DAMF_PROF
    long long _g2 = clock64();
    if (threadIdx.x == 0 && ctarank() == 0) S.gprof[1] += _g2 - _g1;
#endif
    __syncthreads();  // every warp is done with this slot
#if DAMF_PROF
    long long _g3 = clock64();
    if (threadIdx.x == 0 && ctarank() == 0) S.gprof[4] += _g3 - _g2;
#endif

    if (threadIdx.x == 0 && t + 2 < T) issue(t + 2);
#if DAMF_PROF
    long long _g4 = clock64();
    if (threadIdx.x == 0 && ctarank() == 0) S.gprof[5] += _g4 - _g3;
#endif
    if (c == nch - 1) {
      double* Out = jobs[j].Out;
#pragma unroll
      for (int p = 0; p < TPW; ++p) {
        const int tb = warp + NW * p;
        const int col = (tb << 3) + 2 * ac;
#pragma unroll
        for (int h = 0; h < MT; ++h) {
          const int r = 8 * h + ar;
          const double v0 = d0[0][p][h] + d0[1][p][h], v1 = d1[0][p][h] + d1[1][p][h];
          if (r < nt && tb < ntiles) {
            if (col < J) {
              Out[(int64_t)(o0 + r) * ldo + col] = v0;
              frob += v0 * v0;
            }
            if (col + 1 < J) {
              Out[(int64_t)(o0 + r) * ldo + col + 1] = v1;
              frob += v1 * v1;
            }
          }
        }
      }
      if (jobs[j].fro) S.gfro[j] = block_sum(S, frob);
    }
#if DAMF_PROF
    if (threadIdx.x == 0 && ctarank() == 0) S.gprof[6] += clock64() - _g4;
#endif
  }
#if DAMF_PROF
  const long long _g5 = clock64();
#endif
  __syncthreads();
  if (threadIdx.x == 0) {
    S.gq[0] = q0 + (unsigned)((T + 1) >> 1);
    S.gq[1] = q1 + (unsigned)(T >> 1);
  }
  __syncthreads();
#if DAMF_PROF
  if (threadIdx.x == 0 && ctarank() == 0) {
    S.gprof[2] += clock64() - _gs;
    S.gprof[7] += clock64() - _g5;
  }
#endif
}

// Dispatch: the staged form when the shapes fit it, else one rows_gemm each.
template <int C>
DAMF_D void rows_gemms(Smem<C>& S, const GemmJob* jobs, int nj, int ldo, int o0, int ldc, int nt,
                       int ldi, int M, int J) {
  if (nt > 16 || J > 256) {
    for (int j = 0; j < nj; ++j)
      rows_gemm<C>(S, jobs[j].Out, ldo, o0, jobs[j].Coef, ldc, nt, jobs[j].In, ldi, M, J, jobs[j].fro);
    return;
  }
  if (threadIdx.x < nj) S.gjobs[threadIdx.x] = jobs[threadIdx.x];
  __syncthreads();
  if (nt <= 8 && M == 128 && J == 128 && ldi == 132 && ldc == 132 &&
      jobs[0].Coef >= &S.priv[0][0] && jobs[0].Coef < &S.priv[4][0])
    rows_gemm_staged<C, 1, 2, 128>(nj, ldo, o0, ldc, nt, ldi, M, J);
  else if (nt <= 8 && J <= 128)
    rows_gemm_staged<C, 1, 2, 0>(nj, ldo, o0, ldc, nt, ldi, M, J);
  else if (nt <= 16 && J <= 128)
    rows_gemm_staged<C, 2, 2, 0>(nj, ldo, o0, ldc, nt, ldi, M, J);
  else
    rows_gemm_staged<C, 2, 4, 0>(nj, ldo, o0, ldc, nt, ldi, M, J);
  // (the staged call ends with a block barrier: gfro is complete)
  for (int j = 0; j < nj; ++j)
    if (jobs[j].fro) *jobs[j].fro = S.gfro[j];
}

// ---------------------------------------------- exact inverse (one CTA)
// Q = P^-1 (row-major, ld) for P given transposed (PT[j][i] = P[i][j]):
// Gauss-Jordan with partial pivoting in place in Q, pivot row and column
// factors staged in shared memory (prow, fcol, perm: >= k doubles each).
// Used for the rare steps whose kept block is numerically singular (|h| <=
// 1e-12, see rank1_step) or whose H column k is unreliable; returns false if
// P is singular.
DAMF_D bool gj_inverse_cta(const double* PT, double* Q, int k, int ld, double* prow, double* fcol,
                           double* perm, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int x = tid; x < k * k; x += NT) {
    const int i = x / k, j = x % k;
    Q[(int64_t)i * ld + j] = PT[(int64_t)j * ld + i];
  }
  __syncthreads();
  __shared__ int s_piv;
  __shared__ int s_bad;
  if (tid == 0) s_bad = 0;
  for (int c = 0; c < k; ++c) {
    // pivot: argmax_{r >= c} |W[r][c]|
    double bv = -1.0;
    int br = c;
    for (int r = c + tid; r < k; r += NT) {
      const double v = fabs(Q[(int64_t)r * ld + c]);
      if (v > bv) {
        bv = v;
        br = r;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int orr = __shfl_xor_sync(0xffffffffu, br, o);
      if (ov > bv || (ov == bv && orr < br)) {
        bv = ov;
        br = orr;
      }
    }
    if (lane == 0) {
      red[2 * warp] = bv;
      red[2 * warp + 1] = (double)br;
    }
    __syncthreads();
    if (tid == 0) {
      double b = -1.0;
      int r0 = c;
      for (int w = 0; w < NW; ++w)
        if (red[2 * w] > b) {
          b = red[2 * w];
          r0 = (int)red[2 * w + 1];
        }
      s_piv = r0;
      perm[c] = (double)r0;
      if (!(b > 0.0)) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) return false;
    const int p = s_piv;
    // swap rows c <-> p, stage the pivot row
    for (int j = tid; j < k; j += NT) {
      const double a = Q[(int64_t)c * ld + j], b = Q[(int64_t)p * ld + j];
      prow[j] = b;
      if (p != c) Q[(int64_t)p * ld + j] = a;
    }
    __syncthreads();
    const double ip = 1.0 / prow[c];
    for (int j = tid; j < k; j += NT) {
      const double v = j == c ? ip : prow[j] * ip;
      Q[(int64_t)c * ld + j] = v;
    }
    for (int r = tid; r < k; r += NT) fcol[r] = r == c ? 0.0 : Q[(int64_t)r * ld + c];
    __syncthreads();
    for (int j = tid; j < k; j += NT) prow[j] = j == c ? ip : prow[j] * ip;
    __syncthreads();
    for (int x = tid; x < k * k; x += NT) {
      const int r = x / k, j = x % k;
      if (r == c) continue;
      const double w = j == c ? 0.0 : Q[(int64_t)r * ld + j];
      Q[(int64_t)r * ld + j] = w - fcol[r] * prow[j];
    }
    __syncthreads();
  }
  // undo the row interchanges as column interchanges, last first
  for (int c = k - 1; c >= 0; --c) {
    const int p = (int)perm[c];
    if (p != c)
      for (int i = tid; i < k; i += NT) {
        const double a = Q[(int64_t)i * ld + c];
        Q[(int64_t)i * ld + c] = Q[(int64_t)i * ld + p];
        Q[(int64_t)i * ld + p] = a;
      }
    __syncthreads();
  }
  return true;
}

// ------------------------------------------------------------ secular solver
// Branch-free reciprocal: MUFU.RCP64H seed (about 20 bits) and two Newton
// steps, ~1 ulp. The IEEE division nvcc emits carries a slow-path branch per
// call, which serialises the divisions of a secular pass (one per pole per
// lane, each ~150 cycles of dependent latency); these interleave. The seed
// flushes subnormal inputs to zero, so callers re-run a pass with IEEE
// divisions when its result is not finite (never seen outside tests).
DAMF_D double frcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  return r;
}

// One pass of the secular sums at lambda = dorg + tau over the K poles, by a
// 16-lane group (4 poles per lane in flight): psi = sum_{i<=j} z_i^2 / (d_i -
// lambda), phi = sum_{i>j}, and the derivative sums (all before the rho factor).
template <bool FAST>
DAMF_D void secular_pass(const double* kd, const double* kz2, int K, double dorg, double tau, int j,
                         int gl, unsigned gm, double& psi, double& phi, double& dpsi, double& dphi) {
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  if (FAST && K <= 144) {
    // k = 128 (K = 129 poles, the common case) and below: all of a lane's poles
    // (up to 9) in flight at once -- one load / reciprocal latency per pass
    // instead of one per batch of four -- and two accumulator sets
    double r[9], z[9];
#pragma unroll
    for (int u = 0; u < 9; ++u) {
      const int ii = gl + 16 * u;
      const bool in = ii < K;
      const double den = in ? (kd[ii] - dorg) - tau : 1.0;
      z[u] = in ? kz2[ii] : 0.0;
      r[u] = frcp(den);
    }
    double b0 = 0, b1 = 0, b2 = 0, b3 = 0;
#pragma unroll
    for (int u = 0; u < 9; ++u) {
      const double t = z[u] * r[u], dt = t * r[u];
      const bool left = gl + 16 * u <= j;
      if (u & 1) {
        b0 += left ? t : 0.0;
        b1 += left ? 0.0 : t;
        b2 += left ? dt : 0.0;
        b3 += left ? 0.0 : dt;
      } else {
        a0 += left ? t : 0.0;
        a1 += left ? 0.0 : t;
        a2 += left ? dt : 0.0;
        a3 += left ? 0.0 : dt;
      }
    }
    a0 += b0;
    a1 += b1;
    a2 += b2;
    a3 += b3;
  } else {
  int i = gl;
  for (; i + 48 < K; i += 64) {
    double r[4], z[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double den = (kd[i + 16 * u] - dorg) - tau;
      z[u] = kz2[i + 16 * u];
      r[u] = FAST ? frcp(den) : 1.0 / den;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double t = z[u] * r[u], dt = t * r[u];
      const bool left = i + 16 * u <= j;
      a0 += left ? t : 0.0;
      a1 += left ? 0.0 : t;
      a2 += left ? dt : 0.0;
      a3 += left ? 0.0 : dt;
    }
  }
  {
    // tail: up to 4 more poles per lane, the same way with a guard
    double r[4], z[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int ii = i + 16 * u;
      const bool in = ii < K;
      const double den = in ? (kd[ii] - dorg) - tau : 1.0;
      z[u] = in ? kz2[ii] : 0.0;
      r[u] = FAST ? frcp(den) : 1.0 / den;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double t = z[u] * r[u], dt = t * r[u];
      const bool left = i + 16 * u <= j;
      a0 += left ? t : 0.0;
      a1 += left ? 0.0 : t;
      a2 += left ? dt : 0.0;
      a3 += left ? 0.0 : dt;
    }
  }
  }
  // four butterflies interleaved (independent shuffle chains)
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    const double b0 = __shfl_xor_sync(gm, a0, o, 16), b1 = __shfl_xor_sync(gm, a1, o, 16);
    const double b2 = __shfl_xor_sync(gm, a2, o, 16), b3 = __shfl_xor_sync(gm, a3, o, 16);
    a0 += b0;
    a1 += b1;
    a2 += b2;
    a3 += b3;
  }
  psi = a0;
  phi = a1;
  dpsi = a2;
  dphi = a3;
}

// The IEEE-division fallback, out of line (cold).
__device__ __noinline__ void secular_pass_ieee(const double* kd, const double* kz2, int K, double dorg,
                                               double tau, int j, int gl, unsigned gm, double& psi,
                                               double& phi, double& dpsi, double& dphi) {
  secular_pass<false>(kd, kz2, K, dorg, tau, j, gl, gm, psi, phi, dpsi, dphi);
}

// Root in (L, U) of the three-pole model c + sa/(pa-x) + sb/(pb-x) + sh/(ph-x)
// with pa <= L < U <= pb and ph outside [pa, pb]: safeguarded Newton on
// G(x) = F(x) (pa-x)(pb-x), which is smooth on the bracket and decreasing
// through its only zero there. Scalar work (every lane the same); a model
// step only, so a loose tolerance.
DAMF_D double solve3(double c, double pa, double sa, double pb, double sb, double ph, double sh,
                     double L, double U, double x0) {
  // ... cleared of its third pole as well: the cubic
  //   Q(x) = (c (ph-x) + sh)(pa-x)(pb-x) + (ph-x)(sa (pb-x) + sb (pa-x)) = G(x) (ph-x),
  // so an iteration is a handful of dependent FMAs and one reciprocal (the
  // rational form needed two); ph - x keeps its sign on the bracket
  const double sgn = ph > U ? 1.0 : -1.0;
  double lo = L, hi = U;
  double x = (x0 >= L && x0 <= U) ? x0 : 0.5 * (L + U);
#pragma unroll 1
  for (int it = 0; it < 8; ++it) {
    const double a = pa - x, b = pb - x, hh = ph - x;
    const double B = fma(c, hh, sh), ab = a * b, m = fma(sa, b, sb * a);
    const double q = fma(B, ab, hh * m);
    const double dq = -(fma(c, ab, B * (a + b)) + fma(hh, sa + sb, m));
    const double g = sgn * q;
    if (g > 0.0)
      lo = fmax(lo, x);
    else if (g < 0.0)
      hi = fmin(hi, x);
    else
      return x;
    double xn = dq != 0.0 ? x - q * frcp(dq) : 0.5 * (lo + hi);
    if (!(xn > lo && xn < hi)) xn = 0.5 * (lo + hi);
    const bool done = fabs(xn - x) <= 1e-8 * fmax(fabs(xn), fabs(x));
    x = xn;
    if (done) break;
  }
  return x;
}

// Root j of 1 + rho * sum_i kz2[i] / (kd[i] - lambda) = 0 (kd ascending,
// rho > 0, sum kz2 <= 1), one 16-lane group. h: index of a pole that holds
// more than half of the weight (or -1). The interval that receives that
// pole's own moved eigenvalue (the zero of 1/rho + z_h^2/(d_h - l) + rest)
// has a root the two-pole model converges to slowly (the background changes
// sign inside the interval; 7 iterations on the config-5 stream); there the
// heavy pole is kept exact in the model, both in the initial guess and in
// the iteration (solve3), which takes it to 1-2 iterations. Returns tau and the origin pole
// o with lambda = kd[o] + tau, so lambda - kd[i] is formed as
// tau - (kd[i]-kd[o]).
DAMF_D int secular_root(const double* kd, const double* kz2, int K, double rho, double irho,
                        double sumz2, int j, int h, double& tau_out, int& org_out) {
  const int gl = threadIdx.x & 15;
  const unsigned gm = 0xFFFFu << (threadIdx.x & 16);
  int o;
  double lo, hi;
  double tau;
  bool use3 = false;
  if (j < K - 1) {
    // f at the midpoint of (d_j, d_j+1) picks the origin pole; the same sum
    // gives LAPACK dlaed4's initial guess: the two nearest poles exact, the
    // other terms frozen at the midpoint (C), i.e. the root of
    // C + z_j^2/(d_j - l) + z_{j+1}^2/(d_{j+1} - l) = 0 (a quadratic); keeps
    // the slow roots (tiny z, root hugging a pole) from starting at the midpoint
    const double del = kd[j + 1] - kd[j], mid = 0.5 * del;
    double ps, ph, d1, d2;
    secular_pass<true>(kd, kz2, K, kd[j], mid, j, gl, gm, ps, ph, d1, d2);
    double s = ps + ph;
    if (!isfinite(s)) {
      secular_pass_ieee(kd, kz2, K, kd[j], mid, j, gl, gm, ps, ph, d1, d2);
      s = ps + ph;
    }
    if (1.0 + rho * s >= 0.0) {
      o = j;
      lo = 0.0;
      hi = mid;
    } else {
      o = j + 1;
      lo = -mid;
      hi = 0.0;
    }
    tau = 0.5 * (lo + hi);
    const double rmid = frcp(mid);
    const double C = irho + s + kz2[j] * rmid - kz2[j + 1] * rmid;
    if (h >= 0 && h != j && h != j + 1) {
      const double C3 = C - kz2[h] * frcp((kd[h] - kd[j]) - mid);
      const double pa = kd[j] - kd[o], pb = kd[j + 1] - kd[o], ph = kd[h] - kd[o];
      use3 = (C3 + kz2[h] * frcp(ph - pa)) * (C3 + kz2[h] * frcp(ph - pb)) < 0.0;
      if (use3) {
        const double g3 = solve3(C3, pa, kz2[j], pb, kz2[j + 1], ph, kz2[h], fmax(lo, pa), fmin(hi, pb), tau);
        if (g3 > lo && g3 < hi) tau = g3;
      }
    }
    double g;
    if (o == j) {
      const double Aq = C * del + kz2[j] + kz2[j + 1], Bq = kz2[j] * del;
      const double sq = sqrt(fabs(Aq * Aq - 4.0 * Bq * C));
      g = Aq > 0.0 ? 2.0 * Bq * frcp(Aq + sq) : (Aq - sq) * frcp(2.0 * C);
    } else {
      const double Aq = C * del - kz2[j] - kz2[j + 1], Bq = kz2[j + 1] * del;
      const double sq = sqrt(fabs(Aq * Aq + 4.0 * Bq * C));
      g = Aq < 0.0 ? 2.0 * Bq * frcp(Aq - sq) : -(Aq + sq) * frcp(2.0 * C);
    }
    if (!use3 && g > lo && g < hi) tau = g;
  } else {
    o = j;
    lo = 0.0;
    hi = rho * sumz2 * (1.0 + 4.0 * EPS);
    tau = 0.5 * (lo + hi);
    if (K >= 2) {
      // last root: the two-pole model at poles K-2 and K-1 with the other
      // terms frozen at tau = 0, i.e. the positive root of
      // C t^2 - (C dl + a + b) t + b dl = 0 (dl = d_{K-2} - d_{K-1} < 0); kept
      // only when it falls inside the bracket (C > 0)
      double sm = 0;
      for (int i = gl; i < K - 2; i += 16) sm += kz2[i] * frcp(kd[i] - kd[K - 1]);
      sm = gsum(sm, gm);
      const double C = irho + sm, dl = kd[K - 2] - kd[K - 1], a = kz2[K - 2], b = kz2[K - 1];
      if (C > 0.0) {
        const double Bm = C * dl + a + b;
        const double sq = sqrt(fmax(Bm * Bm - 4.0 * C * b * dl, 0.0));
        const double g = Bm > 0.0 ? (Bm + sq) / (2.0 * C) : (2.0 * b * dl) / (Bm - sq);
        if (g > lo && g < hi) tau = g;
      }
    }
  }
  const double dorg = kd[o];
  int it = 0;
  for (; it < 120; ++it) {
    double psi, phi, dpsi, dphi;
    secular_pass<true>(kd, kz2, K, dorg, tau, j, gl, gm, psi, phi, dpsi, dphi);
    if (!isfinite(psi + phi + dpsi + dphi))
      secular_pass_ieee(kd, kz2, K, dorg, tau, j, gl, gm, psi, phi, dpsi, dphi);
    // poles at or below the root contribute negative terms, poles above it
    // positive ones: sum |t| = phi - psi
    const double aerr = rho * (phi - psi);
    psi *= rho;
    phi *= rho;
    dpsi *= rho;
    dphi *= rho;
    const double f = 1.0 + psi + phi;
    if (f < 0.0)
      lo = fmax(lo, tau);
    else
      hi = fmin(hi, tau);
    if (fabs(f) <= 4.0 * EPS * K * (1.0 + aerr)) break;
    const double D1 = (kd[j] - dorg) - tau;
    double nt;
    bool ok = false;
    if (use3) {
      // heavy pole exact, the rest of each side interpolated at its nearest pole
      const double Dh = (kd[h] - dorg) - tau, rh = frcp(Dh), sh = rho * kz2[h];
      const double th = sh * rh, dth = th * rh;
      if (h <= j) {
        psi -= th;
        dpsi -= dth;
      } else {
        phi -= th;
        dphi -= dth;
      }
      const double D2 = (kd[j + 1] - dorg) - tau;
      const double q1 = dpsi * D1 * D1, q2 = dphi * D2 * D2;
      const double c = 1.0 + psi - dpsi * D1 + phi - dphi * D2;
      nt = tau + solve3(c, D1, q1, D2, q2, Dh, sh, fmax(lo - tau, D1), fmin(hi - tau, D2), 0.0);
      ok = true;
    } else if (j < K - 1) {
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
          nt = tau + 2.0 * Cq * frcp(den);  // (a model step: 1 ulp of the quotient is immaterial)
          ok = true;
        }
      }
    } else {
      // last root: Newton on 1/P with P = 1 - f = -(psi + phi) > 0 -- exact
      // for a single pole at any position, so it also converges fast when the
      // weight sits in a cluster of poles below the last one (the cfg-5
      // spectrum after many unit insertions), where a model anchored at the
      // last pole creeps in linearly
      const double P = -(psi + phi), dP = dpsi + dphi;
      if (P > 0.0 && dP > 0.0) {
        nt = tau + (P * P - P) * frcp(dP);
        ok = true;
      }
    }
    if (!ok || !(nt > lo && nt < hi)) {
      // safeguard: bisect, geometrically when the bracket spans many decades
      // of distance from the origin pole (a root hugging it), else in value
      const bool pos = hi > 0.0;
      const double a = fmax(pos ? lo : -hi, 4.0 * EPS * fmax(fabs(dorg), 1e-300)), b = pos ? hi : -lo;
      nt = b > 1e9 * a ? (pos ? sqrt(a * b) : -sqrt(a * b)) : 0.5 * (lo + hi);
    }
    if (nt == tau || hi - lo <= 2.0 * EPS * fmax(fabs(lo), fabs(hi))) {
      tau = nt;
      break;
    }
    tau = nt;
  }
  tau_out = tau;
  org_out = o;
  return it;
}

// ---- look-ahead (side job of a CTA that owns no root in a step's first solve)
// The next event's descriptors, graph rows and base rows are first touched
// on the critical path otherwise (EventDesc / StepDesc reads, the duplicate
// scan, the gather: one to three dependent DRAM latencies each). With K = 129
// roots over 16 CTAs the last CTA has none and waits ~3 us at the barrier
// after the roots; its warp 0 spends that wait pulling the next event's lines
// into L2. Stage 1 (first step of event e): everything addressable from the
// next event's (u, v). Stage 2 (second step, ~80 us later, stage 1's lines
// resident): the dependent part -- the adjacency lists behind off[u] and the
// fp64 side-table rows behind slot[side][row]. Prefetches only: no data is
// consumed, so an event that fails or rebases in between costs nothing.
DAMF_D void pf_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
DAMF_D void pf_l2_span(const void* p, int bytes, int lane0, int lane) {
  // lanes lane0, lane0 + 1, ... take one 128-byte line each
  const char* b = reinterpret_cast<const char*>(p);
  const int i = lane - lane0;
  if (i >= 0 && i * 128 < bytes + 127) pf_l2(b + i * 128);
}
template <int C>
DAMF_D void prefetch_next_event(const EventKernelArgs& A, Smem<C>& S) {
  const int lane = threadIdx.x & 31;
  const int stage = S.pf_stage;
  const int64_t e1 = S.pf_e;
  const EventDesc* evp = A.ev + e1;
  if (stage == 1 && lane == 31 && e1 + 1 < A.e_end) {
    pf_l2(evp + 1);  // the descriptor after it (read by the next look-ahead)
    pf_l2(reinterpret_cast<const char*>(evp + 1) + sizeof(EventDesc) - 1);
  }
  const int kind = evp->kind;
  if (kind != 1 && kind != 2) return;  // edges only
  const int64_t u = evp->u, v = evp->v;
  const int rowb = A.d * 4;
  if (stage == 1) {
    if (lane == 30) {
      pf_l2(A.steps + evp->step0);
      pf_l2(A.steps + evp->step0 + 1);
    }
    const void* direct[12] = {A.out.cnt + u, A.out.off + u, A.out.cap + u, A.deg + u,
                              A.out.cnt + v, A.out.off + v, A.out.cap + v, A.deg + v,
                              A.slot[0] + u, A.slot[1] + v, A.slot[0] + v, A.slot[1] + u};
    if (lane < 12) pf_l2(direct[lane]);
    // base rows X_b[u], Y_b[v] (step 1), X_b[v], Y_b[u] (step 2): 4 lines each up to d = 128
    if (lane >= 12 && lane < 28) {
      const int q = (lane - 12) >> 2, l = (lane - 12) & 3;
      const float* base = (q & 1) ? A.Yb : A.Xb;
      const int64_t row = (q == 0 || q == 3) ? u : v;
      for (int o = l * 128; o < rowb; o += 512) pf_l2(reinterpret_cast<const char*>(base + row * A.d) + o);
    }
  } else {
    if (lane < 2) {
      // adjacency list of u / v (the duplicate / missing-arc scan): first 4 KB
      const int64_t r = lane == 0 ? u : v;
      const int64_t off = A.out.off[r];
      const int bytes = min(A.out.cnt[r], 1024) * 4;
      for (int o = 0; o < bytes; o += 128) pf_l2(reinterpret_cast<const char*>(A.out.ids + off) + o);
    } else if (lane < 6) {
      // fp64 side-table rows
      const int side = lane & 1;
      const int64_t r = (lane == 2 || lane == 5) ? u : v;  // X_b[u], Y_b[v], X_b[v], Y_b[u]
      const int sl = A.slot[side][r];
      if (sl >= 0)
        for (int o = 0; o < A.d * 8; o += 128)
          pf_l2(reinterpret_cast<const char*>(A.rows64[side] + (int64_t)sl * A.ld) + o);
    }
  }
}

// Eigen-decomposition of diag(dd) + rho z z^T over n entries, cluster-wide.
// dd must be descending when rho > 0 and ascending when rho < 0; both map to
// the canonical ascending problem by index reversal (c = n-1-i) and, for
// rho < 0, negation. Outputs the actual eigenvalues in canonical output order
// (lamOut, all CTAs) and eigenvector e as row e of QT (global, ld ldq), for e
// in this CTA's block. Ends WITHOUT a cluster barrier.
template <int C>
DAMF_D void eig_rank1(Smem<C>& S, cg::cluster_group& cl, const double* dd, const double* z,
                      double rho, int n, int elo, int ehi, double* QT, int ldq, int row_off,
                      double* lamOut, unsigned long long* A_prof, double* S_dump = nullptr,
                      const EventKernelArgs* Apf = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)cl.block_rank();
  const bool neg = rho < 0.0;
  long long _pt = clock64();
#define EPROF(slot)                                                        \
  do {                                                                     \
    if (DAMF_PROF && rank == DAMF_PROF_RANK && threadIdx.x == 0) {           \
      const long long _t = clock64();                                      \
      A_prof[slot] += (unsigned long long)(_t - _pt);                      \
      _pt = _t;                                                            \
    }                                                                      \
  } while (0)
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
  EPROF(16);
  const int K = S.K;
#if DAMF_PROF >= 2  // (dump builds only: the extra cluster barrier and global traffic distort the phase timers)
  // dev: dump the first 8 deflated secular problems after a reset
  // (damf_gpu_debug_dump with count < 0): K, rho, sum z^2, kd[K], kz2[K]
  if (S_dump != nullptr) {
    if (rank == 0 && threadIdx.x == 0) {
      const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(S_dump), 1ull);
      S_dump[1] = slot < 8 ? (double)(slot + 1) : 0.0;
      if (slot < 8) {
        double* o = S_dump + 8 + slot * 800;
        o[0] = K; o[1] = rhoN;
        double z2 = 0;
        for (int i = 0; i < K; ++i) { o[8 + i] = S.kd[i]; o[8 + 260 + i] = S.kz2[i]; z2 += S.kz2[i]; }
        o[2] = z2;
      }
    }
    cl.sync();
  }
#endif
  double sz2 = 0;
  for (int j = tid; j < K; j += NT) sz2 += S.kz2[j];
  if (tid == 0) S.heavy = -1;
  sz2 = block_sum(S, sz2);
  // the pole that holds more than half of the weight, if any (at most one)
  for (int j = tid; j < K; j += NT)
    if (S.kz2[j] > 0.5 * sz2) S.heavy = j;
  __syncthreads();
  // --- roots (this CTA's block of K)
  int lo, hi;
  block_range(K, C, rank, lo, hi);
  const int grp = tid >> 4, gl = tid & 15;
  const unsigned gm = 0xFFFFu << (tid & 16);
  constexpr int NG = NT / 16;
  const double irhoN = 1.0 / rhoN;  // (once per solve, not per root)
#if DAMF_PROF
  const long long _r0 = clock64();
  const unsigned long long _t0 = globaltimer();
#endif
  for (int j = lo + grp; j < hi; j += NG) {
    double t;
    int o;
    const int its = secular_root(S.kd, S.kz2, K, rhoN, irhoN, sz2, j, S.heavy, t, o);
#if DAMF_PROF
    const int o_ = o;
#endif
    if (DAMF_PROF && gl == 0 && rank == 0) atomicAdd(&A_prof[13], (unsigned long long)its);
    if (DAMF_PROF && gl == 0 && rank == 0) atomicAdd(&A_prof[14], 1ull);
    if (DAMF_PROF && gl == 0) atomicMax(&A_prof[15], (unsigned long long)its);
    if (DAMF_PROF && gl == 0 && its >= 10) atomicAdd(&A_prof[31], 1ull);
    if (DAMF_PROF && gl == 0) atomicAdd(&A_prof[64 + rank], (unsigned long long)its);
#if DAMF_PROF >= 2
    // dev: record the iteration count of every root of the dumped problems
    if (gl == 0 && S_dump != nullptr) {
      const long long slot = (long long)S_dump[1] - 1;  // this eigensolve's record (set below)
      if (slot >= 0 && slot < 8) S_dump[8 + slot * 800 + 530 + j] = its;
    }
#endif
#if DAMF_PROF
    (void)o_;
#endif
    if (gl < C) {
      *cl.map_shared_rank(S.tau + j, gl) = t;
      *cl.map_shared_rank(S.org + j, gl) = o;
    }
  }
  // (no roots here: look ahead to the next event instead of idling at the barrier)
  if (Apf != nullptr && lo == hi && rank == C - 1 && warp == 0 && S.pf_stage) prefetch_next_event<C>(*Apf, S);
  EPROF(17);
#if DAMF_PROF
  // per-rank: this CTA's root loop (all groups done) and its wait at the barrier
  const unsigned long long _t1 = globaltimer();
  __syncthreads();
  const long long _r1 = clock64();
  const unsigned long long _t2 = globaltimer();
  cl.sync();
  if (threadIdx.x == 0) {
    A_prof[32 + rank] += (unsigned long long)(_r1 - _r0);
    A_prof[48 + rank] += (unsigned long long)(clock64() - _r1);
    if (S.tlog_n < 64) {
      S.tlog[S.tlog_n][0] = _t0;
      S.tlog[S.tlog_n][1] = _t1;
      S.tlog[S.tlog_n][2] = _t2;
      S.tlog[S.tlog_n][3] = globaltimer();
      S.tlog_n += 1;
    }
  }
#else
  cl.sync();
#endif
  EPROF(18);
  // --- Gu-Eisenstat z-hat: zhat_i^2 = prod_j (lam_j - d_i) / prod_{j!=i} (d_j - d_i) / rho
  for (int i = lo + grp; i < hi; i += NG) {
    const double di = S.kd[i];
    double p = 1.0;
    if (K <= 144) {
      // all of a lane's ratios (up to 9) in flight at once, as in secular_pass
      double q[9];
#pragma unroll
      for (int u = 0; u < 9; ++u) {
        const int j = gl + 16 * u;
        const bool in = j < K;
        const double lmd = in ? S.tau[j] - (di - S.kd[S.org[j]]) : 1.0;  // lambda_j - d_i
        q[u] = lmd * frcp(in ? (j == i ? rhoN : S.kd[j] - di) : 1.0);
      }
      p = ((q[0] * q[1]) * (q[2] * q[3])) * ((q[4] * q[5]) * (q[6] * q[7])) * q[8];
    } else
    for (int j0 = gl; j0 < K; j0 += 64) {
      // four ratios in flight per lane (branch-free reciprocals)
      double lmd[4], r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + 16 * u;
        const bool in = j < K;
        lmd[u] = in ? S.tau[j] - (di - S.kd[S.org[j]]) : 1.0;  // lambda_j - d_i
        r[u] = frcp(in ? (j == i ? rhoN : S.kd[j] - di) : 1.0);
      }
      p *= (lmd[0] * r[0]) * (lmd[1] * r[1]) * ((lmd[2] * r[2]) * (lmd[3] * r[3]));
    }
    p = gprod(p, gm);
    const double zh = copysign(sqrt(fmax(p, 0.0)), S.kz[i]);
    if (gl < C) *cl.map_shared_rank(S.zhat + i, gl) = zh;
  }
  EPROF(19);
  cl.sync();
  EPROF(20);
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
  EPROF(21);
  // --- eigenvectors for this CTA's block of output columns
  if (S.nrot == 0) {
    for (int e = elo + grp; e < ehi; e += NG) {
      const int item = S.src[e];
      double* row = QT + (int64_t)(e - row_off) * ldq;
      if (K < n)
        for (int i = gl; i < n; i += 16) row[i] = 0.0;
      __syncwarp(gm);
      if (item < K) {
        const double dj = S.kd[S.org[item]], tj = S.tau[item];
        double nn = 0;
        if (K <= 144) {
          // one pass: the lane's (up to 9) components stay in registers between
          // the norm and the scaled store
          double y[9];
#pragma unroll
          for (int u = 0; u < 9; ++u) {
            const int t = gl + 16 * u;
            const bool in = t < K;
            y[u] = (in ? S.zhat[t] : 0.0) * frcp(in ? (S.kd[t] - dj) - tj : 1.0);
          }
          nn = ((y[0] * y[0] + y[1] * y[1]) + (y[2] * y[2] + y[3] * y[3])) +
               ((y[4] * y[4] + y[5] * y[5]) + (y[6] * y[6] + y[7] * y[7])) + y[8] * y[8];
          const double inv = rsqrt(gsum(nn, gm));
#pragma unroll
          for (int u = 0; u < 9; ++u) {
            const int t = gl + 16 * u;
            if (t < K) row[n - 1 - S.kidx[t]] = y[u] * inv;
          }
          __syncwarp(gm);
          continue;
        }
        for (int t0 = gl; t0 < K; t0 += 64) {
          double y[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int t = t0 + 16 * u;
            const bool in = t < K;
            y[u] = (in ? S.zhat[t] : 0.0) * frcp(in ? (S.kd[t] - dj) - tj : 1.0);
          }
          nn += (y[0] * y[0] + y[1] * y[1]) + (y[2] * y[2] + y[3] * y[3]);
        }
        const double inv = rsqrt(gsum(nn, gm));
        for (int t0 = gl; t0 < K; t0 += 64) {
          double y[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int t = t0 + 16 * u;
            const bool in = t < K;
            y[u] = (in ? S.zhat[t] : 0.0) * frcp(in ? (S.kd[t] - dj) - tj : 1.0);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int t = t0 + 16 * u;
            if (t < K) row[n - 1 - S.kidx[t]] = y[u] * inv;
          }
        }
      } else if (gl == 0) {
        row[n - 1 - (item - K)] = 1.0;
      }
      __syncwarp(gm);
    }
    __syncthreads();
    EPROF(22);
    return;
  }
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
    for (int i = lane; i < n; i += 32) QT[(int64_t)(e - row_off) * ldq + i] = v[n - 1 - i];
    __syncwarp();
  }
  __syncthreads();
  EPROF(22);
}

// --------------------------------------------------------- graph mutation K9
// Cluster-wide scan of row u for target v: returns the position or -1.
template <int C>
DAMF_D long long find_arc(Smem<C>& S, cg::cluster_group& cl, const DevCSR& g, int64_t u,
                          int64_t v, int slot) {
  const int rank = (int)cl.block_rank();
  const long long cnt = g.cnt[u];
  const int64_t base = g.off[u];
  if (cnt <= 4 * NT) {
    // short row: every CTA scans all of it (same answer everywhere), no
    // cluster barrier
    long long pos = -1;
    for (long long p = threadIdx.x; p < cnt; p += NT)
      if (g.ids[base + p] == (int32_t)v) pos = p;
    return block_max_ll<C>(S, pos);
  }
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
#define PROF_MARK(slot)                                                   \
  do {                                                                    \
    if (DAMF_PROF && rank == DAMF_PROF_RANK && threadIdx.x == 0) {        \
      const long long _t = clock64();                                     \
      DAMF_PROF_ADD(S, slot, _t - _pt);                                   \
      _pt = _t;                                                           \
    }                                                                     \
  } while (0)

// ------------------------------------------------------------ rank-1 step
#define PROF_MARK(slot)                                                   \
  do {                                                                    \
    if (DAMF_PROF && rank == DAMF_PROF_RANK && threadIdx.x == 0) {        \
      const long long _t = clock64();                                     \
      DAMF_PROF_ADD(S, slot, _t - _pt);                                   \
      _pt = _t;                                                           \
    }                                                                     \
  } while (0)

// ---- base rows: fp32 storage plus the fp64 side table ----------------------
// Rows written through P^-1 carry components ~cond(P) larger than their
// current value, which fp32 storage would round away; they live in fp64
// (rows64) from their first such write until the next fold, with the fp32
// row kept as a rounded mirror for readers that tolerate it (PPR keys).
DAMF_D double row_val(const EventKernelArgs& A, int side, const float* base, int64_t row, int j) {
  const int sl = A.slot[side][row];
  return sl >= 0 ? A.rows64[side][(int64_t)sl * A.ld + j] : (double)base[row * (int64_t)A.d + j];
}
DAMF_D void row_add(const EventKernelArgs& A, int side, float* base, int64_t row, int j, double delta) {
  const int sl = A.slot[side][row];
  if (sl >= 0) {
    double* p = A.rows64[side] + (int64_t)sl * A.ld + j;
    const double v = *p + delta;
    *p = v;
    base[row * (int64_t)A.d + j] = (float)v;
  } else {
    float* r = base + row * (int64_t)A.d + j;
    *r = (float)((double)*r + delta);
  }
}
DAMF_D void row_set(const EventKernelArgs& A, int side, float* base, int64_t row, int j, double v) {
  const int sl = A.slot[side][row];
  if (sl >= 0) A.rows64[side][(int64_t)sl * A.ld + j] = v;
  base[row * (int64_t)A.d + j] = (float)v;
}
// One warp gives `row` an fp64 slot (initialised from its fp32 value) unless
// it has one; a full table leaves the row in fp32 and requests a rebase.
DAMF_D void row_claim(const EventKernelArgs& A, int side, const float* base, int64_t row) {
  const int lane = threadIdx.x & 31;
  int sl = A.slot[side][row];
  if (sl < 0) {
    long long at = 0;
    if (lane == 0) at = atomicAdd(reinterpret_cast<unsigned long long*>(&A.ctl->dirty_n[side]), 1ull);
    at = __shfl_sync(0xffffffffu, at, 0);
    if (at >= A.dirty_cap) {
      if (lane == 0) A.ctl->need_rebase = 1;
      return;
    }
    for (int j = lane; j < A.d; j += 32)
      A.rows64[side][at * A.ld + j] = (double)base[row * (int64_t)A.d + j];
    if (lane == 0) {
      A.dirty[side][at] = row;
      A.slot[side][row] = (int)at;
    }
  }
}

// Returns false (nothing written) when the bordered system is not finite:
// the reference throws NonFinite from dense_svd_small (svd.cpp:31-32).
template <int C>
DAMF_D bool rank1_step(const EventKernelArgs& A, Smem<C>& S, cg::cluster_group& cl,
                       const StepDesc& st, int64_t ev_index, int64_t step_index) {
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
  long long _pt = clock64();
  // owned output rows and the private (per-CTA) matrices
  int olo, ohi;
  own_range(k, n, C, rank, olo, ohi);
  const int kohi = min(ohi, k);  // owned rows among the kept k
  double* PB[4];
  int pld;
  if (d <= 128) {
    for (int i = 0; i < 4; ++i) PB[i] = S.priv[i];
    pld = PLD;
  } else {
    const int prg = (NMAX + C - 1) / C + 1;
    for (int i = 0; i < 4; ++i) PB[i] = A.ws_priv + ((int64_t)i * C + rank) * prg * ld;
    pld = ld;
  }
  auto prow = [&](int buf, int t) -> double* { return PB[buf] + (int64_t)(t - olo) * pld; };

  // ---- 1. gather (fp64) and w = S^-1/2 (g P), this CTA's columns ---------
  for (int j = tid; j < k; j += NT) {
    double s = 0;
    for (int t = 0; t < st.nb; ++t)
      s += A.sp_vals[st.b_off + t] * row_val(A, sA, baseA, A.sp_rows[st.b_off + t], j);
    S.gA[j] = s;
    S.gB[j] = edge ? st.c_val * row_val(A, sB, baseB, st.c_row, j) : 0.0;
    const double sg = A.sigma[j], rs = sqrt(sg);
    S.sig[j] = sg;
    S.rsig[j] = rs;
    S.irsig[j] = 1.0 / rs;
  }
  __syncthreads();
  {
    int lo, hi;
    block_range(k, C, rank, lo, hi);
    for (int j = lo + warp; j < hi; j += NW) {
      double sa = 0, sb = 0;
      for (int i = lane; i < k; i += 32) {
        sa += S.gA[i] * PTA[(int64_t)j * ld + i];
        if (edge) sb += S.gB[i] * PTB[(int64_t)j * ld + i];
      }
      sa = warp_sum(sa) * S.irsig[j];
      sb = warp_sum(sb) * S.irsig[j];
      if (lane < C) {
        *cl.map_shared_rank(S.wA + j, lane) = sa;
        *cl.map_shared_rank(S.wB + j, lane) = sb;
      }
    }
  }
  cl.sync();  // B1
  // fp64 slots for the rows this step writes (after every CTA's gather; the
  // writes come after B7b): row q of the step is claimed by warp 0 of CTA q % C
  if (warp == 0) {
    for (int q = rank; q <= st.nb; q += C) {
      if (q < st.nb) {
        if (A.sp_vals[st.b_off + q] != 0.0) row_claim(A, sA, baseA, A.sp_rows[st.b_off + q]);
      } else {
        row_claim(A, sB, baseB, st.c_row);
      }
    }
  }
  PROF_MARK(0);
  // ---- 2. bordered system (redundant per CTA) -----------------------------
  double wa2 = 0, wb2 = 0;
  for (int j = tid; j < k; j += NT) {
    wa2 += S.wA[j] * S.wA[j];
    wb2 += S.wB[j] * S.wB[j];
  }
  wa2 = block_sum(S, wa2);
  wb2 = block_sum(S, wb2);
  // M = diag(sigma, 0) + [w_a; r_a][w_b; r_b]^T is finite iff the gathered
  // projections are (sigma > 0 is implied: 1/sqrt(sigma) enters w); the block
  // sums are bit-identical in every CTA, so the cluster agrees on the exit
  if (!isfinite(wa2) || !isfinite(wb2) || !isfinite(st.bnorm2)) {
    if (rank == 0 && tid == 0) {
      A.ctl->err = 7;  // NonFinite
      A.ctl->err_event = ev_index;
    }
    return false;
  }
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
    const double beta = wb2 + rB * rB;
    const double sq = sqrt(beta * beta + 4.0);
    lp = 0.5 * (beta + sq);
    lm = -2.0 / (beta + sq);
  }
  const double np_ = 1.0 / sqrt(lp * lp + 1.0), nm_ = 1.0 / sqrt(lm * lm + 1.0);
  // Entries of the border below 8 eps |M| are set to zero: the same backward
  // perturbation the secular deflation applies to z, made consistent for the
  // closed forms (H = M^T E S^-1, ex, ey). A direction the update does not
  // touch then keeps an exactly zero coupling, and ex / ey come out exactly
  // zero when the reference's SVD leaves them so (the empty dX / dY of
  // types.hpp:101-116, e.g. a node whose base row is numerically zero).
  const double tolM = 8.0 * EPS * fmax(S.sig[0], fmax(bnorm, fabs(st.c_val)));
  for (int i = tid; i < n; i += NT) {
    const double Di = i < k ? S.sig[i] : 0.0;
    double ai = i < k ? S.wA[i] : rA;
    double bi = i < k ? S.wB[i] : rB;
    if (i < k && fabs(ai) <= tolM) ai = 0.0;
    if (i < k && fabs(bi) <= tolM) bi = 0.0;
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
  PROF_MARK(1);
  // ---- 3. eigen step A: D^2 + rho z z^T -> Q1^T rows (L2, shared) ---------
  eig_rank1<C>(S, cl, S.dd, S.zz, edge ? lp : 1.0, n, olo, ohi, A.ws_Q1T, ld, 0, S.lamA,
               DAMF_PROF_PTR(S), DAMF_PROF && d <= 128 ? A.ws_priv : nullptr, &A);
  PROF_MARK(2);
  if (edge) {
    // z2 = Q1^T u_minus for this CTA's columns, broadcast
    for (int e = olo + warp; e < ohi; e += NW) {
      double s = 0;
      for (int i = lane; i < n; i += 32) s += A.ws_Q1T[(int64_t)e * ld + i] * S.um[i];
      s = warp_sum(s);
      if (lane < C) *cl.map_shared_rank(S.zz + e, lane) = s;
    }
  }
  cl.sync();  // B4: Q1^T rows visible (and z2 for edges)
  PROF_MARK(3);
  if (edge) {
    // ---- eigen step B: Lambda1 + lm z2 z2^T -> Q2^T rows (private) ---------
    eig_rank1<C>(S, cl, S.lamA, S.zz, lm, n, olo, ohi, PB[0], pld, olo, S.lamB, DAMF_PROF_PTR(S),
                 DAMF_PROF && d <= 128 ? A.ws_priv : nullptr);
    PROF_MARK(4);
    // E columns t (rows of E^T, private): E^T[t] = sum_e Q2^T[t][e] Q1^T[e]
    {
      // columns [0, n & ~7) on the tensor cores (full 8-column tiles: no
      // third tile group per warp for the one column of the (k+1)-th
      // direction); the last n % 8 columns by warp dot products
      const int jm = n & ~7, nt = ohi - olo;
      const GemmJob job = {PB[1], PB[0], A.ws_Q1T, nullptr};
      rows_gemms<C>(S, &job, 1, pld, 0, pld, nt, ld, n, jm);
      for (int x = warp; x < nt * (n - jm); x += NW) {
        const int r = x / (n - jm), j = jm + x % (n - jm);
        double acc = 0.0;
        for (int e = lane; e < n; e += 32) acc += PB[0][(int64_t)r * pld + e] * A.ws_Q1T[(int64_t)e * ld + j];
        acc = warp_sum(acc);
        if (lane == 0) PB[1][(int64_t)r * pld + j] = acc;
      }
      __syncthreads();
    }
  } else {
    for (int x = tid; x < (ohi - olo) * n; x += NT) {
      const int t = olo + x / n, i = x % n;
      prow(1, t)[i] = A.ws_Q1T[(int64_t)(n - 1 - t) * ld + i];
    }
    __syncthreads();
  }
  PROF_MARK(5);
  const double* lamF = edge ? S.lamB : S.lamA;
  // ---- truncation (update_engine.cpp:39-52, svd.cpp:37-38) ----------------
  // sigma = sqrt(lambda) of M M^T: lambda carries an absolute error of a few
  // eps lambda_max, so singular values below ~sqrt(64 eps) sigma_1 (1.2e-7
  // sigma_1) are indistinguishable from zero here and are treated as zero.
  // The reference's direct SVD resolves them down to its 1e-12 sigma_1 floor
  // (update_engine.cpp:41-44); values in between arise from its in-span
  // clamp (R >= 1e-12, update_engine.cpp:154-155) and contribute < 1.2e-7 of
  // |M| (a documented deviation: the device's rank may then be lower).
  {
    const double lmax = fmax(edge ? lamF[0] : lamF[n - 1], 0.0);
    for (int t = tid; t < n; t += NT) {
      const double l = edge ? lamF[t] : lamF[n - 1 - t];
      const double sv = l > 64.0 * EPS * lmax ? sqrt(l) : 0.0;
      const double rsv = sqrt(sv);
      S.s2[t] = sv;
      S.rs2[t] = rsv;
      S.irs2[t] = sv > 0.0 ? 1.0 / rsv : 0.0;
    }
  }
  __syncthreads();
  int k2 = allow_grow ? n : k;
  while (k2 > 0 && S.s2[k2 - 1] <= 0.0) --k2;
  const double floor_ = k2 > 0 ? 1e-12 * S.s2[0] : 0.0;
  while (k2 > 0 && S.s2[k2 - 1] < floor_) --k2;
  const int tend = min(ohi, k2);
  // ---- 4. per-column H, F, G, ex, ey (one warp per owned column t) --------
  for (int t = olo + warp; t < tend; t += NW) {
    const double* Et = prow(1, t);
    double* Ht = prow(2, t);
    double* Ft = prow(0, t);
    double* Gt = prow(3, t);
    const double rst = S.rs2[t], irst = S.irs2[t], ist = irst * irst;
    double aE = 0;
    for (int i = lane; i < n; i += 32) aE += S.av[i] * Et[i];
    aE = warp_sum(aE);
    double bH = 0;
    for (int i = lane; i < n; i += 32) {
      const double e_i = Et[i];
      const double Hi = (S.Dg[i] * e_i + S.bv[i] * aE) * ist;
      Ht[i] = Hi;
      bH += S.bv[i] * Hi;
      if (i < k) {
        const double rs = S.rsig[i];
        Ft[i] = rs * Hi * irst;                                   // F column t (A side)
        Gt[i] = edge ? rs * e_i * irst : Hi * rst * S.irsig[i];   // G column t (B side)
      }
    }
    bH = warp_sum(bH);
    const double dHt = (S.Dg[k] * Et[k] + S.bv[k] * aE) * ist;  // H[k][t]
    const double dEt = Et[k];
    const double exv = edge ? bH * irst : dHt * irst;   // ex_t
    const double eyv = edge ? aE * irst : dHt * rst;    // ey_t (edge) / appended row (node)
    if (lane < C) {
      *cl.map_shared_rank(S.exv + t, lane) = exv;
      *cl.map_shared_rank(S.eyv + t, lane) = eyv;
      *cl.map_shared_rank(S.dH + t, lane) = dHt;
      *cl.map_shared_rank(S.dE + t, lane) = dEt;
    }
  }
  // The dropped (k+1)-th singular pair, broadcast by its owner (the last CTA):
  // c_H = H[0:k, k], h_H = H[k][k] and (edge) c_E, h_E from E. For the kept
  // k x k block A of an orthogonal (k+1) x (k+1) matrix with bottom row d,
  // A d^T = -c h and 1 - |d|^2 = h^2, so
  //     A^-1 = A^T - d^T c / h
  // whose error grows like 1/|h| = cond(A); the form A^T + d^T (A d^T)^T / (1 - |d|^2)
  // squares it (A d^T is a cancelling sum of size |h|, then divided by h^2).
  // At config 5 the kept block routinely has h ~ 1e-4 (an old direction is
  // dropped for the new one), where the squared form loses 8 digits per step.
  // H's column k = M^T E[:, k] / s_k needs s_k well above zero.
  const bool hk_ok = k2 == k && S.s2[k] > 1e-6 * S.s2[0];
  if (hk_ok && k >= olo && k < ohi) {
    const double* Ek = prow(1, k);
    if (warp == 0) {
      double aEk = 0;
      for (int i = lane; i < n; i += 32) aEk += S.av[i] * Ek[i];
      aEk = warp_sum(aEk);
      if (lane == 0) S.bred[0] = aEk;
    }
    __syncthreads();
    const double aEk = S.bred[0], isk = 1.0 / S.s2[k];
    for (int x = tid; x < C * n; x += NT) {
      const int r = x / n, i = x % n;
      *cl.map_shared_rank(S.cH + i, r) = (S.Dg[i] * Ek[i] + S.bv[i] * aEk) * isk;
      if (edge) *cl.map_shared_rank(S.cE + i, r) = Ek[i];
    }
  }
  __syncthreads();
  // partial column sums over this CTA's kept columns (local smem):
  //  0: sum_t c_t w_t H[i][t]       (row fix, side A: c = ex, w = sqrt(s))
  //  1: sum_t c_t w_t B[i][t]       (row fix, side B: edge c = ey, w = sqrt(s), B = E;
  //                                  node c = vrow, w = 1/sqrt(s), B = H)
  {
    const int tk = min(ohi, k);
    for (int i = tid; i < k; i += NT) {
      double p2 = 0, p3 = 0;
      for (int t = olo; t < tk; ++t) {
        const double Hi = prow(2, t)[i], Ei = prow(1, t)[i];
        const double rs = S.rs2[t];
        p2 += S.exv[t] * rs * Hi;
        p3 += edge ? S.eyv[t] * rs * Ei : S.eyv[t] * S.irs2[t] * Hi;
      }
      S.partL[0][i] = p2;
      S.partL[1][i] = p3;
    }
    if (warp == 0) {
      double q0 = 0, q1 = 0;
      for (int t = olo + lane; t < tk; t += 32) {
        const double rs = S.rs2[t];
        q0 += S.exv[t] * rs * S.dH[t];
        q1 += edge ? S.eyv[t] * rs * S.dE[t] : S.eyv[t] * S.irs2[t] * S.dH[t];
      }
      q0 = warp_sum(q0);
      q1 = warp_sum(q1);
      if (lane == 0) {
        S.partS[0] = q0;
        S.partS[1] = q1;
      }
    }
  }
  cl.sync();  // B7a: partials complete in every CTA
  PROF_MARK(6);
  // reduce-scatter + all-gather over DSMEM: this CTA reduces its block of i
  {
    int lo, hi;
    block_range(k, C, rank, lo, hi);
    const int w = hi - lo;
    for (int x = tid; x < 2 * w; x += NT) {
      const int q = x / w, i = lo + x % w;
      double s = 0;
      for (int r = 0; r < C; ++r) s += *cl.map_shared_rank(&S.partL[q][i], r);
      double* dst = q == 0 ? S.yA1 : S.yB1;
      for (int r = 0; r < C; ++r) *cl.map_shared_rank(dst + i, r) = s;
    }
  }
  double sA_ = 0, sB_ = 0;
  for (int r = 0; r < C; ++r) {
    sA_ += *cl.map_shared_rank(&S.partS[0], r);
    sB_ += *cl.map_shared_rank(&S.partS[1], r);
  }
  cl.sync();  // B7b
  // Modified-row log (DAMF_APPLY_LOG_ROWS): the base rows this step writes,
  // i.e. the row sets of dX = outer(b, ex) and dY = outer(c, ey) / the
  // appended row (types.hpp:101-116: one row per nonzero of b, none when the
  // row vector is exactly zero; update_engine.cpp:93-117,197-202). A growing
  // step has empty dX / dY (update_engine.cpp:98-109,186-196).
  if (A.rowlog && rank == 0 && tid == 0 && k2 <= k) {
    bool exnz = false, eynz = false;
    for (int t = 0; t < k2; ++t) {
      exnz = exnz || S.exv[t] != 0.0;
      eynz = eynz || S.eyv[t] != 0.0;
    }
    auto put = [&](int side, int64_t row) {
      const long long at = A.ctl->rowlog_n++;
      if (at < A.rowlog_cap) {
        A.rowlog[3 * at] = step_index;
        A.rowlog[3 * at + 1] = side;
        A.rowlog[3 * at + 2] = row;
      }
    };
    if (exnz)
      for (int q = 0; q < st.nb; ++q)
        if (A.sp_vals[st.b_off + q] != 0.0) put(sA, A.sp_rows[st.b_off + q]);
    if (eynz && (!edge || st.c_val != 0.0)) put(sB, st.c_row);
  }
  PROF_MARK(7);
  // Closed-form inverses need h well away from 0 (and H's column k, i.e.
  // s_k > 0); otherwise the step stays lazy but P^-1 is recomputed exactly
  // (Gauss-Jordan) and a rebase is requested (the reference folds eagerly
  // when its LU is unreliable, factor_state.cpp:168-177; a rebase is the
  // grid-wide equivalent here). Eager folds remain for rank changes (k2 != k).
  const double hH = hk_ok ? S.cH[k] : 0.0, hE = edge && hk_ok ? S.cE[k] : 1.0;
  // (the stable form's error ~ eps / |h| is what an exact inversion of the
  // ill-conditioned block costs as well; only a numerically singular block,
  // |h| <= 1e-12, where the reference's LU pivot test fails too, needs more:
  // the reference folds eagerly then (factor_state.cpp:168-177). States up to
  // 2^20 rows fold in the cluster (the eager branch below); larger ones take
  // an exact Gauss-Jordan P^-1 and fold over the whole GPU right after the
  // event (a requested rebase).)
  const bool singular_block = k2 == k && !(hk_ok && fabs(hH) > 1e-12 && fabs(hE) > 1e-12);
  const bool small_state = max(A.ctl->rows_x, A.ctl->rows_y) <= (1ll << 20);
  const bool lazy = k2 == k && !(singular_block && small_state);
  const bool exact = lazy && singular_block;
  const int npp = 1 - S.pp[sA], nppB = 1 - S.pp[sB];
  double* PTA_n = A.PT[sA][npp];
  double* PTB_n = A.PT[sB][nppB];
  double* QA_n = A.Q[sA][npp];
  double* QB_n = A.Q[sB][nppB];
  if (lazy) {
    const double ihH = 1.0 / hH, ihE = 1.0 / hE;
    const int fbuf = edge ? 2 : 1, gbuf = edge ? 1 : 2;
    if (!exact) {
    // ---- 5. row fixes from the OLD inverse: y = (ex F^-1) P_old^-1 ----------
    //   ex F^-1 [m] = (1/sqrt(sig_m)) (sum_t ex_t sqrt(s_t) H[m][t]
    //                                  - c_H[m] / h_H * sum_t ex_t sqrt(s_t) dH_t)
    for (int m = tid; m < k; m += NT) {
      const double rsm = S.rsig[m], irsm = S.irsig[m];
      S.yA1[m] = (S.yA1[m] - S.cH[m] * ihH * sA_) * irsm;
      S.yB1[m] = edge ? (S.yB1[m] - S.cE[m] * ihE * sB_) * irsm
                      : (S.yB1[m] - S.cH[m] * ihH * sB_) * rsm;
    }
    __syncthreads();
    {
      int jlo, jhi;
      block_range(k, C, rank, jlo, jhi);
      for (int j = jlo + warp; j < jhi; j += NW) {
        double ya = 0, yb = 0;
        for (int m = lane; m < k; m += 32) {
          ya += S.yA1[m] * QA[(int64_t)m * ld + j];
          yb += S.yB1[m] * QB[(int64_t)m * ld + j];
        }
        ya = warp_sum(ya);
        yb = warp_sum(yb);
        if (lane == 0) {
          for (int q = 0; q < st.nb; ++q)
            row_add(A, sA, baseA, A.sp_rows[st.b_off + q], j, A.sp_vals[st.b_off + q] * ya);
          if (edge)
            row_add(A, sB, baseB, st.c_row, j, st.c_val * yb);
          else
            row_set(A, sB, baseB, st.c_row, j, yb);  // appended row
        }
      }
    }
    // ---- inverse rows (private, in place) ----------------------------------
    //   F^-1[t][m] = sqrt(s_t) (H[m][t] - dH_t c_H[m] / h_H) / sqrt(sig_m)
    //   edge: G^-1[t][m] = sqrt(s_t) (E[m][t] - dE_t c_E[m] / h_E) / sqrt(sig_m)
    //   node: G^-1[t][m] = (H[m][t] - dH_t c_H[m] / h_H) sqrt(sig_m) / sqrt(s_t)
    for (int x = tid; x < (kohi - olo) * k; x += NT) {
      const int t = olo + x / k, m = x % k;
      const double rst = S.rs2[t], rsm = S.rsig[m], irsm = S.irsig[m];
      const double ahinv = prow(2, t)[m] - S.dH[t] * S.cH[m] * ihH;
      double gi;
      if (edge)
        gi = rst * (prow(1, t)[m] - S.dE[t] * S.cE[m] * ihE) * irsm;
      else
        gi = ahinv * rsm * S.irs2[t];
      prow(fbuf, t)[m] = rst * ahinv * irsm;  // edge: over H (read above); node: over E
      prow(gbuf, t)[m] = gi;                 // edge: over E (read above); node: over H
    }
    __syncthreads();
    }  // !exact
    PROF_MARK(8);
    // ---- the four GEMMs on the FP64 tensor cores (owned rows t) -------------
    const int nt = kohi - olo;
    double fro[4] = {0.0, 0.0, 0.0, 0.0};
    {
      const GemmJob jobs[4] = {{PTA_n, prow(0, olo), PTA, &fro[0]},
                               {PTB_n, prow(3, olo), PTB, &fro[2]},
                               {QA_n, prow(fbuf, olo), QA, &fro[1]},
                               {QB_n, prow(gbuf, olo), QB, &fro[3]}};
      rows_gemms<C>(S, jobs, exact ? 2 : 4, ld, olo, pld, nt, ld, k, k);
    }
    if (exact) {
      // exact inverses of the new projections (rank 0: side A, rank 1: side B),
      // then the row fixes y = x_cur P_new^-1 with x_cur = ex / ey / new row
      cl.sync();  // new P^T rows visible
      if (rank < 2) {
        const bool ok = gj_inverse_cta(rank == 0 ? PTA_n : PTB_n, rank == 0 ? QA_n : QB_n, k, ld,
                                       S.yA1, S.yB1, S.cH, S.cE);
        if (!ok && tid == 0) {
          A.ctl->err = 8;  // SingularProjection (factor_state.cpp:21-36)
          A.ctl->err_event = ev_index;
        }
      }
      cl.sync();  // exact inverses visible
      int jlo, jhi;
      block_range(k, C, rank, jlo, jhi);
      for (int j = jlo + warp; j < jhi; j += NW) {
        double ya = 0, yb = 0;
        for (int t = lane; t < k; t += 32) {
          ya += S.exv[t] * QA_n[(int64_t)t * ld + j];
          yb += S.eyv[t] * QB_n[(int64_t)t * ld + j];
        }
        ya = warp_sum(ya);
        yb = warp_sum(yb);
        if (lane == 0) {
          for (int q = 0; q < st.nb; ++q)
            row_add(A, sA, baseA, A.sp_rows[st.b_off + q], j, A.sp_vals[st.b_off + q] * ya);
          if (edge)
            row_add(A, sB, baseB, st.c_row, j, st.c_val * yb);
          else
            row_set(A, sB, baseB, st.c_row, j, yb);  // appended row
        }
      }
    }
    if (tid < 4) *cl.map_shared_rank(&S.pnorm[rank][tid], 0) = fro[tid];
    if (rank == 0)
      for (int t = tid; t < k; t += NT) A.sigma[t] = S.s2[t];
    S.pp[sA] = npp;
    S.pp[sB] = nppB;
    PROF_MARK(9);
    cl.sync();  // B8: new P^T, P^-1, rows and sigma visible
    PROF_MARK(10);
    if (rank == 0 && tid == 0) {
      A.ctl->pp[sA] = npp;
      A.ctl->pp[sB] = nppB;
      A.ctl->rank1 += 1;
      // cond(P_X) <= |P_X|_F |P_X^-1|_F (query-transparent rebase policy)
      const int xA = sA == 0;
      double p2 = 0, q2 = 0;
      for (int r = 0; r < C; ++r) {
        p2 += S.pnorm[r][xA ? 0 : 2];
        q2 += S.pnorm[r][xA ? 1 : 3];
      }
      // cond_2(P) from |P|_F |P^-1|_F (the GEMM epilogues' norms): the bound
      // B satisfies cond_2 <= B <= k cond_2, and B / sqrt(k) is the estimate
      // compared with rebase_cond (the reference runs 10 + 10 power
      // iterations with an LU every event, factor_state.cpp:224-249)
      const double bx = sqrt(p2) * sqrt(q2);
      double p2o = 0, q2o = 0;
      for (int r = 0; r < C; ++r) {
        p2o += S.pnorm[r][xA ? 2 : 0];
        q2o += S.pnorm[r][xA ? 3 : 1];
      }
      const double by = sqrt(p2o) * sqrt(q2o);
      const double rk = sqrt((double)k);
      A.ctl->cond_est = bx / rk;
      A.ctl->cond_est_y = by / rk;
      // P_X as engine.cpp:38-40; P_Y as well (its rows are fp64-slotted the
      // same way and P_Y^-1 is maintained by products too)
      if (fmax(bx, by) / rk > A.rebase_cond) A.ctl->need_rebase = 1;
      // the enhancer's Z_b / r_b are fp32 base-coordinate rows with no fp64
      // side table: with alpha < 1 both projections stay below the fp32
      // storage bound
      if (!A.alpha_is_one && fmax(bx, by) > A.storage_cond) A.ctl->need_rebase = 1;
      if (exact) A.ctl->need_rebase = 1;
    }
  } else {
    // ---- eager fold (rank change or ill-conditioned step) ------------------
    // T_A = P_A F_top (k x k2), stored transposed: TT[t][:] = sum_m FT[t][m] PT[m][:]
    rows_gemm<C>(S, PTA_n, ld, olo, prow(0, olo), pld, tend - olo, PTA, ld, k, k, nullptr);
    rows_gemm<C>(S, PTB_n, ld, olo, prow(3, olo), pld, tend - olo, PTB, ld, k, k, nullptr);
    cl.sync();
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
      const int side = mat == 0 ? sA : mat == 1 ? sB : -1;
      for (long long r = (long long)rank * NW + warp; r < rows; r += (long long)C * NW) {
        for (int i = lane; i < k; i += 32)
          rowv[i] = side >= 0 ? row_val(A, side, base, r, i) : (double)base[r * d + i];
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
    // folded rows are current coordinates now (P = I): back to fp32 storage
    for (int side = 0; side < 2; ++side) {
      const long long ns = min(A.ctl->dirty_n[side], A.dirty_cap);
      for (long long q = (long long)rank * NT + tid; q < ns; q += (long long)C * NT)
        A.slot[side][A.dirty[side][q]] = -1;
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
      for (int q = 0; q < st.nb; ++q)
        row_add(A, sA, baseA, A.sp_rows[st.b_off + q], j, A.sp_vals[st.b_off + q] * S.exv[j]);
      if (edge)
        row_add(A, sB, baseB, st.c_row, j, st.c_val * S.eyv[j]);
      else
        row_set(A, sB, baseB, st.c_row, j, S.eyv[j]);
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
    cl.sync();
    if (rank == 0 && tid == 0) {
      A.ctl->pp[sA] = npp;
      A.ctl->pp[sB] = nppB;
      A.ctl->k = k2;
      A.ctl->rank1 += 1;
      A.ctl->folds += 1;
      A.ctl->cond_est = A.ctl->cond_est_y = 1.0;
      A.ctl->dirty_n[0] = A.ctl->dirty_n[1] = 0;  // folded (fp64 slots read), P = I
    }
  }
  // appended rows (node steps)
  if (!edge && rank == 0 && tid == 0) {
    if (sB == 0)
      A.ctl->rows_x += 1;
    else
      A.ctl->rows_y += 1;
  }
  PROF_MARK(11);
  return true;
}

}  // namespace

// ------------------------------------------------------- fused PPR (cluster)
// For streaming events the enhancer work of one event is small (a few
// touched rows, frontiers of tens to hundreds of rows), so it runs inside
// the same cluster right after the factor update: absorb_structure_delta
// (enhancer.cpp:77-96), s_max = proj_row_bound(P_X) (factor_state.cpp:
// 251-259) and the frontier-synchronous pull push (enhancer.cpp:98-157
// semantics, see ppr.cu). CTA c owns the row chunk [c*n/C, (c+1)*n/C): its
// frontier / affected lists never leave the CTA, so each round needs only
// two cluster barriers (after the pushes, after the pulls + count).
template <int C, class SMT, int PNT>
DAMF_D void ppr_event(const EventKernelArgs& A, SMT& S, cg::cluster_group& cl,
                      const EventDesc& ev) {
  constexpr int PNW = PNT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)cl.block_rank();
  const int k = S.k, d = A.d;
  const double alpha = A.alpha, om = 1.0 - alpha;
  long long _pt = clock64();
  // ---- absorb_structure_delta for the touched rows: one CTA per row, the
  // row's arcs split over its warps (one warp per row walked ~50-100 arcs four
  // at a time: ~9 us per event, with every other warp of the cluster waiting
  // at the next barrier), partial sums combined through the candidate-list
  // storage, which is idle until the lists are built
  float* scr = reinterpret_cast<float*>(&S.plist[0][0]);  // [PNW][kMaxD]
  static_assert(sizeof(S.plist) >= (size_t)PNW * kMaxD * sizeof(float), "absorb scratch");
  for (int q = rank; q < ev.touched_cnt; q += C) {
    const int64_t u = A.touched[ev.touched_off + q];
    float acc[kMaxD / 32];
#pragma unroll
    for (int t = 0; t < kMaxD / 32; ++t) acc[t] = 0.0f;
    const int64_t base = A.out.off[u];
    const int c = A.out.cnt[u];
    const int per = (c + PNW - 1) / PNW;
    const int pb = min(c, warp * per), pe = min(c, pb + per);
    // neighbour ids by lanes, four neighbour rows in flight
    for (int p0 = pb; p0 < pe; p0 += 32) {
      int vl = 0;
      float wl = 0.0f;
      if (p0 + lane < pe) {
        vl = A.out.ids[base + p0 + lane];
        wl = A.out.wts ? (float)A.out.wts[base + p0 + lane] : 1.0f;
      }
      const int cnt = min(32, pe - p0);
      for (int s0 = 0; s0 < cnt; s0 += 4) {
        float zz[4][kMaxD / 32], ww[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int src = s0 + h < cnt ? s0 + h : 0;
          const int v = __shfl_sync(0xffffffffu, vl, src);
          ww[h] = s0 + h < cnt ? __shfl_sync(0xffffffffu, wl, src) : 0.0f;
#pragma unroll
          for (int t = 0; t < kMaxD / 32; ++t) {
            const int j = lane + 32 * t;
            zz[h][t] = j < k ? A.Zb[(int64_t)v * d + j] : 0.0f;
          }
        }
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
          for (int t = 0; t < kMaxD / 32; ++t) acc[t] = fmaf(ww[h], zz[h][t], acc[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < kMaxD / 32; ++t) {
      const int j = lane + 32 * t;
      if (j < k) scr[warp * kMaxD + j] = acc[t];
    }
    __syncthreads();
    const double deg = A.deg[u];
    float m = 0.0f;
    for (int j = tid; j < k; j += PNT) {
      float a = 0.0f;
#pragma unroll
      for (int w = 0; w < PNW; ++w) a += scr[w * kMaxD + j];  // fixed order
      float r = (float)alpha * A.Xb[u * d + j] - A.Zb[u * d + j];
      if (deg > 0.0) r += (float)(om / deg) * a;
      A.rb[u * d + j] = r;
      m = fmaxf(m, fabsf(r));
    }
    m = warp_max(m);
    if (lane == 0) S.bred[warp] = (double)m;
    __syncthreads();
    if (tid == 0) {
      double mm = 0.0;
      for (int w = 0; w < PNW; ++w) mm = fmax(mm, S.bred[w]);
      A.key[u] = (float)(mm / fmax(deg, 1.0));
    }
    __syncthreads();
  }
  PROF_MARK(23);
  if (A.mode & 2) return;  // DAMF_APPLY_DEFER_PUSH: absorb only
  // ---- s_max from P_X: col1 = max_j sum_i |P_ij| (rows of PT), rowinf = max_i sum_j |P_ij|
  {
    const double* PT = A.PT[0][S.pp[0]];
    int lo, hi;
    block_range(k, C, rank, lo, hi);
    double c1 = 0;
    for (int j = lo + warp; j < hi; j += PNW) {
      double s = 0;
      for (int i = lane; i < k; i += 32) s += fabs(PT[(int64_t)j * A.ld + i]);
      c1 = fmax(c1, warp_sum(s));
    }
    for (int i = tid; i < k; i += PNT) {
      double s = 0;
      for (int j = lo; j < hi; ++j) s += fabs(PT[(int64_t)j * A.ld + i]);
      S.partL[0][i] = s;
    }
    if (lane == 0) S.bred[warp] = c1;
    __syncthreads();
    if (tid == 0) {
      double m = 0;
      for (int w = 0; w < PNW; ++w) m = fmax(m, S.bred[w]);
      S.partS[2] = m;
    }
  }
  cl.sync();
  double col1 = 0, rowinf = 0;
  for (int r = 0; r < C; ++r) col1 = fmax(col1, *cl.map_shared_rank(&S.partS[2], r));
  for (int i = tid; i < k; i += PNT) {
    double s = 0;
    for (int r = 0; r < C; ++r) s += *cl.map_shared_rank(&S.partL[0][i], r);
    rowinf = fmax(rowinf, s);
  }
  rowinf = warp_sum(0.0) + rowinf;  // keep lanes converged
  {
    double m = rowinf;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) S.bred[warp] = m;
    __syncthreads();
    m = 0;
    for (int w = 0; w < PNW; ++w) m = fmax(m, S.bred[w]);
    rowinf = m;
  }
  const double smax = k == 0 ? 1.0 : fmax(col1, sqrt(col1 * rowinf));
  const float thr = (float)(alpha * A.eps / smax);
  PROF_MARK(24);
  // ---- rounds (scatter form: small frontiers, no dependent pull chains)
  //   P1  candidate rows (own chunk): key from r (first round: stored key);
  //       over threshold -> delta = r, r = 0, Z += delta, key = 0
  //   --- barrier (frontier counts) ---
  //   P2  every pushed u: r[v] += (1-alpha) w / max(deg v, 1) * delta_u for
  //       v in in(u) (red.global.add), mark[v] = R
  //   --- barrier ---
  //   next candidates: own-chunk rows marked this round
  // Float reductions make the fp32 summation order nondeterministic; the
  // defect bound (the reference's contract) is unaffected.
  const int n = (int)A.ctl->rows_x;
  // block-cyclic ownership: CTA `rank` owns the 32-row blocks b = rank + C*i
  // (balances hot regions; each block is one coalesced 128-byte scan)
  const int nblk = (n + 31) >> 5;
  const int myblk = nblk > rank ? (nblk - rank + C - 1) / C : 0;
  const int maxmine = ((nblk + C - 1) / C) * 32;
  const int seg = (maxmine + PNW - 1) / PNW + 1;  // per-warp segment
  const int stride = seg * PNW;                   // uniform per-CTA list region
  int* Fl = A.listF + (int64_t)rank * stride;
  int* Ll = A.listL + (int64_t)rank * stride;
  int R = (int)A.pstats[2];
  long long pushes = 0;
  int rounds = 0;
  __shared__ int s_cnt[PNW + 1];
  // warp-per-block ballot compaction of own rows into per-warp segments of
  // `out`, then an in-place gather into a contiguous, order-preserving list
  auto compact = [&](auto pred, int* out) -> int {
    int mycnt = 0;
    constexpr int U = 4;
    for (int b0 = warp; b0 < myblk; b0 += PNW * U) {
      bool hit[U];
      int v[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int bi = b0 + q * PNW;
        v[q] = bi < myblk ? ((rank + C * bi) << 5) + lane : n;
        hit[q] = v[q] < n && pred(v[q]);
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const unsigned ball = __ballot_sync(0xffffffffu, hit[q]);
        if (hit[q]) out[warp * seg + mycnt + __popc(ball & ((1u << lane) - 1u))] = v[q];
        mycnt += __popc(ball);
      }
    }
    if (lane == 0) s_cnt[warp] = mycnt;
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < PNW; ++w) {
      if (w < warp) off += s_cnt[w];
      tot += s_cnt[w];
    }
    // gather segments to the front (segments are disjoint and ordered by warp;
    // warp w's destination [off, off+cnt) never overlaps a later segment's
    // unread source because off <= w*seg)
    for (int w = 1; w < PNW; ++w) {
      if (s_cnt[w] == 0) continue;  // (block-uniform: nothing to move, no barrier -- the usual case)
      __syncthreads();
      if (warp == w)
        for (int i = lane; i < mycnt; i += 32) out[off + i] = out[w * seg + i];
    }
    __syncthreads();
    return tot;
  };
  cl.sync();  // touched-row residuals and keys visible
  // first candidates: own rows whose stored key is over threshold
  // round-0 candidates: own rows whose stored key is over threshold, in this
  // CTA's region of list 0; rounds r >= 1 read list r % 3, which the pushes
  // of round r - 1 filled (owner CTA region, DSMEM counters)
  {
    const int c0 = compact([&](int v) { return A.key[v] > thr; }, Ll);
    if (tid == 0) S.lcnt3[0] = c0;
  }
  cl.sync();  // round-0 lists and counts visible cluster-wide
  PROF_MARK(25);
  const DevCSR& in = A.directed ? A.in : A.out;
  int* lists[3] = {A.listL, A.listF, A.listG};
  for (int rr = 0;; ++rr) {
    const int cur = rr % 3, nxt = (rr + 1) % 3, old = (rr + 2) % 3;
    // One phase per round. Each CTA evaluates the candidates of its own
    // list (filled by the previous round's pushes, shared memory with a
    // global overflow); a candidate over threshold is pushed at once: r[u]
    // read-and-zeroed with atomicExch (concurrent contributions are either in
    // this push or stay in r), Z[u] += delta, key = 0, and delta is scattered
    // from registers into r[v], v in in(u) (red.global.add); the first
    // toucher of v appends it to its owner's next list over DSMEM. An
    // asynchronous push in rounds: the contract is the defect bound
    // (enhancer.cpp:98-157); the summation order is nondeterministic.
    const int mycnt = S.lcnt3[cur];
    __syncthreads();
    if (tid == 0) S.lcnt3[old] = 0;  // next filled in round rr + 1 (after this round's barrier)
    int myF = 0;
    for (int q = warp; q < mycnt; q += PNW) {
      const int v = (rr > 0 && q < PCAP) ? S.plist[cur][q] : lists[cur][(int64_t)rank * stride + q];
      // key[v] is an upper bound of |r_v|_inf / max(deg v, 1) (see the
      // scatter below); read it before r, fenced, so every scatter increment
      // it includes is also in the r read
      const float K0 = __ldcg(&A.key[v]);
      __threadfence();
      // independent loads of the candidate, issued together
      const float* rv0 = A.rb + (int64_t)v * d;
      float* zu = A.Zb + (int64_t)v * d;
      float rj[kMaxD / 32], zj[kMaxD / 32];
#pragma unroll
      for (int t = 0; t < kMaxD / 32; ++t) {
        const int j = lane + 32 * t;
        rj[t] = j < k ? rv0[j] : 0.0f;
        zj[t] = j < k ? zu[j] : 0.0f;
      }
      const double degv = A.deg[v];
      const int64_t ib = in.off[v];
      const int c = in.cnt[v];
      float m = 0.0f;
#pragma unroll
      for (int t = 0; t < kMaxD / 32; ++t) m = fmaxf(m, fabsf(rj[t]));
      m = warp_max(m);
      const float key = (float)((double)m / fmax(degv, 1.0));
      const bool push = key > thr;
      if (!push) {
        // exact key of the state read, plus whatever was added since K0
        if (lane == 0) atomicAdd(&A.key[v], key - K0);
        continue;
      }
      // first 32 in-arcs issued alongside the read-and-zero of r[u]
      int vv0 = -1;
      float w0 = 1.0f;
      if (lane < c) {
        vv0 = in.ids[ib + lane];
        if (in.wts) w0 = (float)in.wts[ib + lane];
      }
      float* rv = A.rb + (int64_t)v * d;
#pragma unroll
      for (int t = 0; t < kMaxD / 32; ++t) {
        const int j = lane + 32 * t;
        if (j < k) {
          rj[t] = atomicExch(rv + j, 0.0f);
          zu[j] = zj[t] + rj[t];
        }
      }
      // r_v now holds only what arrived after the exchange: drop the part K0
      // bounded, keep later increments
      if (lane == 0) atomicAdd(&A.key[v], -K0);
      ++myF;
      float dmax = 0.0f;  // |delta|_inf of this push
#pragma unroll
      for (int t = 0; t < kMaxD / 32; ++t) dmax = fmaxf(dmax, fabsf(rj[t]));
      dmax = warp_max(dmax);
      for (int p0 = 0; p0 < c; p0 += 32) {
        const int p = p0 + lane;
        int vv = -1;
        float cf = 0.0f, inc = 0.0f;
        if (p < c) {
          float w = w0;
          vv = vv0;
          if (p0 > 0) {
            vv = in.ids[ib + p];
            w = in.wts ? (float)in.wts[ib + p] : 1.0f;
          }
          const double dg = fmax(A.deg[vv], 1.0);
          cf = (float)(om * w / dg);
          // bound of the key increase of vv (1e-4 slack for fp32 rounding)
          inc = (float)(fabs(om * w) / (dg * dg) * (double)dmax * (1.0 + 1e-4));
        }
        const int cnt = min(32, c - p0);
        for (int s2 = 0; s2 < cnt; ++s2) {
          const int tv = __shfl_sync(0xffffffffu, vv, s2);
          const float cc = __shfl_sync(0xffffffffu, cf, s2);
          float* rt = A.rb + (int64_t)tv * d;
#pragma unroll
          for (int t = 0; t < kMaxD / 32; ++t) {
            const int j = lane + 32 * t;
            if (j < k) atomicAdd(rt + j, cc * rj[t]);  // RED.ADD.F32
          }
        }
        // Candidates for the next round are only the targets whose key bound
        // crosses the threshold (a target under it cannot be over it); the
        // contributions are ordered before the bound update.
        __threadfence();
        if (p < c) {
          const float kb = atomicAdd(&A.key[vv], inc) + inc;
          if (kb > thr && atomicExch(&A.mark[vv], R + 1) != R + 1) {
            const int ow = (vv >> 5) % C;
            const int pos = atomicAdd(cl.map_shared_rank(&S.lcnt3[nxt], ow), 1);
            if (pos < PCAP)
              *cl.map_shared_rank(&S.plist[nxt][pos], ow) = vv;
            else
              lists[nxt][(int64_t)ow * stride + pos] = vv;
          }
        }
      }
    }
    if (lane == 0) s_cnt[warp] = myF;
    __syncthreads();
    int nF = 0;
    for (int w = 0; w < PNW; ++w) nF += s_cnt[w];
    PROF_MARK(26);
    if (tid == 0)
      for (int r = 0; r < C; ++r) *cl.map_shared_rank(&S.found[rank][0], r) = nF;
    cl.sync();  // pushes, contributions and next lists of this round landed
    PROF_MARK(27);
    long long tot = 0;
    for (int r = 0; r < C; ++r) tot += S.found[r][0];
    ++R;
    if (tot == 0) {
      if (tid == 0) S.lcnt3[cur] = 0;  // all counters zero for the next event
      break;
    }
    ++rounds;
    pushes += tot;
    if (pushes > 1000000000LL) {
      if (rank == 0 && tid == 0) A.ctl->err = 9;  // NonConvergence
      break;
    }
    PROF_MARK(30);
  }
  if (rank == 0 && tid == 0) {
    A.pstats[0] += pushes;
    A.pstats[1] += rounds;
    A.pstats[2] = R;
    A.pstats[3] += pushes;
  }
  cl.sync();
}


#if DAMF_PROF
// Flush this CTA's phase counters: rank 0 owns the phase slots, every rank its
// own per-rank slots (32 / 48 / 64 + rank); slot 15 is a maximum.
template <class SMT>
DAMF_D void prof_flush(const EventKernelArgs& A, SMT& S, int rank) {
  if (threadIdx.x != 0) return;
  for (int i = 0; i < 128; ++i) {
    const bool per_rank = i >= 32 && i < 96;
    if (per_rank ? ((i & 15) == rank) : rank == 0) {
      if (i == 15)
        atomicMax(&A.ctl->prof[i], S.lprof[i]);
      else
        atomicAdd(&A.ctl->prof[i], S.lprof[i]);
    }
  }
}
#endif

// ------------------------------------------------------------------ push kernel
// The per-event push as its own cluster kernel (split mode): launched after a
// one-event factor kernel, with its own register budget and twice the warps
// of the factor kernel. A rebase or error requested by an earlier event of
// the batch turns it into a no-op (the factor kernel stops the same way).
constexpr int PPR_NT = 512;
template <int C>
struct PSmem {
  int k, pp[2];
  double partL[1][kMaxD];
  double partS[4];
  double bred[PPR_NT / 32];
  long long found[C][2];
  int lcnt3[3];
  int plist[3][PCAP];
#if DAMF_PROF
  unsigned long long lprof[128];
#endif
};
template <int C>
__global__ void __launch_bounds__(PPR_NT, 1) damf_ppr_kernel(EventKernelArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PSmem<C>& S = *reinterpret_cast<PSmem<C>*>(smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  if (threadIdx.x == 0) {
    S.k = A.ctl->k;
    S.pp[0] = A.ctl->pp[0];
    S.pp[1] = A.ctl->pp[1];
    for (int i = 0; i < 3; ++i) S.lcnt3[i] = 0;
#if DAMF_PROF
    for (int i = 0; i < 128; ++i) S.lprof[i] = 0;
#endif
  }
  __syncthreads();
  cl.sync();
  for (int64_t e = A.e_begin; e < A.e_end; ++e) {
    const long long stop = *(volatile long long*)&A.ctl->stop_event;
    if (*(volatile int*)&A.ctl->err || (stop >= 0 && stop <= e)) break;
    // this event's factor update requested a rebase: Z_b / r_b are fp32 base
    // coordinates, so the absorb and push wait until the host has folded
    // everything to P = I (a rebase is query-transparent for the enhancer,
    // enhancer.cpp:196-206); the host relaunches this kernel for event e
    if (*(volatile int*)&A.ctl->need_rebase) {
      if (rank == 0 && threadIdx.x == 0) A.ctl->ppr_skip = e;
      break;
    }
    const EventDesc ev = A.ev[e];
    ppr_event<C, PSmem<C>, PPR_NT>(A, S, cl, ev);
    if (A.t_end && rank == 0 && threadIdx.x == 0) A.t_end[e] = globaltimer();
  }
#if DAMF_PROF
  prof_flush(A, S, rank);
#endif
}

// ------------------------------------------------------------------ kernel
// FUSED: the per-event PPR push runs in the cluster after each event's
// factor update (alpha < 1 on graphs up to 1 M rows); the factor-only
// instantiation (alpha = 1, or the whole-GPU push afterwards) has no push code.
template <int C, bool FUSED>
__global__ void __launch_bounds__(NT, 1) damf_event_kernel(EventKernelArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<C>& S = *reinterpret_cast<Smem<C>*>(smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  if (threadIdx.x == 0) {
    S.k = A.ctl->k;
    S.pp[0] = A.ctl->pp[0];
    S.pp[1] = A.ctl->pp[1];
    for (int i = 0; i < 3; ++i) S.lcnt3[i] = 0;  // fused-PPR counters
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&S.gbar[i])));
      S.gq[i] = 0;
    }
    for (int i = 0; i < 8; ++i) S.gprof[i] = 0;
#if DAMF_PROF
    for (int i = 0; i < 128; ++i) S.lprof[i] = 0;
    S.tlog_n = 0;
#endif
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (A.reset_stop && rank == 0) A.ctl->stop_event = -1;
  }
  __syncthreads();
  cl.sync();  // counters zeroed (and the stop cleared) before any CTA looks at them
  for (int64_t e = A.e_begin; e < A.e_end; ++e) {
    // (split mode launches one event per kernel: an earlier launch of the
    // batch that stopped for a rebase or failed turns this one into a no-op)
    const long long stop = *(volatile long long*)&A.ctl->stop_event;
    if (*(volatile int*)&A.ctl->err || (stop >= 0 && stop <= e)) break;
    const EventDesc ev = A.ev[e];
    if (A.t_begin && rank == 0 && threadIdx.x == 0) A.t_begin[e] = globaltimer();
    int err = 0;
    long long _pt = clock64();
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
    PROF_MARK(12);
    // ---- factor update (update_engine.cpp:206-226) ----------------------
    if (!(A.mode & 1)) {
      bool fin = true;
      for (int s = 0; s < ev.nsteps && fin; ++s) {
        if (threadIdx.x == 0) {  // (read after several block barriers inside the step)
          S.pf_stage = e + 1 < A.e_end ? (s == 0 ? 1 : s == 1 ? 2 : 0) : 0;
          S.pf_e = e + 1;
        }
        const StepDesc st = A.steps[ev.step0 + s];
        fin = rank1_step<C>(A, S, cl, st, e, ev.step0 + s);
      }
      if (!fin) break;  // NonFinite recorded in ctl; the batch stops here
    }
    if (FUSED) {
      cl.sync();  // factor / graph writes visible to the enhancer
      ppr_event<C, Smem<C>, NT>(A, S, cl, ev);
    }
    if (A.t_end && rank == 0 && threadIdx.x == 0) A.t_end[e] = globaltimer();
    // a rebase was requested: stop after this event; the host rebases over
    // the whole GPU and resumes the batch (engine.cpp:38-40 per-event order)
    cl.sync();
    if (*(volatile int*)&A.ctl->need_rebase || *(volatile int*)&A.ctl->err) {
      if (rank == 0 && threadIdx.x == 0) A.ctl->stop_event = e + 1;
      break;
    }
  }
#if DAMF_PROF
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) S.lprof[28 + i] += (unsigned long long)S.gprof[i];
    for (int i = 3; i < 8; ++i) S.lprof[96 + i] += (unsigned long long)S.gprof[i];
  }
  prof_flush(A, S, rank);
  // barrier timeline of this launch's first 64 eigen-solves (d <= 128: ws_priv is free)
  if (threadIdx.x == 0 && A.d <= 128) {
    double* o = A.ws_priv + 8 + 8 * 800 + rank * 260;
    o[0] = S.tlog_n;
    for (int i = 0; i < S.tlog_n; ++i)
      for (int q = 0; q < 4; ++q) o[4 + 4 * i + q] = (double)(S.tlog[i][q] & 0xFFFFFFFFFFFFull);
  }
#endif
}

// ------------------------------------------------------------------ launch
template <int C, bool FUSED>
static cudaError_t launch_cf(const EventKernelArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(Smem<C>);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(damf_event_kernel<C, FUSED>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (C > 8) {
      e = cudaFuncSetAttribute(damf_event_kernel<C, FUSED>,
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
  return cudaLaunchKernelEx(&cfg, damf_event_kernel<C, FUSED>, a);
}
template <int C>
static cudaError_t launch_c(const EventKernelArgs& a, cudaStream_t s) {
  return a.fused_ppr ? launch_cf<C, true>(a, s) : launch_cf<C, false>(a, s);
}

int event_cluster_size() {
  static int chosen = 0;
  if (chosen) return chosen;
  // Prefer 16 CTAs (non-portable) when the device can co-schedule it.
  int c16 = 0;
  {
    cudaFuncSetAttribute(damf_event_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(Smem<16>));
    cudaFuncSetAttribute(damf_event_kernel<16, true>,
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
    if (cudaOccupancyMaxActiveClusters(&c16, damf_event_kernel<16, true>, &cfg) != cudaSuccess) c16 = 0;
    cudaGetLastError();
  }
  chosen = c16 > 0 ? 16 : 8;
  return chosen;
}

size_t event_kernel_smem(int C) { return C == 16 ? sizeof(Smem<16>) : sizeof(Smem<8>); }

cudaError_t launch_ppr_kernel(const EventKernelArgs& a, cudaStream_t s) {
  constexpr int C = 16;
  const size_t smem = sizeof(PSmem<C>);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(damf_ppr_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(damf_ppr_kernel<C>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(PPR_NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, damf_ppr_kernel<C>, a);
}

cudaError_t launch_event_kernel(const EventKernelArgs& a, cudaStream_t s) {
  return event_cluster_size() == 16 ? launch_c<16>(a, s) : launch_c<8>(a, s);
}

}  // namespace dgpu
