#pragma once
#include "common.cuh"

namespace dgpu {

constexpr int PPR_HEAVY = 256;  // rows with more out-arcs are pulled in chunks
constexpr int PPR_CH = 256;     // arcs per chunk
// In-arcs per scatter item. Short items spread a pushed row's in-list over
// many warps: a warp issues its reductions back to back, so one 512-arc item
// kept a warp busy for ~0.2 ms and set the length of its round (R-MAT scale
// 23, push after 1,000 inserts: 3.4 ms at 512, 1.8 at 64, 1.4 at 32/16/8).
constexpr int PPR_MCH = 32;

// Cross-launch state of a push split into cooperative rounds + standalone
// dense-pull launches (damf_gpu_ppr_init / _push).
struct PprState {
  int phase;         // 0: fresh call, 1: resume after a dense pull
  int pull_pending;  // set when the cooperative kernel exits for a dense pull
  int R, rounds, nH, nchunks, cur, pad;
  long long pushes, narcs;
};

struct PprArgs {
  int64_t n;
  int d, k;
  const float* Xb;
  float* Zb;
  float* rb;
  float* delta;
  float* key;
  int* stamp;
  int* mark;
  int* listF;
  int* listL;
  int* blk;
  long long* blk64;   // scratch (gridDim)
  int* heavy;         // heavy-row list (rows with > HEAVY out-arcs)
  int* hidx;          // row -> heavy index or -1 (n, kept at -1 between calls)
  int* hoff;          // heavy chunk prefix (nH + 1)
  int* cidx;          // chunk -> heavy index (arc pool / CH + nH)
  float* hacc;        // heavy-row pull accumulators (nH x d, kept zero between rounds)
  int* items[2];      // P3 work lists, alternating per round (n + chunks)
  int* hdone;         // per heavy row: chunks finished this round (kept zero between rounds)
  int* mitems;        // marking items (pusher, in-arc chunk) pairs
  PprState* pst;      // split-mode state (device)
  int split;          // 1: exit the cooperative kernel for dense pull rounds
  long long* trace;   // per-round [nF, dense, items, active heavy] of the last call (4 x 1024)
  unsigned long long* wq;  // work counters [P1 grab, P3 grab, big-mark count, push count x3,
                           //  item count, active heavy count]
  DevCSR out, in;
  int directed;
  double* deg;
  double alpha;
  double alpha_eps;   // alpha*eps (enhancer.cpp:104)
  const double* smax; // device s_max = proj_row_bound(P_X); push when key > alpha_eps/s_max
  int round_base;
  const int* cand;    // candidate rows for the first frontier (ncand >= 0)
  int ncand;          // -1: scan all rows
  long long push_guard;
  int force_pull;       // diagnostic (DAMF_PPR_FORCE_PULL=1): pull rounds only, for the scatter-vs-pull A/B
  long long narcs_hint; // arcs of the initial graph: picks the round direction until the exact count is built
  long long* stats;   // [pushes, rounds, next round base, sum|F|, sum|L|,
                      //  sum outdeg(L), matched arcs] (bench accounting)
  unsigned long long* t_end;
  DevCtl* ctl;
};

cudaError_t launch_ppr_push(const PprArgs& a, int grid, cudaStream_t s);
cudaError_t launch_ppr_pull(const PprArgs& a, int nsm, cudaStream_t s);
int ppr_push_max_grid(int nsm, int d);
cudaError_t launch_ppr_absorb(const PprArgs& a, const int64_t* rows, int nrows, cudaStream_t s);
cudaError_t launch_ppr_keys(const PprArgs& a, int nsm, cudaStream_t s);
cudaError_t launch_ppr_init(const PprArgs& a, int nsm, cudaStream_t s);
cudaError_t launch_smax(const double* PT0, const double* PT1, const DevCtl* ctl, int ld,
                        double* out, cudaStream_t s);

}  // namespace dgpu
