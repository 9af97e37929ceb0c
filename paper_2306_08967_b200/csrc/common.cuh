// Shared device-side definitions for the B200 DAMF hot path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define DAMF_HD __host__ __device__ __forceinline__
#define DAMF_D __device__ __forceinline__

namespace dgpu {

constexpr int kMaxD = 256;                // largest supported rank d
constexpr int kWarp = 32;

// Device-resident control block: everything the per-event kernels decide on
// the device (rank, ping-pong buffers, errors) lives here so a whole batch
// runs without host round trips; the host reads it once per batch.
struct DevCtl {
  int k;              // active rank (factor_state.hpp:28)
  int pp[2];          // ping-pong index of P/Q for side X (0) / Y (1)
  int err;            // status code of the first failure (0 = ok)
  long long err_event;
  long long rank1;    // rank-1 steps run
  long long folds;    // eager folds (rank change / ill-conditioned F)
  long long rows_x, rows_y;  // X_b / Y_b row counts
  double cond_est;    // running cond(P_X) estimate (|P|_F |P^-1|_F / sqrt(k))
  double cond_est_y;  // the same for P_Y
  int need_rebase;    // set when cond_est > rebase_cond
  int pad;
  double smax;        // proj_row_bound(P_X) at the end of the last step
  unsigned long long t_begin, t_end;  // %globaltimer stamps of the last event
  long long stop_event;               // first event not processed by a stopped batch
  long long dirty_n[2];               // rows of X_b / Y_b written through P^-1 since the last fold
  long long rowlog_n;                 // entries in the modified-row log (DAMF_APPLY_LOG_ROWS)
  long long ppr_skip;                 // event whose PPR absorb / push waits for a rebase (-1: none)
  unsigned long long prof[128];       // per-phase SM cycles, dev profiling (DAMF_PROF builds)
};

// Slack-per-row CSR (K9): row u occupies ids[off[u] .. off[u]+cnt[u]) inside a
// segment of cap[u] slots; a full row is relocated to the pool top with
// doubled capacity. int64 offsets (2.1e9 arcs at scale 26), int32 ids.
struct DevCSR {
  int64_t* off;
  int32_t* cnt;
  int32_t* cap;
  int32_t* ids;
  double* wts;        // nullptr: all weights 1.0
  int64_t* pool_top;  // device scalar
  int64_t pool_size;
};

// One space-projection step (update_engine.cpp:206-226). Side A receives the
// sparse column b (X for Edge / NodeColumn, Y for NodeRow); side B receives
// c = c_val * e_{c_row} (Edge) or the appended row (Node steps).
enum StepKind : int32_t { kStepEdge = 0, kStepNodeCol = 1, kStepNodeRow = 2 };

struct StepDesc {
  int32_t kind;
  int32_t nb;         // nonzeros of b
  int64_t b_off;      // offset into the sparse (row, val) arrays
  int64_t c_row;      // Edge: row of c; Node: index of the appended B row
  double c_val;       // Edge: +w / -w (patched on device for weighted removals)
  int64_t n_a, n_b;   // rows of side A / side B before the step
  double bnorm2;      // |b|^2
};

// One event's device work list.
struct EventDesc {
  int32_t kind;       // DAMF_ADD_NODE / ADD_EDGE / REMOVE_EDGE
  int32_t nsteps;
  int64_t step0;      // first StepDesc
  int64_t u, v;       // edge endpoints, or new node id for AddNode
  double w;
  int64_t in_off, in_cnt, out_off, out_cnt;  // AddNode neighbour lists
  int64_t touched_off, touched_cnt;          // rows whose defect is recomputed
};

DAMF_D double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
DAMF_D double warp_prod(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v *= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
DAMF_D float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
DAMF_D unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace dgpu
