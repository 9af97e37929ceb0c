// Host-visible interface of the per-event cluster kernel (event_kernel.cu).
#pragma once

#include "common.cuh"

namespace dgpu {

constexpr int kEventThreads = 256;

struct EventKernelArgs {
  // batch
  const EventDesc* ev;
  int64_t e_begin, e_end;
  StepDesc* steps;
  const int64_t* sp_rows;   // sparse b rows
  const double* sp_vals;    // sparse b values
  const int64_t* nb_ids;    // AddNode neighbour ids (flat)
  const double* nb_w;       // AddNode neighbour weights
  unsigned long long* t_begin;  // per-event %globaltimer stamps (or null)
  unsigned long long* t_end;
  int mode;                 // DAMF_APPLY_* bits
  int reset_stop;           // first kernel of a launch group: clear ctl->stop_event
  int64_t* rowlog;          // (step, side 0=X / 1=Y, row) per modified base row, or null
  long long rowlog_cap;     // triples
  // factor state
  DevCtl* ctl;
  int d, ld;
  float* Xb;
  float* Yb;
  float* Zb;
  float* rb;
  float* key;  // enhancer residual keys (refreshed on folds)
  int alpha_is_one;
  // fused per-event enhancer (alpha < 1, n small enough for in-cluster scans)
  int fused_ppr;
  double alpha, eps;
  float* delta;
  int* stamp;
  int* mark;
  int* listF;
  int* listG;   // third candidate-list buffer of the fused push (round mod 3)
  int* listL;
  const int64_t* touched;
  long long* pstats;
  double* PT[2][2];  // [side X/Y][ping-pong]  P transposed
  double* Q[2][2];   // [side][ping-pong]      P^-1
  double* sigma;
  double rebase_cond;
  double storage_cond;
  // fp64 side table of the base rows written through P^-1 (the reference's
  // base rows are fp64; here they are fp32 except these): slot[side][row] =
  // index into rows64[side] (ld doubles per row) or -1; dirty[side][slot] =
  // its row; ctl->dirty_n[side] slots in use out of dirty_cap
  int64_t* dirty[2];
  long long dirty_cap;
  int32_t* slot[2];
  double* rows64[2];
  // graph
  DevCSR out, in;
  int directed, undirected;
  double* deg;
  // workspace (fp64): Q1^T (ld x ld, shared by the cluster) and, for d > 128,
  // the per-CTA private matrices (4 x C x (ceil(257/C)+1) x ld)
  double* ws_Q1T;
  double* ws_priv;
};

cudaError_t launch_event_kernel(const EventKernelArgs& a, cudaStream_t s);
// the per-event push as its own 16-CTA cluster kernel (split mode)
cudaError_t launch_ppr_kernel(const EventKernelArgs& a, cudaStream_t s);
int event_cluster_size();
size_t event_kernel_smem(int C);

}  // namespace dgpu
