// Host orchestration of the B200 DAMF hot path behind the C ABI in
// include/damf_gpu.h. Mirrors damf::Engine (engine.cpp:5-52): graph deltas
// -> space-projection updates -> enhancer absorb + push -> rebase policy,
// with all state device-resident and the per-event work in the cluster
// kernel (event_kernel.cu) and the PPR kernels (ppr.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/damf_gpu.h"
#include "common.cuh"
#include "event_kernel.cuh"
#include "materialize.cuh"
#include "ppr.cuh"
#include "score.cuh"
#include "tsvd.cuh"

using namespace dgpu;

namespace {
// fp64 side-table rows per side between folds (rows written through P^-1;
// a full table requests a rebase): 2 rows per side per edge event, so a
// table outlasts the reference's 50,000-event rebase period
constexpr long long kDirtyCap = 1 << 17;
// DevCtl followed by the 8 push counters (pushes, rounds, round base, ...)
constexpr size_t kCtlOff = (sizeof(dgpu::DevCtl) + 63) & ~size_t(63);
constexpr size_t kCtlBytes = kCtlOff + 8 * sizeof(long long);

#define CK(expr)                                                                       \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) return cuda_fail(h, _e, #expr, __LINE__);                   \
  } while (0)

template <class T>
struct Staged {
  T* h = nullptr;
  T* d = nullptr;
  size_t cap = 0;
  size_t n = 0;
  cudaError_t ensure(size_t want) {
    if (want <= cap) return cudaSuccess;
    const size_t nc = std::max<size_t>(want, cap * 2 + 64);
    T* nh = nullptr;
    T* nd = nullptr;
    cudaError_t e = cudaMallocHost(&nh, nc * sizeof(T));
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&nd, nc * sizeof(T));
    if (e != cudaSuccess) return e;
    if (h && n) std::memcpy(nh, h, n * sizeof(T));  // keep staged content
    if (h) cudaFreeHost(h);
    if (d) cudaFree(d);
    h = nh;
    d = nd;
    cap = nc;
    return cudaSuccess;
  }
  void push(const T& v) { h[n++] = v; }
  cudaError_t upload(cudaStream_t s) {
    return n ? cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s) : cudaSuccess;
  }
  void release() {
    if (h) cudaFreeHost(h);
    if (d) cudaFree(d);
    h = nullptr;
    d = nullptr;
  }
};

// ---- small device kernels ------------------------------------------------
__global__ void csr_expand_kernel(int64_t n, const int64_t* coff, const int32_t* cids,
                                  const double* cw, const int64_t* noff, int32_t* nids,
                                  double* nw, int32_t* cnt, int32_t* cap, int64_t* off) {
  const int64_t u = (int64_t)blockIdx.x;
  for (int64_t r = u; r < n; r += gridDim.x) {
    const int64_t a = coff[r], b = coff[r + 1], o = noff[r];
    for (int64_t p = a + threadIdx.x; p < b; p += blockDim.x) {
      nids[o + (p - a)] = cids[p];
      if (nw) nw[o + (p - a)] = cw ? cw[p] : 1.0;
    }
    if (threadIdx.x == 0) {
      cnt[r] = (int32_t)(b - a);
      cap[r] = (int32_t)(noff[r + 1] - o);
      off[r] = o;
    }
  }
}

__global__ void degree_kernel(int64_t n, DevCSR g, double* deg) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    double s = 0;
    const int64_t o = g.off[u];
    const int c = g.cnt[u];
    if (g.wts)
      for (int p = 0; p < c; ++p) s += g.wts[o + p];
    else
      s = (double)c;
    deg[u] = s;
  }
}

// In-place Gauss-Jordan inverse with partial pivoting of a k x k fp64
// matrix (ld), one CTA; used once at creation for P^-1.
__global__ void gj_inverse_kernel(double* A, double* Inv, int k, int ld, int* singular) {
  __shared__ int piv;
  __shared__ double pval;
  for (int x = threadIdx.x; x < k * k; x += blockDim.x) {
    const int i = x / k, j = x % k;
    Inv[(int64_t)i * ld + j] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int c = 0; c < k; ++c) {
    if (threadIdx.x == 0) {
      int p = c;
      double best = fabs(A[(int64_t)c * ld + c]);
      for (int r = c + 1; r < k; ++r)
        if (fabs(A[(int64_t)r * ld + c]) > best) {
          best = fabs(A[(int64_t)r * ld + c]);
          p = r;
        }
      piv = p;
      pval = A[(int64_t)p * ld + c];
      if (best == 0.0) *singular = 1;
    }
    __syncthreads();
    if (pval == 0.0) return;
    if (piv != c)
      for (int j = threadIdx.x; j < k; j += blockDim.x) {
        double t = A[(int64_t)c * ld + j];
        A[(int64_t)c * ld + j] = A[(int64_t)piv * ld + j];
        A[(int64_t)piv * ld + j] = t;
        t = Inv[(int64_t)c * ld + j];
        Inv[(int64_t)c * ld + j] = Inv[(int64_t)piv * ld + j];
        Inv[(int64_t)piv * ld + j] = t;
      }
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      A[(int64_t)c * ld + j] /= pval;
      Inv[(int64_t)c * ld + j] /= pval;
    }
    __syncthreads();
    for (int x = threadIdx.x; x < k * k; x += blockDim.x) {
      const int r = x / k, j = x % k;
      if (r == c) continue;
      const double f = A[(int64_t)r * ld + c];
      if (j != c) A[(int64_t)r * ld + j] -= f * A[(int64_t)c * ld + j];
      Inv[(int64_t)r * ld + j] -= f * Inv[(int64_t)c * ld + j];
    }
    __syncthreads();
    for (int r = threadIdx.x; r < k; r += blockDim.x)
      if (r != c) A[(int64_t)r * ld + c] = 0.0;
    __syncthreads();
  }
}

__global__ void transpose_kernel(const double* A, double* B, int k, int ld) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < k * k; x += gridDim.x * blockDim.x) {
    const int i = x / k, j = x % k;
    B[(int64_t)j * ld + i] = A[(int64_t)i * ld + j];
  }
}

__global__ void identity_kernel(double* A, int k, int ld) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < k * ld; x += gridDim.x * blockDim.x) {
    const int i = x / ld, j = x % ld;
    A[x] = (i == j && j < k) ? 1.0 : 0.0;
  }
}

// out[q][j] = sum_i base[ids[q]][i] * P[i][j] (P given as PT), fp64 accumulation.
// rows with an fp64 side-table slot (slot != null, slot[r] >= 0) are read
// from rows64 (ld doubles per slot)
__global__ void query_rows_kernel(const float* base, int d, const double* PT, int ld, int k,
                                  const int64_t* ids, int64_t m, float* out, double* out64,
                                  const int32_t* slot, const double* rows64) {
  for (int64_t q = blockIdx.x; q < m; q += gridDim.x) {
    const int64_t r = ids[q];
    const int sl = slot ? slot[r] : -1;
    const double* r64 = sl >= 0 ? rows64 + (int64_t)sl * ld : nullptr;
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      double s = 0;
      for (int i = 0; i < k; ++i)
        s += (r64 ? r64[i] : (double)base[r * d + i]) * PT[(int64_t)j * ld + i];
      if (out) out[q * k + j] = (float)s;
      if (out64) out64[q * k + j] = s;
    }
  }
}

// out[row] = rows64[s] P for every side-table slot s (row = rows[s]), fp64
// products, fp32 result; clear != 0 also releases the slot (a fold).
__global__ void fold_rows64_kernel(const double* rows64, int ld, const int64_t* rows, long long ns,
                                   const double* PT, int k, float* out, int ldo, int32_t* slot,
                                   int clear) {
  extern __shared__ double rv[];
  for (long long s = blockIdx.x; s < ns; s += gridDim.x) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) rv[i] = rows64[s * ld + i];
    __syncthreads();
    const int64_t row = rows[s];
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      double acc = 0;
      for (int i = 0; i < k; ++i) acc += rv[i] * PT[(int64_t)j * ld + i];
      out[row * ldo + j] = (float)acc;
    }
    if (clear && threadIdx.x == 0) slot[row] = -1;
    __syncthreads();
  }
}

// exact base rows (side table aware), fp64, k columns
__global__ void base_rows64_kernel(const float* base, int d, const int32_t* slot, const double* rows64,
                                   int ld, int k, const int64_t* ids, int64_t m, double* out) {
  for (int64_t q = blockIdx.x; q < m; q += gridDim.x) {
    const int64_t r = ids[q];
    const int sl = slot[r];
    for (int j = threadIdx.x; j < k; j += blockDim.x)
      out[q * k + j] = sl >= 0 ? rows64[(int64_t)sl * ld + j] : (double)base[r * d + j];
  }
}

__global__ void count_sum_kernel(const int32_t* cnt, int64_t n, unsigned long long* out) {
  unsigned long long s = 0;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x)
    s += (unsigned long long)cnt[x];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

__global__ void set_slots_kernel(int32_t* slot, const int64_t* rows, long long ns) {
  for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < ns;
       s += (long long)gridDim.x * blockDim.x)
    slot[rows[s]] = (int32_t)s;
}

// After damf_gpu_load_rows rewrote rows [r0, r0 + m) in fp32: refresh the
// side-table copies of those rows.
__global__ void refresh_rows64_kernel(double* rows64, int ld, const int64_t* rows, long long ns,
                                      const float* base, int d, int64_t r0, int64_t m) {
  for (long long s = blockIdx.x; s < ns; s += gridDim.x) {
    const int64_t row = rows[s];
    if (row < r0 || row >= r0 + m) continue;
    for (int j = threadIdx.x; j < d; j += blockDim.x) rows64[s * ld + j] = (double)base[row * d + j];
  }
}

__global__ void pack_rows_kernel(const float* base, int64_t n, int d, int k, float* out) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n * k;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = x / k;
    const int j = (int)(x % k);
    out[x] = base[r * d + j];
  }
}


}  // namespace

struct damf_gpu {
  damf_config cfg{};
  int d = 0, ld = 0, k = 0;
  int64_t n = 0, n_cap = 0, arcs = 0;
  bool alpha1 = false, directed = false;
  cudaStream_t st = nullptr;
  int nsm = 148;
  DevCtl* ctl = nullptr;
  DevCtl* h_ctl = nullptr;  // pinned
  // h_ctl / h_pstats mirror the device exactly: set by sync_ctl, cleared by
  // every entry point that may enqueue device work (apply skips its
  // pre-launch round trip when the mirror is fresh)
  bool ctl_fresh = false;
  // Rows whose residual changed since the last completed push (absorbed
  // structure-only events with a deferred push). While pend_valid, every
  // other row's key is at most the threshold (nothing else changed r, deg or
  // s_max), so damf_gpu_ppr_push can start from these rows instead of
  // checking every key.
  std::vector<int32_t> pend;
  bool pend_valid = false;
  int32_t* pend_d = nullptr;
  float *Xb = nullptr, *Yb = nullptr, *Zb = nullptr, *rb = nullptr, *delta = nullptr,
        *key = nullptr;
  int *stamp = nullptr, *mark = nullptr, *listF = nullptr, *listL = nullptr, *blk = nullptr;
  int* listG = nullptr;
  long long* blk64 = nullptr;
  int *heavy = nullptr, *hidx = nullptr, *hoff = nullptr, *cidx = nullptr;
  float* hacc = nullptr;
  int *items0 = nullptr, *items1 = nullptr, *hdone = nullptr, *mitems = nullptr;
  long long* ptrace = nullptr;
  PprState* pst = nullptr;
  PprState* h_pst = nullptr;  // pinned mirror
  // fp64 side table (see EventKernelArgs): dirty[side][s] = row of slot s,
  // slot[side][row] = s or -1, rows64[side] = kDirtyCap x ld doubles
  int64_t* dirty[2] = {nullptr, nullptr};
  int32_t* slot[2] = {nullptr, nullptr};
  double* rows64[2] = {nullptr, nullptr};
  unsigned long long* wq = nullptr;
  double* PT[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  double* Q[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  double* sigma = nullptr;
  DevCSR out{}, in{};
  double* deg = nullptr;
  double* ws = nullptr;
  double* smax = nullptr;
  long long* pstats = nullptr;  // pushes, rounds, round base
  long long* h_pstats = nullptr;
  Staged<char> pack;  // every descriptor array of one apply, one H2D copy
  EventDesc* d_ev = nullptr;
  StepDesc* d_steps = nullptr;
  int64_t *d_sp_rows = nullptr, *d_nb_ids = nullptr, *d_touched = nullptr;
  double *d_sp_vals = nullptr, *d_nb_w = nullptr;
  Staged<EventDesc> ev;
  Staged<StepDesc> steps;
  Staged<int64_t> sp_rows, nb_ids, touched;
  Staged<double> sp_vals, nb_w;
  unsigned long long *t_begin = nullptr, *t_end = nullptr;
  size_t t_cap = 0;
  std::vector<double> lat_us;
  int64_t lat_pending = 0;            // events whose stamps are still on the device
  cudaEvent_t span0 = nullptr, span1 = nullptr;
  cudaEvent_t mat0 = nullptr, mat1 = nullptr;  // around the last materialisation's X F kernels
  double last_mat_ms = 0.0;
  int64_t* rowlog = nullptr;          // device (step, side, row) triples
  long long rowlog_cap = 0;
  std::vector<int64_t> rowlog_h;      // the last apply's log (DAMF_APPLY_LOG_ROWS)
  uint64_t events_applied = 0;
  int64_t since_rebase = 0;
  int64_t total_pushes = 0;
  int round_base = 0;
  size_t bytes = 0;
  int64_t launches = 0;
  std::string err;
  std::vector<void*> allocs;
};

namespace {

int base_rows_f64(damf_gpu* h, int side, std::vector<double>* out);

int cuda_fail(damf_gpu* h, cudaError_t e, const char* what, int line) {
  if (h) h->err = std::string("CUDA error ") + cudaGetErrorString(e) + " at engine.cu:" +
                  std::to_string(line) + " (" + what + ")";
  return DAMF_E_CUDA;
}

template <class T>
cudaError_t dalloc(damf_gpu* h, T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e == cudaSuccess) {
    h->allocs.push_back(*p);
    h->bytes += count * sizeof(T);
  }
  return e;
}

int fail(damf_gpu* h, int code, const std::string& msg) {
  h->err = msg;
  return code;
}

EventKernelArgs event_args(damf_gpu* h) {
  EventKernelArgs a{};
  a.ev = h->d_ev;
  a.steps = h->d_steps;
  a.sp_rows = h->d_sp_rows;
  a.sp_vals = h->d_sp_vals;
  a.nb_ids = h->d_nb_ids;
  a.nb_w = h->d_nb_w;
  a.ctl = h->ctl;
  a.d = h->d;
  a.ld = h->ld;
  a.Xb = h->Xb;
  a.Yb = h->Yb;
  a.Zb = h->Zb;
  a.rb = h->rb;
  a.alpha_is_one = h->alpha1;
  a.key = h->key;
  a.fused_ppr = 0;
  a.alpha = h->cfg.alpha;
  a.eps = h->cfg.eps;
  a.delta = h->delta;
  a.stamp = h->stamp;
  a.mark = h->mark;
  a.listF = h->listF;
  a.listG = h->listG;
  a.listL = h->listL;
  a.touched = h->d_touched;
  a.pstats = h->pstats;
  for (int s = 0; s < 2; ++s)
    for (int p = 0; p < 2; ++p) {
      a.PT[s][p] = h->PT[s][p];
      a.Q[s][p] = h->Q[s][p];
    }
  a.sigma = h->sigma;
  // Base rows are fp32 (the reference keeps fp64): a row written through
  // solve(P^T, .) carries components ~cond(P) larger than its current value,
  // and the maintained P^-1 drifts in proportion to cond(P), so fp32 storage
  // costs ~6e-8 * cond(P) relative accuracy. Rebasing (an exact change of
  // representation, engine.cpp:38-47) when either projection's Frobenius
  // condition bound passes kStorageSafeCond keeps current-coordinate results
  // within the 1e-4 parity bar; the reference's own trigger (cond(P_X) >
  // rebase_cond) applies as well.
  constexpr double kStorageSafeCond = 1e4;
  a.rebase_cond = h->cfg.rebase_cond;
  a.storage_cond = kStorageSafeCond;
  for (int sd = 0; sd < 2; ++sd) {
    a.dirty[sd] = h->dirty[sd];
    a.slot[sd] = h->slot[sd];
    a.rows64[sd] = h->rows64[sd];
  }
  a.dirty_cap = kDirtyCap;
  a.out = h->out;
  a.in = h->in;
  a.directed = h->directed;
  a.undirected = h->cfg.undirected;
  a.deg = h->deg;
  const size_t m = (size_t)h->ld * h->ld;
  a.ws_Q1T = h->ws;
  a.ws_priv = h->ws + m;
  return a;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

PprArgs ppr_args(damf_gpu* h) {
  PprArgs a{};
  a.n = h->n;
  a.d = h->d;
  a.k = h->k;
  a.Xb = h->Xb;
  a.Zb = h->Zb;
  a.rb = h->rb;
  a.delta = h->delta;
  a.key = h->key;
  a.stamp = h->stamp;
  a.mark = h->mark;
  a.listF = h->listF;
  a.listL = h->listL;
  a.blk = h->blk;
  a.blk64 = h->blk64;
  a.heavy = h->heavy;
  a.hidx = h->hidx;
  a.hoff = h->hoff;
  a.cidx = h->cidx;
  a.hacc = h->hacc;
  a.wq = h->wq;
  a.items[0] = h->items0;
  a.items[1] = h->items1;
  a.hdone = h->hdone;
  a.mitems = h->mitems;
  a.trace = h->ptrace;
  a.pst = h->pst;
  a.split = 0;
  a.out = h->out;
  a.in = h->in;
  a.directed = h->directed;
  a.deg = h->deg;
  a.alpha = h->cfg.alpha;
  a.alpha_eps = h->cfg.alpha * h->cfg.eps;
  a.smax = h->smax;
  a.round_base = h->round_base;
  a.cand = nullptr;
  a.ncand = -1;
  a.push_guard = 1000000000LL;  // enhancer.cpp:8
  a.narcs_hint = h->arcs;
  {
    static const int fp = [] { const char* e = getenv("DAMF_PPR_FORCE_PULL"); return e && *e == '1' ? 1 : 0; }();
    a.force_pull = fp;
  }
  a.stats = h->pstats;
  a.ctl = h->ctl;
  return a;
}

bool ed_absorb_nonempty(damf_gpu* h, int64_t e) { return h->ev.h[e].touched_cnt > 0; }

int sync_ctl(damf_gpu* h) {
  CK(cudaMemcpyAsync(h->h_ctl, h->ctl, kCtlBytes, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  h->k = h->h_ctl->k;
  h->round_base = (int)h->h_pstats[2];
  h->ctl_fresh = true;
  return 0;
}

double* live_PT(damf_gpu* h, int side) { return h->PT[side][h->h_ctl->pp[side]]; }
double* live_Q(damf_gpu* h, int side) { return h->Q[side][h->h_ctl->pp[side]]; }

// PPR push with the current s_max (computed and consumed on the device: no
// host round trip per event); grid sized to the expected work.
// split = 1 (whole-graph calls): dense pull rounds run as a standalone
// kernel with more warps per SM; the cooperative kernel exits before such a
// round and is relaunched after it (one small host read per dense round).
int run_push(damf_gpu* h, int grid, unsigned long long* t_end, int split = 0,
             const int32_t* cand = nullptr, int ncand = -1, bool read_ctl = false) {
  h->launches += 2;
  CK(launch_smax(h->PT[0][0], h->PT[0][1], h->ctl, h->ld, h->smax, h->st));
  PprArgs a = ppr_args(h);
  a.t_end = t_end;
  a.split = split;
  if (cand) {
    a.cand = const_cast<int32_t*>(cand);
    a.ncand = ncand;
  }
  const int gmax = ppr_push_max_grid(h->nsm, h->d);
  for (;;) {
    CK(launch_ppr_push(a, std::min(grid, gmax), h->st));
    if (!split) break;
    CK(cudaMemcpyAsync(h->h_pst, h->pst, sizeof(PprState), cudaMemcpyDeviceToHost, h->st));
    // (split calls end with a control-block read: the same round trip)
    if (read_ctl) CK(cudaMemcpyAsync(h->h_ctl, h->ctl, kCtlBytes, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (read_ctl) {
      h->k = h->h_ctl->k;
      h->round_base = (int)h->h_pstats[2];
      h->ctl_fresh = true;
    }
    if (!h->h_pst->pull_pending) break;
    h->h_pst->pull_pending = 0;
    CK(cudaMemcpyAsync(&h->pst->pull_pending, &h->h_pst->pull_pending, sizeof(int),
                       cudaMemcpyHostToDevice, h->st));
    CK(launch_ppr_pull(a, h->nsm, h->st));
    h->launches += 2;
  }
  return 0;
}

__global__ void fill_f64_kernel(double* p, int64_t n, double v) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x)
    p[x] = v;
}

// Materialise per-arc weights (all 1.0) for an engine built from an
// unweighted CSR, on the first event that carries a non-unit weight: the
// device CSR then stores weights like the reference's adjacency
// (graph.hpp:93-98). Every slot of the pool is set, so relocated and
// appended rows read consistent values.
int ensure_weights(damf_gpu* h) {
  if (h->out.wts) return 0;
  for (int side = 0; side < (h->directed ? 2 : 1); ++side) {
    DevCSR& c = side == 0 ? h->out : h->in;
    CK(dalloc(h, &c.wts, (size_t)c.pool_size));
    fill_f64_kernel<<<h->nsm * 8, 256, 0, h->st>>>(c.wts, c.pool_size, 1.0);
    CK(cudaGetLastError());
  }
  if (!h->directed) h->in = h->out;
  CK(cudaStreamSynchronize(h->st));
  return 0;
}

}  // namespace

extern "C" {

const char* damf_gpu_version(void) {
  return "damf_gpu sm_100a (cluster event update on FP64 tensor cores, tcgen05 materialise, fused + whole-GPU PPR push)";
}

const char* damf_gpu_last_error(const damf_gpu* h) { return h ? h->err.c_str() : "null handle"; }

int damf_gpu_sync(damf_gpu* h) {
  if (h) h->ctl_fresh = false;
  CK(cudaStreamSynchronize(h->st));
  return 0;
}

void damf_gpu_destroy(damf_gpu* h) {
  if (!h) return;
  cudaStreamSynchronize(h->st);
  for (void* p : h->allocs) cudaFree(p);
  if (h->h_ctl) cudaFreeHost(h->h_ctl);  // h_pstats lives in the same block
  if (h->h_pst) cudaFreeHost(h->h_pst);
  h->pack.release();
  h->ev.release();
  h->steps.release();
  h->sp_rows.release();
  h->nb_ids.release();
  h->touched.release();
  h->sp_vals.release();
  h->nb_w.release();
  if (h->t_begin) cudaFree(h->t_begin);
  if (h->t_end) cudaFree(h->t_end);
  if (h->rowlog) cudaFree(h->rowlog);
  if (h->span0) cudaEventDestroy(h->span0);
  if (h->span1) cudaEventDestroy(h->span1);
  if (h->mat0) cudaEventDestroy(h->mat0);
  if (h->mat1) cudaEventDestroy(h->mat1);
  if (h->st) cudaStreamDestroy(h->st);
  delete h;
}

// Engine(g, cfg) (engine.cpp:5-10): FactorState::init_from_graph (device
// randomized t-SVD, csrc/tsvd.cu) followed by the factor-based constructor.
int damf_gpu_create(const damf_csr* g, const damf_config* cfg, damf_gpu** out) {
  *out = nullptr;
  if (!g || !cfg || cfg->d < 1 || cfg->d > kMaxD) return DAMF_E_K_TOO_LARGE;
  const int64_t n = g->n, arcs = g->arcs;
  if (n <= 0 || arcs <= 0) return DAMF_E_ZERO_MATRIX;  // init_from_graph: graph has no edges
  // host views of the CSR (inputs may be device memory)
  std::vector<int64_t> off(n + 1);
  std::vector<int32_t> ids(arcs);
  std::vector<double> w(g->weights ? arcs : 0);
  if (cudaMemcpy(off.data(), g->offsets, (n + 1) * 8, cudaMemcpyDefault) != cudaSuccess ||
      cudaMemcpy(ids.data(), g->targets, arcs * 4, cudaMemcpyDefault) != cudaSuccess ||
      (g->weights && cudaMemcpy(w.data(), g->weights, arcs * 8, cudaMemcpyDefault) != cudaSuccess))
    return DAMF_E_CUDA;
  // A^T as a CSR (the in-adjacency); symmetric graphs reuse A
  std::vector<int64_t> toff;
  std::vector<int32_t> tids;
  std::vector<double> tw;
  if (!cfg->undirected) {
    toff.assign(n + 1, 0);
    for (int64_t p = 0; p < arcs; ++p) toff[ids[p] + 1]++;
    for (int64_t u = 0; u < n; ++u) toff[u + 1] += toff[u];
    tids.resize(arcs);
    if (g->weights) tw.resize(arcs);
    std::vector<int64_t> fill(toff.begin(), toff.end() - 1);
    for (int64_t u = 0; u < n; ++u)
      for (int64_t p = off[u]; p < off[u + 1]; ++p) {
        const int64_t at = fill[ids[p]]++;
        tids[at] = (int32_t)u;
        if (g->weights) tw[at] = w[p];
      }
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return DAMF_E_CUDA;
  std::vector<void*> tmp;
  auto up = [&](const void* src, size_t bytes) -> void* {
    void* p = nullptr;
    if (!bytes) return nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    tmp.push_back(p);
    cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, st);
    return p;
  };
  TsvdGraph tg{};
  tg.n = n;
  tg.arcs = arcs;
  tg.off = (const int64_t*)up(off.data(), (n + 1) * 8);
  tg.ids = (const int32_t*)up(ids.data(), arcs * 4);
  tg.wts = g->weights ? (const double*)up(w.data(), arcs * 8) : nullptr;
  if (cfg->undirected) {
    tg.toff = tg.off;
    tg.tids = tg.ids;
    tg.twts = tg.wts;
  } else {
    tg.toff = (const int64_t*)up(toff.data(), (n + 1) * 8);
    tg.tids = (const int32_t*)up(tids.data(), arcs * 4);
    tg.twts = g->weights ? (const double*)up(tw.data(), arcs * 8) : nullptr;
  }
  int status = 0;
  TsvdResult res;
  if (!tg.off || !tg.ids || !tg.toff || !tg.tids ||
      tsvd_init(tg, (int)cfg->d, cfg->seed, st, nsm, &res, (cfg->flags & DAMF_CFG_REFERENCE_OMEGA) != 0) != cudaSuccess)
    status = DAMF_E_CUDA;
  else if (res.status)
    status = res.status == 6 ? DAMF_E_ZERO_MATRIX : DAMF_E_UNSUPPORTED;
  cudaStreamSynchronize(st);
  for (void* p : tmp) cudaFree(p);
  cudaStreamDestroy(st);
  if (status) return status;
  const int k = res.k;
  std::vector<double> I((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) I[(size_t)i * k + i] = 1.0;
  const float* xb = res.xb_dev ? res.xb_dev : res.xb_host.data();
  const float* yb = res.yb_dev ? res.yb_dev : res.yb_host.data();
  damf_csr hg{n, arcs, off.data(), ids.data(), g->weights ? w.data() : nullptr};
  const int r = damf_gpu_create_from_factors(&hg, cfg, k, xb, yb, I.data(), I.data(),
                                             res.sigma.data(), out);
  if (res.xb_dev) cudaFree(res.xb_dev);
  if (res.yb_dev) cudaFree(res.yb_dev);
  return r;
}

static thread_local bool t_skip_ppr_init = false;  // load_state supplies Z_b / r_b

int damf_gpu_create_from_factors(const damf_csr* g, const damf_config* cfg, int64_t k,
                                 const float* xb, const float* yb, const double* px,
                                 const double* py, const double* sigma, damf_gpu** outp) {
  *outp = nullptr;
  // device-resident inputs may still be produced on other streams
  if (is_device_ptr(g->offsets) || is_device_ptr(g->targets) || is_device_ptr(xb) ||
      is_device_ptr(yb)) {
    if (cudaDeviceSynchronize() != cudaSuccess) return DAMF_E_CUDA;
  }
  auto* h = new damf_gpu();
  h->cfg = *cfg;
  if (cfg->d < 1 || cfg->d > kMaxD || k < 1 || k > cfg->d) {
    int r = fail(h, DAMF_E_K_TOO_LARGE, "d must be in [1,256] and 1 <= k <= d");
    delete h;
    return r;
  }
  h->d = (int)cfg->d;
  h->ld = ((h->d + 1) + 3) & ~3;
  h->k = (int)k;
  h->n = g->n;
  h->arcs = g->arcs;
  h->alpha1 = cfg->alpha == 1.0;
  h->directed = !cfg->undirected;
  const int64_t extra = cfg->node_capacity > 0 ? cfg->node_capacity
                                               : std::max<int64_t>(1024, g->n / 16);
  h->n_cap = g->n + extra;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, dev);
  CK(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
  // the control block and the push counters share one allocation (device and
  // pinned host) so a single copy refreshes both (sync_ctl)
  {
    char* hb = nullptr;
    CK(cudaMallocHost(&hb, kCtlBytes));
    std::memset(hb, 0, kCtlBytes);
    h->h_ctl = reinterpret_cast<DevCtl*>(hb);
    h->h_pstats = reinterpret_cast<long long*>(hb + kCtlOff);
  }
  const int64_t n = g->n, ncap = h->n_cap, d = h->d, ld = h->ld;
  // ---- factor state
  {
    char* db = nullptr;
    CK(dalloc(h, &db, kCtlBytes));
    CK(cudaMemsetAsync(db, 0, kCtlBytes, h->st));
    h->ctl = reinterpret_cast<DevCtl*>(db);
    h->pstats = reinterpret_cast<long long*>(db + kCtlOff);
  }
  for (int sd = 0; sd < 2; ++sd) {
    CK(dalloc(h, &h->dirty[sd], (size_t)kDirtyCap));
    CK(dalloc(h, &h->rows64[sd], (size_t)kDirtyCap * ((h->d + 1 + 3) & ~3)));
    CK(dalloc(h, &h->slot[sd], (size_t)ncap));
    CK(cudaMemsetAsync(h->slot[sd], 0xff, (size_t)ncap * 4, h->st));
  }
  CK(dalloc(h, &h->Xb, (size_t)ncap * d));
  CK(dalloc(h, &h->Yb, (size_t)ncap * d));
  CK(cudaMemsetAsync(h->Xb, 0, (size_t)ncap * d * 4, h->st));
  CK(cudaMemsetAsync(h->Yb, 0, (size_t)ncap * d * 4, h->st));
  // xb / yb: host or device memory (cudaMemcpyDefault); NULL = zero rows,
  // filled later with damf_gpu_load_rows
  if (xb && n) CK(cudaMemcpy2DAsync(h->Xb, d * 4, xb, k * 4, k * 4, n, cudaMemcpyDefault, h->st));
  if (yb && n) CK(cudaMemcpy2DAsync(h->Yb, d * 4, yb, k * 4, k * 4, n, cudaMemcpyDefault, h->st));
  for (int s = 0; s < 2; ++s)
    for (int p = 0; p < 2; ++p) {
      CK(dalloc(h, &h->PT[s][p], (size_t)ld * ld));
      CK(dalloc(h, &h->Q[s][p], (size_t)ld * ld));
      CK(cudaMemsetAsync(h->PT[s][p], 0, (size_t)ld * ld * 8, h->st));
      CK(cudaMemsetAsync(h->Q[s][p], 0, (size_t)ld * ld * 8, h->st));
    }
  CK(dalloc(h, &h->sigma, (size_t)ld));
  CK(cudaMemsetAsync(h->sigma, 0, (size_t)ld * 8, h->st));
  CK(cudaMemcpyAsync(h->sigma, sigma, k * 8, cudaMemcpyHostToDevice, h->st));
  CK(dalloc(h, &h->ws, (size_t)ld * ld + (size_t)4 * 16 * 20 * ld));
  CK(dalloc(h, &h->smax, 1));

  {
    // P (row-major k x k on host) -> device, transpose into PT, invert into Q.
    double* tmp = nullptr;
    double* tmp2 = nullptr;
    int* sing = nullptr;
    CK(cudaMalloc(&tmp, (size_t)ld * ld * 8));
    CK(cudaMalloc(&tmp2, (size_t)ld * ld * 8));
    CK(cudaMalloc(&sing, sizeof(int)));
    for (int s = 0; s < 2; ++s) {
      const double* p = s == 0 ? px : py;
      CK(cudaMemsetAsync(sing, 0, sizeof(int), h->st));
      CK(cudaMemcpy2DAsync(tmp, ld * 8, p, k * 8, k * 8, k, cudaMemcpyHostToDevice, h->st));
      transpose_kernel<<<64, 256, 0, h->st>>>(tmp, h->PT[s][0], (int)k, (int)ld);
      CK(cudaMemcpyAsync(tmp2, tmp, (size_t)ld * ld * 8, cudaMemcpyDeviceToDevice, h->st));
      gj_inverse_kernel<<<1, 256, 0, h->st>>>(tmp2, h->Q[s][0], (int)k, (int)ld, sing);
      int hs = 0;
      CK(cudaMemcpyAsync(&hs, sing, sizeof(int), cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      if (hs) {
        cudaFree(tmp);
        cudaFree(tmp2);
        cudaFree(sing);
        int r = fail(h, DAMF_E_SINGULAR_PROJECTION, "initial projection matrix is singular");
        damf_gpu_destroy(h);
        return r;
      }
    }
    cudaFree(tmp);
    cudaFree(tmp2);
    cudaFree(sing);
  }
  DevCtl c0{};
  c0.k = (int)k;
  c0.rows_x = n;
  c0.rows_y = n;
  c0.cond_est = 1.0;
  c0.cond_est_y = 1.0;
  c0.ppr_skip = -1;
  c0.stop_event = -1;
  *h->h_ctl = c0;
  CK(cudaMemcpyAsync(h->ctl, h->h_ctl, sizeof(DevCtl), cudaMemcpyHostToDevice, h->st));
  // ---- graph (slack CSR)
  {
    const int64_t arcs = g->arcs;
    // CSR arrays may live in host or device memory. Offsets are needed on the
    // host for the slack layout; device targets are expanded in place; a
    // directed graph's in-CSR transpose is built on the host.
    std::vector<int64_t> hoff_v;
    const int64_t* hoff = g->offsets;
    if (is_device_ptr(g->offsets)) {
      hoff_v.resize(n + 1);
      CK(cudaMemcpy(hoff_v.data(), g->offsets, (n + 1) * 8, cudaMemcpyDeviceToHost));
      hoff = hoff_v.data();
    }
    const bool tgt_dev = arcs > 0 && is_device_ptr(g->targets);
    std::vector<int32_t> htgt_v;
    std::vector<double> hw_v;
    const int32_t* htgt = g->targets;
    const double* hw = g->weights;
    if (h->directed && tgt_dev) {
      htgt_v.resize(arcs);
      CK(cudaMemcpy(htgt_v.data(), g->targets, arcs * 4, cudaMemcpyDeviceToHost));
      htgt = htgt_v.data();
      if (g->weights) {
        hw_v.resize(arcs);
        CK(cudaMemcpy(hw_v.data(), g->weights, arcs * 8, cudaMemcpyDeviceToHost));
        hw = hw_v.data();
      }
    }
    std::vector<int64_t> noff(n + 1);
    int64_t pos = 0;
    for (int64_t u = 0; u < n; ++u) {
      noff[u] = pos;
      const int64_t c = hoff[u + 1] - hoff[u];
      pos += c + std::max<int64_t>(4, c >> 3);
    }
    noff[n] = pos;
    const int64_t reserve = cfg->arc_capacity > 0 ? cfg->arc_capacity
                                                  : std::max<int64_t>(1 << 20, arcs / 4) + 64 * extra;
    const bool weighted = g->weights != nullptr;
    for (int side = 0; side < (h->directed ? 2 : 1); ++side) {
      DevCSR& c = side == 0 ? h->out : h->in;
      c.pool_size = pos + reserve;
      CK(dalloc(h, &c.off, (size_t)ncap));
      CK(dalloc(h, &c.cnt, (size_t)ncap));
      CK(dalloc(h, &c.cap, (size_t)ncap));
      CK(dalloc(h, &c.ids, (size_t)c.pool_size));
      if (weighted) CK(dalloc(h, &c.wts, (size_t)c.pool_size));
      CK(dalloc(h, &c.pool_top, 1));
      CK(cudaMemsetAsync(c.cnt, 0, (size_t)ncap * 4, h->st));
      CK(cudaMemsetAsync(c.cap, 0, (size_t)ncap * 4, h->st));
    }
    // out-CSR: compact upload + device expansion into the slack layout
    auto build = [&](DevCSR& c, const std::vector<int64_t>& coff, const int32_t* cids,
                     const double* cw, const std::vector<int64_t>& slack_off) -> int {
      int64_t *d_coff = nullptr, *d_noff = nullptr;
      int32_t* d_cids = nullptr;
      double* d_cw = nullptr;
      const bool dev_in = arcs > 0 && is_device_ptr(cids);
      CK(cudaMalloc(&d_coff, (n + 1) * 8));
      CK(cudaMalloc(&d_noff, (n + 1) * 8));
      if (dev_in) {
        d_cids = const_cast<int32_t*>(cids);
        d_cw = const_cast<double*>(cw);
      } else {
        CK(cudaMalloc(&d_cids, std::max<int64_t>(arcs, 1) * 4));
        if (cw) CK(cudaMalloc(&d_cw, std::max<int64_t>(arcs, 1) * 8));
        if (arcs) CK(cudaMemcpyAsync(d_cids, cids, arcs * 4, cudaMemcpyHostToDevice, h->st));
        if (cw && arcs) CK(cudaMemcpyAsync(d_cw, cw, arcs * 8, cudaMemcpyHostToDevice, h->st));
      }
      CK(cudaMemcpyAsync(d_coff, coff.data(), (n + 1) * 8, cudaMemcpyHostToDevice, h->st));
      CK(cudaMemcpyAsync(d_noff, slack_off.data(), (n + 1) * 8, cudaMemcpyHostToDevice, h->st));
      if (n > 0)
        csr_expand_kernel<<<(int)std::min<int64_t>(n, 65535), 128, 0, h->st>>>(
            n, d_coff, d_cids, d_cw, d_noff, c.ids, c.wts, c.cnt, c.cap, c.off);
      CK(cudaGetLastError());
      int64_t top = slack_off[n];
      CK(cudaMemcpyAsync(c.pool_top, &top, 8, cudaMemcpyHostToDevice, h->st));
      CK(cudaStreamSynchronize(h->st));
      cudaFree(d_coff);
      cudaFree(d_noff);
      if (!dev_in) {
        cudaFree(d_cids);
        if (d_cw) cudaFree(d_cw);
      }
      return 0;
    };
    std::vector<int64_t> coff(hoff, hoff + n + 1);
    if (int r = build(h->out, coff, tgt_dev && !h->directed ? g->targets : htgt,
                      tgt_dev && !h->directed ? g->weights : hw, noff))
      return r;
    if (h->directed) {
      // in-CSR by counting transpose (host; directed graphs are the small
      // reference-test configurations)
      std::vector<int64_t> ioff(n + 1, 0);
      for (int64_t p = 0; p < arcs; ++p) ioff[htgt[p] + 1]++;
      for (int64_t u = 0; u < n; ++u) ioff[u + 1] += ioff[u];
      std::vector<int32_t> iids(std::max<int64_t>(arcs, 1));
      std::vector<double> iw(weighted ? std::max<int64_t>(arcs, 1) : 0);
      std::vector<int64_t> fill(ioff.begin(), ioff.end() - 1);
      for (int64_t u = 0; u < n; ++u)
        for (int64_t p = hoff[u]; p < hoff[u + 1]; ++p) {
          const int64_t at = fill[htgt[p]]++;
          iids[at] = (int32_t)u;
          if (weighted) iw[at] = hw[p];
        }
      std::vector<int64_t> inoff(n + 1);
      int64_t ip = 0;
      for (int64_t u = 0; u < n; ++u) {
        inoff[u] = ip;
        const int64_t c = ioff[u + 1] - ioff[u];
        ip += c + std::max<int64_t>(4, c >> 3);
      }
      inoff[n] = ip;
      if (int r = build(h->in, ioff, iids.data(), weighted ? iw.data() : nullptr, inoff)) return r;
    } else {
      h->in = h->out;
    }
    CK(dalloc(h, &h->deg, (size_t)ncap));
    CK(cudaMemsetAsync(h->deg, 0, (size_t)ncap * 8, h->st));
    degree_kernel<<<h->nsm * 4, 256, 0, h->st>>>(n, h->out, h->deg);
    CK(cudaGetLastError());
  }
  // ---- enhancer (enhancer.cpp:26-47)
  if (h->alpha1) {
    h->Zb = h->Xb;  // Z_b mirrors X_b bit for bit
  } else {
    CK(dalloc(h, &h->Zb, (size_t)ncap * d));
    CK(dalloc(h, &h->rb, (size_t)ncap * d));
    CK(dalloc(h, &h->delta, (size_t)ncap * d));
    CK(dalloc(h, &h->key, (size_t)ncap));
    CK(dalloc(h, &h->stamp, (size_t)ncap));
    CK(dalloc(h, &h->mark, (size_t)ncap));
    // fused in-cluster lists: C regions of (ceil(ceil(n/32)/C)*32/NW + 1)*NW
    CK(dalloc(h, &h->listF, (size_t)ncap + 16 * 32 * 2 + 4096));
    CK(dalloc(h, &h->listG, (size_t)ncap + 16 * 32 * 2 + 4096));
    CK(dalloc(h, &h->listL, (size_t)ncap + 16 * 32 * 2 + 4096));
    CK(dalloc(h, &h->pend_d, (size_t)ncap / 16 + 16));  // damf_gpu_ppr_push's starting rows
    CK(dalloc(h, &h->blk, (size_t)4096));
    CK(dalloc(h, &h->blk64, (size_t)4096));
    {
      // heavy rows have > PPR_HEAVY arcs: at most pool/(PPR_HEAVY+1) of them;
      // chunks of PPR_CH arcs: at most pool/PPR_CH + heavy rows
      const size_t nh = (size_t)(h->out.pool_size / (PPR_HEAVY + 1) + 16);
      const size_t chunks = (size_t)(h->out.pool_size / PPR_CH) + nh;
      CK(dalloc(h, &h->heavy, nh));
      CK(dalloc(h, &h->hoff, nh + 1));
      CK(dalloc(h, &h->cidx, chunks));
      CK(dalloc(h, &h->hacc, nh * (size_t)d));
      CK(dalloc(h, &h->wq, (size_t)2048));
      CK(dalloc(h, &h->ptrace, (size_t)4 * 1024 + 1));
      CK(dalloc(h, &h->pst, (size_t)1));
      CK(cudaMemsetAsync(h->pst, 0, sizeof(PprState), h->st));
      CK(cudaMallocHost(&h->h_pst, sizeof(PprState)));
      CK(dalloc(h, &h->mitems, 2 * ((size_t)ncap + (size_t)(h->out.pool_size / PPR_MCH) + 4096)));
      CK(dalloc(h, &h->hdone, nh));
      CK(cudaMemsetAsync(h->hdone, 0, nh * 4, h->st));
      CK(dalloc(h, &h->items0, (size_t)ncap + chunks + 4096));
      CK(dalloc(h, &h->items1, (size_t)ncap + chunks + 4096));
      CK(cudaMemsetAsync(h->hacc, 0, nh * (size_t)d * 4, h->st));
    }
    CK(dalloc(h, &h->hidx, (size_t)ncap));
    CK(cudaMemsetAsync(h->hidx, 0xff, (size_t)ncap * 4, h->st));
    CK(cudaMemsetAsync(h->Zb, 0, (size_t)ncap * d * 4, h->st));
    CK(cudaMemsetAsync(h->rb, 0, (size_t)ncap * d * 4, h->st));
    CK(cudaMemsetAsync(h->key, 0, (size_t)ncap * 4, h->st));
    CK(cudaMemsetAsync(h->stamp, 0, (size_t)ncap * 4, h->st));
    CK(cudaMemsetAsync(h->mark, 0, (size_t)ncap * 4, h->st));
  }
  CK(cudaStreamSynchronize(h->st));
  *outp = h;
  if (!h->alpha1 && !t_skip_ppr_init) {
    damf_apply_stats s{};
    int r = damf_gpu_ppr_init(h, &s);
    if (r) {
      *outp = nullptr;
      damf_gpu_destroy(h);
      return r;
    }
  }
  return 0;
}

int damf_gpu_ppr_init(damf_gpu* h, damf_apply_stats* stats) {
  if (h) h->ctl_fresh = false;
  if (h->alpha1) return 0;
  if (int r = sync_ctl(h)) return r;
  PprArgs a = ppr_args(h);
  CK(launch_ppr_init(a, h->nsm, h->st));
  CK(launch_ppr_keys(a, h->nsm, h->st));
  const long long p0 = h->h_pstats[0], r0 = h->h_pstats[1];
  h->pend.clear();
  h->pend_valid = false;
  if (int r = run_push(h, 1 << 20, nullptr, 1)) return r;
  if (int r = sync_ctl(h)) return r;
  if (h->h_ctl->err) return fail(h, h->h_ctl->err, "push_to_tolerance: push budget exceeded");
  h->pend_valid = true;
  if (stats) {
    stats->pushes = h->h_pstats[0] - p0;
    stats->push_rounds = h->h_pstats[1] - r0;
  }
  return 0;
}

int damf_gpu_ppr_push(damf_gpu* h, damf_apply_stats* stats) {
  if (h->alpha1) return 0;
  // (after an apply the host mirror of the control block is current)
  if (!h->ctl_fresh)
    if (int r = sync_ctl(h)) return r;
  h->ctl_fresh = false;
  const long long p0 = h->h_pstats[0], r0 = h->h_pstats[1];
  const int32_t* cand = nullptr;
  int ncand = -1;
  if (h->pend_valid && h->pend_d && (int64_t)h->pend.size() * 16 < h->n) {
    std::sort(h->pend.begin(), h->pend.end());
    h->pend.erase(std::unique(h->pend.begin(), h->pend.end()), h->pend.end());
    if (!h->pend.empty())
      CK(cudaMemcpyAsync(h->pend_d, h->pend.data(), h->pend.size() * 4, cudaMemcpyHostToDevice, h->st));
    cand = h->pend_d;
    ncand = (int)h->pend.size();
  }
  h->pend.clear();
  h->pend_valid = false;
  if (int r = run_push(h, 1 << 20, nullptr, 1, cand, ncand, true)) return r;
  if (h->h_ctl->err) return fail(h, h->h_ctl->err, "push_to_tolerance: push budget exceeded");
  h->pend_valid = true;
  if (stats) {
    stats->pushes = h->h_pstats[0] - p0;
    stats->push_rounds = h->h_pstats[1] - r0;
  }
  return 0;
}

int damf_gpu_rebase(damf_gpu* h) {
  if (h) h->ctl_fresh = false;
  if (h) h->pend_valid = false;  // r <- r T and re-keyed: keys may exceed the threshold
  if (int r = sync_ctl(h)) return r;
  const int k = h->k, d = h->d, ld = h->ld;
  // folds use fp64 accumulation: P may be ill-conditioned here (cond up to
  // rebase_cond = 1e8), where fp32 / 3xTF32 products lose the digits
  float* tmp = nullptr;
  if (k > 128) CK(cudaMalloc(&tmp, (size_t)h->n * d * 4));
  // Two tiers: the rows written through P^-1 since the last fold live in the
  // fp64 side table (their base values carry components ~cond(P) larger than
  // their current value); they are folded from their fp64 values with fp64
  // products and leave the table. Every other row is benign and takes the
  // fast HBM-bound path. With an overflowed table (some such rows are fp32
  // only), PPR state or k > 128 the bulk fold runs in fp64 as well.
  // The fast path (3 x TF32 products, fp32 accumulation) errs by ~2^-22 of
  // sum |x_i P_ij|, which exceeds |x P| by up to cond(P): above
  // kFastFoldCond every row is folded with fp64 products instead (DMMA).
  constexpr double kFastFoldCond = 100.0;
  const double condx = h->h_ctl->cond_est, condy = h->h_ctl->cond_est_y;
  auto fold = [&](float* base, const double* PT, int side) -> int {
    const long long nd = side >= 0 ? h->h_ctl->dirty_n[side] : -1;
    const double cond = side == 1 ? condy : condx;
    if (nd >= 0 && nd <= kDirtyCap && k <= 128 && cond <= kFastFoldCond) {
      CK(launch_materialize(base, h->n, k, d, PT, ld, k, base, d, h->st, h->nsm));
    } else if (!tmp) {
      CK(launch_materialize_precise(base, h->n, k, d, PT, ld, k, base, d, h->st, h->nsm));
    } else {
      CK(launch_materialize_precise(base, h->n, k, d, PT, ld, k, tmp, d, h->st, h->nsm));
      CK(cudaMemcpyAsync(base, tmp, (size_t)h->n * d * 4, cudaMemcpyDeviceToDevice, h->st));
    }
    const long long ns = side >= 0 ? std::min<long long>(h->h_ctl->dirty_n[side], kDirtyCap) : 0;
    if (ns > 0) {
      fold_rows64_kernel<<<(int)std::min<long long>(ns, 8 * h->nsm), 128, (size_t)k * 8, h->st>>>(
          h->rows64[side], ld, h->dirty[side], ns, PT, k, base, d, h->slot[side], 1);
      CK(cudaGetLastError());
    }
    return 0;
  };
  if (int r = fold(h->Xb, live_PT(h, 0), 0)) return r;
  if (int r = fold(h->Yb, live_PT(h, 1), 1)) return r;
  if (!h->alpha1) {
    if (int r = fold(h->Zb, live_PT(h, 0), -1)) return r;
    if (int r = fold(h->rb, live_PT(h, 0), -1)) return r;
  }
  h->h_ctl->dirty_n[0] = h->h_ctl->dirty_n[1] = 0;
  CK(cudaMemcpyAsync(h->ctl->dirty_n, h->h_ctl->dirty_n, sizeof(h->h_ctl->dirty_n), cudaMemcpyHostToDevice, h->st));
  for (int s = 0; s < 2; ++s) {
    identity_kernel<<<64, 256, 0, h->st>>>(live_PT(h, s), k, ld);
    identity_kernel<<<64, 256, 0, h->st>>>(live_Q(h, s), k, ld);
  }
  CK(cudaGetLastError());
  if (!h->alpha1) CK(launch_ppr_keys(ppr_args(h), h->nsm, h->st));
  h->launches += (h->alpha1 ? 2 : 5) + 2 + 4;  // folds, side-table folds, P = Q = I
  h->h_ctl->cond_est = h->h_ctl->cond_est_y = 1.0;
  h->h_ctl->need_rebase = 0;
  CK(cudaMemcpyAsync(&h->ctl->cond_est, &h->h_ctl->cond_est, 2 * sizeof(double), cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(&h->ctl->need_rebase, &h->h_ctl->need_rebase, sizeof(int), cudaMemcpyHostToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (tmp) cudaFree(tmp);
  h->since_rebase = 0;
  return 0;
}

int damf_gpu_apply(damf_gpu* h, const damf_event_batch* b, int32_t mode, damf_apply_stats* stats) {
  damf_apply_stats s{};
  s.failed_index = -1;
  const int64_t count = b->count;
  // ---- host validation and descriptor build (graph.cpp:83-207 semantics)
  CK(h->ev.ensure(count + 1));
  CK(h->steps.ensure(2 * count + 2));
  h->ev.n = h->steps.n = h->sp_rows.n = h->sp_vals.n = h->nb_ids.n = h->nb_w.n = h->touched.n = 0;
  int64_t nn = h->n;
  int64_t ok_count = count;
  int vstatus = 0;
  std::string vmsg;
  std::vector<std::pair<int64_t, double>> inl, outl;
  bool need_w = false;  // a non-unit weight arrives at an unweighted engine
  for (int64_t i = 0; i < count && !vstatus; ++i) {
    const int kind = b->kind[i];
    EventDesc e{};
    e.kind = kind;
    e.step0 = (int64_t)h->steps.n;
    e.touched_off = (int64_t)h->touched.n;
    auto need = [&](size_t rows, size_t nbs, size_t tch) -> cudaError_t {
      cudaError_t x = h->sp_rows.ensure(h->sp_rows.n + rows + 2);
      if (x == cudaSuccess) x = h->sp_vals.ensure(h->sp_vals.n + rows + 2);
      if (x == cudaSuccess) x = h->nb_ids.ensure(h->nb_ids.n + nbs + 2);
      if (x == cudaSuccess) x = h->nb_w.ensure(h->nb_w.n + nbs + 2);
      if (x == cudaSuccess) x = h->touched.ensure(h->touched.n + tch + 2);
      return x;
    };
    if (kind == DAMF_ADD_EDGE || kind == DAMF_REMOVE_EDGE) {
      const int64_t u = b->u[i], v = b->v[i];
      const double w = (kind == DAMF_ADD_EDGE && b->w) ? b->w[i] : 1.0;
      if (u < 0 || u >= nn || v < 0 || v >= nn) {
        vstatus = DAMF_E_UNKNOWN_NODE;
        vmsg = "unknown node " + std::to_string(u < 0 || u >= nn ? u : v);
        ok_count = i;
        break;
      }
      // graph.cpp:89-90 rejects w <= 0; NaN and +Inf pass that test, and the
      // reference then inserts the arc and throws NonFinite from the bordered
      // SVD (svd.cpp:31-32). Both are rejected here, before any mutation.
      if (kind == DAMF_ADD_EDGE && !std::isfinite(w) && !(w < 0.0)) {
        vstatus = DAMF_E_NON_FINITE;
        vmsg = "AddEdge: non-finite weight";
        ok_count = i;
        break;
      }
      if (kind == DAMF_ADD_EDGE && !(w > 0.0)) {
        vstatus = DAMF_E_PARSE;
        vmsg = "AddEdge: weight must be > 0";
        ok_count = i;
        break;
      }
      if (w != 1.0) need_w = true;
      CK(need(2, 0, 2));
      const bool two = h->cfg.undirected && u != v;
      e.u = u;
      e.v = v;
      e.w = w;
      e.nsteps = two ? 2 : 1;
      const double cv = kind == DAMF_ADD_EDGE ? w : -1.0;  // removal weight patched on device
      for (int q = 0; q < e.nsteps; ++q) {
        StepDesc sd{};
        sd.kind = kStepEdge;
        sd.nb = 1;
        sd.b_off = (int64_t)h->sp_rows.n;
        h->sp_rows.push(q == 0 ? u : v);
        h->sp_vals.push(1.0);
        sd.c_row = q == 0 ? v : u;
        sd.c_val = cv;
        sd.n_a = nn;
        sd.n_b = nn;
        sd.bnorm2 = 1.0;
        h->steps.push(sd);
      }
      h->touched.push(u);
      if (two) h->touched.push(v);
    } else if (kind == DAMF_ADD_NODE) {
      inl.clear();
      outl.clear();
      if (b->in_off)
        for (int64_t t = b->in_off[i]; t < b->in_off[i + 1]; ++t)
          inl.emplace_back(b->in_ids[t], b->in_w ? b->in_w[t] : 1.0);
      if (b->out_off)
        for (int64_t t = b->out_off[i]; t < b->out_off[i + 1]; ++t)
          outl.emplace_back(b->out_ids[t], b->out_w ? b->out_w[t] : 1.0);
      // touched_by (graph.cpp:199-204): in sources (+ out targets), new id last
      std::vector<int64_t> tch;
      auto addt = [&](int64_t x) {
        if (std::find(tch.begin(), tch.end(), x) == tch.end()) tch.push_back(x);
      };
      for (auto& p : inl) addt(p.first);
      if (h->cfg.undirected)
        for (auto& p : outl) addt(p.first);
      addt(nn);
      if (h->cfg.undirected) {  // graph.cpp:137-141
        for (auto& p : outl) inl.push_back(p);
        outl = inl;
      }
      // graph.cpp:143-152: unknown neighbour, weight <= 0; non-finite weights
      // are rejected up front (the reference throws NonFinite later, svd.cpp:31-32)
      for (const auto* lst : {&inl, &outl})
        for (auto& p : *lst) {
          if (vstatus) break;
          if (p.first < 0 || p.first >= nn) {
            vstatus = DAMF_E_UNKNOWN_NODE;
            vmsg = "AddNode: unknown node " + std::to_string(p.first);
          } else if (!std::isfinite(p.second) && !(p.second < 0.0)) {
            vstatus = DAMF_E_NON_FINITE;
            vmsg = "AddNode: non-finite weight";
          } else if (!(p.second > 0.0)) {
            vstatus = DAMF_E_PARSE;
            vmsg = "AddNode: weight must be > 0";
          }
          if (p.second != 1.0) need_w = true;
        }
      if (nn + 1 > h->n_cap) {
        vstatus = DAMF_E_TOO_LARGE;
        vmsg = "node capacity exhausted (damf_config.node_capacity)";
      }
      if (vstatus) {
        ok_count = i;
        break;
      }
      CK(need(inl.size() + outl.size(), inl.size() + outl.size(), tch.size()));
      e.u = nn;
      e.in_off = (int64_t)h->nb_ids.n;
      e.in_cnt = (int64_t)inl.size();
      for (auto& p : inl) {
        h->nb_ids.push(p.first);
        h->nb_w.push(p.second);
      }
      e.out_off = (int64_t)h->nb_ids.n;
      e.out_cnt = (int64_t)outl.size();
      for (auto& p : outl) {
        h->nb_ids.push(p.first);
        h->nb_w.push(p.second);
      }
      auto sorted_in = inl, sorted_out = outl;
      std::sort(sorted_in.begin(), sorted_in.end());
      std::sort(sorted_out.begin(), sorted_out.end());
      // column step (update_embedding_n, u_is_x = true)
      StepDesc c{};
      c.kind = kStepNodeCol;
      c.nb = (int32_t)sorted_in.size();
      c.b_off = (int64_t)h->sp_rows.n;
      double b2 = 0;
      for (auto& p : sorted_in) {
        h->sp_rows.push(p.first);
        h->sp_vals.push(p.second);
        b2 += p.second * p.second;
      }
      c.bnorm2 = b2;
      c.c_row = nn;  // new Y row
      c.n_a = nn;
      c.n_b = nn;
      h->steps.push(c);
      // row step (u_is_x = false): b over Y rows (now nn + 1)
      StepDesc r{};
      r.kind = kStepNodeRow;
      r.nb = (int32_t)sorted_out.size();
      r.b_off = (int64_t)h->sp_rows.n;
      b2 = 0;
      for (auto& p : sorted_out) {
        h->sp_rows.push(p.first);
        h->sp_vals.push(p.second);
        b2 += p.second * p.second;
      }
      r.bnorm2 = b2;
      r.c_row = nn;  // new X row
      r.n_a = nn + 1;
      r.n_b = nn;
      h->steps.push(r);
      e.nsteps = 2;
      for (int64_t x : tch) h->touched.push(x);
      ++nn;
    } else {
      vstatus = DAMF_E_PARSE;
      vmsg = "unknown event kind";
      ok_count = i;
      break;
    }
    e.touched_cnt = (int64_t)h->touched.n - e.touched_off;
    h->ev.push(e);
  }
  // an engine created from an unweighted CSR stores no weights (all 1.0);
  // the first non-unit weight materialises them (graph.hpp: weights are f64)
  if (need_w && !h->out.wts)
    if (int r = ensure_weights(h)) return r;
  // ---- upload
  {
    // one pinned staging block and one copy for all descriptor arrays (a
    // batch of one event costs one H2D call, not seven)
    size_t off = 0;
    auto place = [&](size_t bytes) {
      const size_t o = off;
      off += (bytes + 15) & ~size_t(15);
      return o;
    };
    const size_t o_ev = place(h->ev.n * sizeof(EventDesc)), o_st = place(h->steps.n * sizeof(StepDesc));
    const size_t o_sr = place(h->sp_rows.n * 8), o_sv = place(h->sp_vals.n * 8);
    const size_t o_ni = place(h->nb_ids.n * 8), o_nw = place(h->nb_w.n * 8);
    const size_t o_tc = place(h->touched.n * 8);
    CK(h->pack.ensure(off + 16));
    char* hp = h->pack.h;
    std::memcpy(hp + o_ev, h->ev.h, h->ev.n * sizeof(EventDesc));
    std::memcpy(hp + o_st, h->steps.h, h->steps.n * sizeof(StepDesc));
    std::memcpy(hp + o_sr, h->sp_rows.h, h->sp_rows.n * 8);
    std::memcpy(hp + o_sv, h->sp_vals.h, h->sp_vals.n * 8);
    std::memcpy(hp + o_ni, h->nb_ids.h, h->nb_ids.n * 8);
    std::memcpy(hp + o_nw, h->nb_w.h, h->nb_w.n * 8);
    std::memcpy(hp + o_tc, h->touched.h, h->touched.n * 8);
    if (off) CK(cudaMemcpyAsync(h->pack.d, hp, off, cudaMemcpyHostToDevice, h->st));
    char* dp = h->pack.d;
    h->d_ev = reinterpret_cast<EventDesc*>(dp + o_ev);
    h->d_steps = reinterpret_cast<StepDesc*>(dp + o_st);
    h->d_sp_rows = reinterpret_cast<int64_t*>(dp + o_sr);
    h->d_sp_vals = reinterpret_cast<double*>(dp + o_sv);
    h->d_nb_ids = reinterpret_cast<int64_t*>(dp + o_ni);
    h->d_nb_w = reinterpret_cast<double*>(dp + o_nw);
    h->d_touched = reinterpret_cast<int64_t*>(dp + o_tc);
  }
  const bool timing = mode & DAMF_APPLY_TIME_EVENTS;
  if (timing && (size_t)ok_count > h->t_cap) {
    if (h->t_begin) cudaFree(h->t_begin);
    if (h->t_end) cudaFree(h->t_end);
    h->t_cap = (size_t)ok_count + 1024;
    CK(cudaMalloc(&h->t_begin, h->t_cap * 8));
    CK(cudaMalloc(&h->t_end, h->t_cap * 8));
  }
  if (!h->ctl_fresh)
    if (int r = sync_ctl(h)) return r;
  const bool log_rows = mode & DAMF_APPLY_LOG_ROWS;
  if (log_rows) {
    // every modified row is a nonzero of some b, or one c / appended row
    const long long need = (long long)h->sp_rows.n + (long long)h->steps.n + 16;
    if (need > h->rowlog_cap) {
      if (h->rowlog) cudaFree(h->rowlog);
      h->rowlog_cap = need;
      CK(cudaMalloc(&h->rowlog, (size_t)need * 3 * sizeof(int64_t)));
    }
    h->h_ctl->rowlog_n = 0;
    CK(cudaMemcpyAsync(&h->ctl->rowlog_n, &h->h_ctl->rowlog_n, sizeof(long long),
                       cudaMemcpyHostToDevice, h->st));
  }
  if (timing) {
    // device span of the call: from the first launch (descriptors already
    // uploaded) to the completion of its last kernel, rebases included
    if (!h->span0) {
      CK(cudaEventCreate(&h->span0));
      CK(cudaEventCreate(&h->span1));
    }
    CK(cudaEventRecord(h->span0, h->st));
  }
  const long long rank1_0 = h->h_ctl->rank1, folds0 = h->h_ctl->folds;
  const long long p0 = h->h_pstats[0], r0 = h->h_pstats[1];
  EventKernelArgs ea = event_args(h);
  ea.mode = mode;
  ea.t_begin = timing ? h->t_begin : nullptr;
  ea.t_end = timing ? h->t_end : nullptr;
  ea.rowlog = log_rows ? h->rowlog : nullptr;
  ea.rowlog_cap = log_rows ? h->rowlog_cap : 0;
  const bool ppr = !h->alpha1;
  const bool push_each = ppr && !(mode & DAMF_APPLY_DEFER_PUSH);
  int64_t rebases = 0;
  int64_t i = 0;
  int64_t n_before = h->n;
  const bool split_mode = ppr && event_cluster_size() == 16;
  // the PPR absorb / push of one event on its own (after a rebase it waited for)
  auto event_ppr = [&](int64_t e) -> int {
    const bool fused_e = h->n_cap <= (1 << 20) || (mode & DAMF_APPLY_DEFER_PUSH);
    if (fused_e && split_mode) {
      ea.e_begin = e;
      ea.e_end = e + 1;
      CK(launch_ppr_kernel(ea, h->st));
      h->launches += 1;
    } else {
      const EventDesc& ed = h->ev.h[e];
      PprArgs pa = ppr_args(h);
      pa.k = h->k;
      CK(launch_ppr_absorb(pa, h->d_touched + ed.touched_off, (int)ed.touched_cnt, h->st));
      h->launches += 1;
      if (push_each)
        if (int r = run_push(h, 8 * h->nsm, timing ? h->t_end + e : nullptr)) return r;
    }
    return 0;
  };
  int64_t host_ppr_skip = -1;  // the whole-GPU path records it on the host
  auto pending_ppr = [&]() -> int {
    const int64_t e = host_ppr_skip >= 0 ? host_ppr_skip : h->h_ctl->ppr_skip;
    host_ppr_skip = -1;
    if (!ppr || e < 0) return 0;
    h->h_ctl->ppr_skip = -1;
    h->h_ctl->stop_event = -1;
    CK(cudaMemcpyAsync(&h->ctl->stop_event, &h->h_ctl->stop_event, sizeof(long long),
                       cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(&h->ctl->ppr_skip, &h->h_ctl->ppr_skip, sizeof(long long), cudaMemcpyHostToDevice,
                       h->st));
    if (int r = event_ppr(e)) return r;
    return sync_ctl(h);
  };
  while (i < ok_count) {
    // events up to the next rebase_every boundary (engine.cpp:37-40)
    int64_t j = ok_count;
    if (h->cfg.rebase_every > 0) j = std::min<int64_t>(j, i + (h->cfg.rebase_every - h->since_rebase));
    // In-cluster enhancer when its per-round row scans are cheap (n <= 1M) or
    // when only absorption is requested; otherwise one cooperative push
    // kernel per event over the whole GPU.
    const bool fused = ppr && (h->n_cap <= (1 << 20) || (mode & DAMF_APPLY_DEFER_PUSH));
    h->ctl_fresh = false;
    // Split mode (16-CTA clusters): per event a factor-only kernel, then the
    // push as its own kernel -- 76 registers and 16 warps per CTA instead of
    // sharing the factor kernel's 255-register, 8-warp budget (cfg-2 mean
    // event 300 -> 283 us, same-box A/B). The in-kernel fused push remains
    // for 8-CTA clusters.
    const bool split = fused && event_cluster_size() == 16;
    // no stop recorded yet for this launch group (the kernels stop at an
    // event that requests a rebase and skip everything after it): the
    // group's first event kernel clears it before any CTA looks at it
    h->h_ctl->stop_event = -1;
    ea.reset_stop = 1;
    if (split) {
      // one-event factor kernel, then the push kernel for that event
      ea.fused_ppr = 0;
      for (int64_t e = i; e < j; ++e) {
        ea.e_begin = e;
        ea.e_end = e + 1;
        CK(launch_event_kernel(ea, h->st));
        ea.reset_stop = 0;
        CK(launch_ppr_kernel(ea, h->st));
        h->launches += 2;
      }
    } else if (!ppr || fused) {
      ea.e_begin = i;
      ea.e_end = j;
      ea.fused_ppr = fused ? 1 : 0;
      CK(launch_event_kernel(ea, h->st));
      ea.reset_stop = 0;
      h->launches += 1;
    } else {
      // whole-GPU push per event (large graphs): the host reads the control
      // block after every event, so an event that requests a rebase (or
      // fails) ends the launch group right there -- the kernels of later
      // events would be no-ops (stop_event) and their absorb / push must not run
      for (int64_t e = i; e < j; ++e) {
        ea.e_begin = e;
        ea.e_end = e + 1;
        CK(launch_event_kernel(ea, h->st));
        ea.reset_stop = 0;
        h->launches += 1;
        if (int r = sync_ctl(h)) return r;
        if (h->h_ctl->err) break;
        // rows appended by AddNode are visible to the enhancer from here
        if (h->ev.h[e].kind == DAMF_ADD_NODE) h->n = h->ev.h[e].u + 1;
        if (h->h_ctl->need_rebase) {
          // absorb / push after the fold (see damf_ppr_kernel)
          host_ppr_skip = e;
          h->h_ctl->stop_event = e + 1;
          break;
        }
        if (int r = event_ppr(e)) return r;
      }
    }
    if (int r = sync_ctl(h)) return r;
    // a launch group stops right after an event that requested a rebase
    // (cond trigger, storage bound or an exact-inverse step): rebase over the
    // whole GPU and resume with the next event, as engine.cpp:38-40 orders it
    int64_t done = j;
    const bool stopped = !h->h_ctl->err && h->h_ctl->need_rebase && h->h_ctl->stop_event > i &&
                         h->h_ctl->stop_event < j;
    if (stopped) done = h->h_ctl->stop_event;
    for (int64_t e = i; e < done; ++e)
      if (h->ev.h[e].kind == DAMF_ADD_NODE) h->n = h->ev.h[e].u + 1;
    if (h->h_ctl->err) break;
    h->events_applied += (uint64_t)(done - i);
    h->since_rebase += (done - i);
    if (stopped || (h->cfg.rebase_every > 0 && h->since_rebase >= h->cfg.rebase_every)) {
      if (int r = damf_gpu_rebase(h)) return r;
      ++rebases;
      if (int r = pending_ppr()) return r;
      if (h->h_ctl->err) break;
    }
    i = done;
  }
  if (!h->ctl_fresh)
    if (int r = sync_ctl(h)) return r;
  int status = 0;
  if (h->h_ctl->err) {
    const int64_t fe = h->h_ctl->err_event;
    status = h->h_ctl->err;
    s.failed_index = fe;
    // events before fe were applied; rewind the node count to the device view
    h->n = n_before;
    for (int64_t e = 0; e < fe; ++e)
      if (h->ev.h[e].kind == DAMF_ADD_NODE) h->n = h->ev.h[e].u + 1;
    h->err = status == DAMF_E_DUPLICATE_EDGE ? "AddEdge: edge already present"
             : status == DAMF_E_MISSING_EDGE ? "RemoveEdge: edge not present"
             : status == DAMF_E_NON_CONVERGENCE ? "push_to_tolerance: push budget exceeded"
                                                : "event failed on device";
    for (int64_t e2 = 0; e2 < fe; ++e2) (void)e2;
    h->events_applied += (uint64_t)std::max<int64_t>(0, fe - i);
    h->since_rebase += std::max<int64_t>(0, fe - i);
    // clear the device error for subsequent calls
    h->h_ctl->err = 0;
    CK(cudaMemcpyAsync(&h->ctl->err, &h->h_ctl->err, sizeof(int), cudaMemcpyHostToDevice, h->st));
    s.applied = fe;
  } else {
    s.applied = ok_count;
    if (vstatus) {
      status = vstatus;
      s.failed_index = ok_count;
      h->err = vmsg;
    }
  }
  // deferred cond-triggered rebase (engine.cpp:38-40; query-transparent)
  if (!status && h->h_ctl->need_rebase) {
    if (int r = damf_gpu_rebase(h)) return r;
    ++rebases;
    if (int r = pending_ppr()) return r;
  }
  if (log_rows) {
    // rebases inside the call do not touch the log; the mirror is fresh here
    if (!h->ctl_fresh)
      if (int r = sync_ctl(h)) return r;
    const long long m = std::min<long long>(h->h_ctl->rowlog_n, h->rowlog_cap);
    h->rowlog_h.resize((size_t)m * 3);
    if (m) CK(cudaMemcpy(h->rowlog_h.data(), h->rowlog, (size_t)m * 3 * sizeof(int64_t),
                         cudaMemcpyDeviceToHost));
  } else {
    h->rowlog_h.clear();
  }
  if (timing) {
    // per-event stamps stay on the device until damf_gpu_event_latencies
    h->lat_pending = s.applied;
    h->lat_us.clear();
    CK(cudaEventRecord(h->span1, h->st));
    CK(cudaEventSynchronize(h->span1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->span0, h->span1));
    s.device_ms = ms;
  }
  if (!h->alpha1) {
    if (!(mode & DAMF_APPLY_DEFER_PUSH)) {
      // every event was pushed to tolerance (fused or whole-GPU)
      h->pend.clear();
      h->pend_valid = status == 0;
    } else if (!(mode & DAMF_APPLY_GRAPH_AND_PPR_ONLY)) {
      h->pend_valid = false;  // factor updates moved s_max: every key must be re-checked
    } else if (h->pend_valid) {
      for (int64_t e = 0; e < s.applied; ++e) {
        const EventDesc& ed = h->ev.h[e];
        for (int64_t t = 0; t < ed.touched_cnt; ++t) h->pend.push_back((int32_t)h->touched.h[ed.touched_off + t]);
      }
    }
  }
  s.rank1_updates = h->h_ctl->rank1 - rank1_0;
  s.eager_folds = h->h_ctl->folds - folds0;
  s.rebases = rebases;
  s.pushes = h->h_pstats[0] - p0;
  s.push_rounds = h->h_pstats[1] - r0;
  h->total_pushes = h->h_pstats[0];
  if (stats) *stats = s;
  return status;
}

int damf_gpu_apply_edge(damf_gpu* h, int32_t kind, int64_t u, int64_t v, double w, int32_t mode,
                        damf_apply_stats* stats) {
  damf_event_batch b{};
  b.count = 1;
  b.kind = &kind;
  b.u = &u;
  b.v = &v;
  b.w = &w;
  return damf_gpu_apply(h, &b, mode, stats);
}

int64_t damf_gpu_row_log(damf_gpu* h, int64_t* out, int64_t max) {
  const int64_t m = (int64_t)h->rowlog_h.size() / 3;
  for (int64_t i = 0; i < 3 * std::min(m, max); ++i) out[i] = h->rowlog_h[i];
  return m;
}

int64_t damf_gpu_event_latencies(damf_gpu* h, double* out, int64_t max) {
  if (h->lat_pending > 0) {
    const int64_t m = h->lat_pending;
    std::vector<unsigned long long> tb(m), te(m);
    if (cudaMemcpy(tb.data(), h->t_begin, m * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(te.data(), h->t_end, m * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
      cuda_fail(h, cudaGetLastError(), "event latency read-back", __LINE__);
      return -1;
    }
    h->lat_us.resize(m);
    for (int64_t e = 0; e < m; ++e) h->lat_us[e] = (double)(te[e] - tb[e]) * 1e-3;
    h->lat_pending = 0;
  }
  const int64_t m = (int64_t)h->lat_us.size();
  for (int64_t i = 0; i < std::min(m, max); ++i) out[i] = h->lat_us[i];
  return m;
}

int damf_gpu_load_rows(damf_gpu* h, int32_t which, int64_t row0, int64_t m, const float* src) {
  if (h) h->ctl_fresh = false;
  if (!h) return DAMF_E_SHAPE_MISMATCH;
  if (which != DAMF_XB && which != DAMF_YB)
    return fail(h, DAMF_E_SHAPE_MISMATCH, "load_rows: which must be DAMF_XB or DAMF_YB");
  if (row0 < 0 || m < 0 || row0 + m > h->n)
    return fail(h, DAMF_E_UNKNOWN_NODE, "load_rows: rows out of range");
  if (m == 0) return 0;
  float* dst = (which == DAMF_XB ? h->Xb : h->Yb) + row0 * h->d;
  // device sources may still be written by work on other streams (the
  // caller's framework stream): order against all prior device work
  if (is_device_ptr(src)) CK(cudaDeviceSynchronize());
  CK(cudaMemcpy2DAsync(dst, (size_t)h->d * 4, src, (size_t)h->k * 4, (size_t)h->k * 4, m,
                       cudaMemcpyDefault, h->st));
  if (int r = sync_ctl(h)) return r;
  const int side = which == DAMF_XB ? 0 : 1;
  const long long ns = std::min<long long>(h->h_ctl->dirty_n[side], kDirtyCap);
  if (ns > 0) {
    refresh_rows64_kernel<<<(int)std::min<long long>(ns, 8 * h->nsm), 128, 0, h->st>>>(
        h->rows64[side], h->ld, h->dirty[side], ns, which == DAMF_XB ? h->Xb : h->Yb, h->d, row0, m);
    CK(cudaGetLastError());
  }
  CK(cudaStreamSynchronize(h->st));
  if (h->alpha1 && which == DAMF_XB) return 0;  // Z_b aliases X_b
  return 0;
}

int damf_gpu_query_rows(damf_gpu* h, int32_t which, const int64_t* ids, int64_t m, float* out) {
  if (int r = sync_ctl(h)) return r;
  for (int64_t q = 0; q < m; ++q)
    if (ids[q] < 0 || ids[q] >= h->n) return fail(h, DAMF_E_UNKNOWN_NODE, "query: unknown node " + std::to_string(ids[q]));
  if (which == DAMF_XB || which == DAMF_YB || which == DAMF_ZB || which == DAMF_RB) {
    // raw base-coordinate rows (no projection)
    const float* src = which == DAMF_XB ? h->Xb : which == DAMF_YB ? h->Yb
                     : which == DAMF_ZB ? h->Zb : h->rb;
    if (!src) return fail(h, DAMF_E_SHAPE_MISMATCH, "matrix not allocated (alpha == 1)");
    for (int64_t q = 0; q < m; ++q)
      CK(cudaMemcpyAsync(out + q * h->k, src + ids[q] * h->d, (size_t)h->k * 4, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return 0;
  }
  const float* base = which == DAMF_Y ? h->Yb : which == DAMF_Z ? h->Zb : h->Xb;
  const double* PT = live_PT(h, which == DAMF_Y ? 1 : 0);
  int64_t* dids = nullptr;
  float* dout = nullptr;
  CK(cudaMalloc(&dids, std::max<int64_t>(m, 1) * 8));
  CK(cudaMalloc(&dout, std::max<int64_t>(m, 1) * h->k * 4));
  CK(cudaMemcpyAsync(dids, ids, m * 8, cudaMemcpyHostToDevice, h->st));
  const int qs = which == DAMF_Y ? 1 : which == DAMF_X || (which == DAMF_Z && h->alpha1) ? 0 : -1;
  query_rows_kernel<<<(int)std::min<int64_t>(std::max<int64_t>(m, 1), 4096), 128, 0, h->st>>>(
      base, h->d, PT, h->ld, h->k, dids, m, dout, nullptr, qs >= 0 ? h->slot[qs] : nullptr,
      qs >= 0 ? h->rows64[qs] : nullptr);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, dout, m * h->k * 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  cudaFree(dids);
  cudaFree(dout);
  return 0;
}

int damf_gpu_query_rows64(damf_gpu* h, int32_t which, const int64_t* ids, int64_t m, double* out) {
  if (int r = sync_ctl(h)) return r;
  if (which != DAMF_XB && which != DAMF_YB)
    return fail(h, DAMF_E_SHAPE_MISMATCH, "query_rows64: which must be DAMF_XB or DAMF_YB");
  for (int64_t q = 0; q < m; ++q)
    if (ids[q] < 0 || ids[q] >= h->n) return fail(h, DAMF_E_UNKNOWN_NODE, "query: unknown node " + std::to_string(ids[q]));
  if (m == 0) return 0;
  const int side = which == DAMF_XB ? 0 : 1;
  int64_t* dids = nullptr;
  double* dout = nullptr;
  CK(cudaMalloc(&dids, m * 8));
  CK(cudaMalloc(&dout, m * h->k * 8));
  CK(cudaMemcpyAsync(dids, ids, m * 8, cudaMemcpyHostToDevice, h->st));
  base_rows64_kernel<<<(int)std::min<int64_t>(m, 4096), 128, 0, h->st>>>(
      side ? h->Yb : h->Xb, h->d, h->slot[side], h->rows64[side], h->ld, h->k, dids, m, dout);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, dout, m * h->k * 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  cudaFree(dids);
  cudaFree(dout);
  return 0;
}

// pair_score over a batch (eval.cpp:211-215) and the top-K of a pair set
// (eval.cpp:336-371). ids: host arrays. flags: DAMF_SCORE_*.
namespace {
int score_batch(damf_gpu* h, const int64_t* u, const int64_t* v, int64_t m, int32_t flags,
                double** dscores) {
  if (int r = sync_ctl(h)) return r;
  for (int64_t q = 0; q < m; ++q)
    if (u[q] < 0 || u[q] >= h->n || v[q] < 0 || v[q] >= h->n)
      return fail(h, DAMF_E_UNKNOWN_NODE, "score: unknown node");
  const int k = h->k;
  float *A = nullptr, *B = nullptr;
  int64_t *du = nullptr, *dv = nullptr;
  CK(cudaMalloc(&A, (size_t)std::max<int64_t>(h->n, 1) * k * 4));
  CK(cudaMalloc(&B, (size_t)std::max<int64_t>(h->n, 1) * k * 4));
  CK(cudaMalloc(&du, std::max<int64_t>(m, 1) * 8));
  CK(cudaMalloc(&dv, std::max<int64_t>(m, 1) * 8));
  CK(cudaMalloc(dscores, std::max<int64_t>(m, 1) * 8));
  int r = damf_gpu_materialize(h, (flags & DAMF_SCORE_ENHANCED) ? DAMF_Z : DAMF_X, A, 1);
  if (!r) r = damf_gpu_materialize(h, DAMF_Y, B, 1);
  if (!r) {
    CK(cudaMemcpyAsync(du, u, m * 8, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(dv, v, m * 8, cudaMemcpyHostToDevice, h->st));
    CK(launch_pair_scores(A, B, k, du, dv, m, (flags & DAMF_SCORE_SYMMETRIC_MAX) ? 1 : 0, *dscores,
                          h->st, h->nsm));
    CK(cudaStreamSynchronize(h->st));
    h->launches += 3;
  }
  cudaFree(A);
  cudaFree(B);
  cudaFree(du);
  cudaFree(dv);
  return r;
}
}  // namespace

int damf_gpu_score_pairs(damf_gpu* h, const int64_t* u, const int64_t* v, int64_t m, int32_t flags,
                         double* out) {
  if (!h) return DAMF_E_SHAPE_MISMATCH;
  if (m <= 0) return 0;
  double* ds = nullptr;
  int r = score_batch(h, u, v, m, flags, &ds);
  if (!r) CK(cudaMemcpy(out, ds, m * 8, cudaMemcpyDeviceToHost));
  if (ds) cudaFree(ds);
  return r;
}

int damf_gpu_topk_pairs(damf_gpu* h, const int64_t* u, const int64_t* v, int64_t m, int32_t flags,
                        int64_t K, int64_t* idx_out, double* score_out) {
  if (!h) return DAMF_E_SHAPE_MISMATCH;
  if (m <= 0 || K <= 0) return 0;
  double* ds = nullptr;
  int r = score_batch(h, u, v, m, flags, &ds);
  if (!r) {
    CK(topk_indices(ds, m, K, idx_out, score_out, h->st));
    CK(cudaStreamSynchronize(h->st));
  }
  if (ds) cudaFree(ds);
  return r;
}

int damf_gpu_score(damf_gpu* h, int64_t u, int64_t v, int32_t enhanced, double* out) {
  if (int r = sync_ctl(h)) return r;
  if (u < 0 || u >= h->n || v < 0 || v >= h->n) return fail(h, DAMF_E_UNKNOWN_NODE, "score: unknown node");
  int64_t ids[2] = {u, v};
  int64_t* dids = nullptr;
  double* dout = nullptr;
  CK(cudaMalloc(&dids, 16));
  CK(cudaMalloc(&dout, 2 * h->k * 8));
  CK(cudaMemcpyAsync(dids, ids, 16, cudaMemcpyHostToDevice, h->st));
  const bool zs = enhanced && !h->alpha1;  // Z_b rows have no side table
  query_rows_kernel<<<1, 128, 0, h->st>>>(enhanced ? h->Zb : h->Xb, h->d, live_PT(h, 0), h->ld, h->k,
                                          dids, 1, nullptr, dout, zs ? nullptr : h->slot[0],
                                          zs ? nullptr : h->rows64[0]);
  query_rows_kernel<<<1, 128, 0, h->st>>>(h->Yb, h->d, live_PT(h, 1), h->ld, h->k, dids + 1, 1,
                                          nullptr, dout + h->k, h->slot[1], h->rows64[1]);
  CK(cudaGetLastError());
  std::vector<double> hv(2 * h->k);
  CK(cudaMemcpyAsync(hv.data(), dout, 2 * h->k * 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  double s = 0;
  for (int j = 0; j < h->k; ++j) s += hv[j] * hv[h->k + j];
  *out = s;
  cudaFree(dids);
  cudaFree(dout);
  return 0;
}

int damf_gpu_materialize(damf_gpu* h, int32_t which, float* dst, int32_t dst_is_device) {
  if (h) h->ctl_fresh = false;
  if (int r = sync_ctl(h)) return r;
  const float* base = which == DAMF_Y ? h->Yb : which == DAMF_Z ? h->Zb : h->Xb;
  const double* PT = live_PT(h, which == DAMF_Y ? 1 : 0);
  float* out = dst;
  if (!dst_is_device) CK(cudaMalloc(&out, (size_t)std::max<int64_t>(h->n, 1) * h->k * 4));
  // The fast paths (3xTF32 tensor cores / fp32 SIMT) lose ~log10(cond P)
  // digits to cancellation; above kPreciseCond the fp64-accumulating fold
  // keeps query_all at fp32 storage accuracy.
  // (benign rows) and, above kPreciseCond, the dirty rows (written through
  // P^-1 since the last fold) are recomputed in fp64 and patched in; without
  // a usable dirty list (PPR state, overflow) the whole fold is fp64.
  // Two tiers, as for a rebase but without the cond switch: the rows whose
  // base values carry cond(P)-sized cancelling components are exactly the
  // side-table rows (written through P^-1 since the last fold), patched from
  // their fp64 values with fp64 products; every other row was set by a fold
  // and is benign for the fast path (~sqrt(k) 2^-22 relative). Without a
  // usable table (overflow, PPR state Z_b above cond 100, k > 128) every row
  // takes fp64 products.
  constexpr double kPreciseCond = 100.0;
  const int side = which == DAMF_Y ? 1 : (which == DAMF_Z && !h->alpha1) ? -1 : 0;
  const long long nd = side >= 0 ? h->h_ctl->dirty_n[side] : -1;
  const double cond = side == 1 ? h->h_ctl->cond_est_y : h->h_ctl->cond_est;
  if (!h->mat0) {
    CK(cudaEventCreate(&h->mat0));
    CK(cudaEventCreate(&h->mat1));
  }
  CK(cudaEventRecord(h->mat0, h->st));
  if (cond <= kPreciseCond || (nd >= 0 && nd <= kDirtyCap && h->k <= 128)) {
    CK(launch_materialize(base, h->n, h->k, h->d, PT, h->ld, h->k, out, h->k, h->st, h->nsm));
  } else {
    CK(launch_materialize_precise(base, h->n, h->k, h->d, PT, h->ld, h->k, out, h->k, h->st, h->nsm));
  }
  CK(cudaEventRecord(h->mat1, h->st));
  // side-table rows from their fp64 base values with fp64 products
  const long long ns = side >= 0 ? std::min<long long>(nd, kDirtyCap) : 0;
  if (ns > 0) {
    fold_rows64_kernel<<<(int)std::min<long long>(ns, 8 * h->nsm), 128, (size_t)h->k * 8, h->st>>>(
        h->rows64[side], h->ld, h->dirty[side], ns, PT, h->k, out, h->k, nullptr, 0);
    CK(cudaGetLastError());
  }
  if (!dst_is_device) {
    CK(cudaMemcpyAsync(dst, out, (size_t)h->n * h->k * 4, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    cudaFree(out);
  }
  CK(cudaStreamSynchronize(h->st));
  {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, h->mat0, h->mat1) == cudaSuccess) h->last_mat_ms = ms;
  }
  return 0;
}

int damf_gpu_get_state(damf_gpu* h, int32_t which, void* out) {
  if (int r = sync_ctl(h)) return r;
  const int k = h->k, d = h->d, ld = h->ld;
  switch (which) {
    case DAMF_XB:
    case DAMF_YB:
    case DAMF_ZB:
    case DAMF_RB: {
      const float* base = which == DAMF_XB ? h->Xb : which == DAMF_YB ? h->Yb
                          : which == DAMF_ZB ? h->Zb : h->rb;
      if (!base) return fail(h, DAMF_E_SHAPE_MISMATCH, "matrix not allocated (alpha == 1)");
      CK(cudaMemcpy2D(out, k * 4, base, d * 4, k * 4, h->n, cudaMemcpyDeviceToHost));
      return 0;
    }
    case DAMF_PX:
    case DAMF_PY: {
      std::vector<double> t((size_t)k * ld);
      CK(cudaMemcpy(t.data(), live_PT(h, which == DAMF_PY), (size_t)k * ld * 8, cudaMemcpyDeviceToHost));
      double* o = static_cast<double*>(out);
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) o[i * k + j] = t[(size_t)j * ld + i];
      return 0;
    }
    case DAMF_QX:
    case DAMF_QY:
      CK(cudaMemcpy2D(out, k * 8, live_Q(h, which == DAMF_QY), ld * 8, k * 8, k, cudaMemcpyDeviceToHost));
      return 0;
    case DAMF_SIGMA:
      CK(cudaMemcpy(out, h->sigma, k * 8, cudaMemcpyDeviceToHost));
      return 0;
    case DAMF_XB64:
    case DAMF_YB64: {
      std::vector<double> r64;
      if (int r = base_rows_f64(h, which == DAMF_XB64 ? 0 : 1, &r64)) return r;
      std::memcpy(out, r64.data(), r64.size() * 8);
      return 0;
    }
    case DAMF_X:
    case DAMF_Y:
    case DAMF_Z:
      return damf_gpu_materialize(h, which, static_cast<float*>(out), 0);
  }
  return fail(h, DAMF_E_SHAPE_MISMATCH, "unknown matrix id");
}

int damf_gpu_get_graph(damf_gpu* h, int64_t* offsets, int32_t* targets, double* degree) {
  if (int r = sync_ctl(h)) return r;
  const int64_t n = h->n;
  std::vector<int64_t> off(n);
  std::vector<int32_t> cnt(n);
  CK(cudaMemcpy(off.data(), h->out.off, n * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cnt.data(), h->out.cnt, n * 4, cudaMemcpyDeviceToHost));
  if (degree) CK(cudaMemcpy(degree, h->deg, n * 8, cudaMemcpyDeviceToHost));
  int64_t top = 0;
  CK(cudaMemcpy(&top, h->out.pool_top, 8, cudaMemcpyDeviceToHost));
  std::vector<int32_t> ids(std::max<int64_t>(top, 1));
  CK(cudaMemcpy(ids.data(), h->out.ids, top * 4, cudaMemcpyDeviceToHost));
  int64_t pos = 0;
  for (int64_t u = 0; u < n; ++u) {
    if (offsets) offsets[u] = pos;
    if (targets) {
      std::copy(ids.begin() + off[u], ids.begin() + off[u] + cnt[u], targets + pos);
      std::sort(targets + pos, targets + pos + cnt[u]);
    }
    pos += cnt[u];
  }
  if (offsets) offsets[n] = pos;
  return 0;
}

}  // extern "C"
namespace {
// X_b (side 0) / Y_b (side 1) as fp64 row-major n x k: the fp32 rows widened,
// with the side-table rows' fp64 values in place.
int base_rows_f64(damf_gpu* h, int side, std::vector<double>* out) {
  const int64_t n = h->n, k = h->k;
  std::vector<float> rows((size_t)n * k);
  if (int r = damf_gpu_get_state(h, side == 0 ? DAMF_XB : DAMF_YB, rows.data())) return r;
  out->assign(rows.begin(), rows.end());
  const long long ns = std::min<long long>(h->h_ctl->dirty_n[side], kDirtyCap);
  if (ns > 0) {
    std::vector<int64_t> ids((size_t)ns);
    std::vector<double> r64((size_t)ns * h->ld);
    CK(cudaMemcpy(ids.data(), h->dirty[side], ns * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r64.data(), h->rows64[side], ns * h->ld * 8, cudaMemcpyDeviceToHost));
    for (long long q = 0; q < ns; ++q)
      for (int64_t j = 0; j < k; ++j) (*out)[(size_t)ids[q] * k + j] = r64[(size_t)q * h->ld + j];
  }
  return 0;
}

// Rows of an fp64 file (n x k row-major) that fp32 cannot hold exactly go to
// the side table, so a saved engine resumes bit-identically; when they do
// not fit, every row stays fp32 (rounded).
int seed_rows64(damf_gpu* h, int side, const std::vector<double>& rm) {
  const int64_t n = h->n, k = h->k;
  std::vector<int64_t> ids;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < k; ++j) {
      const double v = rm[(size_t)i * k + j];
      if ((double)(float)v != v) {
        ids.push_back(i);
        break;
      }
    }
  if (ids.empty() || (long long)ids.size() > kDirtyCap) return 0;
  std::vector<double> r64(ids.size() * (size_t)h->ld, 0.0);
  for (size_t q = 0; q < ids.size(); ++q)
    for (int64_t j = 0; j < k; ++j) r64[q * h->ld + j] = rm[(size_t)ids[q] * k + j];
  CK(cudaMemcpy(h->dirty[side], ids.data(), ids.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->rows64[side], r64.data(), r64.size() * 8, cudaMemcpyHostToDevice));
  set_slots_kernel<<<(int)std::min<size_t>(ids.size(), 4096), 128>>>(h->slot[side], h->dirty[side],
                                                                      (long long)ids.size());
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  h->h_ctl->dirty_n[side] = (long long)ids.size();
  CK(cudaMemcpy(&h->ctl->dirty_n[side], &h->h_ctl->dirty_n[side], 8, cudaMemcpyHostToDevice));
  h->ctl_fresh = false;
  return 0;
}
}  // namespace
extern "C" {

// ---- state persistence: the reference's DAMF v1 binary (io.cpp:182-264) --
// magic "DAMF", u32 version 1, RunConfig, u64 events_applied, i64
// events_since_rebase, sigma (i64 n + f64), X_b, Y_b, P_X, P_Y, Z_b, r_b
// (i64 rows, i64 cols, f64 row-major: DenseMatrix is Eigen RowMajor,
// types.hpp:17-18, and write_matrix dumps m.data(), io.cpp:51-56), then the
// out-adjacency (i64 n; per node i64 count and (i64 v, f64 w) pairs). Files
// written here load in the reference and vice versa (fp32 rows widen to fp64
// exactly; fp64 rows from the reference are rounded to fp32 on load).
}  // extern "C"
namespace {
template <typename T>
void putv(std::FILE* f, T v) {
  std::fwrite(&v, sizeof(T), 1, f);
}
template <typename T>
bool getv(std::FILE* f, T* v) {
  return std::fread(v, sizeof(T), 1, f) == 1;
}
void put_rows(std::FILE* f, const std::vector<float>& rm, int64_t n, int64_t k) {
  // write_matrix (io.cpp:51-56) dumps Eigen RowMajor storage (types.hpp:17-18)
  putv<int64_t>(f, n);
  putv<int64_t>(f, k);
  std::vector<double> row((size_t)k);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < k; ++j) row[j] = rm[(size_t)i * k + j];
    std::fwrite(row.data(), 8, (size_t)k, f);
  }
}
// read_matrix (io.cpp:58-65): i64 rows, i64 cols, fp64 row-major
bool get_matrix(std::FILE* f, int64_t* r, int64_t* c, std::vector<double>* rowmajor) {
  if (!getv(f, r) || !getv(f, c) || *r < 0 || *c < 0) return false;
  rowmajor->resize((size_t)(*r * *c));
  return (size_t)(*r * *c) == 0 ||
         std::fread(rowmajor->data(), 8, (size_t)(*r * *c), f) == (size_t)(*r * *c);
}
}  // namespace
extern "C" {

int damf_gpu_save_state(damf_gpu* h, const char* path) {
  if (!h) return DAMF_E_SHAPE_MISMATCH;
  if (int r = sync_ctl(h)) return r;
  const int64_t n = h->n, k = h->k;
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return fail(h, DAMF_E_IO, std::string("cannot write ") + path);
  std::fwrite("DAMF", 1, 4, f);
  putv<uint32_t>(f, 1);
  putv<int64_t>(f, h->cfg.d);
  putv<double>(f, h->cfg.alpha);
  putv<double>(f, h->cfg.eps);
  putv<uint64_t>(f, h->cfg.seed);
  putv<double>(f, h->cfg.rebase_cond);
  putv<int64_t>(f, h->cfg.rebase_every);
  putv<uint8_t>(f, h->cfg.undirected ? 1 : 0);
  putv<uint64_t>(f, h->events_applied);
  putv<int64_t>(f, h->since_rebase);
  std::vector<double> sig((size_t)k);
  CK(cudaMemcpy(sig.data(), h->sigma, k * 8, cudaMemcpyDeviceToHost));
  putv<int64_t>(f, k);
  std::fwrite(sig.data(), 8, (size_t)k, f);
  std::vector<float> rows((size_t)n * k);
  for (int which : {DAMF_XB, DAMF_YB}) {
    // the base rows exactly: fp32 rows widened, side-table rows in fp64
    std::vector<double> r64;
    if (int r = base_rows_f64(h, which == DAMF_XB ? 0 : 1, &r64)) { std::fclose(f); return r; }
    putv<int64_t>(f, n);
    putv<int64_t>(f, k);
    std::fwrite(r64.data(), 8, r64.size(), f);
  }
  std::vector<double> P((size_t)k * k);
  for (int which : {DAMF_PX, DAMF_PY}) {
    if (int r = damf_gpu_get_state(h, which, P.data())) { std::fclose(f); return r; }
    putv<int64_t>(f, k);
    putv<int64_t>(f, k);
    std::fwrite(P.data(), 8, P.size(), f);  // row-major, as get_state returns it
  }
  if (h->alpha1) {  // enhancer.cpp:34-38: Z_b mirrors X_b, r_b = 0
    if (int r = damf_gpu_get_state(h, DAMF_XB, rows.data())) { std::fclose(f); return r; }
    put_rows(f, rows, n, k);
    std::fill(rows.begin(), rows.end(), 0.0f);
    put_rows(f, rows, n, k);
  } else {
    for (int which : {DAMF_ZB, DAMF_RB}) {
      if (int r = damf_gpu_get_state(h, which, rows.data())) { std::fclose(f); return r; }
      put_rows(f, rows, n, k);
    }
  }
  // adjacency (insertion order of the device rows; weights 1.0 when unweighted)
  std::vector<int64_t> off(n);
  std::vector<int32_t> cnt(n);
  CK(cudaMemcpy(off.data(), h->out.off, n * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cnt.data(), h->out.cnt, n * 4, cudaMemcpyDeviceToHost));
  int64_t top = 0;
  CK(cudaMemcpy(&top, h->out.pool_top, 8, cudaMemcpyDeviceToHost));
  std::vector<int32_t> ids((size_t)std::max<int64_t>(top, 1));
  std::vector<double> w(h->out.wts ? (size_t)std::max<int64_t>(top, 1) : 0);
  CK(cudaMemcpy(ids.data(), h->out.ids, top * 4, cudaMemcpyDeviceToHost));
  if (h->out.wts) CK(cudaMemcpy(w.data(), h->out.wts, top * 8, cudaMemcpyDeviceToHost));
  putv<int64_t>(f, n);
  for (int64_t u = 0; u < n; ++u) {
    putv<int64_t>(f, cnt[u]);
    for (int32_t p = 0; p < cnt[u]; ++p) {
      putv<int64_t>(f, ids[off[u] + p]);
      putv<double>(f, h->out.wts ? w[off[u] + p] : 1.0);
    }
  }
  const bool ok = std::ferror(f) == 0;
  if (std::fclose(f) != 0 || !ok) return fail(h, DAMF_E_IO, std::string("write failed: ") + path);
  return 0;
}

int damf_gpu_load_state(const char* path, const damf_config* sizing, damf_gpu** out) {
  *out = nullptr;
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return DAMF_E_IO;
  auto bad = [&](int code) {
    std::fclose(f);
    return code;
  };
  char magic[4];
  uint32_t version = 0;
  if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "DAMF", 4) != 0) return bad(DAMF_E_PARSE);
  if (!getv(f, &version) || version != 1) return bad(DAMF_E_PARSE);
  damf_config cfg{};
  uint8_t und = 0;
  uint64_t applied = 0;
  int64_t since = 0;
  if (!getv(f, &cfg.d) || !getv(f, &cfg.alpha) || !getv(f, &cfg.eps) || !getv(f, &cfg.seed) ||
      !getv(f, &cfg.rebase_cond) || !getv(f, &cfg.rebase_every) || !getv(f, &und) ||
      !getv(f, &applied) || !getv(f, &since))
    return bad(DAMF_E_PARSE);
  cfg.undirected = und ? 1 : 0;
  if (sizing) {
    cfg.node_capacity = sizing->node_capacity;
    cfg.arc_capacity = sizing->arc_capacity;
    cfg.flags = sizing->flags;
  }
  int64_t k = 0;
  if (!getv(f, &k) || k < 1 || k > cfg.d) return bad(DAMF_E_PARSE);
  std::vector<double> sig((size_t)k);
  if (std::fread(sig.data(), 8, (size_t)k, f) != (size_t)k) return bad(DAMF_E_PARSE);
  int64_t r = 0, c = 0;
  std::vector<double> xb, yb, px, py, zb, rb;
  if (!get_matrix(f, &r, &c, &xb) || c != k) return bad(DAMF_E_PARSE);
  const int64_t n = r;
  if (!get_matrix(f, &r, &c, &yb) || r != n || c != k) return bad(DAMF_E_PARSE);
  if (!get_matrix(f, &r, &c, &px) || r != k || c != k) return bad(DAMF_E_PARSE);
  if (!get_matrix(f, &r, &c, &py) || r != k || c != k) return bad(DAMF_E_PARSE);
  if (!get_matrix(f, &r, &c, &zb) || r != n || c != k) return bad(DAMF_E_PARSE);
  if (!get_matrix(f, &r, &c, &rb) || r != n || c != k) return bad(DAMF_E_PARSE);
  int64_t gn = 0;
  if (!getv(f, &gn) || gn != n) return bad(DAMF_E_PARSE);
  std::vector<int64_t> off((size_t)n + 1, 0);
  std::vector<int32_t> tgt;
  std::vector<double> wts;
  bool weighted = false;
  for (int64_t u = 0; u < n; ++u) {
    int64_t cnt = 0;
    if (!getv(f, &cnt) || cnt < 0) return bad(DAMF_E_PARSE);
    for (int64_t i = 0; i < cnt; ++i) {
      int64_t v = 0;
      double w = 0;
      if (!getv(f, &v) || !getv(f, &w) || v < 0 || v >= n) return bad(DAMF_E_PARSE);
      tgt.push_back((int32_t)v);
      wts.push_back(w);
      weighted = weighted || w != 1.0;
    }
    off[u + 1] = (int64_t)tgt.size();
  }
  std::fclose(f);
  // fp64 row-major -> fp32 row-major (X_b, Y_b); P stays fp64 row-major
  auto rows32 = [&](const std::vector<double>& rm) {
    std::vector<float> o((size_t)n * k);
    for (size_t x = 0; x < o.size(); ++x) o[x] = (float)rm[x];
    return o;
  };
  const std::vector<float> x32 = rows32(xb), y32 = rows32(yb);
  const std::vector<double>& pxr = px;
  const std::vector<double>& pyr = py;
  damf_csr g{n, (int64_t)tgt.size(), off.data(), tgt.data(), weighted ? wts.data() : nullptr};
  const std::vector<float> z32 = rows32(zb), r32 = rows32(rb);
  const int st = damf_gpu_resume(&g, &cfg, k, x32.data(), y32.data(), pxr.data(), pyr.data(),
                                 sig.data(), z32.data(), r32.data(), applied, since, out);
  if (st) return st;
  if (int r = seed_rows64(*out, 0, xb)) return r;
  return seed_rows64(*out, 1, yb);
}

// Engine(g, fs, es, cfg, events_applied, events_since_rebase) (engine.hpp:32-34):
// the factor state plus a saved enhancer, no init_propagate.
int damf_gpu_resume(const damf_csr* g, const damf_config* cfg, int64_t k, const float* xb,
                    const float* yb, const double* px, const double* py, const double* sigma,
                    const float* zb, const float* rb, uint64_t events_applied,
                    int64_t events_since_rebase, damf_gpu** out) {
  *out = nullptr;
  t_skip_ppr_init = true;
  const int st = damf_gpu_create_from_factors(g, cfg, k, xb, yb, px, py, sigma, out);
  t_skip_ppr_init = false;
  if (st) return st;
  damf_gpu* h = *out;
  h->events_applied = events_applied;
  h->since_rebase = events_since_rebase;
  if (!h->alpha1) {
    // alpha == 1 mirrors Z_b = X_b (enhancer.cpp:34-38); otherwise the saved
    // Z_b / r_b, re-keyed like EnhancerState's constructor (enhancer.cpp:11-24)
    if (!zb || !rb) return fail(h, DAMF_E_SHAPE_MISMATCH, "resume: Z_b and r_b are required when alpha != 1");
    CK(cudaMemcpy2D(h->Zb, (size_t)h->d * 4, zb, (size_t)k * 4, (size_t)k * 4, g->n,
                    cudaMemcpyDefault));
    CK(cudaMemcpy2D(h->rb, (size_t)h->d * 4, rb, (size_t)k * 4, (size_t)k * 4, g->n,
                    cudaMemcpyDefault));
    CK(launch_ppr_keys(ppr_args(h), h->nsm, h->st));
    CK(cudaStreamSynchronize(h->st));
  }
  return 0;
}

int damf_gpu_diagnostics(damf_gpu* h, damf_diag* o) {
  if (int r = sync_ctl(h)) return r;
  o->n = h->n;
  o->k = h->k;
  o->d = h->d;
  unsigned long long* dsum = nullptr;
  CK(cudaMalloc(&dsum, 8));
  CK(cudaMemsetAsync(dsum, 0, 8, h->st));
  count_sum_kernel<<<h->nsm * 4, 256, 0, h->st>>>(h->out.cnt, h->n, dsum);
  CK(cudaGetLastError());
  unsigned long long arcs = 0;
  CK(cudaMemcpyAsync(&arcs, dsum, 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  cudaFree(dsum);
  o->arcs = (int64_t)arcs;
  o->events_applied = (int64_t)h->events_applied;
  o->events_since_rebase = h->since_rebase;
  o->cond_estimate = h->h_ctl->cond_est;
  CK(launch_smax(h->PT[0][0], h->PT[0][1], h->ctl, h->ld, h->smax, h->st));
  double sm = 0;
  CK(cudaMemcpy(&sm, h->smax, 8, cudaMemcpyDeviceToHost));
  o->proj_row_bound = sm;
  o->total_pushes = h->h_pstats[0];
  o->device_bytes = (int64_t)h->bytes;
  o->kernel_launches = h->launches;
  o->last_materialize_ms = h->last_mat_ms;
  return 0;
}

int damf_gpu_get_config(const damf_gpu* h, damf_config* out) {
  if (!h || !out) return DAMF_E_SHAPE_MISMATCH;
  *out = h->cfg;
  return 0;
}

void* damf_gpu_stream(damf_gpu* h) { return (void*)h->st; }

// Dev: per-round trace of the last whole-GPU push ([nF, dense, items, active
// heavy] x rounds); returns the round count (or -1).
int damf_gpu_ppr_trace(damf_gpu* h, int64_t* out, int cap) {
  if (!h || !h->ptrace) return -1;
  long long buf[4 * 1024 + 1];
  if (cudaMemcpy(buf, h->ptrace, sizeof(buf), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  const int r = (int)std::min<long long>(buf[4 * 1024], 1024);
  for (int i = 0; i < 4 * std::min(r, cap); ++i) out[i] = buf[i];
  return r;
}

// Dev (DAMF_PROF builds): the slow-secular-root dump kept in the d > 128
// workspace: 8 header doubles, then up to 8 records of 600 doubles.
int damf_gpu_debug_dump(damf_gpu* h, double* out, int64_t count) {
  double* src = h->ws + (size_t)h->ld * h->ld;
  if (count < 0) {  // reset
    CK(cudaMemset(src, 0, 16));
    return 0;
  }
  const int64_t m = std::min<int64_t>(count, 8 + 8 * 800 + 16 * 260);
  CK(cudaMemcpy(out, src, m * 8, cudaMemcpyDeviceToHost));
  return 0;
}

int damf_gpu_profile_counters(damf_gpu* h, uint64_t* out16) {
  if (int r = sync_ctl(h)) return r;
  for (int i = 0; i < 128; ++i) out16[i] = h->h_ctl->prof[i];
  return 0;
}

int damf_gpu_push_counters(damf_gpu* h, int64_t* out4) {
  if (int r = sync_ctl(h)) return r;
  for (int i = 0; i < 4; ++i) out4[i] = h->h_pstats[3 + i];
  return 0;
}

int damf_materialize_dev(const float* x, int64_t n, int64_t d, const double* f_host, float* z,
                         void* stream, float* ms_out) {
  damf_gpu* h = nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int ld = (int)d;
  double* FT = nullptr;
  std::vector<double> ft((size_t)d * d);
  for (int64_t i = 0; i < d; ++i)
    for (int64_t j = 0; j < d; ++j) ft[j * d + i] = f_host[i * d + j];
  CK(cudaMalloc(&FT, (size_t)d * d * 8));
  CK(cudaMemcpyAsync(FT, ft.data(), (size_t)d * d * 8, cudaMemcpyHostToDevice, s));
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  CK(launch_materialize(x, n, (int)d, (int)d, FT, ld, (int)d, z, (int)d, s, nsm));
  cudaEventRecord(e1, s);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  if (ms_out) *ms_out = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(FT);
  return 0;
}

}  // extern "C"
