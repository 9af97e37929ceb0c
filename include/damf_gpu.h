/*
 * damf_gpu.h — C ABI of the B200-native DAMF hot path.
 *
 * This is the drop-in boundary. The reference (arxiv 2306.08967, DAMF) is a
 * C++ library whose hot path is reached through damf::Engine
 * (/root/reference/proj/include/damf/engine.hpp:26-61). It has no FFI, so
 * every entry point below names the reference member function it replaces;
 * the header-only C++ facade (paper_2306_08967_b200/csrc/damf_engine.hpp)
 * restores the Engine API on top of it, and INTEGRATION.md shows the
 * ctypes / pybind binding a maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only; no CUDA or torch types cross the ABI.
 *    Buffers named *_host are host memory; *_dev are device pointers.
 *  - Every call returns a status: 0 = ok, otherwise damf::Error::Kind
 *    ordinal + 1 (types.hpp:21-41), so DAMF_E_UNKNOWN_NODE == 2, etc.
 *    DAMF_E_CUDA / DAMF_E_UNSUPPORTED are ABI-specific. No exception ever
 *    crosses the ABI; damf_gpu_last_error() returns the message.
 *  - One CUDA stream per handle; calls on one handle are externally
 *    serialised (single writer).
 *  - Node ids are dense int64 in [0, n); AddNode ids are implicit (= n).
 */
#ifndef DAMF_GPU_H_
#define DAMF_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: Error::Kind ordinal + 1 (types.hpp:21-41) ----------- */
enum {
  DAMF_OK = 0,
  DAMF_E_PARSE = 1,
  DAMF_E_UNKNOWN_NODE = 2,
  DAMF_E_DUPLICATE_EDGE = 3,
  DAMF_E_MISSING_EDGE = 4,
  DAMF_E_SHAPE_MISMATCH = 5,
  DAMF_E_ZERO_MATRIX = 6,
  DAMF_E_NON_FINITE = 7,
  DAMF_E_SINGULAR_PROJECTION = 8,
  DAMF_E_NON_CONVERGENCE = 9,
  DAMF_E_DEGENERATE_LABELS = 10,
  DAMF_E_K_TOO_LARGE = 11,
  DAMF_E_GRAPH_TOO_SMALL = 12,
  DAMF_E_TOO_LARGE = 13,
  DAMF_E_IO = 14,
  DAMF_E_CUDA = 100,
  DAMF_E_UNSUPPORTED = 101
};

/* GraphEvent::Kind order (graph.hpp:17). */
enum { DAMF_ADD_NODE = 0, DAMF_ADD_EDGE = 1, DAMF_REMOVE_EDGE = 2 };

/* Matrices addressable by the query / state calls. */
enum {
  DAMF_XB = 0,     /* base context rows  X_b  (n x k, fp32)  factor_state.hpp:68 */
  DAMF_YB = 1,     /* base content rows  Y_b  (n x k, fp32)                      */
  DAMF_PX = 2,     /* projection P_X (k x k, fp64)           factor_state.hpp:69 */
  DAMF_PY = 3,     /* projection P_Y (k x k, fp64)                               */
  DAMF_SIGMA = 4,  /* spectrum (k, fp64)                     factor_state.hpp:70 */
  DAMF_ZB = 5,     /* enhancer Z_b (n x k, fp32)             enhancer.hpp:67     */
  DAMF_RB = 6,     /* enhancer r_b (n x k, fp32)                                 */
  DAMF_X = 7,      /* current X = X_b P_X  (query_all / query_context)           */
  DAMF_Y = 8,      /* current Y = Y_b P_Y  (query_all / query_content)           */
  DAMF_Z = 9,      /* enhanced Z = Z_b P_X (query_enhanced)                      */
  DAMF_QX = 10,    /* maintained inverse P_X^{-1} (k x k, fp64; GPU-only state)  */
  DAMF_QY = 11,
  DAMF_XB64 = 12,  /* X_b exactly, fp64 (n x k): the fp32 rows widened, the rows
                      written through P^-1 since the last fold at their fp64
                      values (the reference's X_b is fp64, types.hpp:15-19)     */
  DAMF_YB64 = 13
};

/* RunConfig (engine.hpp:13-21) plus device sizing. */
typedef struct damf_config {
  int64_t d;             /* target rank                                   */
  double alpha;          /* PPR restart (enhancer.hpp:14-17)              */
  double eps;            /* PPR push threshold                            */
  uint64_t seed;         /* init sketch seed                              */
  double rebase_cond;    /* rebase when cond(P_X) exceeds this (1e8)      */
  int64_t rebase_every;  /* rebase every this many events (50000)         */
  int32_t undirected;    /* DynamicGraph(n, undirected)                   */
  int32_t flags;         /* DAMF_CFG_* bits, 0 by default                 */
  int64_t node_capacity; /* rows to reserve beyond n for AddNode (0=auto) */
  int64_t arc_capacity;  /* arc slots to reserve beyond arcs (0=auto)     */
} damf_config;

/* damf_config.flags */
enum {
  DAMF_CFG_REFERENCE_OMEGA = 1 /* damf_gpu_create: always draw the sketch from the
                                  reference's Gaussian stream (rng.hpp) on the host;
                                  by default sketches above 2^26 values use a
                                  device counter-based generator */
};

/* Out-adjacency in CSR form. Arrays may be host or device memory (detected
 * with cudaPointerGetAttributes; device arrays are consumed in place).
 * weights may be NULL (all 1.0). */
typedef struct damf_csr {
  int64_t n;
  int64_t arcs;
  const int64_t* offsets; /* n+1 */
  const int32_t* targets; /* arcs */
  const double* weights;  /* arcs or NULL */
} damf_csr;

/* A batch of GraphEvents (graph.hpp:14-47), applied SEQUENTIALLY exactly as
 * `for (e : batch) engine.apply(e)`. AddNode neighbour lists use offsets
 * into flat arrays (in_off/out_off have count+1 entries; NULL if unused).
 * All pointers are host memory; w / in_w / out_w may be NULL (1.0). */
typedef struct damf_event_batch {
  int64_t count;
  const int32_t* kind;
  const int64_t* u;
  const int64_t* v;
  const double* w;
  const int64_t* in_off;
  const int64_t* in_ids;
  const double* in_w;
  const int64_t* out_off;
  const int64_t* out_ids;
  const double* out_w;
} damf_event_batch;

/* Apply modes (bit flags). The default (0) is Engine::apply. */
enum {
  DAMF_APPLY_GRAPH_AND_PPR_ONLY = 1, /* structure-only events: graph mutation
                                        + absorb_structure_delta + push, no
                                        factor update   */
  DAMF_APPLY_DEFER_PUSH = 2,         /* absorb only; caller pushes later   */
  DAMF_APPLY_TIME_EVENTS = 4,        /* record per-event device latency    */
  DAMF_APPLY_LOG_ROWS = 8            /* record the modified base rows of
                                        every rank-1 step (damf_gpu_row_log) */
};

typedef struct damf_apply_stats {
  int64_t applied;       /* events fully applied                          */
  int64_t failed_index;  /* index of the failing event, or -1             */
  int64_t rank1_updates; /* space-projection steps run                    */
  int64_t rebases;       /* rebases triggered inside this call            */
  int64_t eager_folds;   /* rank change / ill-conditioned folds           */
  int64_t push_rounds;   /* frontier rounds of the PPR push               */
  int64_t pushes;        /* rows pushed                                   */
  double device_ms;      /* DAMF_APPLY_TIME_EVENTS: device span of the call
                            (CUDA events from the first launch to the end of
                            its last kernel, rebases included), else 0     */
} damf_apply_stats;

typedef struct damf_diag {
  int64_t n, k, d, arcs;
  int64_t events_applied, events_since_rebase;
  double cond_estimate;   /* factor_state.cpp:224-249 (estimator differs) */
  double proj_row_bound;  /* factor_state.cpp:251-259                      */
  int64_t total_pushes;   /* enhancer.hpp:41                               */
  int64_t device_bytes;   /* HBM held by the handle                        */
  int64_t kernel_launches;/* kernels this handle has launched (all calls)  */
  double last_materialize_ms; /* device time of the last damf_gpu_materialize's X F
                                 kernels (CUDA events on the handle's stream around
                                 the launch; 0 before the first call)            */
} damf_diag;

typedef struct damf_gpu damf_gpu; /* opaque handle: owns all device memory */

/* Engine(g, fs, es, cfg, 0, 0) with fs = FactorState(xb, yb, px, py, sigma, d)
 * (factor_state.hpp:22-23, engine.hpp:32-34) followed by
 * EnhancerState::init_propagate (enhancer.cpp:26-47). xb/yb: n x k fp32
 * row-major arrays in host or device memory, or NULL for zero rows to be
 * filled with damf_gpu_load_rows; px/py: k x k fp64 host; sigma: k fp64
 * host, nonincreasing. */
int damf_gpu_create_from_factors(const damf_csr* g, const damf_config* cfg, int64_t k,
                                 const float* xb, const float* yb,
                                 const double* px_host, const double* py_host,
                                 const double* sigma_host, damf_gpu** out);

/* Engine(g, cfg) (engine.cpp:5-10): FactorState::init_from_graph
 * (factor_state.cpp:84-102) — randomized t-SVD of the adjacency on the device
 * (svd.cpp:47-96: l = d + 10, 4 power iterations, the reference's Gaussian
 * stream for Omega; graphs with n <= 600 take the exact dense SVD), then
 * the factor-based constructor. A numerically rank-deficient sketch
 * (rank(A) < l) is orthogonalised by Gram-Schmidt with basis completion, as
 * the reference's Householder QR does, and the rank is clamped
 * (svd.cpp:84-89). DAMF_E_ZERO_MATRIX for an empty graph. */
int damf_gpu_create(const damf_csr* g, const damf_config* cfg, damf_gpu** out);

/* Engine(g, fs, es, cfg, events_applied, events_since_rebase)
 * (engine.hpp:32-34, engine.cpp:12-16): resume from a factor state AND a saved
 * enhancer (zb / rb: n x k fp32 host or device; ignored when alpha == 1, where
 * Z_b mirrors X_b) with the engine's counters; no init_propagate runs.
 * damf_gpu_load_state is this call fed from a DAMF v1 file. */
int damf_gpu_resume(const damf_csr* g, const damf_config* cfg, int64_t k, const float* xb,
                    const float* yb, const double* px_host, const double* py_host,
                    const double* sigma_host, const float* zb, const float* rb,
                    uint64_t events_applied, int64_t events_since_rebase, damf_gpu** out);

void damf_gpu_destroy(damf_gpu* h);
const char* damf_gpu_last_error(const damf_gpu* h);
int damf_gpu_sync(damf_gpu* h);

/* Engine::apply (engine.cpp:22-41) over a batch, sequentially. On error the
 * failing index is reported and earlier events stay applied, as with the
 * reference's per-event throw. stats may be NULL. */
int damf_gpu_apply(damf_gpu* h, const damf_event_batch* batch, int32_t mode,
                   damf_apply_stats* stats);

/* Engine::apply(GraphEvent::add_edge(u, v, w)) / remove_edge(u, v)
 * (engine.cpp:22-41, graph.hpp:14-47) for ONE edge event, without building
 * a damf_event_batch: kind = DAMF_ADD_EDGE or DAMF_REMOVE_EDGE (w ignored for
 * removals). Same semantics and errors as a batch of one. */
int damf_gpu_apply_edge(damf_gpu* h, int32_t kind, int64_t u, int64_t v, double w, int32_t mode,
                        damf_apply_stats* stats);

/* Batched scoring. flags: DAMF_SCORE_ENHANCED scores
 * <Z[u], Y[v]> instead of <X[u], Y[v]> (Engine::score, engine.cpp:49-52);
 * DAMF_SCORE_SYMMETRIC_MAX takes max(s(u,v), s(v,u)) as pair_score does for
 * undirected graphs (eval.cpp:211-215). u, v, out: host arrays of m. */
enum { DAMF_SCORE_ENHANCED = 1, DAMF_SCORE_SYMMETRIC_MAX = 2 };
int damf_gpu_score_pairs(damf_gpu* h, const int64_t* u, const int64_t* v, int64_t m,
                         int32_t flags, double* out);

/* The K best pairs of (u[i], v[i]) by score descending, pair index ascending
 * on ties (run_graph_reconstruction's heap order, eval.cpp:336-371): writes
 * min(K, m) indices into idx_out (host or device) and their scores into
 * score_out (may be NULL). */
int damf_gpu_topk_pairs(damf_gpu* h, const int64_t* u, const int64_t* v, int64_t m,
                        int32_t flags, int64_t K, int64_t* idx_out, double* score_out);

/* State persistence in the reference's DAMF v1 binary format (io.cpp:182-264:
 * save_state / load_state). Files are interchangeable with the reference.
 * load: `sizing` (may be NULL) supplies node/arc headroom and flags; the
 * RunConfig comes from the file. */
int damf_gpu_save_state(damf_gpu* h, const char* path);
int damf_gpu_load_state(const char* path, const damf_config* sizing, damf_gpu** out);

/* FactorState(xb, yb, ...) row by row: copy m rows (m x k fp32, host or
 * device memory) into X_b (which = DAMF_XB) or Y_b (DAMF_YB) starting at
 * row0. Lets a caller build huge states (config 5: 34 GB per factor) in
 * pieces after damf_gpu_create_from_factors(..., xb = yb = NULL, ...).
 * With alpha != 1 call damf_gpu_ppr_init afterwards. */
int damf_gpu_load_rows(damf_gpu* h, int32_t which, int64_t row0, int64_t m, const float* src);

/* Per-event device latency (microseconds) of the last apply with
 * DAMF_APPLY_TIME_EVENTS (%globaltimer stamps at each event's start and end,
 * read back here, not inside apply): fills min(max, count) values, returns
 * count. */
int64_t damf_gpu_event_latencies(damf_gpu* h, double* out_us_host, int64_t max);

/* The base rows the last apply with DAMF_APPLY_LOG_ROWS modified, one
 * (step, side, row) int64 triple per row: step = rank-1 step index within
 * that call (deltas in handle_event order, update_engine.cpp:206-226), side
 * 0 = X_b (the row set of ProjectionUpdate::dX), 1 = Y_b (dY), in the order
 * the device wrote them (projection_update.hpp:17-36, types.hpp:101-116).
 * Fills min(max, count) triples into out3_host, returns count. */
int64_t damf_gpu_row_log(damf_gpu* h, int64_t* out3_host, int64_t max);

/* Engine::context/content/enhanced (engine.hpp:45-47) for m rows:
 * out_host[m x k] fp32 (which = DAMF_X, DAMF_Y or DAMF_Z). which = DAMF_XB /
 * DAMF_YB / DAMF_ZB / DAMF_RB returns the raw base-coordinate rows. */
int damf_gpu_query_rows(damf_gpu* h, int32_t which, const int64_t* ids_host, int64_t m,
                        float* out_host);

/* The base rows X_b (DAMF_XB) or Y_b (DAMF_YB) of m nodes exactly, fp64
 * (out_host m x k): fp32 rows widened, side-table rows at their fp64 values. */
int damf_gpu_query_rows64(damf_gpu* h, int32_t which, const int64_t* ids_host, int64_t m,
                          double* out_host);

/* Engine::score (engine.cpp:49-52). */
int damf_gpu_score(damf_gpu* h, int64_t u, int64_t v, int32_t enhanced, double* out);

/* FactorState::query_all (factor_state.cpp:120-123) / full Z = Z_b P_X:
 * dst = base(which) * P into a caller buffer of n x k fp32, device or host. */
int damf_gpu_materialize(damf_gpu* h, int32_t which, float* dst, int32_t dst_is_device);

/* Raw state download for parity checks (DAMF_XB..DAMF_QY), host buffer of
 * the natural size/type (fp32 for row matrices, fp64 for P/Q/sigma). */
int damf_gpu_get_state(damf_gpu* h, int32_t which, void* out_host);

/* Sorted out-neighbour sets and weighted out-degrees (graph.cpp bookkeeping):
 * offsets_host[n+1], targets_host[arcs] (sorted per row), degree_host[n]. */
int damf_gpu_get_graph(damf_gpu* h, int64_t* offsets_host, int32_t* targets_host,
                       double* degree_host);

/* EnhancerState::init_propagate / push_to_tolerance (enhancer.cpp:26-47,
 * 98-157). init_propagate resets Z_b = 0, r_b = alpha X_b and pushes. */
int damf_gpu_ppr_init(damf_gpu* h, damf_apply_stats* stats);
int damf_gpu_ppr_push(damf_gpu* h, damf_apply_stats* stats);

/* Engine::rebase (engine.cpp:43-47). */
int damf_gpu_rebase(damf_gpu* h);

int damf_gpu_diagnostics(damf_gpu* h, damf_diag* out);

/* Engine::config() (engine.hpp:43): the RunConfig the handle runs with. */
int damf_gpu_get_config(const damf_gpu* h, damf_config* out);

/* The handle's CUDA stream (cudaStream_t as void*), for callers that time
 * or order work against it. */
void* damf_gpu_stream(damf_gpu* h);

/* Cumulative PPR push work since creation, for algorithmic-byte accounting:
 * out4 = {sum |frontier|, sum |affected|, sum outdeg(affected), pulled arcs}. */
int damf_gpu_push_counters(damf_gpu* h, int64_t* out4);

/* Developer profiling: cumulative SM cycles per phase of the per-event
 * kernel, 128 slots (see event_kernel.cu PROF_MARK; nonzero only in
 * -DDAMF_PROF=1 builds). */
int damf_gpu_profile_counters(damf_gpu* h, uint64_t* out16);

/* Development: per-round trace of the last whole-GPU push, 4 int64 per round
 * [frontier size, dense round, P3 items, active heavy rows]; returns rounds. */
int damf_gpu_ppr_trace(damf_gpu* h, int64_t* out, int cap);

/* Standalone materialisation kernel, Z = X * F (cfg 4): x_dev/z_dev are
 * n x d fp32 device buffers (may alias for in-place), f_host is d x d fp64.
 * stream is a cudaStream_t passed as void* (NULL = default stream). The
 * returned kernel time (ms, CUDA events on that stream) is written to
 * *ms_out when non-NULL. */
int damf_materialize_dev(const float* x_dev, int64_t n, int64_t d, const double* f_host,
                         float* z_dev, void* stream, float* ms_out);

/* Library build info: "sm_100a <git> <flags>". */
const char* damf_gpu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DAMF_GPU_H_ */
