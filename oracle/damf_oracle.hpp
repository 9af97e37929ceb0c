// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// A CPU fp64 restatement of the DAMF reference library's hot path
// (/root/reference/proj, read-only), used ONLY by tests/, by
// __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
// --impl reference leg. The product path (paper_2306_08967_b200/) never
// links or calls anything here.
//
// Each declaration cites the reference file:line it follows. The reference
// itself cannot be compiled here (it needs Eigen3, proj/CMakeLists.txt:12,
// and CLI11/doctest from an absent vendor/ directory), so Eigen's dense
// routines are restated in la.hpp.
#pragma once

#include <cstdint>
#include <deque>
#include <functional>
#include <optional>
#include <queue>
#include <random>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

#include "la.hpp"

namespace damf_oracle {

// ---- rng.hpp:11-35 ---------------------------------------------------------
using Rng = std::mt19937_64;
inline double rand_unit(Rng& rng) {
  return static_cast<double>(rng() >> 11) * 0x1.0p-53;
}
inline std::uint64_t rand_index(Rng& rng, std::uint64_t n) {
  const std::uint64_t bound = ~std::uint64_t{0} - (~std::uint64_t{0} % n);
  std::uint64_t x;
  do {
    x = rng();
  } while (x >= bound);
  return x % n;
}
inline double rand_gaussian(Rng& rng) {
  double u1;
  do {
    u1 = rand_unit(rng);
  } while (u1 <= 0.0);
  const double u2 = rand_unit(rng);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

// ---- types.hpp:21-41 (kinds in the same order: the C ABI status is ordinal+1)
struct Error : std::runtime_error {
  enum class Kind {
    ParseError,
    UnknownNode,
    DuplicateEdge,
    MissingEdge,
    ShapeMismatch,
    ZeroMatrix,
    NonFinite,
    SingularProjection,
    NonConvergence,
    DegenerateLabels,
    KTooLarge,
    GraphTooSmall,
    TooLarge,
    IoError,
  };
  Error(Kind k, const std::string& msg) : std::runtime_error(msg), kind(k) {}
  Kind kind;
};

// ---- types.hpp:44-66 --------------------------------------------------------
struct SparseVec {
  Index size = 0;
  std::vector<std::pair<Index, double>> nz;
  static SparseVec unit(Index size, Index i, double v = 1.0) {
    SparseVec b;
    b.size = size;
    if (v != 0.0) b.nz.emplace_back(i, v);
    return b;
  }
  double norm2sq() const {
    double s = 0.0;
    for (const auto& p : nz) s += p.second * p.second;
    return s;
  }
  Vec to_dense() const {
    Vec x(static_cast<size_t>(size), 0.0);
    for (const auto& p : nz) x[p.first] = p.second;
    return x;
  }
};

// ---- types.hpp:68-123 -------------------------------------------------------
struct SparseRowMatrix {
  Index rows = 0, cols = 0;
  std::vector<Index> idx;
  Mat vals;  // idx.size() x cols
  Index nnz_rows() const { return static_cast<Index>(idx.size()); }
  static SparseRowMatrix zero(Index rows, Index cols) {
    SparseRowMatrix m;
    m.rows = rows;
    m.cols = cols;
    m.vals = Mat(0, cols);
    return m;
  }
  static SparseRowMatrix from_column(const SparseVec& b);
  // types.hpp:101-116: exact-zero row vector -> empty.
  static SparseRowMatrix outer(const SparseVec& b, const Vec& r);
  Mat to_dense() const;
};

// ---- graph.hpp:14-58 --------------------------------------------------------
struct GraphEvent {
  enum class Kind { AddNode, AddEdge, RemoveEdge };
  Kind kind = Kind::AddEdge;
  Index u = 0, v = 0;
  double w = 1.0;
  std::vector<std::pair<Index, double>> in_edges, out_edges;
  static GraphEvent add_edge(Index u, Index v, double w = 1.0) {
    GraphEvent e;
    e.kind = Kind::AddEdge;
    e.u = u;
    e.v = v;
    e.w = w;
    return e;
  }
  static GraphEvent remove_edge(Index u, Index v) {
    GraphEvent e;
    e.kind = Kind::RemoveEdge;
    e.u = u;
    e.v = v;
    return e;
  }
  static GraphEvent add_node(std::vector<std::pair<Index, double>> in,
                             std::vector<std::pair<Index, double>> out) {
    GraphEvent e;
    e.kind = Kind::AddNode;
    e.in_edges = std::move(in);
    e.out_edges = std::move(out);
    return e;
  }
};

struct DeltaVectors {
  enum class Step { NodeColumn, NodeRow, Edge };
  SparseVec b;
  std::optional<SparseVec> c;
  Index delta_m = 0;
  Step step = Step::Edge;
};

// ---- graph.hpp:62-104, graph.cpp:16-207 -------------------------------------
class DynamicGraph {
 public:
  explicit DynamicGraph(Index n = 0, bool undirected = false);
  Index node_count() const { return static_cast<Index>(out_adj_.size()); }
  Index arc_count() const { return arcs_; }
  bool undirected() const { return undirected_; }
  double out_degree(Index u) const;
  const std::vector<std::pair<Index, double>>& out_neighbors(Index u) const;
  const std::vector<std::pair<Index, double>>& in_neighbors(Index u) const;
  bool has_edge(Index u, Index v) const;
  double edge_weight(Index u, Index v) const;
  std::vector<DeltaVectors> apply_event(const GraphEvent& e);
  std::vector<Index> touched_by(const GraphEvent& e) const;
  void add_arc_raw(Index u, Index v, double w);

 private:
  void check_node(Index u, const char* who) const;
  void insert_arc(Index u, Index v, double w);
  void erase_arc(Index u, Index v);
  bool undirected_ = false;
  Index arcs_ = 0;
  std::vector<std::vector<std::pair<Index, double>>> out_adj_, in_adj_;
  std::vector<double> out_deg_;
  std::unordered_set<std::uint64_t> edge_keys_;
};

// ---- projection_update.hpp:17-36 --------------------------------------------
struct ProjectionUpdate {
  Mat F, G;
  SparseRowMatrix dX, dY;
  Vec sigma2;
  std::optional<SparseVec> grow_x, grow_y;
  Index append_x = -1, append_y = -1;
};

struct AppliedDelta {
  std::optional<Mat> x_transform;
  Index x_rows_appended = 0;
  std::optional<SparseVec> x_grow_col;
  SparseRowMatrix x_base_rows;
};

// ---- kernels.hpp / kernels.cpp:7-65 -----------------------------------------
Mat mult_sparseT_dense(const SparseRowMatrix& b, const Mat& a);
SparseRowMatrix mult_sparse_dense(const SparseRowMatrix& b, const Mat& c);
struct ResidualNorm {
  double r = 0.0;
  Vec w;
};
ResidualNorm ortho_residual_norm(const Mat& xb, const Mat& p, const Vec& sigma,
                                 const SparseVec& b);

// ---- svd.hpp / svd.cpp:12-96 ------------------------------------------------
struct SparseOp {
  Index rows = 0, cols = 0;
  std::function<Mat(const Mat&)> apply, apply_t;
  static SparseOp from_dense(const Mat& a);
};
SvdTriple dense_svd_small(const Mat& m, Index keep);
SvdTriple randomized_tsvd(const SparseOp& a, Index d, Index oversample = 10,
                          Index power_iters = 4, std::uint64_t seed = 0);
Mat qr_orthonormalize(const Mat& m);

// ---- factor_state.hpp:16-75, factor_state.cpp ------------------------------
class FactorState {
 public:
  FactorState() = default;
  FactorState(Mat xb, Mat yb, Mat px, Mat py, Vec sigma, Index d);
  static FactorState init_from_graph(const DynamicGraph& g, Index d,
                                     std::uint64_t seed);
  Index rank() const { return static_cast<Index>(sigma_.size()); }
  Index dim() const { return d_; }
  Index rows_x() const { return xb_.r; }
  Index rows_y() const { return yb_.r; }
  const Vec& sigma() const { return sigma_; }
  const Mat& xb() const { return xb_; }
  const Mat& yb() const { return yb_; }
  const Mat& px() const { return px_; }
  const Mat& py() const { return py_; }
  AppliedDelta apply_update(const ProjectionUpdate& u);
  Vec query_context(Index u) const;
  Vec query_content(Index u) const;
  void query_all(Mat& x, Mat& y) const;
  double reconstruct_entry(Index u, Index v) const;
  Mat rebase();
  double cond_estimate() const;
  double proj_row_bound() const;
  double ortho_defect_x() const;
  double ortho_defect_y() const;
  // Counters used by the parity harness (not in the reference).
  std::uint64_t eager_folds = 0;
  // Harness mode (not in the reference): the device's storage model -- base
  // rows rounded to fp32 whenever a fold writes them (rebase, eager fold),
  // rows written through the lazy solve kept in fp64 until then -- so
  // storage-precision effects can be told apart from logic differences.
  bool fp32_base = false;
  void round_base();

 private:
  Mat xb_, yb_, px_, py_;
  Vec sigma_;
  Index d_ = 0;
};
SparseOp adjacency_op(const DynamicGraph& g);

// ---- update_engine.hpp / update_engine.cpp:12-226 ---------------------------
ProjectionUpdate update_embedding_n(const FactorState& s, const SparseVec& b,
                                    bool u_is_x = true);
ProjectionUpdate update_embedding_e(const FactorState& s, const SparseVec& b,
                                    const SparseVec& c);
struct HandledEvent {
  std::vector<ProjectionUpdate> updates;
  std::vector<AppliedDelta> applied;
};
HandledEvent handle_event(FactorState& s, const std::vector<DeltaVectors>& deltas);

// ---- enhancer.hpp:14-76, enhancer.cpp:11-206 --------------------------------
struct EnhancerParams {
  double alpha = 0.3;
  double eps = 1e-5;
};
class EnhancerState {
 public:
  EnhancerState() = default;
  EnhancerState(EnhancerParams params, Mat zb, Mat rb);
  static EnhancerState init_propagate(const DynamicGraph& g, const FactorState& s,
                                      EnhancerParams params);
  double alpha() const { return params_.alpha; }
  double eps() const { return params_.eps; }
  const Mat& zb() const { return zb_; }
  const Mat& rb() const { return rb_; }
  std::uint64_t total_pushes() const { return total_pushes_; }
  void absorb_signal_delta(const SparseRowMatrix& dxb);
  void absorb_structure_delta(const DynamicGraph& g, const FactorState& s,
                              const std::vector<Index>& touched);
  void push_to_tolerance(const DynamicGraph& g, const FactorState& s);
  Vec query_enhanced(const FactorState& s, Index u) const;
  void append_rows(Index count);
  void grow_column(const SparseVec& col);
  void apply_transform(const Mat& t);

 private:
  double row_key(Index u, double deg) const;
  void note_residual(Index u, double key);
  EnhancerParams params_;
  Mat zb_, rb_;
  std::deque<Index> fifo_;
  std::vector<char> in_fifo_;
  std::priority_queue<std::pair<double, Index>> index_;
  std::vector<double> index_key_;
  std::uint64_t total_pushes_ = 0;
};

// ---- engine.hpp:13-61, engine.cpp:5-52 --------------------------------------
struct RunConfig {
  Index d = 128;
  double alpha = 0.3;
  double eps = 1e-5;
  std::uint64_t seed = 0;
  double rebase_cond = 1e8;
  Index rebase_every = 50000;
  bool undirected = false;
};

class Engine {
 public:
  Engine() = default;
  Engine(DynamicGraph g, const RunConfig& cfg);
  Engine(DynamicGraph g, FactorState fs, EnhancerState es, const RunConfig& cfg,
         std::uint64_t events_applied, Index events_since_rebase);
  void apply(const GraphEvent& e);
  const DynamicGraph& graph() const { return g_; }
  const FactorState& state() const { return fs_; }
  const EnhancerState& enhancer() const { return es_; }
  const RunConfig& config() const { return cfg_; }
  std::uint64_t events_applied() const { return events_applied_; }
  Index events_since_rebase() const { return events_since_rebase_; }
  Vec context(Index u) const { return fs_.query_context(u); }
  Vec content(Index u) const { return fs_.query_content(u); }
  Vec enhanced(Index u) const { return es_.query_enhanced(fs_, u); }
  double score(Index u, Index v, bool enhanced = true) const;
  void rebase();
  std::uint64_t rebases = 0;  // counter for the harness
  // Harness hook (not in the reference): when set, apply() appends one
  // (step, side, row) triple per row of every ProjectionUpdate's dX (side 0)
  // and dY (side 1), steps numbered by *row_log_step across calls.
  std::vector<std::int64_t>* row_log = nullptr;
  std::int64_t row_log_step = 0;

 private:
  DynamicGraph g_;
  FactorState fs_;
  EnhancerState es_;
  RunConfig cfg_;
  std::uint64_t events_applied_ = 0;
  Index events_since_rebase_ = 0;
};

// ---- eval.hpp:69-111, eval.cpp:405-610 --------------------------------------
class OracleTsvd {
 public:
  OracleTsvd(const DynamicGraph& g0, Index d);
  void apply_deltas(const std::vector<DeltaVectors>& deltas);
  const Vec& sigma() const { return sigma_; }
  Mat product() const;
  bool last_gap_ok() const { return gap_ok_; }
  double product_rel_dist(const FactorState& s) const;
  double sigma_rel_dist(const Vec& engine_sigma) const;

 private:
  void step(const SparseVec& b, const std::optional<SparseVec>& c, bool swapped);
  Mat u_, v_;
  Vec sigma_;
  Index d_ = 0;
  bool gap_ok_ = true;
};

struct DriftReport {
  double drift = 0.0, c_diag = 0.0;
};
DriftReport drift_report(const FactorState& s, const DynamicGraph& g);
double dense_defect_bound(const DynamicGraph& g, const FactorState& s,
                          const EnhancerState& e);

// ---- eval.cpp:616-705 (generators the reference tests use) ------------------
DynamicGraph gen_random_graph(Index n, Index arcs, std::uint64_t seed,
                              bool undirected = false);
DynamicGraph gen_sbm(Index n, double p_in, double p_out, std::uint64_t seed);
struct StreamCase {
  DynamicGraph g0;
  std::vector<GraphEvent> events;
};
StreamCase gen_mixed_stream(Index n_total, Index n0, Index m0, Index n_events,
                            std::uint64_t seed);

}  // namespace damf_oracle
