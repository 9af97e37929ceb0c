// ORACLE / TEST INFRASTRUCTURE ONLY — see damf_oracle.hpp.
// Line-by-line restatement of /root/reference/proj/src/*.cpp for the hot path.
#include "damf_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

namespace damf_oracle {

// ============================================================ types.hpp:68-123
SparseRowMatrix SparseRowMatrix::from_column(const SparseVec& b) {
  SparseRowMatrix m;
  m.rows = b.size;
  m.cols = 1;
  m.vals = Mat(static_cast<Index>(b.nz.size()), 1);
  for (size_t i = 0; i < b.nz.size(); ++i) {
    m.idx.push_back(b.nz[i].first);
    m.vals(static_cast<Index>(i), 0) = b.nz[i].second;
  }
  return m;
}

SparseRowMatrix SparseRowMatrix::outer(const SparseVec& b, const Vec& r) {
  SparseRowMatrix m;
  m.rows = b.size;
  m.cols = static_cast<Index>(r.size());
  bool zero = true;
  for (double v : r) zero = zero && v == 0.0;
  if (zero) {
    m.vals = Mat(0, m.cols);
    return m;
  }
  m.vals = Mat(static_cast<Index>(b.nz.size()), m.cols);
  for (size_t i = 0; i < b.nz.size(); ++i) {
    m.idx.push_back(b.nz[i].first);
    for (Index j = 0; j < m.cols; ++j)
      m.vals(static_cast<Index>(i), j) = b.nz[i].second * r[j];
  }
  return m;
}

Mat SparseRowMatrix::to_dense() const {
  Mat d(rows, cols);
  for (Index i = 0; i < nnz_rows(); ++i)
    for (Index j = 0; j < cols; ++j) d(idx[i], j) = vals(i, j);
  return d;
}

// ============================================================ graph.cpp:10-207
namespace {
std::uint64_t edge_key(Index u, Index v) {
  return (static_cast<std::uint64_t>(u) << 32) | static_cast<std::uint64_t>(v);
}
}  // namespace

DynamicGraph::DynamicGraph(Index n, bool undirected)
    : undirected_(undirected), out_adj_(n), in_adj_(n), out_deg_(n, 0.0) {}

void DynamicGraph::check_node(Index u, const char* who) const {
  if (u < 0 || u >= node_count())
    throw Error(Error::Kind::UnknownNode,
                std::string(who) + ": unknown node " + std::to_string(u));
}

double DynamicGraph::out_degree(Index u) const {
  check_node(u, "out_degree");
  return out_deg_[u];
}

const std::vector<std::pair<Index, double>>& DynamicGraph::out_neighbors(Index u) const {
  check_node(u, "out_neighbors");
  return out_adj_[u];
}

const std::vector<std::pair<Index, double>>& DynamicGraph::in_neighbors(Index u) const {
  check_node(u, "in_neighbors");
  return in_adj_[u];
}

bool DynamicGraph::has_edge(Index u, Index v) const {
  return edge_keys_.count(edge_key(u, v)) != 0;
}

double DynamicGraph::edge_weight(Index u, Index v) const {
  if (!has_edge(u, v)) return 0.0;
  for (const auto& p : out_adj_[u])
    if (p.first == v) return p.second;
  return 0.0;
}

void DynamicGraph::insert_arc(Index u, Index v, double w) {
  out_adj_[u].emplace_back(v, w);
  in_adj_[v].emplace_back(u, w);
  out_deg_[u] += w;
  edge_keys_.insert(edge_key(u, v));
  ++arcs_;
}

void DynamicGraph::erase_arc(Index u, Index v) {
  auto& out = out_adj_[u];
  auto it = std::find_if(out.begin(), out.end(),
                         [v](const auto& e) { return e.first == v; });
  out_deg_[u] -= it->second;
  out.erase(it);
  auto& in = in_adj_[v];
  in.erase(std::find_if(in.begin(), in.end(),
                        [u](const auto& e) { return e.first == u; }));
  edge_keys_.erase(edge_key(u, v));
  --arcs_;
}

void DynamicGraph::add_arc_raw(Index u, Index v, double w) {
  check_node(u, "add_arc_raw");
  check_node(v, "add_arc_raw");
  insert_arc(u, v, w);
}

std::vector<DeltaVectors> DynamicGraph::apply_event(const GraphEvent& e) {
  std::vector<DeltaVectors> deltas;
  switch (e.kind) {
    case GraphEvent::Kind::AddEdge: {  // graph.cpp:86-109
      check_node(e.u, "AddEdge");
      check_node(e.v, "AddEdge");
      if (e.w <= 0.0) throw Error(Error::Kind::ParseError, "AddEdge: weight must be > 0");
      if (has_edge(e.u, e.v))
        throw Error(Error::Kind::DuplicateEdge, "AddEdge: edge already present");
      const Index dm = undirected_ && e.u != e.v ? 2 : 1;
      insert_arc(e.u, e.v, e.w);
      deltas.push_back({SparseVec::unit(node_count(), e.u),
                        SparseVec::unit(node_count(), e.v, e.w), dm,
                        DeltaVectors::Step::Edge});
      if (undirected_ && e.u != e.v) {
        if (has_edge(e.v, e.u))
          throw Error(Error::Kind::DuplicateEdge, "AddEdge: reverse arc already present");
        insert_arc(e.v, e.u, e.w);
        deltas.push_back({SparseVec::unit(node_count(), e.v),
                          SparseVec::unit(node_count(), e.u, e.w), dm,
                          DeltaVectors::Step::Edge});
      }
      break;
    }
    case GraphEvent::Kind::RemoveEdge: {  // graph.cpp:110-131
      check_node(e.u, "RemoveEdge");
      check_node(e.v, "RemoveEdge");
      if (!has_edge(e.u, e.v))
        throw Error(Error::Kind::MissingEdge, "RemoveEdge: edge not present");
      const Index dm = undirected_ && e.u != e.v ? 2 : 1;
      const double w = edge_weight(e.u, e.v);
      erase_arc(e.u, e.v);
      deltas.push_back({SparseVec::unit(node_count(), e.u),
                        SparseVec::unit(node_count(), e.v, -w), dm,
                        DeltaVectors::Step::Edge});
      if (undirected_ && e.u != e.v) {
        const double wr = edge_weight(e.v, e.u);
        erase_arc(e.v, e.u);
        deltas.push_back({SparseVec::unit(node_count(), e.v),
                          SparseVec::unit(node_count(), e.u, -wr), dm,
                          DeltaVectors::Step::Edge});
      }
      break;
    }
    case GraphEvent::Kind::AddNode: {  // graph.cpp:132-182
      const Index old_n = node_count();
      std::vector<std::pair<Index, double>> in = e.in_edges, out = e.out_edges;
      if (undirected_) {
        for (const auto& p : e.out_edges) in.emplace_back(p.first, p.second);
        out = in;
      }
      for (const auto& p : in) {
        check_node(p.first, "AddNode");
        if (p.second <= 0.0) throw Error(Error::Kind::ParseError, "AddNode: weight must be > 0");
      }
      for (const auto& p : out) {
        check_node(p.first, "AddNode");
        if (p.second <= 0.0) throw Error(Error::Kind::ParseError, "AddNode: weight must be > 0");
      }
      out_adj_.emplace_back();
      in_adj_.emplace_back();
      out_deg_.push_back(0.0);
      const Index dm = static_cast<Index>(in.size() + out.size());
      DeltaVectors col;
      col.b.size = old_n;
      col.delta_m = dm;
      col.step = DeltaVectors::Step::NodeColumn;
      auto sorted_in = in;
      std::sort(sorted_in.begin(), sorted_in.end());
      for (const auto& p : sorted_in) col.b.nz.emplace_back(p.first, p.second);
      DeltaVectors row;
      row.b.size = old_n + 1;
      row.delta_m = dm;
      row.step = DeltaVectors::Step::NodeRow;
      auto sorted_out = out;
      std::sort(sorted_out.begin(), sorted_out.end());
      for (const auto& p : sorted_out) row.b.nz.emplace_back(p.first, p.second);
      for (const auto& p : in) insert_arc(p.first, old_n, p.second);
      for (const auto& p : out) insert_arc(old_n, p.first, p.second);
      deltas.push_back(std::move(col));
      deltas.push_back(std::move(row));
      break;
    }
  }
  return deltas;
}

std::vector<Index> DynamicGraph::touched_by(const GraphEvent& e) const {
  std::vector<Index> touched;
  auto add = [&touched](Index u) {
    if (std::find(touched.begin(), touched.end(), u) == touched.end()) touched.push_back(u);
  };
  switch (e.kind) {
    case GraphEvent::Kind::AddEdge:
    case GraphEvent::Kind::RemoveEdge:
      add(e.u);
      if (undirected_ && e.u != e.v) add(e.v);
      break;
    case GraphEvent::Kind::AddNode:
      for (const auto& p : e.in_edges) add(p.first);
      if (undirected_)
        for (const auto& p : e.out_edges) add(p.first);
      add(node_count());
      break;
  }
  return touched;
}

// ============================================================ kernels.cpp:7-65
Mat mult_sparseT_dense(const SparseRowMatrix& b, const Mat& a) {
  if (b.rows != a.r)
    throw Error(Error::Kind::ShapeMismatch, "mult_sparseT_dense: row mismatch");
  const Index q = b.cols, p = a.c;
  Mat out(q, p);
  for (Index t = 0; t < b.nnz_rows(); ++t) {
    const Index l = b.idx[t];
    for (Index i = 0; i < q; ++i) {
      const double bv = b.vals(t, i);
      if (bv == 0.0) continue;
      for (Index j = 0; j < p; ++j) out(i, j) += a(l, j) * bv;
    }
  }
  return out;
}

SparseRowMatrix mult_sparse_dense(const SparseRowMatrix& b, const Mat& c) {
  if (b.cols != c.r)
    throw Error(Error::Kind::ShapeMismatch, "mult_sparse_dense: col mismatch");
  SparseRowMatrix out;
  out.rows = b.rows;
  out.cols = c.c;
  std::vector<Vec> kept;
  for (Index t = 0; t < b.nnz_rows(); ++t) {
    Vec row(static_cast<size_t>(c.c), 0.0);
    for (Index i = 0; i < b.cols; ++i) {
      const double bv = b.vals(t, i);
      if (bv == 0.0) continue;
      for (Index j = 0; j < c.c; ++j) row[j] += bv * c(i, j);
    }
    bool z = true;
    for (double v : row) z = z && v == 0.0;
    if (z) continue;
    out.idx.push_back(b.idx[t]);
    kept.push_back(row);
  }
  out.vals = Mat(static_cast<Index>(kept.size()), c.c);
  for (size_t t = 0; t < kept.size(); ++t)
    for (Index j = 0; j < c.c; ++j) out.vals(static_cast<Index>(t), j) = kept[t][j];
  return out;
}

ResidualNorm ortho_residual_norm(const Mat& xb, const Mat& p, const Vec& sigma,
                                 const SparseVec& b) {
  SparseRowMatrix bcol = SparseRowMatrix::from_column(b);
  Mat bt_x = mult_sparseT_dense(bcol, xb);  // 1 x k
  Mat wrow = matmul(bt_x, p);
  ResidualNorm res;
  res.w.resize(static_cast<size_t>(wrow.c));
  double wsq = 0.0;
  for (Index i = 0; i < wrow.c; ++i) {
    res.w[i] = wrow(0, i) / std::sqrt(sigma[i]);
    wsq += res.w[i] * res.w[i];
  }
  res.r = std::sqrt(std::max(0.0, b.norm2sq() - wsq));
  return res;
}

// ============================================================ svd.cpp:12-96
SparseOp SparseOp::from_dense(const Mat& a) {
  SparseOp op;
  op.rows = a.r;
  op.cols = a.c;
  op.apply = [a](const Mat& x) { return matmul(a, x); };
  op.apply_t = [a](const Mat& x) { return matmul(transpose(a), x); };
  return op;
}

Mat qr_orthonormalize(const Mat& m) { return HouseholderQR(m).Q; }

SvdTriple dense_svd_small(const Mat& m, Index keep) {
  if (!m.all_finite()) throw Error(Error::Kind::NonFinite, "dense_svd_small: non-finite input");
  SvdTriple svd = jacobi_svd_full(m);
  Index k = std::min<Index>(keep, svd.rank());
  while (k > 0 && svd.sigma[k - 1] <= 0.0) --k;
  return svd_head(svd, k);
}

SvdTriple randomized_tsvd(const SparseOp& a, Index d, Index oversample,
                          Index power_iters, std::uint64_t seed) {
  const Index n = a.rows, m = a.cols;
  const Index min_dim = std::min(n, m);
  const Index l = min_dim <= 600 ? min_dim : std::min(min_dim, d + oversample);
  Rng rng(seed);
  Mat omega(m, l);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < l; ++j) omega(i, j) = rand_gaussian(rng);
  Mat y = a.apply(omega);
  if (y.frob() == 0.0) throw Error(Error::Kind::ZeroMatrix, "randomized_tsvd: all-zero matrix");
  Mat q = qr_orthonormalize(y);
  if (l < min_dim) {
    for (Index it = 0; it < power_iters; ++it) {
      q = qr_orthonormalize(a.apply_t(q));
      q = qr_orthonormalize(a.apply(q));
    }
  }
  Mat bt = a.apply_t(q);  // m x l
  HouseholderQR qr(bt);
  const Mat& q2 = qr.Q;  // m x l
  Mat r2(l, l);
  for (Index i = 0; i < std::min(l, qr.R.r); ++i)
    for (Index j = i; j < l; ++j) r2(i, j) = qr.R(i, j);
  SvdTriple core = dense_svd_small(transpose(r2), l);
  Index k = std::min<Index>(d, core.rank());
  const double floor = 1e-12 * (core.rank() > 0 ? core.sigma[0] : 0.0);
  while (k > 0 && core.sigma[k - 1] <= floor) --k;
  if (k == 0) throw Error(Error::Kind::ZeroMatrix, "randomized_tsvd: zero-rank matrix");
  SvdTriple ch = svd_head(core, k);
  SvdTriple out;
  out.U = matmul(q, ch.U);
  out.sigma = ch.sigma;
  out.V = matmul(q2, ch.V);
  return out;
}

// ============================================================ factor_state.cpp
namespace {
struct ProjSolver {
  std::optional<PartialPivLU> lu;
  bool reliable = true;
  bool singular = false;
};

// factor_state.cpp:21-36
ProjSolver lu_of_transpose(const Mat& p) {
  ProjSolver s;
  s.lu.emplace(transpose(p));
  const Vec diag = s.lu->diag();
  double dmax = 0.0, dmin = std::numeric_limits<double>::infinity();
  for (double d : diag) {
    dmax = std::max(dmax, std::abs(d));
    dmin = std::min(dmin, std::abs(d));
  }
  if (!diag.empty()) {
    s.singular = !(dmin > 0.0) || !std::isfinite(dmax);
    s.reliable = !s.singular && dmin > dmax * 1e-12;
  }
  return s;
}

void append_column(Mat& m, const SparseVec& col) {
  m.append_zero_col();
  for (const auto& p : col.nz) m(p.first, m.c - 1) = p.second;
}

Mat blkdiag_one(const Mat& p) {
  Mat out(p.r + 1, p.c + 1);
  for (Index i = 0; i < p.r; ++i)
    for (Index j = 0; j < p.c; ++j) out(i, j) = p(i, j);
  out(p.r, p.c) = 1.0;
  return out;
}
}  // namespace

FactorState::FactorState(Mat xb, Mat yb, Mat px, Mat py, Vec sigma, Index d)
    : xb_(std::move(xb)), yb_(std::move(yb)), px_(std::move(px)), py_(std::move(py)),
      sigma_(std::move(sigma)), d_(d) {}

// factor_state.cpp:67-84
SparseOp adjacency_op(const DynamicGraph& g) {
  SparseOp op;
  op.rows = g.node_count();
  op.cols = g.node_count();
  const DynamicGraph* gp = &g;
  op.apply = [gp](const Mat& x) {
    Mat y(gp->node_count(), x.c);
    for (Index u = 0; u < gp->node_count(); ++u)
      for (const auto& p : gp->out_neighbors(u)) {
        const double* xr = x.row(p.first);
        double* yr = y.row(u);
        for (Index j = 0; j < x.c; ++j) yr[j] += p.second * xr[j];
      }
    return y;
  };
  op.apply_t = [gp](const Mat& x) {
    Mat y(gp->node_count(), x.c);
    for (Index u = 0; u < gp->node_count(); ++u)
      for (const auto& p : gp->out_neighbors(u)) {
        const double* xr = x.row(u);
        double* yr = y.row(p.first);
        for (Index j = 0; j < x.c; ++j) yr[j] += p.second * xr[j];
      }
    return y;
  };
  return op;
}

// factor_state.cpp:86-102
FactorState FactorState::init_from_graph(const DynamicGraph& g, Index d, std::uint64_t seed) {
  if (g.node_count() == 0 || g.arc_count() == 0)
    throw Error(Error::Kind::ZeroMatrix, "init_from_graph: graph has no edges");
  SvdTriple svd = randomized_tsvd(adjacency_op(g), d, 10, 4, seed);
  const Index k = svd.rank();
  FactorState s;
  s.xb_ = svd.U;
  s.yb_ = svd.V;
  for (Index i = 0; i < s.xb_.r; ++i)
    for (Index j = 0; j < k; ++j) s.xb_(i, j) *= std::sqrt(svd.sigma[j]);
  for (Index i = 0; i < s.yb_.r; ++i)
    for (Index j = 0; j < k; ++j) s.yb_(i, j) *= std::sqrt(svd.sigma[j]);
  s.px_ = Mat::eye(k);
  s.py_ = Mat::eye(k);
  s.sigma_ = svd.sigma;
  s.d_ = d;
  return s;
}

namespace {
Vec row_times(const Mat& base, Index u, const Mat& p) {
  Vec out(static_cast<size_t>(p.c), 0.0);
  const double* br = base.row(u);
  for (Index i = 0; i < p.r; ++i) {
    const double bi = br[i];
    for (Index j = 0; j < p.c; ++j) out[j] += bi * p(i, j);
  }
  return out;
}
void check_row(Index u, Index n, const char* who) {
  if (u < 0 || u >= n)
    throw Error(Error::Kind::UnknownNode, std::string(who) + ": unknown node " + std::to_string(u));
}
}  // namespace

Vec FactorState::query_context(Index u) const {  // factor_state.cpp:110-113
  check_row(u, rows_x(), "query_context");
  return row_times(xb_, u, px_);
}
Vec FactorState::query_content(Index u) const {  // factor_state.cpp:115-118
  check_row(u, rows_y(), "query_content");
  return row_times(yb_, u, py_);
}
void FactorState::query_all(Mat& x, Mat& y) const {  // factor_state.cpp:120-123
  x = matmul(xb_, px_);
  y = matmul(yb_, py_);
}
double FactorState::reconstruct_entry(Index u, Index v) const {
  Vec a = query_context(u), b = query_content(v);
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// factor_state.cpp:129-213
AppliedDelta FactorState::apply_update(const ProjectionUpdate& u) {
  const Index k_old = rank();
  const Index k2 = static_cast<Index>(u.sigma2.size());
  const bool grown = u.grow_x.has_value();
  AppliedDelta out;
  if (u.append_x >= 0) {
    if (u.append_x != rows_x()) throw Error(Error::Kind::ShapeMismatch, "apply_update: bad row append");
    xb_.append_zero_row();
    out.x_rows_appended = 1;
  }
  if (u.append_y >= 0) {
    if (u.append_y != rows_y()) throw Error(Error::Kind::ShapeMismatch, "apply_update: bad row append");
    yb_.append_zero_row();
  }
  if (grown) {
    if (k2 != k_old + 1 || !u.grow_y.has_value())
      throw Error(Error::Kind::ShapeMismatch, "apply_update: inconsistent rank growth");
    append_column(xb_, *u.grow_x);
    append_column(yb_, *u.grow_y);
    px_ = blkdiag_one(px_);
    py_ = blkdiag_one(py_);
    out.x_grow_col = u.grow_x;
  }
  if (u.F.r != px_.c || u.G.r != py_.c || u.F.c != k2 || u.G.c != k2)
    throw Error(Error::Kind::ShapeMismatch, "apply_update: projection shape");
  Mat px_new = matmul(px_, u.F);
  Mat py_new = matmul(py_, u.G);
  bool eager = k2 < k_old;
  ProjSolver lux, luy;
  if (!eager && k2 > 0) {
    lux = lu_of_transpose(px_new);
    luy = lu_of_transpose(py_new);
    if (lux.singular || luy.singular)
      throw Error(Error::Kind::SingularProjection, "apply_update: projection matrix is singular");
    eager = !lux.reliable || !luy.reliable;
  }
  if (eager) {
    ++eager_folds;
    xb_ = matmul(xb_, px_new);
    yb_ = matmul(yb_, py_new);
    if (fp32_base) round_base();
    for (Index t = 0; t < u.dX.nnz_rows(); ++t)
      for (Index j = 0; j < k2; ++j) xb_(u.dX.idx[t], j) += u.dX.vals(t, j);
    for (Index t = 0; t < u.dY.nnz_rows(); ++t)
      for (Index j = 0; j < k2; ++j) yb_(u.dY.idx[t], j) += u.dY.vals(t, j);
    px_ = Mat::eye(k2);
    py_ = Mat::eye(k2);
    out.x_transform = px_new;
    out.x_base_rows = u.dX;
    sigma_ = u.sigma2;
    return out;
  }
  px_ = px_new;
  py_ = py_new;
  out.x_base_rows = SparseRowMatrix::zero(rows_x(), k2);
  if (u.dX.nnz_rows() > 0) {
    out.x_base_rows.idx = u.dX.idx;
    out.x_base_rows.vals = Mat(u.dX.nnz_rows(), k2);
    for (Index t = 0; t < u.dX.nnz_rows(); ++t) {
      Vec rhs(u.dX.vals.row(t), u.dX.vals.row(t) + k2);
      Vec z = lux.lu->solve(rhs);  // (P^T)^{-1} dX_t^T
      for (Index j = 0; j < k2; ++j) {
        out.x_base_rows.vals(t, j) = z[j];
        xb_(u.dX.idx[t], j) += z[j];
      }
    }
  }
  if (u.dY.nnz_rows() > 0) {
    for (Index t = 0; t < u.dY.nnz_rows(); ++t) {
      Vec rhs(u.dY.vals.row(t), u.dY.vals.row(t) + k2);
      Vec z = luy.lu->solve(rhs);
      for (Index j = 0; j < k2; ++j) yb_(u.dY.idx[t], j) += z[j];
    }
  }
  sigma_ = u.sigma2;
  return out;
}

Mat FactorState::rebase() {  // factor_state.cpp:215-222
  Mat tx = px_;
  xb_ = matmul(xb_, px_);
  yb_ = matmul(yb_, py_);
  px_ = Mat::eye(rank());
  py_ = Mat::eye(rank());
  if (fp32_base) round_base();
  return tx;
}

void FactorState::round_base() {  // harness fp32 storage mode
  for (double& v : xb_.a) v = static_cast<double>(static_cast<float>(v));
  for (double& v : yb_.a) v = static_cast<double>(static_cast<float>(v));
}

double FactorState::cond_estimate() const {  // factor_state.cpp:224-249
  const Index k = rank();
  if (k == 0) return 1.0;
  Vec v(static_cast<size_t>(k), 1.0 / std::sqrt(double(k)));
  double smax_sq = 1.0;
  const Mat pt = transpose(px_);
  auto mv = [](const Mat& m, const Vec& x) {
    Vec y(static_cast<size_t>(m.r), 0.0);
    for (Index i = 0; i < m.r; ++i) y[i] = dot(m.row(i), x.data(), m.c);
    return y;
  };
  auto norm = [](const Vec& x) { return std::sqrt(dot(x.data(), x.data(), (Index)x.size())); };
  for (int it = 0; it < 10; ++it) {
    Vec w = mv(pt, mv(px_, v));
    smax_sq = norm(w);
    if (smax_sq == 0.0) return std::numeric_limits<double>::infinity();
    for (Index i = 0; i < k; ++i) v[i] = w[i] / smax_sq;
  }
  PartialPivLU lu(px_);
  for (double dg : lu.diag())
    if (dg == 0.0) return std::numeric_limits<double>::infinity();
  Vec v2(static_cast<size_t>(k), 1.0 / std::sqrt(double(k)));
  double inv_smin_sq = 1.0;
  for (int it = 0; it < 10; ++it) {
    Vec w = lu.solve(lu.solve_transpose(v2));
    inv_smin_sq = norm(w);
    for (Index i = 0; i < k; ++i) v2[i] = w[i] / inv_smin_sq;
  }
  return std::sqrt(smax_sq) * std::sqrt(inv_smin_sq);
}

double FactorState::proj_row_bound() const {  // factor_state.cpp:251-259
  const Index k = rank();
  if (k == 0) return 1.0;
  double col1 = 0.0, rowinf = 0.0;
  for (Index j = 0; j < k; ++j) {
    double s = 0;
    for (Index i = 0; i < px_.r; ++i) s += std::abs(px_(i, j));
    col1 = std::max(col1, s);
  }
  for (Index i = 0; i < px_.r; ++i) {
    double s = 0;
    for (Index j = 0; j < k; ++j) s += std::abs(px_(i, j));
    rowinf = std::max(rowinf, s);
  }
  return std::max(col1, std::sqrt(col1 * rowinf));
}

namespace {
double ortho_defect(const Mat& base, const Mat& p, const Vec& sigma) {  // :262-273
  if (sigma.empty()) return 0.0;
  Mat u = matmul(base, p);
  for (Index i = 0; i < u.r; ++i)
    for (Index j = 0; j < u.c; ++j) u(i, j) /= std::sqrt(sigma[j]);
  Mat g = matmul(transpose(u), u);
  double worst = 0;
  for (Index i = 0; i < g.r; ++i)
    for (Index j = 0; j < g.c; ++j)
      worst = std::max(worst, std::abs(g(i, j) - (i == j ? 1.0 : 0.0)));
  return worst;
}
}  // namespace

double FactorState::ortho_defect_x() const { return ortho_defect(xb_, px_, sigma_); }
double FactorState::ortho_defect_y() const { return ortho_defect(yb_, py_, sigma_); }

// ============================================================ update_engine.cpp
namespace {
constexpr double kSigmaFloor = 1e-12;  // update_engine.cpp:12
constexpr double kGrowFloor = 1e-6;    // update_engine.cpp:17

// update_engine.cpp:24-31
Mat scale_projection(const Mat& inner, const Vec& s1, const Vec& s2) {
  Mat out(inner.r, inner.c);
  for (Index i = 0; i < inner.r; ++i)
    for (Index j = 0; j < inner.c; ++j) out(i, j) = inner(i, j) * std::sqrt(s2[j] / s1[i]);
  return out;
}

struct SmallSvd {
  Mat e_top, h_top;
  Vec e_bot, h_bot, sigma2;
};

// update_engine.cpp:39-52
SmallSvd split_small_svd(const Mat& m, Index k, Index keep) {
  SvdTriple svd = dense_svd_small(m, keep);
  Index k2 = svd.rank();
  const double floor = k2 > 0 ? kSigmaFloor * svd.sigma[0] : 0.0;
  while (k2 > 0 && svd.sigma[k2 - 1] < floor) --k2;
  SmallSvd out;
  out.e_top = Mat(k, k2);
  out.h_top = Mat(k, k2);
  out.e_bot.assign(static_cast<size_t>(k2), 0.0);
  out.h_bot.assign(static_cast<size_t>(k2), 0.0);
  for (Index j = 0; j < k2; ++j) {
    for (Index i = 0; i < k; ++i) {
      out.e_top(i, j) = svd.U(i, j);
      out.h_top(i, j) = svd.V(i, j);
    }
    out.e_bot[j] = svd.U(k, j);
    out.h_bot[j] = svd.V(k, j);
  }
  out.sigma2.assign(svd.sigma.begin(), svd.sigma.begin() + k2);
  return out;
}

// inner = top - (w / r) * bot (outer product)
Mat corrected(const Mat& top, const Vec& w, double r, const Vec& bot) {
  Mat out = top;
  for (Index i = 0; i < top.r; ++i)
    for (Index j = 0; j < top.c; ++j) out(i, j) -= (w[i] / r) * bot[j];
  return out;
}
}  // namespace

// update_engine.cpp:56-142
ProjectionUpdate update_embedding_n(const FactorState& s, const SparseVec& b, bool u_is_x) {
  const Index k = s.rank();
  const Index n_u = u_is_x ? s.rows_x() : s.rows_y();
  const Index n_v = u_is_x ? s.rows_y() : s.rows_x();
  if (b.size != n_u) throw Error(Error::Kind::ShapeMismatch, "update_embedding_n: column size");
  ResidualNorm res = u_is_x ? ortho_residual_norm(s.xb(), s.px(), s.sigma(), b)
                            : ortho_residual_norm(s.yb(), s.py(), s.sigma(), b);
  const double bnorm = std::sqrt(b.norm2sq());
  const double delta_r = 1e-12 * std::max(1.0, bnorm);
  const double r_b = std::max(res.r, delta_r);
  Mat m(k + 1, k + 1);
  for (Index i = 0; i < k; ++i) {
    m(i, i) = s.sigma()[i];
    m(i, k) = res.w[i];
  }
  m(k, k) = r_b;
  const Index rank_cap = std::min(n_u, n_v + 1);
  const bool allow_grow =
      k < s.dim() && k < rank_cap && res.r >= kGrowFloor * std::max(1.0, bnorm);
  SmallSvd small = split_small_svd(m, k, allow_grow ? k + 1 : k);
  const Index k2 = static_cast<Index>(small.sigma2.size());
  Vec s2root(static_cast<size_t>(k2));
  for (Index j = 0; j < k2; ++j) s2root[j] = std::sqrt(small.sigma2[j]);
  Mat inner_f = corrected(small.e_top, res.w, r_b, small.e_bot);
  Mat f_top = scale_projection(inner_f, s.sigma(), small.sigma2);
  Mat g_top = scale_projection(small.h_top, s.sigma(), small.sigma2);
  Vec ex(static_cast<size_t>(k2)), vrow(static_cast<size_t>(k2));
  for (Index j = 0; j < k2; ++j) {
    ex[j] = (small.e_bot[j] * s2root[j]) / r_b;
    vrow[j] = small.h_bot[j] * s2root[j];
  }
  ProjectionUpdate pu;
  pu.sigma2 = small.sigma2;
  const bool grown = k2 == k + 1;
  Mat f_u, g_v;
  SparseRowMatrix d_u = SparseRowMatrix::zero(n_u, k2);
  SparseRowMatrix d_v = SparseRowMatrix::zero(n_v + 1, k2);
  if (grown) {
    f_u = Mat(k + 1, k2);
    g_v = Mat(k + 1, k2);
    for (Index j = 0; j < k2; ++j) {
      for (Index i = 0; i < k; ++i) {
        f_u(i, j) = f_top(i, j);
        g_v(i, j) = g_top(i, j);
      }
      f_u(k, j) = ex[j];
      g_v(k, j) = vrow[j];
    }
  } else {
    f_u = f_top;
    g_v = g_top;
    d_u = SparseRowMatrix::outer(b, ex);
    bool vz = true;
    for (double v : vrow) vz = vz && v == 0.0;
    if (!vz) {
      d_v.idx.push_back(n_v);
      d_v.vals = Mat(1, k2);
      for (Index j = 0; j < k2; ++j) d_v.vals(0, j) = vrow[j];
    }
  }
  if (u_is_x) {
    pu.F = f_u;
    pu.G = g_v;
    pu.dX = d_u;
    pu.dY = d_v;
    pu.append_y = n_v;
    if (grown) {
      pu.grow_x = b;
      pu.grow_y = SparseVec::unit(n_v + 1, n_v);
    }
  } else {
    pu.F = g_v;
    pu.G = f_u;
    pu.dX = d_v;
    pu.dY = d_u;
    pu.append_x = n_v;
    if (grown) {
      pu.grow_x = SparseVec::unit(n_v + 1, n_v);
      pu.grow_y = b;
    }
  }
  return pu;
}

// update_engine.cpp:144-204
ProjectionUpdate update_embedding_e(const FactorState& s, const SparseVec& b, const SparseVec& c) {
  const Index k = s.rank();
  if (b.size != s.rows_x() || c.size != s.rows_y())
    throw Error(Error::Kind::ShapeMismatch, "update_embedding_e: column size");
  ResidualNorm res_b = ortho_residual_norm(s.xb(), s.px(), s.sigma(), b);
  ResidualNorm res_c = ortho_residual_norm(s.yb(), s.py(), s.sigma(), c);
  const double bnorm = std::sqrt(b.norm2sq());
  const double cnorm = std::sqrt(c.norm2sq());
  const double r_b = std::max(res_b.r, 1e-12 * std::max(1.0, bnorm));
  const double r_c = std::max(res_c.r, 1e-12 * std::max(1.0, cnorm));
  Vec wb(static_cast<size_t>(k + 1)), wc(static_cast<size_t>(k + 1));
  for (Index i = 0; i < k; ++i) {
    wb[i] = res_b.w[i];
    wc[i] = res_c.w[i];
  }
  wb[k] = r_b;
  wc[k] = r_c;
  Mat m(k + 1, k + 1);
  for (Index i = 0; i < k; ++i) m(i, i) = s.sigma()[i];
  for (Index i = 0; i <= k; ++i)
    for (Index j = 0; j <= k; ++j) m(i, j) += wb[i] * wc[j];
  const bool allow_grow = k < s.dim() && k < std::min(s.rows_x(), s.rows_y()) &&
                          res_b.r >= kGrowFloor * std::max(1.0, bnorm) &&
                          res_c.r >= kGrowFloor * std::max(1.0, cnorm);
  SmallSvd small = split_small_svd(m, k, allow_grow ? k + 1 : k);
  const Index k2 = static_cast<Index>(small.sigma2.size());
  Vec s2root(static_cast<size_t>(k2));
  for (Index j = 0; j < k2; ++j) s2root[j] = std::sqrt(small.sigma2[j]);
  Mat inner_f = corrected(small.e_top, res_b.w, r_b, small.e_bot);
  Mat inner_g = corrected(small.h_top, res_c.w, r_c, small.h_bot);
  Mat f_top = scale_projection(inner_f, s.sigma(), small.sigma2);
  Mat g_top = scale_projection(inner_g, s.sigma(), small.sigma2);
  Vec ex(static_cast<size_t>(k2)), ey(static_cast<size_t>(k2));
  for (Index j = 0; j < k2; ++j) {
    ex[j] = (small.e_bot[j] * s2root[j]) / r_b;
    ey[j] = (small.h_bot[j] * s2root[j]) / r_c;
  }
  ProjectionUpdate pu;
  pu.sigma2 = small.sigma2;
  if (k2 == k + 1) {
    pu.F = Mat(k + 1, k2);
    pu.G = Mat(k + 1, k2);
    for (Index j = 0; j < k2; ++j) {
      for (Index i = 0; i < k; ++i) {
        pu.F(i, j) = f_top(i, j);
        pu.G(i, j) = g_top(i, j);
      }
      pu.F(k, j) = ex[j];
      pu.G(k, j) = ey[j];
    }
    pu.grow_x = b;
    pu.grow_y = c;
    pu.dX = SparseRowMatrix::zero(s.rows_x(), k2);
    pu.dY = SparseRowMatrix::zero(s.rows_y(), k2);
  } else {
    pu.F = f_top;
    pu.G = g_top;
    pu.dX = SparseRowMatrix::outer(b, ex);
    pu.dY = SparseRowMatrix::outer(c, ey);
  }
  return pu;
}

// update_engine.cpp:206-226
HandledEvent handle_event(FactorState& s, const std::vector<DeltaVectors>& deltas) {
  HandledEvent out;
  for (const DeltaVectors& dv : deltas) {
    ProjectionUpdate pu;
    switch (dv.step) {
      case DeltaVectors::Step::Edge:
        pu = update_embedding_e(s, dv.b, *dv.c);
        break;
      case DeltaVectors::Step::NodeColumn:
        pu = update_embedding_n(s, dv.b, true);
        break;
      case DeltaVectors::Step::NodeRow:
        pu = update_embedding_n(s, dv.b, false);
        break;
    }
    out.applied.push_back(s.apply_update(pu));
    out.updates.push_back(std::move(pu));
  }
  return out;
}

// ============================================================ enhancer.cpp
namespace {
constexpr std::uint64_t kPushGuard = 1000000000ull;  // enhancer.cpp:8
double row_inf(const Mat& m, Index u) {
  double s = 0;
  for (Index j = 0; j < m.c; ++j) s = std::max(s, std::abs(m(u, j)));
  return s;
}
}  // namespace

EnhancerState::EnhancerState(EnhancerParams params, Mat zb, Mat rb)  // enhancer.cpp:11-24
    : params_(params), zb_(std::move(zb)), rb_(std::move(rb)) {
  in_fifo_.assign(static_cast<size_t>(zb_.r), 0);
  index_key_.assign(static_cast<size_t>(zb_.r), 0.0);
  for (Index u = 0; u < rb_.r; ++u) {
    const double key = rb_.c > 0 ? row_inf(rb_, u) : 0.0;
    if (key > 0.0) {
      index_.emplace(key, u);
      index_key_[u] = key;
    }
  }
}

EnhancerState EnhancerState::init_propagate(const DynamicGraph& g, const FactorState& s,
                                            EnhancerParams params) {  // enhancer.cpp:26-47
  EnhancerState e;
  e.params_ = params;
  const Index n = s.rows_x();
  e.in_fifo_.assign(static_cast<size_t>(n), 0);
  e.index_key_.assign(static_cast<size_t>(n), 0.0);
  if (params.alpha == 1.0) {
    e.zb_ = s.xb();
    e.rb_ = Mat(n, s.rank());
    return e;
  }
  e.zb_ = Mat(n, s.rank());
  e.rb_ = s.xb();
  for (double& v : e.rb_.a) v *= params.alpha;
  for (Index u = 0; u < n; ++u) {
    e.fifo_.push_back(u);
    e.in_fifo_[u] = 1;
  }
  e.push_to_tolerance(g, s);
  return e;
}

double EnhancerState::row_key(Index u, double deg) const {  // enhancer.cpp:49-52
  if (rb_.c == 0) return 0.0;
  return row_inf(rb_, u) / std::max(deg, 1.0);
}

void EnhancerState::note_residual(Index u, double key) {  // enhancer.cpp:54-59
  if (key > index_key_[u]) {
    index_.emplace(key, u);
    index_key_[u] = key;
  }
}

void EnhancerState::absorb_signal_delta(const SparseRowMatrix& dxb) {  // :61-75
  if (params_.alpha == 1.0) {
    for (Index t = 0; t < dxb.nnz_rows(); ++t)
      for (Index j = 0; j < dxb.cols; ++j) zb_(dxb.idx[t], j) += dxb.vals(t, j);
    return;
  }
  for (Index t = 0; t < dxb.nnz_rows(); ++t) {
    const Index u = dxb.idx[t];
    for (Index j = 0; j < dxb.cols; ++j) rb_(u, j) += params_.alpha * dxb.vals(t, j);
    if (!in_fifo_[u]) {
      fifo_.push_back(u);
      in_fifo_[u] = 1;
    }
  }
}

void EnhancerState::absorb_structure_delta(const DynamicGraph& g, const FactorState& s,
                                           const std::vector<Index>& touched) {  // :77-96
  if (params_.alpha == 1.0) return;
  const double one_minus = 1.0 - params_.alpha;
  const Index k = zb_.c;
  Vec acc(static_cast<size_t>(k)), nb(static_cast<size_t>(k));
  for (Index u : touched) {
    const double deg = g.out_degree(u);
    for (Index j = 0; j < k; ++j) acc[j] = params_.alpha * s.xb()(u, j) - zb_(u, j);
    if (deg > 0.0) {
      std::fill(nb.begin(), nb.end(), 0.0);
      for (const auto& p : g.out_neighbors(u))
        for (Index j = 0; j < k; ++j) nb[j] += p.second * zb_(p.first, j);
      for (Index j = 0; j < k; ++j) acc[j] += (one_minus / deg) * nb[j];
    }
    for (Index j = 0; j < k; ++j) rb_(u, j) = acc[j];
    if (!in_fifo_[u]) {
      fifo_.push_back(u);
      in_fifo_[u] = 1;
    }
  }
}

void EnhancerState::push_to_tolerance(const DynamicGraph& g, const FactorState& s) {  // :98-157
  if (params_.alpha == 1.0) return;
  const double smax = s.proj_row_bound();
  const double eps = params_.alpha * params_.eps;
  const double one_minus = 1.0 - params_.alpha;
  while (!index_.empty() && index_.top().first * smax > eps) {
    auto [key, u] = index_.top();
    index_.pop();
    if (index_key_[u] == key) index_key_[u] = 0.0;
    const double cur = row_key(u, g.out_degree(u));
    if (cur * smax > eps) {
      if (!in_fifo_[u]) {
        fifo_.push_back(u);
        in_fifo_[u] = 1;
      }
    } else {
      note_residual(u, cur);
    }
  }
  std::uint64_t pushes = 0;
  const Index k = rb_.c;
  Vec delta(static_cast<size_t>(k));
  while (!fifo_.empty()) {
    const Index u = fifo_.front();
    fifo_.pop_front();
    in_fifo_[u] = 0;
    const double deg_u = g.out_degree(u);
    const double cur = row_key(u, deg_u);
    if (cur * smax <= eps) {
      if (cur > 0.0) note_residual(u, cur);
      continue;
    }
    if (++pushes > kPushGuard)
      throw Error(Error::Kind::NonConvergence, "push_to_tolerance: push budget exceeded; eps too small");
    for (Index j = 0; j < k; ++j) {
      delta[j] = rb_(u, j);
      rb_(u, j) = 0.0;
      zb_(u, j) += delta[j];
    }
    for (const auto& p : g.in_neighbors(u)) {
      const Index v = p.first;
      const double deg_v = std::max(g.out_degree(v), 1.0);
      const double f = one_minus * p.second / deg_v;
      for (Index j = 0; j < k; ++j) rb_(v, j) += f * delta[j];
      const double key_v = row_key(v, g.out_degree(v));
      if (key_v * smax > eps) {
        if (!in_fifo_[v]) {
          fifo_.push_back(v);
          in_fifo_[v] = 1;
        }
      } else if (key_v > 0.0) {
        note_residual(v, key_v);
      }
    }
  }
  total_pushes_ += pushes;
}

Vec EnhancerState::query_enhanced(const FactorState& s, Index u) const {  // :159-164
  if (u < 0 || u >= zb_.r)
    throw Error(Error::Kind::UnknownNode, "query_enhanced: unknown node " + std::to_string(u));
  return row_times(zb_, u, s.px());
}

void EnhancerState::append_rows(Index count) {  // :166-176
  for (Index i = 0; i < count; ++i) {
    zb_.append_zero_row();
    rb_.append_zero_row();
  }
  in_fifo_.resize(static_cast<size_t>(zb_.r), 0);
  index_key_.resize(static_cast<size_t>(zb_.r), 0.0);
}

void EnhancerState::grow_column(const SparseVec& col) {  // :178-194
  zb_.append_zero_col();
  rb_.append_zero_col();
  if (params_.alpha == 1.0) {
    for (const auto& p : col.nz) zb_(p.first, zb_.c - 1) = p.second;
    return;
  }
  for (const auto& p : col.nz) {
    rb_(p.first, rb_.c - 1) += params_.alpha * p.second;
    if (!in_fifo_[p.first]) {
      fifo_.push_back(p.first);
      in_fifo_[p.first] = 1;
    }
  }
}

void EnhancerState::apply_transform(const Mat& t) {  // :196-206
  zb_ = matmul(zb_, t);
  rb_ = matmul(rb_, t);
  if (params_.alpha == 1.0) return;
  for (Index u = 0; u < rb_.r; ++u) {
    const double key = rb_.c > 0 ? row_inf(rb_, u) : 0.0;
    note_residual(u, key);
  }
}

// ============================================================ engine.cpp:5-52
Engine::Engine(DynamicGraph g, const RunConfig& cfg) : g_(std::move(g)), cfg_(cfg) {
  fs_ = FactorState::init_from_graph(g_, cfg.d, cfg.seed);
  es_ = EnhancerState::init_propagate(g_, fs_, EnhancerParams{cfg.alpha, cfg.eps});
}

Engine::Engine(DynamicGraph g, FactorState fs, EnhancerState es, const RunConfig& cfg,
               std::uint64_t events_applied, Index events_since_rebase)
    : g_(std::move(g)), fs_(std::move(fs)), es_(std::move(es)), cfg_(cfg),
      events_applied_(events_applied), events_since_rebase_(events_since_rebase) {}

void Engine::apply(const GraphEvent& e) {
  std::vector<Index> touched = g_.touched_by(e);
  std::vector<DeltaVectors> deltas = g_.apply_event(e);
  HandledEvent handled = handle_event(fs_, deltas);
  for (const ProjectionUpdate& pu : handled.updates) {  // harness hook
    if (row_log) {
      for (Index r : pu.dX.idx) row_log->insert(row_log->end(), {row_log_step, 0, r});
      for (Index r : pu.dY.idx) row_log->insert(row_log->end(), {row_log_step, 1, r});
    }
    ++row_log_step;
  }
  for (const AppliedDelta& ad : handled.applied) {
    if (ad.x_transform) es_.apply_transform(*ad.x_transform);
    if (ad.x_rows_appended > 0) es_.append_rows(ad.x_rows_appended);
    if (ad.x_grow_col) es_.grow_column(*ad.x_grow_col);
    if (ad.x_base_rows.nnz_rows() > 0) es_.absorb_signal_delta(ad.x_base_rows);
  }
  es_.absorb_structure_delta(g_, fs_, touched);
  es_.push_to_tolerance(g_, fs_);
  ++events_applied_;
  if (++events_since_rebase_ >= cfg_.rebase_every || fs_.cond_estimate() > cfg_.rebase_cond)
    rebase();
}

void Engine::rebase() {
  Mat t = fs_.rebase();
  es_.apply_transform(t);
  events_since_rebase_ = 0;
  ++rebases;
}

double Engine::score(Index u, Index v, bool enhanced) const {
  Vec zu = enhanced ? es_.query_enhanced(fs_, u) : fs_.query_context(u);
  Vec yv = fs_.query_content(v);
  double s = 0;
  for (size_t i = 0; i < zu.size(); ++i) s += zu[i] * yv[i];
  return s;
}

// ============================================================ eval.cpp:405-610
namespace {
SvdTriple jacobi_svd_keep(const Mat& m, Index keep) {  // eval.cpp:407-418
  SvdTriple svd = jacobi_svd_full(m);
  Index k = std::min<Index>(keep, svd.rank());
  while (k > 0 && svd.sigma[k - 1] <= 0.0) --k;
  return svd_head(svd, k);
}
Mat dense_adjacency(const DynamicGraph& g) {
  const Index n = g.node_count();
  Mat a(n, n);
  for (Index u = 0; u < n; ++u)
    for (const auto& p : g.out_neighbors(u)) a(u, p.first) += p.second;
  return a;
}
Vec matT_vec(const Mat& m, const Vec& x) {  // m^T x
  Vec y(static_cast<size_t>(m.c), 0.0);
  for (Index i = 0; i < m.r; ++i)
    for (Index j = 0; j < m.c; ++j) y[j] += m(i, j) * x[i];
  return y;
}
Vec mat_vec(const Mat& m, const Vec& x) {
  Vec y(static_cast<size_t>(m.r), 0.0);
  for (Index i = 0; i < m.r; ++i) y[i] = dot(m.row(i), x.data(), m.c);
  return y;
}
double vnorm(const Vec& x) { return std::sqrt(dot(x.data(), x.data(), (Index)x.size())); }
}  // namespace

OracleTsvd::OracleTsvd(const DynamicGraph& g0, Index d) : d_(d) {  // eval.cpp:422-436
  const Index n = g0.node_count();
  if (n > 500) throw Error(Error::Kind::TooLarge, "OracleTsvd: graph too large");
  SvdTriple svd = jacobi_svd_keep(dense_adjacency(g0), d);
  Index k = svd.rank();
  const double floor = k > 0 ? 1e-12 * svd.sigma[0] : 0.0;
  while (k > 0 && svd.sigma[k - 1] < floor) --k;
  SvdTriple h = svd_head(svd, k);
  u_ = h.U;
  sigma_ = h.sigma;
  v_ = h.V;
}

void OracleTsvd::apply_deltas(const std::vector<DeltaVectors>& deltas) {  // :438-453
  gap_ok_ = true;
  for (const DeltaVectors& dv : deltas) {
    switch (dv.step) {
      case DeltaVectors::Step::Edge: step(dv.b, dv.c, false); break;
      case DeltaVectors::Step::NodeColumn: step(dv.b, std::nullopt, false); break;
      case DeltaVectors::Step::NodeRow: step(dv.b, std::nullopt, true); break;
    }
  }
}

void OracleTsvd::step(const SparseVec& b, const std::optional<SparseVec>& c, bool swapped) {
  // eval.cpp:455-540
  Mat& ub = swapped ? v_ : u_;
  Mat& vb = swapped ? u_ : v_;
  const Index k = static_cast<Index>(sigma_.size());
  Vec bd = b.to_dense();
  Vec w = matT_vec(ub, bd);
  Vec q = bd;
  {
    Vec uw = mat_vec(ub, w);
    for (size_t i = 0; i < q.size(); ++i) q[i] -= uw[i];
    Vec w2 = matT_vec(ub, q);
    Vec uw2 = mat_vec(ub, w2);
    for (size_t i = 0; i < q.size(); ++i) q[i] -= uw2[i];
    for (Index i = 0; i < k; ++i) w[i] += w2[i];
  }
  double r = vnorm(q);
  const double tiny = 1e-6 * std::max(1.0, vnorm(bd));
  Vec qn(q.size(), 0.0);
  if (r > tiny)
    for (size_t i = 0; i < q.size(); ++i) qn[i] = q[i] / r;
  if (r <= tiny) r = 0.0;
  Mat m(k + 1, k + 1);
  for (Index i = 0; i < k; ++i) m(i, i) = sigma_[i];
  Vec cq;
  if (c) {
    Vec cd = c->to_dense();
    Vec cw = matT_vec(vb, cd);
    cq = cd;
    Vec vw = mat_vec(vb, cw);
    for (size_t i = 0; i < cq.size(); ++i) cq[i] -= vw[i];
    Vec cw2 = matT_vec(vb, cq);
    Vec vw2 = mat_vec(vb, cw2);
    for (size_t i = 0; i < cq.size(); ++i) cq[i] -= vw2[i];
    for (Index i = 0; i < k; ++i) cw[i] += cw2[i];
    double rc = vnorm(cq);
    const double tiny_c = 1e-6 * std::max(1.0, vnorm(cd));
    if (rc > tiny_c) {
      for (double& v : cq) v /= rc;
    } else {
      rc = 0.0;
      std::fill(cq.begin(), cq.end(), 0.0);
    }
    Vec wb(static_cast<size_t>(k + 1)), wc(static_cast<size_t>(k + 1));
    for (Index i = 0; i < k; ++i) {
      wb[i] = w[i];
      wc[i] = cw[i];
    }
    wb[k] = r;
    wc[k] = rc;
    for (Index i = 0; i <= k; ++i)
      for (Index j = 0; j <= k; ++j) m(i, j) += wb[i] * wc[j];
  } else {
    for (Index i = 0; i < k; ++i) m(i, k) = w[i];
    m(k, k) = r;
  }
  SvdTriple small = jacobi_svd_keep(m, k + 1);
  Index k2 = std::min<Index>(d_, small.rank());
  const double floor = small.rank() > 0 ? 1e-12 * small.sigma[0] : 0.0;
  while (k2 > 0 && small.sigma[k2 - 1] < floor) --k2;
  const double s1 = small.rank() > 0 ? small.sigma[0] : 0.0;
  const double skept = k2 > 0 ? small.sigma[k2 - 1] : 0.0;
  const double snext = k2 < small.rank() ? small.sigma[k2] : 0.0;
  if (!(skept - snext > 1e-6 * s1)) gap_ok_ = false;
  // U2 = [Ub, qn] * small.U[:, :k2]
  Mat u2(ub.r, k2);
  for (Index i = 0; i < ub.r; ++i)
    for (Index j = 0; j < k2; ++j) {
      double s = qn[i] * small.U(k, j);
      for (Index t = 0; t < k; ++t) s += ub(i, t) * small.U(t, j);
      u2(i, j) = s;
    }
  Mat v2;
  if (c) {
    v2 = Mat(vb.r, k2);
    for (Index i = 0; i < vb.r; ++i)
      for (Index j = 0; j < k2; ++j) {
        double s = cq[i] * small.V(k, j);
        for (Index t = 0; t < k; ++t) s += vb(i, t) * small.V(t, j);
        v2(i, j) = s;
      }
  } else {
    v2 = Mat(vb.r + 1, k2);
    for (Index i = 0; i < vb.r; ++i)
      for (Index j = 0; j < k2; ++j) {
        double s = 0;
        for (Index t = 0; t < k; ++t) s += vb(i, t) * small.V(t, j);
        v2(i, j) = s;
      }
    for (Index j = 0; j < k2; ++j) v2(vb.r, j) = small.V(k, j);
  }
  ub = u2;
  vb = v2;
  sigma_.assign(small.sigma.begin(), small.sigma.begin() + k2);
}

Mat OracleTsvd::product() const {  // eval.cpp:542-544
  Mat us = u_;
  for (Index i = 0; i < us.r; ++i)
    for (Index j = 0; j < us.c; ++j) us(i, j) *= sigma_[j];
  return matmul(us, transpose(v_));
}

double OracleTsvd::product_rel_dist(const FactorState& s) const {  // eval.cpp:546-559
  Mat x, y;
  s.query_all(x, y);
  double norm_o_sq = 0;
  for (double v : sigma_) norm_o_sq += v * v;
  Mat xtx = matmul(transpose(x), x), yty = matmul(transpose(y), y);
  Mat p = matmul(xtx, yty);
  double norm_e_sq = 0;
  for (Index i = 0; i < p.r; ++i) norm_e_sq += p(i, i);
  Mat xtu = matmul(transpose(x), u_);
  for (Index i = 0; i < xtu.r; ++i)
    for (Index j = 0; j < xtu.c; ++j) xtu(i, j) *= sigma_[j];
  Mat cr = matmul(xtu, matmul(transpose(v_), y));
  double cross = 0;
  for (Index i = 0; i < cr.r; ++i) cross += cr(i, i);
  const double dist_sq = std::max(0.0, norm_e_sq - 2.0 * cross + norm_o_sq);
  if (norm_o_sq == 0.0) return std::sqrt(norm_e_sq);
  return std::sqrt(dist_sq / norm_o_sq);
}

double OracleTsvd::sigma_rel_dist(const Vec& es) const {  // eval.cpp:561-568
  const size_t k = std::max(es.size(), sigma_.size());
  Vec a(k, 0.0), b(k, 0.0);
  std::copy(es.begin(), es.end(), a.begin());
  std::copy(sigma_.begin(), sigma_.end(), b.begin());
  double num = 0, den = 0;
  for (size_t i = 0; i < k; ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  if (den == 0.0) {
    double an = 0;
    for (double v : a) an += v * v;
    return std::sqrt(an);
  }
  return std::sqrt(num / den);
}

DriftReport drift_report(const FactorState& s, const DynamicGraph& g) {  // :570-589
  const Index n = g.node_count();
  if (n > 500) throw Error(Error::Kind::TooLarge, "drift_report");
  Mat a = dense_adjacency(g);
  SvdTriple svd = jacobi_svd_keep(a, s.dim());
  Mat best = svd.reconstruct();
  Mat x, y;
  s.query_all(x, y);
  DriftReport r;
  const double an = a.frob();
  Mat xy = matmul(x, transpose(y));
  for (size_t i = 0; i < xy.a.size(); ++i) xy.a[i] -= best.a[i];
  r.drift = an == 0.0 ? 0.0 : xy.frob() / an;
  for (Index u = 0; u < n; ++u) {
    double mx = 0;
    for (Index j = 0; j < x.c; ++j) mx = std::max(mx, std::abs(x(u, j)));
    r.c_diag = std::max(r.c_diag, g.out_degree(u) * mx);
  }
  return r;
}

double dense_defect_bound(const DynamicGraph& g, const FactorState& s,
                          const EnhancerState& e) {  // eval.cpp:591-610
  const Index n = g.node_count();
  const double alpha = e.alpha();
  Mat z = matmul(e.zb(), s.px());
  Mat x = matmul(s.xb(), s.px());
  double worst = 0.0;
  const Index k = z.c;
  Vec def(static_cast<size_t>(k)), nb(static_cast<size_t>(k));
  for (Index u = 0; u < n; ++u) {
    for (Index j = 0; j < k; ++j) def[j] = alpha * x(u, j) - z(u, j);
    const double deg = g.out_degree(u);
    if (deg > 0.0) {
      std::fill(nb.begin(), nb.end(), 0.0);
      for (const auto& p : g.out_neighbors(u))
        for (Index j = 0; j < k; ++j) nb[j] += p.second * z(p.first, j);
      for (Index j = 0; j < k; ++j) def[j] += ((1.0 - alpha) / deg) * nb[j];
    }
    double mx = 0;
    for (double v : def) mx = std::max(mx, std::abs(v));
    worst = std::max(worst, mx / std::max(deg, 1.0));
  }
  return worst;
}

// ============================================================ eval.cpp:616-705
DynamicGraph gen_random_graph(Index n, Index arcs, std::uint64_t seed, bool undirected) {
  DynamicGraph g(n, undirected);
  Rng rng(seed);
  Index placed = 0;
  while (placed < arcs) {
    Index u = static_cast<Index>(rand_index(rng, n));
    Index v = static_cast<Index>(rand_index(rng, n));
    if (u == v) continue;
    if (g.has_edge(u, v) || (undirected && g.has_edge(v, u))) continue;
    g.add_arc_raw(u, v, 1.0);
    if (undirected) g.add_arc_raw(v, u, 1.0);
    ++placed;
  }
  return g;
}

DynamicGraph gen_sbm(Index n, double p_in, double p_out, std::uint64_t seed) {
  DynamicGraph g(n, true);
  Rng rng(seed);
  const Index half = n / 2;
  for (Index u = 0; u < n; ++u)
    for (Index v = u + 1; v < n; ++v) {
      const bool same = (u < half) == (v < half);
      if (rand_unit(rng) < (same ? p_in : p_out)) {
        g.add_arc_raw(u, v, 1.0);
        g.add_arc_raw(v, u, 1.0);
      }
    }
  return g;
}

StreamCase gen_mixed_stream(Index n_total, Index n0, Index m0, Index n_events,
                            std::uint64_t seed) {
  StreamCase sc{gen_random_graph(n0, m0, seed), {}};
  DynamicGraph mirror = sc.g0;
  Rng rng(seed ^ 0xabcdef1234567890ull);
  std::vector<std::pair<Index, Index>> arcs;
  for (Index u = 0; u < n0; ++u)
    for (const auto& p : mirror.out_neighbors(u)) arcs.emplace_back(u, p.first);
  for (Index t = 0; t < n_events; ++t) {
    const Index remaining = n_events - t;
    const bool add_node =
        mirror.node_count() < n_total &&
        rand_index(rng, remaining) < static_cast<std::uint64_t>(n_total - mirror.node_count());
    GraphEvent ev;
    if (add_node) {
      ev.kind = GraphEvent::Kind::AddNode;
      const Index n = mirror.node_count();
      const Index fan_in = 1 + static_cast<Index>(rand_index(rng, 3));
      const Index fan_out = static_cast<Index>(rand_index(rng, 3));
      std::unordered_set<std::uint64_t> used;
      for (Index i = 0; i < fan_in; ++i) {
        Index s = static_cast<Index>(rand_index(rng, n));
        if (!used.insert(s).second) continue;
        ev.in_edges.emplace_back(s, 1.0);
        arcs.emplace_back(s, n);
      }
      used.clear();
      for (Index i = 0; i < fan_out; ++i) {
        Index d2 = static_cast<Index>(rand_index(rng, n));
        if (!used.insert(d2).second) continue;
        ev.out_edges.emplace_back(d2, 1.0);
        arcs.emplace_back(n, d2);
      }
    } else if (!arcs.empty() && rand_unit(rng) < 0.3) {
      const size_t pick = rand_index(rng, arcs.size());
      ev = GraphEvent::remove_edge(arcs[pick].first, arcs[pick].second);
      arcs[pick] = arcs.back();
      arcs.pop_back();
      if (arcs.empty()) ev = GraphEvent::add_edge(0, 1, 1.0);
    } else {
      const Index n = mirror.node_count();
      Index u, v;
      do {
        u = static_cast<Index>(rand_index(rng, n));
        v = static_cast<Index>(rand_index(rng, n));
      } while (u == v || mirror.has_edge(u, v));
      ev = GraphEvent::add_edge(u, v, 1.0);
      arcs.emplace_back(u, v);
    }
    mirror.apply_event(ev);
    sc.events.push_back(std::move(ev));
  }
  return sc;
}

}  // namespace damf_oracle
