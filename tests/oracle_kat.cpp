// Known-answer tests for the CPU oracle, ported case by case from the
// reference's doctest suite (/root/reference/proj/tests/*.cpp) with the same
// inputs, seeds and tolerances. This pins the restatement (oracle/) before
// anything on the GPU is compared against it. Built and run by
// tests/test_oracle_kat.py; prints one line per case and exits non-zero on
// any failure.
#include <chrono>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "../oracle/damf_oracle.hpp"

using namespace damf_oracle;

namespace {

int g_fail = 0, g_checks = 0;
std::string g_case;

#define CHECK(...)                                                                  \
  do {                                                                              \
    ++g_checks;                                                                     \
    if (!(__VA_ARGS__)) {                                                               \
      ++g_fail;                                                                     \
      std::printf("  FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #__VA_ARGS__); \
    }                                                                               \
  } while (0)

#define CHECK_THROWS(expr)             \
  do {                                 \
    bool thrown = false;               \
    try {                              \
      (void)(expr);                    \
    } catch (const Error&) {           \
      thrown = true;                   \
    }                                  \
    CHECK(thrown);                     \
  } while (0)

bool approx(double a, double b, double eps = 1e-5) {
  // doctest::Approx: |a-b| < eps * (scale + max(|a|,|b|)), scale = 1
  return std::abs(a - b) < eps * (1.0 + std::max(std::abs(a), std::abs(b)));
}

// ---- tests/helpers.hpp:13-119 ----------------------------------------------
Mat random_dense(Index r, Index c, Rng& rng) {
  Mat m(r, c);
  for (Index i = 0; i < r; ++i)
    for (Index j = 0; j < c; ++j) m(i, j) = rand_gaussian(rng);
  return m;
}
Mat random_orthonormal(Index r, Index c, Rng& rng) {
  return HouseholderQR(random_dense(r, c, rng)).Q;
}
SparseRowMatrix random_sparse_rows(Index rows, Index cols, Index t, Rng& rng) {
  SparseRowMatrix m;
  m.rows = rows;
  m.cols = cols;
  std::vector<Index> picked;
  while (static_cast<Index>(picked.size()) < t) {
    Index r = static_cast<Index>(rand_index(rng, rows));
    bool dup = false;
    for (Index p : picked) dup = dup || p == r;
    if (!dup) picked.push_back(r);
  }
  std::sort(picked.begin(), picked.end());
  m.idx = picked;
  m.vals = random_dense(t, cols, rng);
  return m;
}
SparseVec random_sparse_vec(Index size, Index t, Rng& rng) {
  SparseRowMatrix rows = random_sparse_rows(size, 1, t, rng);
  SparseVec b;
  b.size = size;
  for (Index i = 0; i < rows.nnz_rows(); ++i) b.nz.emplace_back(rows.idx[i], rows.vals(i, 0));
  return b;
}
SvdTriple jacobi_tsvd(const Mat& m, Index d) {
  SvdTriple svd = jacobi_svd_full(m);
  Index k = std::min<Index>(d, svd.rank());
  while (k > 0 && svd.sigma[k - 1] <= 1e-13 * svd.sigma[0]) --k;
  return svd_head(svd, k);
}
FactorState state_from_dense(const Mat& m, Index d) {
  SvdTriple svd = jacobi_tsvd(m, d);
  const Index k = svd.rank();
  Mat x = svd.U, y = svd.V;
  for (Index i = 0; i < x.r; ++i)
    for (Index j = 0; j < k; ++j) x(i, j) *= std::sqrt(svd.sigma[j]);
  for (Index i = 0; i < y.r; ++i)
    for (Index j = 0; j < k; ++j) y(i, j) *= std::sqrt(svd.sigma[j]);
  return FactorState(x, y, Mat::eye(k), Mat::eye(k), svd.sigma, d);
}
double frob_diff(const Mat& a, const Mat& b) {
  double s = 0;
  for (size_t i = 0; i < a.a.size(); ++i) s += (a.a[i] - b.a[i]) * (a.a[i] - b.a[i]);
  return std::sqrt(s);
}
double rel_frob_dist(const Mat& a, const Mat& b) {
  const double den = b.frob();
  return den == 0.0 ? a.frob() : frob_diff(a, b) / den;
}
Mat engine_product(const FactorState& s) {
  Mat x, y;
  s.query_all(x, y);
  return matmul(x, transpose(y));
}
Mat mat_add(Mat a, const Mat& b, double f = 1.0) {
  for (size_t i = 0; i < a.a.size(); ++i) a.a[i] += f * b.a[i];
  return a;
}
double vec_inf(const Vec& a, const Vec& b) {
  double m = 0;
  for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return m;
}
double vnorm(const Vec& a) {
  double s = 0;
  for (double v : a) s += v * v;
  return std::sqrt(s);
}
ProjectionUpdate identity_update(const FactorState& s) {
  const Index k = s.rank();
  ProjectionUpdate u;
  u.F = Mat::eye(k);
  u.G = Mat::eye(k);
  u.dX = SparseRowMatrix::zero(s.rows_x(), k);
  u.dY = SparseRowMatrix::zero(s.rows_y(), k);
  u.sigma2 = s.sigma();
  return u;
}

std::vector<std::pair<std::string, std::function<void()>>> g_cases;
struct Reg {
  Reg(const char* n, std::function<void()> f) { g_cases.emplace_back(n, f); }
};
#define TEST_CASE(name, id) static void id(); static Reg reg_##id(name, id); static void id()

// ======================================================= test_graph.cpp:8-158
TEST_CASE("graph: add edge emits a rank-1 delta", g1) {
  DynamicGraph g(2);
  auto d = g.apply_event(GraphEvent::add_edge(0, 1, 1.0));
  CHECK(d.size() == 1);
  CHECK(d[0].step == DeltaVectors::Step::Edge);
  CHECK(d[0].delta_m == 1);
  CHECK(d[0].b.nz.size() == 1 && d[0].b.nz[0] == std::make_pair<Index, double>(0, 1.0));
  CHECK(d[0].c.has_value() && d[0].c->nz[0] == std::make_pair<Index, double>(1, 1.0));
}
TEST_CASE("graph: remove edge negates the delta", g2) {
  DynamicGraph g(2);
  g.apply_event(GraphEvent::add_edge(0, 1, 1.0));
  auto d = g.apply_event(GraphEvent::remove_edge(0, 1));
  CHECK(d.size() == 1);
  CHECK(d[0].c->nz[0] == std::make_pair<Index, double>(1, -1.0));
  CHECK(g.out_degree(0) == 0.0);
  CHECK(!g.has_edge(0, 1));
}
TEST_CASE("graph: add node column delta", g3) {
  DynamicGraph g(3);
  auto d = g.apply_event(GraphEvent::add_node({{0, 1.0}, {2, 1.0}}, {}));
  CHECK(d.size() == 2);
  CHECK(d[0].step == DeltaVectors::Step::NodeColumn && d[0].b.size == 3);
  CHECK(d[0].b.nz.size() == 2 && d[0].b.nz[0].first == 0 && d[0].b.nz[1].first == 2);
  CHECK(d[0].delta_m == 2);
  CHECK(d[1].step == DeltaVectors::Step::NodeRow && d[1].b.size == 4 && d[1].b.nz.empty());
  CHECK(g.node_count() == 4);
  CHECK(g.out_degree(0) == 1.0);
  CHECK(g.in_neighbors(3).size() == 2);
}
TEST_CASE("graph: accessors on a directed path", g4) {
  DynamicGraph g(3);
  g.apply_event(GraphEvent::add_edge(0, 1));
  g.apply_event(GraphEvent::add_edge(1, 2));
  CHECK(g.out_degree(0) == 1.0);
  CHECK(g.out_neighbors(1).size() == 1 && g.out_neighbors(1)[0].first == 2);
  CHECK(g.in_neighbors(1).size() == 1 && g.in_neighbors(1)[0].first == 0);
  g.apply_event(GraphEvent::remove_edge(0, 1));
  CHECK(g.out_degree(0) == 0.0);
}
TEST_CASE("graph: event errors", g5) {
  DynamicGraph g(2);
  CHECK_THROWS(g.apply_event(GraphEvent::add_edge(0, 5)));
  CHECK_THROWS(g.apply_event(GraphEvent::remove_edge(0, 1)));
  g.apply_event(GraphEvent::add_edge(0, 1));
  CHECK_THROWS(g.apply_event(GraphEvent::add_edge(0, 1)));
  CHECK_THROWS(g.out_degree(9));
}
TEST_CASE("graph: undirected edges become two deltas", g6) {
  DynamicGraph g(3, true);
  auto d = g.apply_event(GraphEvent::add_edge(0, 2, 2.0));
  CHECK(d.size() == 2 && d[0].delta_m == 2 && d[1].b.nz[0].first == 2);
  CHECK(g.has_edge(0, 2) && g.has_edge(2, 0));
  auto rm = g.apply_event(GraphEvent::remove_edge(0, 2));
  CHECK(rm.size() == 2 && !g.has_edge(2, 0) && g.arc_count() == 0);
}
TEST_CASE("graph: undirected add node mirrors", g7) {
  DynamicGraph g(2, true);
  auto d = g.apply_event(GraphEvent::add_node({{0, 1.0}}, {{1, 1.0}}));
  CHECK(d.size() == 2 && d[0].b.nz.size() == 2 && d[1].b.nz.size() == 2);
  CHECK(d[0].delta_m == 4);
  CHECK(g.has_edge(2, 0) && g.has_edge(0, 2) && g.has_edge(2, 1) && g.has_edge(1, 2));
}
TEST_CASE("graph: replayed stream keeps mirrors consistent", g8) {
  Rng rng(21);
  DynamicGraph g(5);
  std::vector<std::pair<Index, Index>> arcs;
  for (int t = 0; t < 300; ++t) {
    const double roll = rand_unit(rng);
    if (roll < 0.15) {
      const Index n = g.node_count();
      std::vector<std::pair<Index, double>> in{{static_cast<Index>(rand_index(rng, n)), 1.0}};
      GraphEvent ev = GraphEvent::add_node(in, {});
      for (auto& p : ev.in_edges) arcs.emplace_back(p.first, n);
      g.apply_event(ev);
    } else if (roll < 0.45 && !arcs.empty()) {
      const size_t pick = rand_index(rng, arcs.size());
      if (g.has_edge(arcs[pick].first, arcs[pick].second)) {
        auto d = g.apply_event(GraphEvent::remove_edge(arcs[pick].first, arcs[pick].second));
        for (auto& x : d) CHECK(static_cast<Index>(x.b.nz.size()) <= x.delta_m);
      }
      arcs[pick] = arcs.back();
      arcs.pop_back();
    } else {
      const Index n = g.node_count();
      Index u = static_cast<Index>(rand_index(rng, n));
      Index v = static_cast<Index>(rand_index(rng, n));
      if (u == v || g.has_edge(u, v)) continue;
      auto d = g.apply_event(GraphEvent::add_edge(u, v));
      for (auto& x : d) CHECK(static_cast<Index>(x.b.nz.size()) <= x.delta_m);
      arcs.emplace_back(u, v);
    }
  }
  for (Index u = 0; u < g.node_count(); ++u) {
    double sum = 0;
    for (auto& p : g.out_neighbors(u)) {
      sum += p.second;
      bool mirrored = false;
      for (auto& q : g.in_neighbors(p.first)) mirrored = mirrored || (q.first == u && q.second == p.second);
      CHECK(mirrored);
    }
    CHECK(approx(g.out_degree(u), sum, 1e-12));
  }
}

// ======================================================= test_kernels.cpp
TEST_CASE("kernels: sparseT_dense single scaled row", k1) {
  Rng rng(1);
  Mat a = random_dense(4, 3, rng);
  SparseRowMatrix b;
  b.rows = 4;
  b.cols = 1;
  b.idx = {0};
  b.vals = Mat(1, 1, 2.0);
  Mat r = mult_sparseT_dense(b, a);
  double d = 0;
  for (Index j = 0; j < 3; ++j) d += std::abs(r(0, j) - 2.0 * a(0, j));
  CHECK(r.r == 1 && d == 0.0);
}
TEST_CASE("kernels: sparseT_dense empty gives zero", k2) {
  Rng rng(2);
  Mat a = random_dense(6, 2, rng);
  Mat r = mult_sparseT_dense(SparseRowMatrix::zero(6, 3), a);
  CHECK(r.r == 3 && r.c == 2 && r.frob() == 0.0);
}
TEST_CASE("kernels: sparseT_dense matches dense", k3) {
  Rng rng(3);
  for (int rep = 0; rep < 100; ++rep) {
    SparseRowMatrix b = random_sparse_rows(1000, 4, 5, rng);
    Mat a = random_dense(1000, 6, rng);
    CHECK(rel_frob_dist(mult_sparseT_dense(b, a), matmul(transpose(b.to_dense()), a)) < 1e-12);
  }
}
TEST_CASE("kernels: shape mismatch throws", k4) {
  CHECK_THROWS(mult_sparseT_dense(SparseRowMatrix::zero(5, 2), Mat(4, 2)));
}
TEST_CASE("kernels: sparse_dense matches dense", k5) {
  Rng rng(6);
  for (int rep = 0; rep < 100; ++rep) {
    SparseRowMatrix b = random_sparse_rows(200, 5, 4, rng);
    Mat c = random_dense(5, 7, rng);
    CHECK(rel_frob_dist(mult_sparse_dense(b, c).to_dense(), matmul(b.to_dense(), c)) < 1e-12);
  }
}
TEST_CASE("kernels: ortho_residual_norm pythagorean (3,4)", k6) {
  Mat xb(2, 1);
  xb(0, 0) = 1.0;
  SparseVec b;
  b.size = 2;
  b.nz = {{0, 3.0}, {1, 4.0}};
  ResidualNorm r = ortho_residual_norm(xb, Mat::eye(1), Vec{1.0}, b);
  CHECK(r.w.size() == 1 && approx(r.w[0], 3.0) && approx(r.r, 4.0));
}
TEST_CASE("kernels: ortho_residual_norm vanishes in span", k7) {
  Rng rng(7);
  Mat q = random_orthonormal(50, 4, rng);
  Vec sigma{4.0, 3.0, 2.0, 1.0};
  Mat xb = q;
  for (Index i = 0; i < 50; ++i)
    for (Index j = 0; j < 4; ++j) xb(i, j) *= std::sqrt(sigma[j]);
  Vec coeff{0.3, -1.2, 0.5, 2.0};
  SparseVec b;
  b.size = 50;
  double bn = 0;
  for (Index i = 0; i < 50; ++i) {
    double v = 0;
    for (Index j = 0; j < 4; ++j) v += q(i, j) * coeff[j];
    if (v != 0.0) b.nz.emplace_back(i, v);
    bn += v * v;
  }
  ResidualNorm r = ortho_residual_norm(xb, Mat::eye(4), sigma, b);
  CHECK(r.r <= 1e-7 * std::sqrt(bn));
  double e = 0;
  for (Index j = 0; j < 4; ++j) e += (r.w[j] - coeff[j]) * (r.w[j] - coeff[j]);
  CHECK(std::sqrt(e) < 1e-10);
}
TEST_CASE("kernels: ortho_residual_norm matches explicit projector", k8) {
  Rng rng(8);
  for (int rep = 0; rep < 100; ++rep) {
    Mat q = random_orthonormal(100, 8, rng);
    Vec sigma(8);
    for (Index i = 0; i < 8; ++i) sigma[i] = 9.0 - double(i);
    Mat p = random_dense(8, 8, rng);
    for (Index i = 0; i < 8; ++i) p(i, i) += 8.0;
    // xb = q sqrt(S) p^{-1}
    Mat qs = q;
    for (Index i = 0; i < 100; ++i)
      for (Index j = 0; j < 8; ++j) qs(i, j) *= std::sqrt(sigma[j]);
    PartialPivLU lu(p);
    Mat xb(100, 8);
    for (Index i = 0; i < 100; ++i) {
      Vec row(qs.row(i), qs.row(i) + 8);
      Vec z = lu.solve_transpose(row);  // row * p^{-1}
      for (Index j = 0; j < 8; ++j) xb(i, j) = z[j];
    }
    SparseVec b = random_sparse_vec(100, 6, rng);
    ResidualNorm res = ortho_residual_norm(xb, p, sigma, b);
    Vec bd = b.to_dense();
    Vec qtb(8, 0.0);
    for (Index i = 0; i < 100; ++i)
      for (Index j = 0; j < 8; ++j) qtb[j] += q(i, j) * bd[i];
    double want = 0, bsq = 0, wsq = 0;
    for (Index i = 0; i < 100; ++i) {
      double pr = bd[i];
      for (Index j = 0; j < 8; ++j) pr -= q(i, j) * qtb[j];
      want += pr * pr;
      bsq += bd[i] * bd[i];
    }
    want = std::sqrt(want);
    for (double v : res.w) wsq += v * v;
    CHECK(approx(res.r, want, 1e-8));
    CHECK(approx(res.r * res.r + wsq, bsq, 1e-9));
  }
}

// ======================================================= test_svd.cpp
TEST_CASE("svd: identity truncation", s1) {
  SvdTriple s = dense_svd_small(Mat::eye(3), 2);
  CHECK(s.rank() == 2 && approx(s.sigma[0], 1.0) && approx(s.sigma[1], 1.0));
}
TEST_CASE("svd: known 2x2 spectrum", s2) {
  Mat m(2, 2);
  m(0, 0) = 2;
  m(0, 1) = 1;
  m(1, 1) = 1;
  SvdTriple s = dense_svd_small(m, 2);
  CHECK(s.rank() == 2);
  CHECK(approx(s.sigma[0], std::sqrt(3.0 + std::sqrt(5.0)), 1e-12));
  CHECK(approx(s.sigma[1], std::sqrt(3.0 - std::sqrt(5.0)), 1e-12));
}
TEST_CASE("svd: full-rank reconstruction exact", s3) {
  Rng rng(11);
  for (int rep = 0; rep < 20; ++rep) {
    Mat m = random_dense(9, 9, rng);
    SvdTriple s = dense_svd_small(m, 9);
    CHECK(frob_diff(s.reconstruct(), m) <= 1e-12 * m.frob());
    Mat utu = matmul(transpose(s.U), s.U);
    double worst = 0;
    for (Index i = 0; i < utu.r; ++i)
      for (Index j = 0; j < utu.c; ++j) worst = std::max(worst, std::abs(utu(i, j) - (i == j)));
    CHECK(worst < 1e-12);
    for (Index i = 0; i + 1 < s.rank(); ++i) CHECK(s.sigma[i] >= s.sigma[i + 1]);
    CHECK(s.sigma[s.rank() - 1] > 0.0);
  }
}
TEST_CASE("svd: planted spectrum", s4) {
  Rng rng(12);
  Mat u = random_orthonormal(17, 17, rng), v = random_orthonormal(17, 17, rng);
  Vec sigma(17);
  for (Index i = 0; i < 17; ++i) sigma[i] = std::pow(10.0, -0.5 * double(i));
  Mat us = u;
  for (Index i = 0; i < 17; ++i)
    for (Index j = 0; j < 17; ++j) us(i, j) *= sigma[j];
  SvdTriple s = dense_svd_small(matmul(us, transpose(v)), 17);
  CHECK(s.rank() == 17);
  for (Index i = 0; i < 17; ++i) CHECK(std::abs(s.sigma[i] - sigma[i]) < 1e-13 * sigma[0]);
}
TEST_CASE("svd: rejects non-finite", s5) {
  Mat m(2, 2);
  m(0, 0) = std::numeric_limits<double>::quiet_NaN();
  CHECK_THROWS(dense_svd_small(m, 2));
}
TEST_CASE("svd: randomized diagonal example", s6) {
  Mat a(3, 3);
  a(0, 0) = 3;
  a(1, 1) = 2;
  a(2, 2) = 1;
  SvdTriple s = randomized_tsvd(SparseOp::from_dense(a), 2, 10, 4, 42);
  CHECK(s.rank() == 2 && approx(s.sigma[0], 3.0, 1e-10) && approx(s.sigma[1], 2.0, 1e-10));
  Mat want(3, 3);
  want(0, 0) = 3;
  want(1, 1) = 2;
  CHECK(frob_diff(s.reconstruct(), want) < 1e-9);
}
TEST_CASE("svd: randomized wide rank-one", s7) {
  Mat a(1, 2, 1.0);
  SvdTriple s = randomized_tsvd(SparseOp::from_dense(a), 1, 10, 4, 7);
  CHECK(s.rank() == 1 && approx(s.sigma[0], std::sqrt(2.0), 1e-12));
  CHECK(frob_diff(s.reconstruct(), a) < 1e-12);
}
TEST_CASE("svd: randomized exact low rank", s8) {
  Rng rng(13);
  Mat p = random_dense(50, 8, rng), q = random_dense(50, 8, rng);
  Mat a = matmul(p, transpose(q));
  SvdTriple s = randomized_tsvd(SparseOp::from_dense(a), 8, 10, 4, 99);
  CHECK(frob_diff(s.reconstruct(), a) <= 1e-8 * a.frob());
}
TEST_CASE("svd: randomized clamps rank", s9) {
  Rng rng(14);
  Mat p = random_dense(20, 3, rng), q = random_dense(20, 3, rng);
  SvdTriple s = randomized_tsvd(SparseOp::from_dense(matmul(p, transpose(q))), 10, 10, 4, 3);
  CHECK(s.rank() == 3);
}
TEST_CASE("svd: randomized rejects zero", s10) {
  CHECK_THROWS(randomized_tsvd(SparseOp::from_dense(Mat(4, 4)), 2, 10, 4, 1));
}
TEST_CASE("svd: randomized near-optimal on decaying spectra", s11) {
  Rng rng(15);
  for (int rep = 0; rep < 10; ++rep) {
    Mat u = random_orthonormal(60, 60, rng), v = random_orthonormal(60, 60, rng);
    Vec sigma(60);
    for (Index i = 0; i < 60; ++i) sigma[i] = std::pow(0.8, double(i));
    Mat us = u;
    for (Index i = 0; i < 60; ++i)
      for (Index j = 0; j < 60; ++j) us(i, j) *= sigma[j];
    Mat a = matmul(us, transpose(v));
    SvdTriple s = randomized_tsvd(SparseOp::from_dense(a), 10, 10, 4, 1000 + rep);
    double best = 0;
    for (Index i = 10; i < 60; ++i) best += sigma[i] * sigma[i];
    CHECK(frob_diff(s.reconstruct(), a) <= 1.1 * std::sqrt(best));
  }
}

// ======================================================= test_factor_state.cpp
TEST_CASE("state: init on a directed star", f1) {
  DynamicGraph g(4);
  for (Index leaf = 1; leaf < 4; ++leaf) g.apply_event(GraphEvent::add_edge(0, leaf));
  FactorState s = FactorState::init_from_graph(g, 1, 5);
  CHECK(s.rank() == 1 && approx(s.sigma()[0], std::sqrt(3.0), 1e-10));
  for (Index leaf = 1; leaf < 4; ++leaf) CHECK(approx(s.reconstruct_entry(0, leaf), 1.0, 1e-8));
}
TEST_CASE("state: disjoint edges flat spectrum", f2) {
  DynamicGraph g(6);
  g.apply_event(GraphEvent::add_edge(0, 1));
  g.apply_event(GraphEvent::add_edge(2, 3));
  g.apply_event(GraphEvent::add_edge(4, 5));
  FactorState s = FactorState::init_from_graph(g, 3, 1);
  CHECK(s.rank() == 3);
  for (Index i = 0; i < 3; ++i) CHECK(approx(s.sigma()[i], 1.0, 1e-10));
}
TEST_CASE("state: init clamps rank below d", f3) {
  DynamicGraph g(3);
  g.apply_event(GraphEvent::add_edge(0, 1));
  FactorState s = FactorState::init_from_graph(g, 4, 2);
  CHECK(s.rank() == 1 && approx(s.sigma()[0], 1.0, 1e-10));
}
TEST_CASE("state: rejects edgeless", f4) {
  DynamicGraph g(3);
  CHECK_THROWS(FactorState::init_from_graph(g, 2, 0));
}
TEST_CASE("state: identity update bit-exact", f5) {
  Rng rng(31);
  FactorState s = state_from_dense(random_dense(12, 12, rng), 6);
  Mat x0, y0, x1, y1;
  s.query_all(x0, y0);
  s.apply_update(identity_update(s));
  s.query_all(x1, y1);
  CHECK(frob_diff(x0, x1) == 0.0 && frob_diff(y0, y1) == 0.0);
}
TEST_CASE("state: single-row delta moves only that row", f6) {
  Rng rng(32);
  FactorState s = state_from_dense(random_dense(10, 10, rng), 5);
  const Index k = s.rank();
  std::vector<Vec> before;
  for (Index u = 0; u < 10; ++u) before.push_back(s.query_context(u));
  ProjectionUpdate u = identity_update(s);
  u.dX.idx = {5};
  u.dX.vals = Mat(1, k, 1.0);
  AppliedDelta ad = s.apply_update(u);
  CHECK(ad.x_base_rows.nnz_rows() == 1);
  for (Index v = 0; v < 10; ++v) {
    Vec after = s.query_context(v);
    if (v == 5) {
      Vec d(after);
      for (Index j = 0; j < k; ++j) d[j] -= before[v][j];
      CHECK(vnorm(d) > 0.1);
    } else {
      CHECK(vec_inf(after, before[v]) == 0.0);
    }
  }
}
TEST_CASE("state: projection-only update equals dense", f7) {
  Rng rng(33);
  FactorState s = state_from_dense(random_dense(15, 15, rng), 6);
  const Index k = s.rank();
  Mat x0, y0;
  s.query_all(x0, y0);
  ProjectionUpdate u = identity_update(s);
  u.F = mat_add(random_orthonormal(k, k, rng), random_dense(k, k, rng), 0.05);
  u.G = random_orthonormal(k, k, rng);
  s.apply_update(u);
  Mat want = matmul(x0, u.F);
  for (Index i = 0; i < 15; ++i) {
    Vec got = s.query_context(i);
    Vec w(want.row(i), want.row(i) + k);
    Vec d(got);
    for (Index j = 0; j < k; ++j) d[j] -= w[j];
    CHECK(vnorm(d) <= 1e-10 * (vnorm(w) + 1.0));
  }
}
TEST_CASE("state: rebase transparency", f8) {
  Rng rng(34);
  FactorState s = state_from_dense(random_dense(20, 20, rng), 8);
  s.rebase();
  CHECK(approx(s.cond_estimate(), 1.0));
  for (int t = 0; t < 40; ++t) {
    ProjectionUpdate u = identity_update(s);
    const Index k = s.rank();
    u.F = mat_add(random_orthonormal(k, k, rng), random_dense(k, k, rng), 0.02);
    u.G = random_orthonormal(k, k, rng);
    s.apply_update(u);
  }
  Mat x0, y0, x1, y1;
  s.query_all(x0, y0);
  s.rebase();
  s.query_all(x1, y1);
  CHECK(rel_frob_dist(x1, x0) <= 1e-9 && rel_frob_dist(y1, y0) <= 1e-9);
  CHECK(approx(s.cond_estimate(), 1.0));
}
TEST_CASE("state: planted condition number", f9) {
  Mat p(2, 2);
  p(0, 0) = 10;
  p(1, 1) = 1;
  FactorState s(Mat::eye(4, 2), Mat::eye(4, 2), p, p, Vec{1, 1}, 2);
  CHECK(s.cond_estimate() >= 9.5 && s.cond_estimate() <= 10.5);
}
TEST_CASE("state: proj_row_bound dominates", f10) {
  Rng rng(35);
  for (int rep = 0; rep < 50; ++rep) {
    const Index k = 6;
    Mat p = random_dense(k, k, rng);
    FactorState s(Mat::eye(8, k), Mat::eye(8, k), p, p, Vec(k, 1.0), k);
    const double bound = s.proj_row_bound();
    Mat r = random_dense(1, k, rng);
    Mat rp = matmul(r, p);
    double amp = 0, rin = 0;
    for (Index j = 0; j < k; ++j) {
      amp = std::max(amp, std::abs(rp(0, j)));
      rin = std::max(rin, std::abs(r(0, j)));
    }
    CHECK(amp <= bound * rin * (1.0 + 1e-12));
  }
}
TEST_CASE("state: unknown node throws", f11) {
  Rng rng(36);
  FactorState s = state_from_dense(random_dense(5, 5, rng), 3);
  CHECK_THROWS(s.query_context(17));
  CHECK_THROWS(s.query_content(-1));
}

// ======================================================= test_update_engine.cpp
TEST_CASE("update: append column to 1x1", u1) {
  FactorState s(Mat(1, 1, 1.0), Mat(1, 1, 1.0), Mat::eye(1), Mat::eye(1), Vec{1.0}, 2);
  ProjectionUpdate u = update_embedding_n(s, SparseVec::unit(1, 0, 1.0));
  s.apply_update(u);
  CHECK(s.rank() == 1 && approx(s.sigma()[0], std::sqrt(2.0), 1e-10));
  Mat prod = engine_product(s);
  CHECK(prod.c == 2 && approx(prod(0, 0), 1.0, 1e-10) && approx(prod(0, 1), 1.0, 1e-10));
}
TEST_CASE("update: zero column adds isolated node", u2) {
  Rng rng(41);
  Mat a = matmul(random_dense(6, 4, rng), random_dense(4, 6, rng));
  FactorState s = state_from_dense(a, 4);
  const Index k = s.rank();
  SparseVec b;
  b.size = 6;
  ProjectionUpdate u = update_embedding_n(s, b);
  CHECK(frob_diff(u.F, Mat::eye(k)) < 1e-11 && frob_diff(u.G, Mat::eye(k)) < 1e-11);
  CHECK(u.dX.nnz_rows() == 0);
  Mat before = engine_product(s);
  s.apply_update(u);
  Mat after = engine_product(s);
  CHECK(after.c == 7);
  double col6 = 0;
  Mat left(6, 6);
  for (Index i = 0; i < 6; ++i) {
    col6 += after(i, 6) * after(i, 6);
    for (Index j = 0; j < 6; ++j) left(i, j) = after(i, j);
  }
  CHECK(std::sqrt(col6) < 1e-12);
  CHECK(rel_frob_dist(left, before) < 1e-12);
}
TEST_CASE("update: node change vs dense truncation", u3) {
  Rng rng(42);
  for (int rep = 0; rep < 10; ++rep) {
    Mat a = matmul(random_dense(20, 6, rng), random_dense(6, 20, rng));
    FactorState s = state_from_dense(a, 6);
    SparseVec b = random_sparse_vec(20, 3, rng);
    ProjectionUpdate u = update_embedding_n(s, b);
    for (size_t i = 0; i + 1 < u.sigma2.size(); ++i) CHECK(u.sigma2[i] >= u.sigma2[i + 1]);
    s.apply_update(u);
    Mat upd(20, 21);
    Vec bd = b.to_dense();
    for (Index i = 0; i < 20; ++i) {
      for (Index j = 0; j < 20; ++j) upd(i, j) = a(i, j);
      upd(i, 20) = bd[i];
    }
    CHECK(rel_frob_dist(engine_product(s), jacobi_tsvd(upd, 6).reconstruct()) <= 1e-8);
    CHECK(s.ortho_defect_x() < 1e-6 && s.ortho_defect_y() < 1e-6);
  }
}
TEST_CASE("update: known 2x2 edge update", u4) {
  Mat xb(2, 2);
  xb(0, 0) = std::sqrt(2.0);
  xb(1, 1) = 1.0;
  FactorState s(xb, xb, Mat::eye(2), Mat::eye(2), Vec{2.0, 1.0}, 2);
  s.apply_update(update_embedding_e(s, SparseVec::unit(2, 0), SparseVec::unit(2, 1, 1.0)));
  CHECK(approx(s.sigma()[0], std::sqrt(3.0 + std::sqrt(5.0)), 1e-10));
  CHECK(approx(s.sigma()[1], std::sqrt(3.0 - std::sqrt(5.0)), 1e-10));
  Mat want(2, 2);
  want(0, 0) = 2;
  want(0, 1) = 1;
  want(1, 1) = 1;
  CHECK(rel_frob_dist(engine_product(s), want) <= 1e-10);
}
TEST_CASE("update: add then remove restores", u5) {
  Rng rng(43);
  Mat a = matmul(random_dense(12, 5, rng), random_dense(5, 12, rng));
  FactorState s = state_from_dense(a, 6);
  Mat before = engine_product(s);
  SparseVec b = SparseVec::unit(12, 3);
  s.apply_update(update_embedding_e(s, b, SparseVec::unit(12, 7, 1.0)));
  s.apply_update(update_embedding_e(s, b, SparseVec::unit(12, 7, -1.0)));
  CHECK(rel_frob_dist(engine_product(s), before) <= 1e-8);
}
TEST_CASE("update: in-subspace edge update stays clamped", u6) {
  Rng rng(44);
  Mat a = matmul(random_dense(15, 6, rng), random_dense(6, 15, rng));
  FactorState s = state_from_dense(a, 6);
  const Index k = s.rank();
  Mat x, y;
  s.query_all(x, y);
  Mat cu = random_dense(k, 1, rng), cv = random_dense(k, 1, rng);
  Vec bd(15, 0.0), cd(15, 0.0);
  for (Index i = 0; i < 15; ++i)
    for (Index j = 0; j < k; ++j) {
      bd[i] += x(i, j) / std::sqrt(s.sigma()[j]) * cu(j, 0);
      cd[i] += y(i, j) / std::sqrt(s.sigma()[j]) * cv(j, 0);
    }
  auto sparsify = [](const Vec& v) {
    SparseVec o;
    o.size = static_cast<Index>(v.size());
    for (size_t i = 0; i < v.size(); ++i)
      if (v[i] != 0.0) o.nz.emplace_back(static_cast<Index>(i), v[i]);
    return o;
  };
  ProjectionUpdate u = update_embedding_e(s, sparsify(bd), sparsify(cd));
  CHECK(static_cast<Index>(u.sigma2.size()) == k);
  s.apply_update(u);
  Mat upd = a;
  for (Index i = 0; i < 15; ++i)
    for (Index j = 0; j < 15; ++j) upd(i, j) += bd[i] * cd[j];
  CHECK(rel_frob_dist(engine_product(s), jacobi_tsvd(upd, 6).reconstruct()) <= 1e-8);
}
TEST_CASE("update: random edges vs oracle", u7) {
  Rng rng(45);
  for (int rep = 0; rep < 10; ++rep) {
    Mat a = matmul(random_dense(18, 6, rng), random_dense(6, 18, rng));
    FactorState s = state_from_dense(a, 6);
    const Index un = static_cast<Index>(rand_index(rng, 18));
    Index vn = static_cast<Index>(rand_index(rng, 18));
    if (vn == un) vn = (vn + 1) % 18;
    const double w = rand_unit(rng) > 0.5 ? 1.0 : -0.5;
    s.apply_update(update_embedding_e(s, SparseVec::unit(18, un), SparseVec::unit(18, vn, w)));
    Mat upd = a;
    upd(un, vn) += w;
    SvdTriple o = jacobi_tsvd(upd, 6);
    CHECK(rel_frob_dist(engine_product(s), o.reconstruct()) <= 1e-8);
    double num = 0, den = 0;
    for (size_t i = 0; i < o.sigma.size(); ++i) {
      num += (s.sigma()[i] - o.sigma[i]) * (s.sigma()[i] - o.sigma[i]);
      den += o.sigma[i] * o.sigma[i];
    }
    CHECK(std::sqrt(num / den) <= 1e-8);
  }
}
TEST_CASE("update: isolated node leaves old queries", u8) {
  DynamicGraph g(4);
  g.apply_event(GraphEvent::add_edge(0, 1));
  g.apply_event(GraphEvent::add_edge(2, 3));
  g.apply_event(GraphEvent::add_edge(1, 2));
  FactorState s = FactorState::init_from_graph(g, 3, 7);
  Mat x0, y0, x1, y1;
  s.query_all(x0, y0);
  handle_event(s, g.apply_event(GraphEvent::add_node({}, {})));
  CHECK(s.rows_x() == 5 && s.rows_y() == 5);
  CHECK(vnorm(s.query_context(4)) == 0.0 && vnorm(s.query_content(4)) == 0.0);
  s.query_all(x1, y1);
  Mat xt(4, x1.c), yt(4, y1.c);
  for (Index i = 0; i < 4; ++i)
    for (Index j = 0; j < x1.c; ++j) {
      xt(i, j) = x1(i, j);
      yt(i, j) = y1(i, j);
    }
  CHECK(rel_frob_dist(xt, x0) <= 1e-10 && rel_frob_dist(yt, y0) <= 1e-10);
}
TEST_CASE("update: rank grows on a fresh edge", u9) {
  DynamicGraph g(2);
  g.apply_event(GraphEvent::add_edge(1, 0));
  FactorState s = FactorState::init_from_graph(g, 2, 9);
  CHECK(s.rank() == 1);
  handle_event(s, g.apply_event(GraphEvent::add_edge(0, 1)));
  CHECK(s.rank() == 2);
  CHECK(approx(s.reconstruct_entry(0, 1), 1.0, 1e-10) && approx(s.reconstruct_entry(1, 0), 1.0, 1e-10));
}
TEST_CASE("update: random stream stays on oracle recursion", u10) {
  StreamCase sc = gen_mixed_stream(100, 80, 300, 500, 4242);
  DynamicGraph g = sc.g0;
  FactorState s = FactorState::init_from_graph(g, 16, 4242);
  OracleTsvd oracle(sc.g0, 16);
  Index compared = 0;
  double worst_p = 0, worst_s = 0;
  for (const GraphEvent& ev : sc.events) {
    auto deltas = g.apply_event(ev);
    HandledEvent he = handle_event(s, deltas);
    oracle.apply_deltas(deltas);
    for (size_t i = 0; i < he.updates.size(); ++i) {
      CHECK(he.updates[i].dX.nnz_rows() <= deltas[i].delta_m);
      CHECK(he.updates[i].dY.nnz_rows() <= deltas[i].delta_m);
    }
    if (oracle.last_gap_ok()) {
      worst_p = std::max(worst_p, oracle.product_rel_dist(s));
      worst_s = std::max(worst_s, oracle.sigma_rel_dist(s.sigma()));
      ++compared;
    }
    CHECK(s.ortho_defect_x() <= 1e-6 && s.ortho_defect_y() <= 1e-6);
  }
  std::printf("    compared %lld, worst product %.3g, worst sigma %.3g\n", (long long)compared,
              worst_p, worst_s);
  CHECK(worst_p <= 1e-6 && worst_s <= 1e-8);
  CHECK(compared > 400);
}

// ======================================================= test_enhancer.cpp
FactorState two_cycle_state() {
  Mat xb(2, 1);
  xb(0, 0) = 1.0;
  return FactorState(xb, xb, Mat::eye(1), Mat::eye(1), Vec{1.0}, 1);
}
DynamicGraph two_cycle_graph() {
  DynamicGraph g(2);
  g.apply_event(GraphEvent::add_edge(0, 1));
  g.apply_event(GraphEvent::add_edge(1, 0));
  return g;
}
TEST_CASE("ppr: alpha=1 collapses to X bit-exact", e1) {
  DynamicGraph g = two_cycle_graph();
  FactorState s = two_cycle_state();
  EnhancerState e = EnhancerState::init_propagate(g, s, {1.0, 1e-5});
  for (Index u = 0; u < 2; ++u) CHECK(vec_inf(e.query_enhanced(s, u), s.query_context(u)) == 0.0);
}
TEST_CASE("ppr: two-cycle fixed point", e2) {
  DynamicGraph g = two_cycle_graph();
  FactorState s = two_cycle_state();
  EnhancerState e = EnhancerState::init_propagate(g, s, {0.5, 1e-9});
  CHECK(std::abs(e.query_enhanced(s, 0)[0] - 2.0 / 3.0) < 1e-7);
  CHECK(std::abs(e.query_enhanced(s, 1)[0] - 1.0 / 3.0) < 1e-7);
}
TEST_CASE("ppr: isolated node keeps Z = alpha X", e3) {
  DynamicGraph g(3);
  g.apply_event(GraphEvent::add_edge(0, 1));
  FactorState s = FactorState::init_from_graph(g, 2, 3);
  EnhancerState e = EnhancerState::init_propagate(g, s, {0.3, 1e-8});
  Vec z = e.query_enhanced(s, 2), x = s.query_context(2);
  for (auto& v : x) v *= 0.3;
  CHECK(vec_inf(z, x) <= 1e-12);
}
TEST_CASE("ppr: signal delta accumulates", e4) {
  DynamicGraph g = two_cycle_graph();
  FactorState s = two_cycle_state();
  EnhancerState e = EnhancerState::init_propagate(g, s, {0.5, 1e-9});
  Mat r0 = e.rb();
  e.absorb_signal_delta(SparseRowMatrix::zero(2, 1));
  CHECK(frob_diff(e.rb(), r0) == 0.0);
  SparseRowMatrix d = SparseRowMatrix::zero(2, 1);
  d.idx = {1};
  d.vals = Mat(1, 1, 0.8);
  e.absorb_signal_delta(d);
  CHECK(approx(e.rb()(1, 0), r0(1, 0) + 0.5 * 0.8));
}
TEST_CASE("ppr: structure delta for rows that lost all edges", e5) {
  DynamicGraph g = two_cycle_graph();
  FactorState s = two_cycle_state();
  EnhancerState e = EnhancerState::init_propagate(g, s, {0.5, 1e-9});
  e.absorb_structure_delta(g, s, {});
  g.apply_event(GraphEvent::remove_edge(0, 1));
  e.absorb_structure_delta(g, s, {0});
  CHECK(approx(e.rb()(0, 0), 0.5 * s.xb()(0, 0) - e.zb()(0, 0), 1e-12));
}
TEST_CASE("ppr: defect bound after structural churn", e6) {
  Rng rng(55);
  RunConfig cfg;
  cfg.d = 6;
  cfg.alpha = 0.3;
  cfg.eps = 1e-5;
  cfg.seed = 555;
  Engine eng(gen_random_graph(30, 120, 555), cfg);
  CHECK(dense_defect_bound(eng.graph(), eng.state(), eng.enhancer()) <= cfg.eps * (1.0 + 1e-6));
  for (int t = 0; t < 60; ++t) {
    const Index n = eng.graph().node_count();
    Index u = static_cast<Index>(rand_index(rng, n));
    Index v = static_cast<Index>(rand_index(rng, n));
    if (u == v) continue;
    eng.apply(eng.graph().has_edge(u, v) ? GraphEvent::remove_edge(u, v) : GraphEvent::add_edge(u, v));
    CHECK(dense_defect_bound(eng.graph(), eng.state(), eng.enhancer()) <= cfg.eps * (1.0 + 1e-6));
  }
}
TEST_CASE("ppr: enhanced query matches dense linear solve", e7) {
  RunConfig cfg;
  cfg.d = 8;
  cfg.alpha = 0.3;
  cfg.eps = 1e-7;
  cfg.seed = 77;
  Engine eng(gen_random_graph(30, 140, 77), cfg);
  const Index n = eng.graph().node_count();
  Mat x, y;
  eng.state().query_all(x, y);
  Mat op = Mat::eye(n);
  double maxdeg = 1.0;
  for (Index u = 0; u < n; ++u) {
    const double deg = eng.graph().out_degree(u);
    maxdeg = std::max(maxdeg, deg);
    if (deg == 0.0) continue;
    for (auto& p : eng.graph().out_neighbors(u)) op(u, p.first) -= (1.0 - cfg.alpha) * p.second / deg;
  }
  PartialPivLU lu(op);
  Mat z_exact(n, x.c);
  for (Index j = 0; j < x.c; ++j) {
    Vec rhs(n);
    for (Index i = 0; i < n; ++i) rhs[i] = cfg.alpha * x(i, j);
    Vec sol = lu.solve(rhs);
    for (Index i = 0; i < n; ++i) z_exact(i, j) = sol[i];
  }
  for (Index u = 0; u < n; ++u) {
    Vec z = eng.enhanced(u);
    Vec ze(z_exact.row(u), z_exact.row(u) + x.c);
    CHECK(vec_inf(z, ze) <= cfg.eps * (1.0 + maxdeg));
  }
}
TEST_CASE("ppr: alpha=1 scores identical to raw context", e8) {
  RunConfig cfg;
  cfg.d = 8;
  cfg.alpha = 1.0;
  cfg.seed = 99;
  Engine eng(gen_random_graph(40, 160, 99), cfg);
  Rng rng(42);
  for (int t = 0; t < 25; ++t) {
    Index u = static_cast<Index>(rand_index(rng, 40));
    Index v = static_cast<Index>(rand_index(rng, 40));
    if (u == v || eng.graph().has_edge(u, v)) continue;
    eng.apply(GraphEvent::add_edge(u, v));
  }
  for (Index u = 0; u < 40; ++u)
    for (Index v = 0; v < 40; ++v) CHECK(eng.score(u, v, true) == eng.score(u, v, false));
}
TEST_CASE("ppr: lazy base coordinates commute with eager rebasing", e9) {
  StreamCase sc = gen_mixed_stream(60, 50, 200, 200, 777);
  RunConfig cfg;
  cfg.d = 8;
  cfg.alpha = 0.3;
  cfg.eps = 1e-12;
  cfg.seed = 777;
  Engine lazy(sc.g0, cfg), eager(sc.g0, cfg);
  for (const GraphEvent& ev : sc.events) {
    lazy.apply(ev);
    eager.apply(ev);
    eager.rebase();
  }
  for (Index u = 0; u < lazy.graph().node_count(); ++u) {
    Vec zl = lazy.enhanced(u), ze = eager.enhanced(u);
    CHECK(vec_inf(zl, ze) <= 1e-8 * (1.0 + vnorm(ze)));
  }
  Engine clone = lazy;
  clone.rebase();
  for (Index u = 0; u < lazy.graph().node_count(); ++u)
    CHECK(vec_inf(clone.enhanced(u), lazy.enhanced(u)) <= 1e-10);
}

// ======================================================= acceptance_main.cpp
// Criteria 1+2 (acceptance_main.cpp:55-112), reduced to 4 streams x 1000
// events for CI time; the full 20-stream run is `oracle_kat --full`.
int g_streams = 4;
TEST_CASE("acceptance 1+2: oracle equivalence and sparsity", a1) {
  const Index d = 16;
  double worst_p = 0, worst_s = 0;
  long long compared = 0, skipped = 0;
  bool sparsity_ok = true;
  for (int stream = 0; stream < g_streams; ++stream) {
    StreamCase sc = gen_mixed_stream(300, 250, 900, 1000, 9000 + stream);
    DynamicGraph g = sc.g0;
    FactorState s = FactorState::init_from_graph(g, d, 9000 + stream);
    OracleTsvd oracle(sc.g0, d);
    Index since = 0;
    for (const GraphEvent& ev : sc.events) {
      auto deltas = g.apply_event(ev);
      HandledEvent he = handle_event(s, deltas);
      oracle.apply_deltas(deltas);
      for (size_t i = 0; i < he.updates.size(); ++i) {
        const auto& pu = he.updates[i];
        if (pu.dX.nnz_rows() > deltas[i].delta_m || pu.dY.nnz_rows() > deltas[i].delta_m)
          sparsity_ok = false;
      }
      if (oracle.last_gap_ok()) {
        worst_p = std::max(worst_p, oracle.product_rel_dist(s));
        worst_s = std::max(worst_s, oracle.sigma_rel_dist(s.sigma()));
        ++compared;
      } else {
        ++skipped;
      }
      if (++since >= 300 || s.cond_estimate() > 1e8) {
        s.rebase();
        since = 0;
      }
    }
  }
  std::printf("    streams %d, compared %lld, gap-skipped %lld, worst product %.3g, worst sigma %.3g\n",
              g_streams, compared, skipped, worst_p, worst_s);
  CHECK(worst_p <= 1e-6 && worst_s <= 1e-8 && sparsity_ok);
}
// Criterion 4 (acceptance_main.cpp:222-287): PPR correctness, 50 graphs x
// 30 events with node additions, plus the 2-cycle fixed point.
TEST_CASE("acceptance 4: ppr correctness", a4) {
  bool ok = true;
  double worst = 0;
  for (int rep = 0; rep < 50; ++rep) {
    Rng rng(500 + rep);
    const Index n = 20 + static_cast<Index>(rand_index(rng, 181));
    RunConfig cfg;
    cfg.d = 8;
    cfg.alpha = 0.3;
    cfg.eps = 1e-5;
    cfg.seed = 500 + rep;
    Engine eng(gen_random_graph(n, 4 * n, 500 + rep), cfg);
    const double bound = cfg.eps * (1.0 + 1e-6);
    for (int t = 0; t < 30; ++t) {
      const Index nn = eng.graph().node_count();
      const double roll = rand_unit(rng);
      if (roll < 0.15) {
        std::vector<std::pair<Index, double>> in{{static_cast<Index>(rand_index(rng, nn)), 1.0}};
        std::vector<std::pair<Index, double>> out{{static_cast<Index>(rand_index(rng, nn)), 1.0}};
        eng.apply(GraphEvent::add_node(in, out));
      } else {
        Index u = static_cast<Index>(rand_index(rng, nn)), v = static_cast<Index>(rand_index(rng, nn));
        if (u == v) continue;
        eng.apply(eng.graph().has_edge(u, v) ? GraphEvent::remove_edge(u, v) : GraphEvent::add_edge(u, v));
      }
      const double defect = dense_defect_bound(eng.graph(), eng.state(), eng.enhancer());
      worst = std::max(worst, defect);
      if (defect > bound) ok = false;
    }
  }
  for (double eps : {1e-6, 1e-7}) {
    DynamicGraph g = two_cycle_graph();
    FactorState s = two_cycle_state();
    EnhancerState e = EnhancerState::init_propagate(g, s, {0.5, eps});
    if (std::abs(e.query_enhanced(s, 0)[0] - 2.0 / 3.0) > eps ||
        std::abs(e.query_enhanced(s, 1)[0] - 1.0 / 3.0) > eps)
      ok = false;
  }
  std::printf("    max scaled defect %.3g vs bound %.3g\n", worst, 1e-5 * (1.0 + 1e-6));
  CHECK(ok);
}
// Criterion 7 (acceptance_main.cpp:351-400): eager mirror vs lazy state.
TEST_CASE("acceptance 7: lazy vs eager maintenance", a7) {
  StreamCase sc = gen_mixed_stream(120, 100, 350, 500, 7777);
  DynamicGraph g = sc.g0;
  FactorState s = FactorState::init_from_graph(g, 16, 7777);
  Mat ex, ey;
  s.query_all(ex, ey);
  double worst = 0;
  for (const GraphEvent& ev : sc.events) {
    auto deltas = g.apply_event(ev);
    HandledEvent he = handle_event(s, deltas);
    for (const ProjectionUpdate& u : he.updates) {
      if (u.append_x >= 0) ex.append_zero_row();
      if (u.append_y >= 0) ey.append_zero_row();
      if (u.grow_x) {
        auto grow = [](const Mat& m, const Mat& F, const SparseVec& gv) {
          Mat ftop(m.c, F.c);
          for (Index i = 0; i < m.c; ++i)
            for (Index j = 0; j < F.c; ++j) ftop(i, j) = F(i, j);
          Mat out = matmul(m, ftop);
          for (auto& p : gv.nz)
            for (Index j = 0; j < F.c; ++j) out(p.first, j) += p.second * F(F.r - 1, j);
          return out;
        };
        ex = grow(ex, u.F, *u.grow_x);
        ey = grow(ey, u.G, *u.grow_y);
      } else {
        ex = matmul(ex, u.F);
        ey = matmul(ey, u.G);
        for (Index t = 0; t < u.dX.nnz_rows(); ++t)
          for (Index j = 0; j < ex.c; ++j) ex(u.dX.idx[t], j) += u.dX.vals(t, j);
        for (Index t = 0; t < u.dY.nnz_rows(); ++t)
          for (Index j = 0; j < ey.c; ++j) ey(u.dY.idx[t], j) += u.dY.vals(t, j);
      }
    }
    Mat lx, ly;
    s.query_all(lx, ly);
    worst = std::max(worst, frob_diff(lx, ex) / std::max(1.0, ex.frob()));
    worst = std::max(worst, frob_diff(ly, ey) / std::max(1.0, ey.frob()));
  }
  Mat x0, y0, x1, y1;
  s.query_all(x0, y0);
  s.rebase();
  s.query_all(x1, y1);
  const double rb = std::max(frob_diff(x1, x0) / std::max(1.0, x0.frob()),
                             frob_diff(y1, y0) / std::max(1.0, y0.frob()));
  std::printf("    max eager/lazy divergence %.3g, rebase transparency %.3g\n", worst, rb);
  CHECK(worst <= 1e-8 && rb <= 1e-9);
}

}  // namespace

int main(int argc, char** argv) {
  std::string filter;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--full") g_streams = 20;
    else filter = a;
  }
  for (auto& [name, fn] : g_cases) {
    if (!filter.empty() && name.find(filter) == std::string::npos) continue;
    g_case = name;
    const int before = g_fail;
    auto t0 = std::chrono::steady_clock::now();
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  FAIL [%s] unexpected exception: %s\n", name.c_str(), e.what());
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("[%s] %s (%.2fs)\n", g_fail == before ? "PASS" : "FAIL", name.c_str(), s);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
