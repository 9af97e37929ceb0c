// ORACLE / TEST INFRASTRUCTURE ONLY: a C ABI over the fp64 restatement so
// the Python parity tests (tests/) and bench.py's cpu_baseline leg can drive
// it with the same seeded inputs the GPU path receives. Status codes follow
// the product ABI (include/damf_gpu.h): 0 ok, Error::Kind ordinal + 1.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "damf_oracle.hpp"

using namespace damf_oracle;

namespace {
thread_local std::string g_err;

int fail(const Error& e) {
  g_err = e.what();
  return static_cast<int>(e.kind) + 1;
}
int fail_other(const std::exception& e) {
  g_err = e.what();
  return 99;
}

struct OEngine {
  Engine eng;
  double last_apply_ms = 0;
  std::vector<std::int64_t> row_log;
};

DynamicGraph build_graph(int64_t n, int undirected, int64_t arcs, const int64_t* src,
                         const int64_t* dst, const double* w) {
  DynamicGraph g(n, undirected != 0);
  for (int64_t i = 0; i < arcs; ++i) g.add_arc_raw(src[i], dst[i], w ? w[i] : 1.0);
  return g;
}

Mat from_ptr(const double* p, int64_t r, int64_t c) {
  Mat m(r, c);
  if (r * c) std::memcpy(m.a.data(), p, sizeof(double) * r * c);
  return m;
}

GraphEvent decode(int64_t i, const int32_t* kind, const int64_t* u, const int64_t* v,
                  const double* w, const int64_t* in_off, const int64_t* in_ids,
                  const double* in_w, const int64_t* out_off, const int64_t* out_ids,
                  const double* out_w) {
  GraphEvent e;
  switch (kind[i]) {
    case 0: {
      std::vector<std::pair<Index, double>> in, out;
      if (in_off)
        for (int64_t t = in_off[i]; t < in_off[i + 1]; ++t)
          in.emplace_back(in_ids[t], in_w ? in_w[t] : 1.0);
      if (out_off)
        for (int64_t t = out_off[i]; t < out_off[i + 1]; ++t)
          out.emplace_back(out_ids[t], out_w ? out_w[t] : 1.0);
      e = GraphEvent::add_node(in, out);
      break;
    }
    case 1:
      e = GraphEvent::add_edge(u[i], v[i], w ? w[i] : 1.0);
      break;
    default:
      e = GraphEvent::remove_edge(u[i], v[i]);
      break;
  }
  return e;
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

int oracle_engine_create(int64_t n, int undirected, int64_t arcs, const int64_t* src,
                         const int64_t* dst, const double* w, int64_t d, double alpha,
                         double eps, uint64_t seed, double rebase_cond, int64_t rebase_every,
                         void** out) {
  try {
    RunConfig cfg;
    cfg.d = d;
    cfg.alpha = alpha;
    cfg.eps = eps;
    cfg.seed = seed;
    cfg.rebase_cond = rebase_cond;
    cfg.rebase_every = rebase_every;
    cfg.undirected = undirected != 0;
    auto* h = new OEngine{Engine(build_graph(n, undirected, arcs, src, dst, w), cfg)};
    *out = h;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_other(e);
  }
}

// State from explicit factors (factor_state.hpp:22-23) + init_propagate.
int oracle_engine_create_from_factors(int64_t n, int undirected, int64_t arcs,
                                      const int64_t* src, const int64_t* dst, const double* w,
                                      int64_t k, int64_t d, const double* xb, const double* yb,
                                      const double* px, const double* py, const double* sigma,
                                      double alpha, double eps, double rebase_cond,
                                      int64_t rebase_every, void** out) {
  try {
    RunConfig cfg;
    cfg.d = d;
    cfg.alpha = alpha;
    cfg.eps = eps;
    cfg.rebase_cond = rebase_cond;
    cfg.rebase_every = rebase_every;
    cfg.undirected = undirected != 0;
    DynamicGraph g = build_graph(n, undirected, arcs, src, dst, w);
    FactorState fs(from_ptr(xb, n, k), from_ptr(yb, n, k), from_ptr(px, k, k),
                   from_ptr(py, k, k), Vec(sigma, sigma + k), d);
    EnhancerState es = EnhancerState::init_propagate(g, fs, EnhancerParams{alpha, eps});
    auto* h = new OEngine{Engine(std::move(g), std::move(fs), std::move(es), cfg, 0, 0)};
    *out = h;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_other(e);
  }
}

void oracle_engine_destroy(void* h) { delete static_cast<OEngine*>(h); }

void* oracle_engine_clone(void* h) { return new OEngine(*static_cast<OEngine*>(h)); }

// Applies events sequentially; on error *failed = index, earlier events stay.
int oracle_engine_apply(void* hp, int64_t count, const int32_t* kind, const int64_t* u,
                        const int64_t* v, const double* w, const int64_t* in_off,
                        const int64_t* in_ids, const double* in_w, const int64_t* out_off,
                        const int64_t* out_ids, const double* out_w, int64_t* failed,
                        double* lat_ms) {
  auto* h = static_cast<OEngine*>(hp);
  *failed = -1;
  for (int64_t i = 0; i < count; ++i) {
    try {
      GraphEvent e = decode(i, kind, u, v, w, in_off, in_ids, in_w, out_off, out_ids, out_w);
      auto t0 = std::chrono::steady_clock::now();
      h->eng.apply(e);
      if (lat_ms)
        lat_ms[i] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                        .count();
    } catch (const Error& e) {
      *failed = i;
      return fail(e);
    } catch (const std::exception& e) {
      *failed = i;
      return fail_other(e);
    }
  }
  return 0;
}

void oracle_engine_dims(void* hp, int64_t* n, int64_t* k, int64_t* arcs, int64_t* d) {
  auto* h = static_cast<OEngine*>(hp);
  *n = h->eng.state().rows_x();
  *k = h->eng.state().rank();
  *arcs = h->eng.graph().arc_count();
  *d = h->eng.state().dim();
}

// which: 0 xb, 1 yb, 2 px, 3 py, 4 sigma, 5 zb, 6 rb, 7 X=xb px, 8 Y=yb py, 9 Z=zb px
int oracle_engine_get(void* hp, int which, double* out) {
  auto* h = static_cast<OEngine*>(hp);
  const FactorState& s = h->eng.state();
  const EnhancerState& e = h->eng.enhancer();
  Mat m;
  switch (which) {
    case 0: m = s.xb(); break;
    case 1: m = s.yb(); break;
    case 2: m = s.px(); break;
    case 3: m = s.py(); break;
    case 4: std::memcpy(out, s.sigma().data(), sizeof(double) * s.sigma().size()); return 0;
    case 5: m = e.zb(); break;
    case 6: m = e.rb(); break;
    case 7: m = matmul(s.xb(), s.px()); break;
    case 8: m = matmul(s.yb(), s.py()); break;
    case 9: m = matmul(e.zb(), s.px()); break;
    default: return 5;
  }
  if (!m.a.empty()) std::memcpy(out, m.a.data(), sizeof(double) * m.a.size());
  return 0;
}

// 0 defect bound, 1 cond, 2 proj_row_bound, 3 ortho_x, 4 ortho_y, 5 pushes,
// 6 eager folds, 7 rebases, 8 events applied
double oracle_engine_stat(void* hp, int which) {
  auto* h = static_cast<OEngine*>(hp);
  const auto& s = h->eng.state();
  switch (which) {
    case 0: return dense_defect_bound(h->eng.graph(), s, h->eng.enhancer());
    case 1: return s.cond_estimate();
    case 2: return s.proj_row_bound();
    case 3: return s.ortho_defect_x();
    case 4: return s.ortho_defect_y();
    case 5: return static_cast<double>(h->eng.enhancer().total_pushes());
    case 6: return static_cast<double>(s.eager_folds);
    case 7: return static_cast<double>(h->eng.rebases);
    case 8: return static_cast<double>(h->eng.events_applied());
  }
  return 0;
}

void oracle_engine_rebase(void* hp) { static_cast<OEngine*>(hp)->eng.rebase(); }

// Adjacency export: out-degree (double) per node, and sorted out-neighbour
// lists in CSR form (offsets n+1, ids) — the bit-exact graph comparison.
void oracle_engine_graph(void* hp, double* out_deg, int64_t* off, int64_t* ids) {
  const auto& g = static_cast<OEngine*>(hp)->eng.graph();
  int64_t pos = 0;
  for (Index u = 0; u < g.node_count(); ++u) {
    if (out_deg) out_deg[u] = g.out_degree(u);
    if (off) off[u] = pos;
    std::vector<Index> nb;
    for (auto& p : g.out_neighbors(u)) nb.push_back(p.first);
    std::sort(nb.begin(), nb.end());
    for (Index v : nb) {
      if (ids) ids[pos] = v;
      ++pos;
    }
  }
  if (off) off[g.node_count()] = pos;
}

int oracle_engine_query(void* hp, int which, int64_t u, double* out) {
  auto* h = static_cast<OEngine*>(hp);
  try {
    Vec r = which == 0 ? h->eng.context(u) : which == 1 ? h->eng.content(u) : h->eng.enhanced(u);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

double oracle_engine_score(void* hp, int64_t u, int64_t v, int enhanced) {
  return static_cast<OEngine*>(hp)->eng.score(u, v, enhanced != 0);
}

// Materialisation timing leg for the CPU baseline: out = in (rows x k) * T.
double oracle_materialize(const double* in, int64_t rows, int64_t k, const double* t,
                          double* out) {
  auto t0 = std::chrono::steady_clock::now();
  Mat a = from_ptr(in, rows, k), b = from_ptr(t, k, k);
  Mat c = matmul(a, b);
  std::memcpy(out, c.a.data(), sizeof(double) * c.a.size());
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// Row-local oracle for one rank-1 edge update (Appendix B of SURVEY.md):
// only rows u of X_b and v of Y_b, P_X, P_Y and sigma are read
// (kernels.cpp:55-65, update_engine.cpp:144-204, factor_state.cpp:194-211).
// Outputs the new sigma (k2), F, G (k x k2), and the updated base rows.
int oracle_edge_update_rowlocal(int64_t k, int64_t d, const double* xu, const double* yv,
                                const double* px, const double* py, const double* sigma,
                                double w, int same_row, double* sigma2, double* F, double* G,
                                double* xu_new, double* yv_new, int64_t* k2_out) {
  try {
    // Two-row base matrices: row 0 = u (X side), row 1 = v (Y side); when
    // u == v the single row serves both.
    Mat xb(2, k), yb(2, k);
    for (int64_t j = 0; j < k; ++j) {
      xb(0, j) = xu[j];
      yb(1, j) = yv[j];
    }
    FactorState s(xb, yb, from_ptr(px, k, k), from_ptr(py, k, k), Vec(sigma, sigma + k), d);
    (void)same_row;
    ProjectionUpdate pu = update_embedding_e(s, SparseVec::unit(2, 0), SparseVec::unit(2, 1, w));
    s.apply_update(pu);
    const int64_t k2 = static_cast<int64_t>(pu.sigma2.size());
    *k2_out = k2;
    std::memcpy(sigma2, pu.sigma2.data(), sizeof(double) * k2);
    std::memcpy(F, pu.F.a.data(), sizeof(double) * pu.F.a.size());
    std::memcpy(G, pu.G.a.data(), sizeof(double) * pu.G.a.size());
    for (int64_t j = 0; j < k2; ++j) {
      xu_new[j] = s.xb()(0, j);
      yv_new[j] = s.yb()(1, j);
    }
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// Same update, also returning the projections after apply_update (which may
// have folded eagerly): current rows are xu_new * px_new, yv_new * py_new.
int oracle_edge_update_rowlocal_p(int64_t k, int64_t d, const double* xu, const double* yv,
                                  const double* px, const double* py, const double* sigma,
                                  double w, double* sigma2, double* F, double* G, double* xu_new,
                                  double* yv_new, double* px_new, double* py_new,
                                  int64_t* k2_out) {
  try {
    Mat xb(2, k), yb(2, k);
    for (int64_t j = 0; j < k; ++j) {
      xb(0, j) = xu[j];
      yb(1, j) = yv[j];
    }
    FactorState s(xb, yb, from_ptr(px, k, k), from_ptr(py, k, k), Vec(sigma, sigma + k), d);
    ProjectionUpdate pu = update_embedding_e(s, SparseVec::unit(2, 0), SparseVec::unit(2, 1, w));
    s.apply_update(pu);
    const int64_t k2 = static_cast<int64_t>(pu.sigma2.size());
    *k2_out = k2;
    std::memcpy(sigma2, pu.sigma2.data(), sizeof(double) * k2);
    std::memcpy(F, pu.F.a.data(), sizeof(double) * pu.F.a.size());
    std::memcpy(G, pu.G.a.data(), sizeof(double) * pu.G.a.size());
    for (int64_t j = 0; j < k2; ++j) {
      xu_new[j] = s.xb()(0, j);
      yv_new[j] = s.yb()(1, j);
    }
    for (int64_t i = 0; i < k2; ++i)
      for (int64_t j = 0; j < k2; ++j) {
        px_new[i * k2 + j] = s.px()(i, j);
        py_new[i * k2 + j] = s.py()(i, j);
      }
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// ---- generators (eval.cpp:616-705) -----------------------------------------
struct OStream {
  StreamCase sc;
};

void* oracle_gen_mixed_stream(int64_t n_total, int64_t n0, int64_t m0, int64_t n_events,
                              uint64_t seed) {
  return new OStream{gen_mixed_stream(n_total, n0, m0, n_events, seed)};
}
void* oracle_gen_random_graph(int64_t n, int64_t arcs, uint64_t seed, int undirected) {
  return new OStream{StreamCase{gen_random_graph(n, arcs, seed, undirected != 0), {}}};
}
void* oracle_gen_sbm2(int64_t n, double p_in, double p_out, uint64_t seed) {
  return new OStream{StreamCase{gen_sbm(n, p_in, p_out, seed), {}}};
}
void oracle_stream_destroy(void* h) { delete static_cast<OStream*>(h); }
// Sizes: n, arcs, events, total in-list entries, total out-list entries.
void oracle_stream_sizes(void* hp, int64_t* n, int64_t* arcs, int64_t* events, int64_t* nin,
                         int64_t* nout) {
  auto* h = static_cast<OStream*>(hp);
  *n = h->sc.g0.node_count();
  *arcs = h->sc.g0.arc_count();
  *events = static_cast<int64_t>(h->sc.events.size());
  int64_t a = 0, b = 0;
  for (auto& e : h->sc.events) {
    a += static_cast<int64_t>(e.in_edges.size());
    b += static_cast<int64_t>(e.out_edges.size());
  }
  *nin = a;
  *nout = b;
}
// Arcs in insertion order per source node (graph.cpp:56-63 order).
void oracle_stream_graph(void* hp, int64_t* src, int64_t* dst, double* w) {
  auto* h = static_cast<OStream*>(hp);
  int64_t pos = 0;
  for (Index u = 0; u < h->sc.g0.node_count(); ++u)
    for (auto& p : h->sc.g0.out_neighbors(u)) {
      src[pos] = u;
      dst[pos] = p.first;
      w[pos] = p.second;
      ++pos;
    }
}
void oracle_stream_events(void* hp, int32_t* kind, int64_t* u, int64_t* v, double* w,
                          int64_t* in_off, int64_t* in_ids, double* in_w, int64_t* out_off,
                          int64_t* out_ids, double* out_w) {
  auto* h = static_cast<OStream*>(hp);
  int64_t a = 0, b = 0, i = 0;
  for (auto& e : h->sc.events) {
    kind[i] = static_cast<int32_t>(e.kind);
    u[i] = e.u;
    v[i] = e.v;
    w[i] = e.w;
    in_off[i] = a;
    out_off[i] = b;
    for (auto& p : e.in_edges) {
      in_ids[a] = p.first;
      in_w[a++] = p.second;
    }
    for (auto& p : e.out_edges) {
      out_ids[b] = p.first;
      out_w[b++] = p.second;
    }
    ++i;
  }
  in_off[i] = a;
  out_off[i] = b;
}

}  // extern "C"

// ---- harness: modified-row log (see Engine::row_log) -----------------------
extern "C" {
// fp32 base-row storage model (FactorState::fp32_base); rounds the current
// base rows once when switched on.
void oracle_engine_set_fp32_base(void* hp, int on) {
  auto* h = static_cast<OEngine*>(hp);
  auto& fs = const_cast<FactorState&>(h->eng.state());
  fs.fp32_base = on != 0;
  if (on) fs.round_base();
}
// Start (on != 0) or stop logging; starting clears the log and the step count.
void oracle_engine_row_log_enable(void* hp, int on) {
  auto* h = static_cast<OEngine*>(hp);
  if (on) {
    h->row_log.clear();
    h->eng.row_log = &h->row_log;
    h->eng.row_log_step = 0;
  } else {
    h->eng.row_log = nullptr;
  }
}
// Copies min(max, count) (step, side, row) triples; returns count.
int64_t oracle_engine_row_log(void* hp, int64_t* out, int64_t max) {
  auto* h = static_cast<OEngine*>(hp);
  const int64_t m = static_cast<int64_t>(h->row_log.size() / 3);
  for (int64_t i = 0; i < 3 * std::min(m, max); ++i) out[i] = h->row_log[i];
  return m;
}
}

// ---- io.cpp:182-269 save_state / load_state, restated ------------------------
namespace {
const char kMagic[4] = {'D', 'A', 'M', 'F'};
template <typename T>
void wpod(std::FILE* f, T v) { std::fwrite(&v, sizeof(T), 1, f); }
template <typename T>
T rpod(std::FILE* f) {
  T v{};
  if (std::fread(&v, sizeof(T), 1, f) != 1) throw Error(Error::Kind::ParseError, "truncated state file");
  return v;
}
void wmat(std::FILE* f, const Mat& m) {  // io.cpp:51-56: rows, cols, row-major data
  wpod<std::int64_t>(f, m.r);
  wpod<std::int64_t>(f, m.c);
  if (!m.a.empty()) std::fwrite(m.a.data(), sizeof(double), m.a.size(), f);
}
Mat rmat(std::FILE* f) {  // io.cpp:58-65
  const auto r = rpod<std::int64_t>(f);
  const auto c = rpod<std::int64_t>(f);
  Mat m(r, c);
  if (!m.a.empty() && std::fread(m.a.data(), sizeof(double), m.a.size(), f) != m.a.size())
    throw Error(Error::Kind::ParseError, "truncated state file");
  return m;
}
}  // namespace

extern "C" {
int oracle_engine_save_state(void* hp, const char* path) {
  auto* h = static_cast<OEngine*>(hp);
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return fail(Error(Error::Kind::IoError, std::string("cannot write ") + path));
  const Engine& e = h->eng;
  const RunConfig& cfg = e.config();
  std::fwrite(kMagic, 1, 4, f);
  wpod<std::uint32_t>(f, 1);
  wpod<std::int64_t>(f, cfg.d);
  wpod<double>(f, cfg.alpha);
  wpod<double>(f, cfg.eps);
  wpod<std::uint64_t>(f, cfg.seed);
  wpod<double>(f, cfg.rebase_cond);
  wpod<std::int64_t>(f, cfg.rebase_every);
  wpod<std::uint8_t>(f, cfg.undirected ? 1 : 0);
  wpod<std::uint64_t>(f, e.events_applied());
  wpod<std::int64_t>(f, e.events_since_rebase());
  const FactorState& fs = e.state();
  wpod<std::int64_t>(f, static_cast<std::int64_t>(fs.sigma().size()));  // io.cpp:67-71
  std::fwrite(fs.sigma().data(), sizeof(double), fs.sigma().size(), f);
  wmat(f, fs.xb());
  wmat(f, fs.yb());
  wmat(f, fs.px());
  wmat(f, fs.py());
  wmat(f, e.enhancer().zb());
  wmat(f, e.enhancer().rb());
  const DynamicGraph& g = e.graph();
  wpod<std::int64_t>(f, g.node_count());
  for (Index u = 0; u < g.node_count(); ++u) {
    const auto& nb = g.out_neighbors(u);
    wpod<std::int64_t>(f, static_cast<std::int64_t>(nb.size()));
    for (const auto& [v, w] : nb) {
      wpod<std::int64_t>(f, v);
      wpod<double>(f, w);
    }
  }
  const bool ok = std::ferror(f) == 0;
  if (std::fclose(f) != 0 || !ok) return fail(Error(Error::Kind::IoError, std::string("write failed: ") + path));
  return 0;
}

int oracle_engine_load_state(const char* path, void** out) {
  *out = nullptr;
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return fail(Error(Error::Kind::IoError, std::string("cannot open ") + path));
  try {
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, kMagic, 4) != 0)
      throw Error(Error::Kind::ParseError, std::string(path) + ": not a DAMF state file");
    if (rpod<std::uint32_t>(f) != 1) throw Error(Error::Kind::ParseError, "unsupported version");
    RunConfig cfg;
    cfg.d = rpod<std::int64_t>(f);
    cfg.alpha = rpod<double>(f);
    cfg.eps = rpod<double>(f);
    cfg.seed = rpod<std::uint64_t>(f);
    cfg.rebase_cond = rpod<double>(f);
    cfg.rebase_every = rpod<std::int64_t>(f);
    cfg.undirected = rpod<std::uint8_t>(f) != 0;
    const auto applied = rpod<std::uint64_t>(f);
    const auto since = rpod<std::int64_t>(f);
    const auto ks = rpod<std::int64_t>(f);
    Vec sigma(static_cast<size_t>(ks));
    if (ks && std::fread(sigma.data(), sizeof(double), sigma.size(), f) != sigma.size())
      throw Error(Error::Kind::ParseError, "truncated state file");
    Mat xb = rmat(f), yb = rmat(f), px = rmat(f), py = rmat(f), zb = rmat(f), rb = rmat(f);
    const auto n = rpod<std::int64_t>(f);
    DynamicGraph g(n, cfg.undirected);
    for (Index u = 0; u < n; ++u) {
      const auto cnt = rpod<std::int64_t>(f);
      for (std::int64_t i = 0; i < cnt; ++i) {
        const auto v = rpod<std::int64_t>(f);
        const double w = rpod<double>(f);
        g.add_arc_raw(u, v, w);
      }
    }
    std::fclose(f);
    FactorState fs(std::move(xb), std::move(yb), std::move(px), std::move(py), std::move(sigma), cfg.d);
    EnhancerState es(EnhancerParams{cfg.alpha, cfg.eps}, std::move(zb), std::move(rb));
    auto* h = new OEngine{Engine(std::move(g), std::move(fs), std::move(es), cfg, applied, since)};
    *out = h;
    return 0;
  } catch (const Error& e) {
    std::fclose(f);
    return fail(e);
  }
}
}
