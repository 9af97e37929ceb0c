// Header-only C++ facade that restores the reference's damf::Engine API
// (/root/reference/proj/include/damf/engine.hpp:26-61) on top of the C ABI in
// include/damf_gpu.h. A caller of the reference swaps
//     damf::Engine eng(std::move(g), cfg);  eng.apply(e);  eng.enhanced(u);
// for
//     damf::gpu::Engine eng(g, cfg);  eng.apply(e);  eng.enhanced(u);
// Errors are rethrown as damf::gpu::Error carrying the reference's
// Error::Kind (types.hpp:21-41); nothing but plain pointers crosses the ABI.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/damf_gpu.h"

namespace damf {
namespace gpu {

struct Error : std::runtime_error {
  // same order as damf::Error::Kind (types.hpp:21-41)
  enum class Kind {
    ParseError, UnknownNode, DuplicateEdge, MissingEdge, ShapeMismatch, ZeroMatrix, NonFinite,
    SingularProjection, NonConvergence, DegenerateLabels, KTooLarge, GraphTooSmall, TooLarge,
    IoError, Cuda, Unsupported
  };
  Error(int status, const std::string& msg, int64_t index = -1)
      : std::runtime_error(msg), kind(to_kind(status)), status(status), event_index(index) {}
  static Kind to_kind(int s) {
    if (s >= 1 && s <= 14) return static_cast<Kind>(s - 1);
    return s == DAMF_E_UNSUPPORTED ? Kind::Unsupported : Kind::Cuda;
  }
  Kind kind;
  int status;
  int64_t event_index;
};

// RunConfig (engine.hpp:13-21)
struct RunConfig {
  int64_t d = 128;
  double alpha = 0.3;
  double eps = 1e-5;
  uint64_t seed = 0;
  double rebase_cond = 1e8;
  int64_t rebase_every = 50000;
  bool undirected = false;
};

// GraphEvent (graph.hpp:14-47)
struct GraphEvent {
  enum class Kind { AddNode = DAMF_ADD_NODE, AddEdge = DAMF_ADD_EDGE, RemoveEdge = DAMF_REMOVE_EDGE };
  Kind kind = Kind::AddEdge;
  int64_t u = 0, v = 0;
  double w = 1.0;
  std::vector<std::pair<int64_t, double>> in_edges, out_edges;
  static GraphEvent add_edge(int64_t u, int64_t v, double w = 1.0) {
    GraphEvent e;
    e.u = u;
    e.v = v;
    e.w = w;
    return e;
  }
  static GraphEvent remove_edge(int64_t u, int64_t v) {
    GraphEvent e;
    e.kind = Kind::RemoveEdge;
    e.u = u;
    e.v = v;
    return e;
  }
  static GraphEvent add_node(std::vector<std::pair<int64_t, double>> in,
                             std::vector<std::pair<int64_t, double>> out) {
    GraphEvent e;
    e.kind = Kind::AddNode;
    e.in_edges = std::move(in);
    e.out_edges = std::move(out);
    return e;
  }
};

// Out-adjacency (DynamicGraph's arcs) in CSR form.
struct Csr {
  int64_t n = 0;
  std::vector<int64_t> offsets;  // n + 1
  std::vector<int32_t> targets;
  std::vector<double> weights;   // empty = all 1.0
};

// FactorState(xb, yb, px, py, sigma, d) (factor_state.hpp:22-23), row-major.
struct Factors {
  int64_t k = 0;
  std::vector<float> xb, yb;      // n x k
  std::vector<double> px, py;     // k x k
  std::vector<double> sigma;      // k
};

// EnhancerState(params, zb, rb) (enhancer.hpp:24-25): base-coordinate PPR rows.
struct Enhancer {
  std::vector<float> zb, rb;      // n x k
};

class Engine {
 public:
  // Engine(DynamicGraph g, const RunConfig&) (engine.hpp:29, engine.cpp:5-10):
  // randomized t-SVD init on the device, then init_propagate.
  Engine(const Csr& g, const RunConfig& cfg) : cfg_(cfg) {
    damf_csr c = csr(g);
    damf_config dc = config(cfg);
    check(damf_gpu_create(&c, &dc, &h_));
  }
  // Engine(g, FactorState(...), EnhancerState::init_propagate(...), cfg, 0, 0)
  Engine(const Csr& g, const RunConfig& cfg, const Factors& f) : cfg_(cfg) {
    damf_csr c = csr(g);
    damf_config dc = config(cfg);
    check(damf_gpu_create_from_factors(&c, &dc, f.k, f.xb.data(), f.yb.data(), f.px.data(),
                                       f.py.data(), f.sigma.data(), &h_));
  }
  // Engine(g, fs, es, cfg, events_applied, events_since_rebase) (engine.hpp:32-34)
  Engine(const Csr& g, const Factors& f, const Enhancer& es, const RunConfig& cfg,
         uint64_t events_applied, int64_t events_since_rebase)
      : cfg_(cfg) {
    damf_csr c = csr(g);
    damf_config dc = config(cfg);
    check(damf_gpu_resume(&c, &dc, f.k, f.xb.data(), f.yb.data(), f.px.data(), f.py.data(),
                          f.sigma.data(), es.zb.empty() ? nullptr : es.zb.data(),
                          es.rb.empty() ? nullptr : es.rb.data(), events_applied,
                          events_since_rebase, &h_));
  }
  // load_state (io.cpp:221-269) / save_state (io.cpp:182-219): DAMF v1 files
  static Engine load_state(const std::string& path) {
    Engine e;
    e.check(damf_gpu_load_state(path.c_str(), nullptr, &e.h_));
    damf_config c{};
    e.check(damf_gpu_get_config(e.h_, &c));
    e.cfg_ = RunConfig{c.d, c.alpha, c.eps, c.seed, c.rebase_cond, c.rebase_every, c.undirected != 0};
    return e;
  }
  void save_state(const std::string& path) const { check(damf_gpu_save_state(h_, path.c_str())); }

  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  Engine(Engine&& o) noexcept : h_(std::exchange(o.h_, nullptr)), cfg_(o.cfg_) {}
  ~Engine() { damf_gpu_destroy(h_); }

  // Engine::apply (engine.cpp:22-41)
  void apply(const GraphEvent& e) { apply(std::vector<GraphEvent>{e}); }

  // A batch, applied sequentially; on error earlier events stay applied.
  damf_apply_stats apply(const std::vector<GraphEvent>& evs, int32_t mode = 0) {
    const size_t m = evs.size();
    std::vector<int32_t> kind(m);
    std::vector<int64_t> u(m), v(m), in_off(m + 1, 0), out_off(m + 1, 0), in_ids, out_ids;
    std::vector<double> w(m), in_w, out_w;
    for (size_t i = 0; i < m; ++i) {
      const GraphEvent& e = evs[i];
      kind[i] = static_cast<int32_t>(e.kind);
      u[i] = e.u;
      v[i] = e.v;
      w[i] = e.w;
      for (auto& p : e.in_edges) {
        in_ids.push_back(p.first);
        in_w.push_back(p.second);
      }
      for (auto& p : e.out_edges) {
        out_ids.push_back(p.first);
        out_w.push_back(p.second);
      }
      in_off[i + 1] = (int64_t)in_ids.size();
      out_off[i + 1] = (int64_t)out_ids.size();
    }
    damf_event_batch b{(int64_t)m,     kind.data(),    u.data(),      v.data(),
                       w.data(),       in_off.data(),  in_ids.data(), in_w.data(),
                       out_off.data(), out_ids.data(), out_w.data()};
    damf_apply_stats s{};
    const int st = damf_gpu_apply(h_, &b, mode, &s);
    if (st) throw Error(st, damf_gpu_last_error(h_), s.failed_index);
    return s;
  }

  std::vector<float> context(int64_t u) const { return row(DAMF_X, u); }   // engine.hpp:45
  std::vector<float> content(int64_t u) const { return row(DAMF_Y, u); }   // engine.hpp:46
  std::vector<float> enhanced(int64_t u) const { return row(DAMF_Z, u); }  // engine.hpp:47

  // Link score <Z[u], Y[v]> (engine.cpp:49-52)
  double score(int64_t u, int64_t v, bool enhanced = true) const {
    double s = 0;
    check(damf_gpu_score(h_, u, v, enhanced ? 1 : 0, &s));
    return s;
  }

  void rebase() { check(damf_gpu_rebase(h_)); }  // engine.cpp:43-47

  damf_diag diagnostics() const {
    damf_diag d{};
    check(damf_gpu_diagnostics(h_, &d));
    return d;
  }

  // FactorState::query_all (factor_state.cpp:120-123), into device or host memory
  void materialize(int32_t which, float* dst, bool dst_is_device) const {
    check(damf_gpu_materialize(h_, which, dst, dst_is_device ? 1 : 0));
  }

  damf_gpu* handle() const { return h_; }

  // Accessors (engine.hpp:38-43), as host copies of the device state.
  const RunConfig& config() const { return cfg_; }
  uint64_t events_applied() const { return (uint64_t)diagnostics().events_applied; }
  int64_t events_since_rebase() const { return diagnostics().events_since_rebase; }
  // graph(): the out-adjacency, sorted per row, with weighted out-degrees
  Csr graph(std::vector<double>* out_degree = nullptr) const {
    const damf_diag d = diagnostics();
    Csr g;
    g.n = d.n;
    g.offsets.resize((size_t)d.n + 1);
    g.targets.resize((size_t)d.arcs);
    std::vector<double> deg((size_t)d.n);
    check(damf_gpu_get_graph(h_, g.offsets.data(), g.targets.data(), deg.data()));
    if (out_degree) *out_degree = std::move(deg);
    return g;
  }
  // state(): X_b, Y_b, P_X, P_Y, sigma (FactorState, factor_state.hpp:68-71)
  Factors state() const {
    const damf_diag d = diagnostics();
    Factors f;
    f.k = d.k;
    f.xb.resize((size_t)(d.n * d.k));
    f.yb.resize((size_t)(d.n * d.k));
    f.px.resize((size_t)(d.k * d.k));
    f.py.resize((size_t)(d.k * d.k));
    f.sigma.resize((size_t)d.k);
    check(damf_gpu_get_state(h_, DAMF_XB, f.xb.data()));
    check(damf_gpu_get_state(h_, DAMF_YB, f.yb.data()));
    check(damf_gpu_get_state(h_, DAMF_PX, f.px.data()));
    check(damf_gpu_get_state(h_, DAMF_PY, f.py.data()));
    check(damf_gpu_get_state(h_, DAMF_SIGMA, f.sigma.data()));
    return f;
  }
  // enhancer(): Z_b, r_b (EnhancerState, enhancer.hpp:67); alpha == 1 mirrors X_b, r_b = 0
  Enhancer enhancer() const {
    const damf_diag d = diagnostics();
    Enhancer e;
    e.zb.resize((size_t)(d.n * d.k));
    e.rb.assign((size_t)(d.n * d.k), 0.0f);
    if (cfg_.alpha == 1.0) {
      check(damf_gpu_get_state(h_, DAMF_XB, e.zb.data()));
    } else {
      check(damf_gpu_get_state(h_, DAMF_ZB, e.zb.data()));
      check(damf_gpu_get_state(h_, DAMF_RB, e.rb.data()));
    }
    return e;
  }

 private:
  Engine() = default;
  static damf_csr csr(const Csr& g) {
    return damf_csr{g.n, (int64_t)g.targets.size(), g.offsets.data(), g.targets.data(),
                    g.weights.empty() ? nullptr : g.weights.data()};
  }
  static damf_config config(const RunConfig& cfg) {
    return damf_config{cfg.d, cfg.alpha, cfg.eps, cfg.seed, cfg.rebase_cond, cfg.rebase_every,
                       cfg.undirected ? 1 : 0, 0, 0, 0};
  }
  std::vector<float> row(int32_t which, int64_t u) const {
    const int64_t k = diagnostics().k;
    std::vector<float> out((size_t)k);
    check(damf_gpu_query_rows(h_, which, &u, 1, out.data()));
    return out;
  }
  void check(int st) const {
    if (st) throw Error(st, h_ ? damf_gpu_last_error(h_) : "engine construction failed");
  }
  damf_gpu* h_ = nullptr;
  RunConfig cfg_;
};

}  // namespace gpu
}  // namespace damf
