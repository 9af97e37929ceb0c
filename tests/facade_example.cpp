// The C++ facade (damf::gpu::Engine) used the way a reference caller uses
// damf::Engine: the known 2x2 edge update of test_update_engine.cpp:79-98,
// an error of the reference's kind, Engine(g, cfg) (device t-SVD init,
// engine.cpp:5-10), the resume constructor (engine.hpp:32-34) fed from the
// accessors (engine.hpp:38-43) and a save/load round trip (io.cpp:182-269).
// Built by tests/test_facade.py.
#include <cmath>
#include <cstdio>

#include "../paper_2306_08967_b200/csrc/damf_engine.hpp"

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "/tmp/facade_state.damf";
  damf::gpu::Csr g;
  g.n = 2;
  g.offsets = {0, 0, 0};
  damf::gpu::RunConfig cfg;
  cfg.d = 2;
  cfg.alpha = 1.0;
  damf::gpu::Factors f;
  f.k = 2;
  f.xb = {(float)std::sqrt(2.0), 0.f, 0.f, 1.f};
  f.yb = f.xb;
  f.px = {1, 0, 0, 1};
  f.py = {1, 0, 0, 1};
  f.sigma = {2.0, 1.0};
  damf::gpu::Engine eng(g, cfg, f);
  eng.apply(damf::gpu::GraphEvent::add_edge(0, 1));
  const double s01 = eng.score(0, 1, false), s00 = eng.score(0, 0, false);
  const double s10 = eng.score(1, 0, false), s11 = eng.score(1, 1, false);
  std::printf("product [[%.6f %.6f] [%.6f %.6f]]\n", s00, s01, s10, s11);
  bool ok = std::abs(s00 - 2) < 1e-5 && std::abs(s01 - 1) < 1e-5 && std::abs(s10) < 1e-5 &&
            std::abs(s11 - 1) < 1e-5;
  try {
    eng.apply(damf::gpu::GraphEvent::add_edge(0, 1));
    ok = false;
  } catch (const damf::gpu::Error& e) {
    std::printf("caught %s (kind %d)\n", e.what(), (int)e.kind);
    ok = ok && e.kind == damf::gpu::Error::Kind::DuplicateEdge && e.event_index == 0;
  }

  // Engine(g, cfg) on a 6-cycle plus chords (undirected), then the resume
  // constructor from its own accessors: both answer the same queries
  damf::gpu::Csr ring;
  ring.n = 6;
  std::vector<std::vector<int32_t>> adj(6);
  auto link = [&](int a, int b) { adj[a].push_back(b); adj[b].push_back(a); };
  for (int i = 0; i < 6; ++i) link(i, (i + 1) % 6);
  link(0, 3);
  link(1, 4);
  ring.offsets.push_back(0);
  for (auto& r : adj) {
    for (int v : r) ring.targets.push_back(v);
    ring.offsets.push_back((int64_t)ring.targets.size());
  }
  damf::gpu::RunConfig rc;
  rc.d = 3;
  rc.alpha = 0.3;
  rc.eps = 1e-7;
  rc.undirected = true;
  damf::gpu::Engine a(ring, rc);
  a.apply(damf::gpu::GraphEvent::add_edge(2, 5));
  damf::gpu::Engine b(a.graph(), a.state(), a.enhancer(), a.config(), a.events_applied(),
                      a.events_since_rebase());
  double diff = 0;
  for (int u = 0; u < 6; ++u)
    for (int v = 0; v < 6; ++v) diff = std::fmax(diff, std::abs(a.score(u, v) - b.score(u, v)));
  std::printf("Engine(g, cfg): k=%lld events=%llu; resumed copy max score diff %.3g\n",
              (long long)a.diagnostics().k, (unsigned long long)b.events_applied(), diff);
  ok = ok && diff < 1e-6 && b.events_applied() == 1;
  a.save_state(path);
  damf::gpu::Engine c = damf::gpu::Engine::load_state(path);
  double diff2 = 0;
  for (int u = 0; u < 6; ++u) diff2 = std::fmax(diff2, std::abs(a.score(u, u) - c.score(u, u)));
  std::printf("load_state: alpha %.2f, max score diff %.3g\n", c.config().alpha, diff2);
  ok = ok && diff2 < 1e-6 && c.config().alpha == 0.3 && c.config().undirected;
  std::printf(ok ? "facade ok\n" : "facade FAILED\n");
  return ok ? 0 : 1;
}
