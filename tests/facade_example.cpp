// The C++ facade (damf::gpu::Engine) used the way a reference caller uses
// damf::Engine: the known 2x2 edge update of test_update_engine.cpp:79-98
// and an error of the reference's kind. Built by tests/test_facade.py.
#include <cmath>
#include <cstdio>

#include "../paper_2306_08967_b200/csrc/damf_engine.hpp"

int main() {
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
  std::printf(ok ? "facade ok\n" : "facade FAILED\n");
  return ok ? 0 : 1;
}
