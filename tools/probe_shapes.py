"""Dev: odd ranks / directedness / alpha against the oracle on small streams."""
import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle
from helpers import gpu_from_oracle, sampled_product_rel, sigma_rel, dense_defect
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200.workloads import EventList
F = ("kind", "u", "v", "w", "in_off", "in_ids", "in_w", "out_off", "out_ids", "out_w")
for d in (5, 13, 33, 100):
    for alpha in (1.0, 0.3):
        g, ev = oracle.gen_mixed_stream(260, 180, 1000, 120, 17 + d)
        try:
            oe = oracle.OracleEngine(g, d=d, alpha=alpha, eps=1e-6, seed=d)
            e = gpu_from_oracle(g, oe, d=d, alpha=alpha, eps=1e-6, node_capacity=128)
            st = e.apply(EventList(*(getattr(ev, f) for f in F)))
            oe.apply(ev)
            p = sampled_product_rel(e.get(ge.X), e.get(ge.Y), oe.get(oe.X), oe.get(oe.Y))
            s = sigma_rel(e.get(ge.SIGMA), oe.get(oe.SIGMA))
            off, ids, deg = e.graph_sets()
            dfc = dense_defect(e.n, off, ids, deg, e.get(ge.X), e.get(ge.Z), alpha) if alpha < 1 else 0.0
            ok = p <= 1e-4 and s <= 1e-6 and dfc <= 1e-6 * (1 + 1e-6) + 2e-7
            print(d, alpha, "OK" if ok else "BAD", st["applied"], len(ev), f"prod {p:.2e} sigma {s:.2e} defect {dfc:.2e}", flush=True)
        except Exception as ex:
            print(d, alpha, "ERROR", repr(ex)[:300], flush=True)
