"""Dev: a failing event in the middle of an enhanced (alpha < 1) batch, then
the rest of the stream: device vs oracle (which also stops at the failing
event) and the defect bound."""
import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle
from helpers import gpu_from_oracle, sampled_product_rel, sigma_rel, dense_defect
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200.workloads import EventList
F = ("kind", "u", "v", "w", "in_off", "in_ids", "in_w", "out_off", "out_ids", "out_w")
for undirected, alpha in ((True, 0.3), (False, 0.25), (True, 1.0)):
    g = oracle.gen_random_graph(300, 2400, 9, undirected=undirected)
    oe = oracle.OracleEngine(g, d=12, alpha=alpha, eps=1e-6, seed=9)
    e = gpu_from_oracle(g, oe, d=12, alpha=alpha, eps=1e-6)
    off, tgt, _ = g.csr()
    rng = np.random.default_rng(2)
    us, vs = [], []
    while len(us) < 30:
        a, b = (int(x) for x in rng.integers(0, g.n, 2))
        if a != b and not np.any(tgt[off[a]:off[a + 1]] == b) and (a, b) not in zip(us, vs) and (b, a) not in zip(us, vs):
            us.append(a); vs.append(b)
    dup = (us[3], vs[3])
    bu = us[:10] + [dup[0]] + us[10:20]
    bv = vs[:10] + [dup[1]] + vs[10:20]
    ev = oracle.Events.edges(1, bu, bv)
    gev = EventList(*(getattr(ev, f) for f in F))
    kinds = []
    try:
        e.apply(gev)
    except ge.DamfError as ex:
        kinds.append((ex.kind, ex.index))
    try:
        oe.apply(ev)
    except oracle.OracleError as ex:
        kinds.append(("oracle", str(ex)[:40]))
    rest = oracle.Events.edges(1, us[20:], vs[20:])
    e.apply(EventList(*(getattr(rest, f) for f in F)))
    oe.apply(rest)
    p = sampled_product_rel(e.get(ge.X), e.get(ge.Y), oe.get(oe.X), oe.get(oe.Y))
    s = sigma_rel(e.get(ge.SIGMA), oe.get(oe.SIGMA))
    o1, i1, d1 = e.graph_sets()
    o2, i2, d2 = oe.graph_sets()
    gs = np.array_equal(o1, o2) and np.array_equal(i1.astype(np.int64), i2)
    dfc = dense_defect(e.n, o1, i1, d1, e.get(ge.X), e.get(ge.Z), alpha) if alpha < 1 else 0.0
    ok = p <= 1e-4 and s <= 1e-6 and gs and dfc <= 1e-6 * (1 + 1e-6) + 2e-7
    print(undirected, alpha, "OK" if ok else "BAD", kinds, f"prod {p:.2e} sigma {s:.2e} graph {gs} defect {dfc:.2e}", flush=True)
