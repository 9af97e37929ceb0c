import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, oracle
from helpers import dense_defect, gpu_from_oracle
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200.workloads import EventList
rng = np.random.default_rng(500)
n = 20 + int(rng.integers(181))
g = oracle.gen_random_graph(n, 4 * n, 500)
oe = oracle.OracleEngine(g, d=8, alpha=0.3, eps=1e-5, seed=500)
e = gpu_from_oracle(g, oe, d=8, alpha=0.3, eps=1e-5)
off, ids, deg = e.graph_sets()
print("n", n, "init defect", dense_defect(e.n, off, ids, deg, e.get(ge.X), e.get(ge.Z), 0.3))
for t in range(30):
    nn = e.n
    off, ids, deg = e.graph_sets()
    if rng.random() < 0.15:
        a, b = int(rng.integers(nn)), int(rng.integers(nn))
        ev = EventList(np.array([ge.ADD_NODE], np.int32), np.array([nn]), np.array([0]), np.ones(1), np.array([0, 1]), np.array([a]), np.ones(1), np.array([0, 1]), np.array([b]), np.ones(1)); kind = f"node({a},{b})"
    else:
        u, v = int(rng.integers(nn)), int(rng.integers(nn))
        if u == v: continue
        has = v in ids[off[u]:off[u + 1]]
        ev = EventList.edges(ge.REMOVE_EDGE if has else ge.ADD_EDGE, [u], [v]); kind = f"{'rm' if has else 'add'}({u},{v})"
    st = e.apply(ev)
    off, ids, deg = e.graph_sets()
    dfc = dense_defect(e.n, off, ids, deg, e.get(ge.X), e.get(ge.Z), 0.3)
    print(t, kind, "n", e.n, "defect %.3g" % dfc, "pushes", st["pushes"], "rounds", st["push_rounds"])
