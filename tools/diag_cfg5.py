"""Dev diagnostic: cfg-5-like stream (R-MAT, orthonormal U/V, sigma_i = i^-1/2,
degree-proportional inserts) against the compact fp64 oracle, per chunk:
product / sigma error, device cond estimate, |P Q - I| per side, rebases."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from helpers import sampled_product_rel, sigma_rel
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
from test_gpu_configs import cfg5_like

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
m = int(sys.argv[2]) if len(sys.argv) > 2 else 600
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 10
d = 128
e, su, sv = cfg5_like(scale, d, m, seed=4)
rng = np.random.default_rng(5)
rows = np.unique(np.concatenate([su, sv, rng.integers(0, e.n, 1024)]))
oe = oracle.OracleEngine(oracle.Graph(len(rows), np.zeros(0, np.int64), np.zeros(0, np.int64), None, True),
                         d=d, alpha=1.0, factors=(e.query64(ge.XB, rows), e.query64(ge.YB, rows),
                                                  e.get(ge.PX), e.get(ge.PY), e.get(ge.SIGMA)))
lu, lv = np.searchsorted(rows, su), np.searchsorted(rows, sv)
reb = 0
for a in range(0, m, chunk):
    b = min(m, a + chunk)
    oe.apply(W.EventList.edges(1, lu[a:b], lv[a:b]))
    st = e.apply(W.EventList.edges(1, su[a:b], sv[a:b]))
    reb += st["rebases"]
    xg = e.query(ge.X, rows).astype(np.float64); yg = e.query(ge.Y, rows).astype(np.float64)
    wp = sampled_product_rel(xg, yg, oe.get(oe.X), oe.get(oe.Y), m=100000, seed=a)
    ws = sigma_rel(e.get(ge.SIGMA), oe.get(oe.SIGMA))
    px, qx, py, qy = e.get(ge.PX), e.get(ge.QX), e.get(ge.PY), e.get(ge.QY)
    I = np.eye(len(px))
    dx = np.abs(px @ qx - I).max(); dy = np.abs(py @ qy - I).max()
    sx = np.linalg.svd(px, compute_uv=False); sy = np.linalg.svd(py, compute_uv=False)
    print(f"{b:5d} prod {wp:.2e} sig {ws:.2e} est {e.diag()['cond_estimate']:.2e} "
          f"condX {sx[0]/sx[-1]:.2e} condY {sy[0]/sy[-1]:.2e} |PQ-I| {dx:.1e} {dy:.1e} "
          f"dev_reb {reb} ora_reb {int(oe.stat(7))} ora_fold {int(oe.stat(6))}", flush=True)
