"""Dev diagnostic: per-event error at config 5 from the device's exact
pre-state (row-local fp64 oracle replays both rank-1 steps of each insertion),
split into untouched sampled rows and the two touched rows."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
from test_gpu_configs import cfg5_like

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
m0 = int(sys.argv[2]) if len(sys.argv) > 2 else 100
m1 = int(sys.argv[3]) if len(sys.argv) > 3 else 160
d = 128
e, su, sv = cfg5_like(scale, d, m1, seed=4)
e.apply(W.EventList.edges(1, su[:m0], sv[:m0]))
rng = np.random.default_rng(1)
sample = rng.integers(0, e.n, 400)
for i in range(m0, m1):
    u, v = int(su[i]), int(sv[i])
    px, py, sig = e.get(ge.PX), e.get(ge.PY), e.get(ge.SIGMA)
    rows = np.concatenate([[u, v], sample]).astype(np.int64)
    xb, yb = e.query64(ge.XB, rows), e.query64(ge.YB, rows)
    r1 = oracle.edge_update_rowlocal_p(len(sig), d, xb[0], yb[1], px, py, sig, 1.0)
    P1x, P1y = px @ r1["F"], py @ r1["G"]
    xv1 = (xb[1] @ P1x) @ np.linalg.inv(r1["px"]); yu1 = (yb[0] @ P1y) @ np.linalg.inv(r1["py"])
    r2 = oracle.edge_update_rowlocal_p(len(r1["sigma2"]), d, xv1, yu1, r1["px"], r1["py"], r1["sigma2"], 1.0)
    Xo = (xb @ px) @ r1["F"] @ r2["F"]; Yo = (yb @ py) @ r1["G"] @ r2["G"]
    Xo[0] = r1["xu"] @ r1["px"] @ r2["F"]; Xo[1] = r2["xu"] @ r2["px"]
    Yo[1] = r1["yv"] @ r1["py"] @ r2["G"]; Yo[0] = r2["yv"] @ r2["py"]
    st = e.apply(W.EventList.edges(1, [u], [v]))
    Xg, Yg = e.query(ge.X, rows).astype(np.float64), e.query(ge.Y, rows).astype(np.float64)
    Pg, Po = Xg @ Yg.T, Xo @ Yo.T
    eu = np.linalg.norm(Pg[2:, 2:] - Po[2:, 2:]) / np.linalg.norm(Po[2:, 2:])
    et = np.linalg.norm(Pg[:2] - Po[:2]) / np.linalg.norm(Po[:2])
    print(f"event {i}: reb {st['rebases']} cond {e.diag()['cond_estimate']:.1e} untouched {eu:.1e} touched {et:.1e} "
          f"sigma {np.abs(e.get(ge.SIGMA) - r2['sigma2']).max() / sig[0]:.1e} oracle condP {np.linalg.cond(r2['px']):.1e}", flush=True)
