"""Dev diagnostic: single rank-1 steps (directed edge events) from P = I on a
cfg-5-like state: device F, G (= P_X, P_Y after the step) vs the row-local
fp64 oracle (edge_update_rowlocal_p)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W

scale = 20
d = 128
n = 1 << scale
keys = W.rmat_keys_device(scale, 16, 4)
off, tgt = W.csr_from_keys_device(n, keys)
su, sv = W.degree_proportional_inserts(keys, tgt, 40, seed=4)
sig = np.arange(1, d + 1, dtype=np.float64) ** -0.5
e = ge.Engine(n, off, tgt, None, d, d, None, None, np.eye(d), np.eye(d), sig, alpha=1.0,
              undirected=False, node_capacity=1024, arc_capacity=1 << 22)
W.orthonormal_rows_into(e, ge.XB, n, d, sig, seed=40)
W.orthonormal_rows_into(e, ge.YB, n, d, sig, seed=41)
for i in range(12):
    e.rebase()
    u, v = int(su[i]), int(sv[i])
    xu = e.query64(ge.XB, [u])[0]; yv = e.query64(ge.YB, [v])[0]
    s0 = e.get(ge.SIGMA)
    r = oracle.edge_update_rowlocal_p(d, d, xu, yv, np.eye(d), np.eye(d), s0, 1.0)
    e.apply(W.EventList.edges(1, [u], [v]))
    F, G, s2 = e.get(ge.PX), e.get(ge.PY), e.get(ge.SIGMA)
    FG = F @ G.T; FGo = r["F"] @ r["G"].T
    ds = np.abs(s2 - r["sigma2"]) / s2[0]
    # column-sign-invariant comparison of F
    sg = np.sign(np.sum(F * r["F"], axis=0))
    dF = np.abs(F * sg - r["F"]).max() / np.abs(r["F"]).max()
    wsz = np.linalg.norm(xu)
    print(f"step {i}: |xu| {wsz:.2e} sigma err {ds.max():.1e} FG^T rel {np.abs(FG - FGo).max() / np.abs(FGo).max():.1e} "
          f"F rel {dF:.1e} oracle |F| {np.abs(r['F']).max():.1e} gapk {(r['sigma2'][-2]-r['sigma2'][-1]):.2e} s2min {r['sigma2'][-1]:.3e}", flush=True)
