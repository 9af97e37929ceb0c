"""Dev diagnostic: per-step error given identical pre-states. Directed cfg-5-
like engine, P accumulating (no rebase). Before each step the device's exact
pre-state (rows, P_X, P_Y, sigma) feeds the row-local fp64 oracle; after the
step the device's current rows (touched u / v and a random sample) are
compared with the oracle's."""
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
              undirected=False, node_capacity=1024, arc_capacity=1 << 22, rebase_cond=1e30)
W.orthonormal_rows_into(e, ge.XB, n, d, sig, seed=40)
W.orthonormal_rows_into(e, ge.YB, n, d, sig, seed=41)
rng = np.random.default_rng(1)
sample = rng.integers(0, n, 300)
for i in range(30):
    u, v = int(su[i]), int(sv[i])
    px, py, s0 = e.get(ge.PX), e.get(ge.PY), e.get(ge.SIGMA)
    xs = e.query64(ge.XB, sample); ys = e.query64(ge.YB, sample)
    xu = e.query64(ge.XB, [u])[0]; yv = e.query64(ge.YB, [v])[0]
    r = oracle.edge_update_rowlocal_p(d, d, xu, yv, px, py, s0, 1.0)
    st = e.apply(W.EventList.edges(1, [u], [v]))
    Xs_o = xs @ px @ r["F"]; Ys_o = ys @ py @ r["G"]
    Xu_o = r["xu"] @ r["px"]; Yv_o = r["yv"] @ r["py"]
    Xs_d = e.query(ge.X, sample).astype(np.float64); Ys_d = e.query(ge.Y, sample).astype(np.float64)
    Xu_d = e.query(ge.X, [u])[0].astype(np.float64); Yv_d = e.query(ge.Y, [v])[0].astype(np.float64)
    # sign-invariant: products among sample + touched
    Xo = np.vstack([Xs_o, Xu_o]); Yo = np.vstack([Ys_o, Yv_o]); Xd = np.vstack([Xs_d, Xu_d]); Yd = np.vstack([Ys_d, Yv_d])
    Po, Pd = Xo @ Yo.T, Xd @ Yd.T
    err_s = np.linalg.norm(Pd[:-1, :-1] - Po[:-1, :-1]) / np.linalg.norm(Po[:-1, :-1])
    err_t = np.linalg.norm(Pd[-1] - Po[-1]) / np.linalg.norm(Po[-1])
    pq = np.abs(px @ e.get(ge.QX) - np.eye(d)).max() if False else 0
    cx = np.linalg.svd(e.get(ge.PX), compute_uv=False)
    print(f"step {i}: rebases {st['rebases']} cond(P_X) {cx[0]/cx[-1]:.1e} sample-product err {err_s:.1e} "
          f"touched-row err {err_t:.1e} sigma err {np.abs(e.get(ge.SIGMA) - r['sigma2']).max()/s0[0]:.1e}", flush=True)
