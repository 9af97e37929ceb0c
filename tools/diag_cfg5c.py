"""Dev diagnostic: where does the device deviate after a few cfg-5-like
events? Per-row errors of X = X_b P (device query vs host fp64 from the
device's own exact base rows and P) and vs the accurate compact oracle."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W

scale, m = 20, int(sys.argv[1]) if len(sys.argv) > 1 else 5
d = 128
n = 1 << scale
keys = W.rmat_keys_device(scale, 16, 4)
off, tgt = W.csr_from_keys_device(n, keys)
su, sv = W.degree_proportional_inserts(keys, tgt, 40, seed=4)
sig = np.arange(1, d + 1, dtype=np.float64) ** -0.5
e = ge.Engine(n, off, tgt, None, d, d, None, None, np.eye(d), np.eye(d), sig, alpha=1.0,
              undirected=True, node_capacity=1024, arc_capacity=1 << 22)
W.orthonormal_rows_into(e, ge.XB, n, d, sig, seed=40)
W.orthonormal_rows_into(e, ge.YB, n, d, sig, seed=41)
rng = np.random.default_rng(5)
rows = np.unique(np.concatenate([su, sv, rng.integers(0, n, 256)]))
o = oracle.OracleEngine(oracle.Graph(len(rows), np.zeros(0, np.int64), np.zeros(0, np.int64), None, True),
                        d=d, alpha=1.0, rebase_cond=1e2,
                        factors=(e.query64(ge.XB, rows), e.query64(ge.YB, rows), np.eye(d), np.eye(d), sig))
lu, lv = np.searchsorted(rows, su), np.searchsorted(rows, sv)
touched = set()
for i in range(m):
    o.apply(W.EventList.edges(1, lu[i:i+1], lv[i:i+1]))
    st = e.apply(W.EventList.edges(1, su[i:i+1], sv[i:i+1]))
    touched |= {int(su[i]), int(sv[i])}
    xq = e.query(ge.X, rows).astype(np.float64)
    xh = e.query64(ge.XB, rows) @ e.get(ge.PX)
    xo = o.get(o.X)
    yq = e.query(ge.Y, rows).astype(np.float64)
    yo = o.get(o.Y)
    nrm = np.linalg.norm(xo, axis=1)
    eq = np.linalg.norm(xq - xh, axis=1) / nrm
    eo = np.abs(np.abs((xq * 1).sum(1)) - 0)  # placeholder
    # sign-invariant: compare Gram rows X X^T restricted to a few columns
    G = xq @ yq.T; Go = xo @ yo.T
    rel_rows = np.linalg.norm(G - Go, axis=1) / np.linalg.norm(Go, axis=1).clip(1e-300)
    tmask = np.isin(rows, list(touched))
    print(f"event {i}: rebases {st['rebases']} cond {e.diag()['cond_estimate']:.2e} "
          f"query-vs-host max {eq.max():.1e} | product row err touched max {rel_rows[tmask].max():.1e} "
          f"untouched max {rel_rows[~tmask].max():.1e} median {np.median(rel_rows[~tmask]):.1e}", flush=True)
