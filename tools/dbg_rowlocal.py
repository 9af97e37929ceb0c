import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch, oracle
from paper_2306_08967_b200 import engine as ge, workloads as W
from helpers import rel_frob, product
import test_gpu_configs as T
scale, d = 12, 16
n = 1 << scale
u, v = W.rmat_edges(scale, 8, 3)
rng = np.random.default_rng(1)
Q, _ = np.linalg.qr(rng.standard_normal((n, d))); Q2, _ = np.linalg.qr(rng.standard_normal((n, d)))
sig = np.arange(1, d + 1) ** -0.5
xb, yb = Q * np.sqrt(sig), Q2 * np.sqrt(sig)
off, tgt = W.undirected_csr(n, u, v)
g = oracle.Graph(n, np.concatenate([u, v]), np.concatenate([v, u]), None, True)
oe = oracle.OracleEngine(g, d=d, alpha=1.0, factors=(xb, yb, np.eye(d), np.eye(d), sig))
for mode in ("host", "load"):
    if mode == "host":
        e = ge.Engine(n, off, tgt, None, d, d, xb.astype(np.float32), yb.astype(np.float32), np.eye(d), np.eye(d), sig, alpha=1.0, undirected=True)
    else:
        e = ge.Engine(n, off, tgt, None, d, d, None, None, np.eye(d), np.eye(d), sig, alpha=1.0, undirected=True)
        e.load_rows(ge.XB, 0, xb.astype(np.float32)); e.load_rows(ge.YB, 0, yb.astype(np.float32))
    print(mode, "init X diff", np.abs(e.get(ge.X) - xb).max(), "XB query", np.abs(e.query(ge.XB, [3, 5]) - xb[[3, 5]]).max())
    keys = set(zip(u.tolist(), v.tolist()))
    r2 = np.random.default_rng(5)
    for t in range(6):
        while True:
            a, b = map(int, r2.integers(0, n, 2))
            if a != b and (min(a, b), max(a, b)) not in keys: break
        keys.add((min(a, b), max(a, b)))
        wp, ws = T.rowlocal_insert_check(e, a, b, r2.integers(0, n, 10), d)
        print(mode, t, a, b, "rowlocal", wp, ws)
    e.close()
