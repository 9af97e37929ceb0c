import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch, oracle
from paper_2306_08967_b200 import engine as ge, workloads as W
from helpers import rel_frob, product, sampled_product_rel, sigma_rel
import test_gpu_configs as T
scale = int(sys.argv[1]); d = int(sys.argv[2]); mode = sys.argv[3]
n = 1 << scale
keys = W.rmat_keys_device(scale, 16, 7)
off, tgt = W.csr_from_keys_device(n, keys)
su, sv = W.degree_proportional_inserts(keys, tgt, 12, seed=7)
kk = keys.cpu().numpy(); u, v = kk >> 32, kk & 0xFFFFFFFF
rng = np.random.default_rng(1)
Q, _ = np.linalg.qr(rng.standard_normal((n, d))); Q2, _ = np.linalg.qr(rng.standard_normal((n, d)))
sig = np.arange(1, d + 1) ** -0.5
xb, yb = Q * np.sqrt(sig), Q2 * np.sqrt(sig)
g = oracle.Graph(n, np.concatenate([u, v]), np.concatenate([v, u]), None, True)
oe = oracle.OracleEngine(g, d=d, alpha=1.0, factors=(xb, yb, np.eye(d), np.eye(d), sig))
e = ge.Engine(n, off.cpu().numpy(), tgt.cpu().numpy(), None, d, d, xb.astype(np.float32), yb.astype(np.float32), np.eye(d), np.eye(d), sig, alpha=1.0, undirected=True)
deg = np.diff(off.cpu().numpy())
for t in range(12):
    a, b = int(su[t]), int(sv[t])
    if mode == "rl":
        wp, ws = T.rowlocal_insert_check(e, a, b, rng.integers(0, n, 10), d)
        oe.apply(W.EventList.edges(1, [a], [b]))
    else:
        ev = W.EventList.edges(1, [a], [b]); e.apply(ev); oe.apply(ev); wp = ws = 0
    P = sampled_product_rel(e.get(ge.X), e.get(ge.Y), oe.get(oe.X), oe.get(oe.Y), seed=t)
    print(t, a, b, "deg", deg[a], deg[b], "rl", wp, ws, "full", P, sigma_rel(e.get(ge.SIGMA), oe.get(oe.SIGMA)))
