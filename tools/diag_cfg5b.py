"""Dev diagnostic: two device engines (rebase_cond 1e8 / 1e2) and two compact
oracles (rebase_cond 1e8 / 1e2) on the same cfg-5-like stream; pairwise
sampled-product distances per chunk (the rc=1e2 oracle is the accurate
reference: P stays well conditioned)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from helpers import sampled_product_rel, sigma_rel
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
m = int(sys.argv[2]) if len(sys.argv) > 2 else 300
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 5
d = 128
n = 1 << scale
keys = W.rmat_keys_device(scale, 16, 4)
off, tgt = W.csr_from_keys_device(n, keys)
su, sv = W.degree_proportional_inserts(keys, tgt, m, seed=4)
sig = np.arange(1, d + 1, dtype=np.float64) ** -0.5
devs = {}
for rc in (1e8, 1e2):
    e = ge.Engine(n, off, tgt, None, d, d, None, None, np.eye(d), np.eye(d), sig, alpha=1.0,
                  undirected=True, node_capacity=1024, arc_capacity=1 << 22, rebase_cond=rc)
    W.orthonormal_rows_into(e, ge.XB, n, d, sig, seed=40)
    W.orthonormal_rows_into(e, ge.YB, n, d, sig, seed=41)
    devs[rc] = e
rng = np.random.default_rng(5)
rows = np.unique(np.concatenate([su, sv, rng.integers(0, n, 1024)]))
e0 = devs[1e8]
ors = {rc: oracle.OracleEngine(oracle.Graph(len(rows), np.zeros(0, np.int64), np.zeros(0, np.int64), None, True),
                               d=d, alpha=1.0, rebase_cond=rc,
                               factors=(e0.query64(ge.XB, rows), e0.query64(ge.YB, rows), np.eye(d), np.eye(d), sig))
       for rc in (1e8, 1e2)}
lu, lv = np.searchsorted(rows, su), np.searchsorted(rows, sv)
for a in range(0, m, chunk):
    b = min(m, a + chunk)
    for o in ors.values():
        o.apply(W.EventList.edges(1, lu[a:b], lv[a:b]))
    for e in devs.values():
        e.apply(W.EventList.edges(1, su[a:b], sv[a:b]))
    ref = ors[1e2]
    xr, yr, sr = ref.get(ref.X), ref.get(ref.Y), ref.get(ref.SIGMA)
    out = []
    for name, (x, y, s) in [("O8", (ors[1e8].get(ref.X), ors[1e8].get(ref.Y), ors[1e8].get(ref.SIGMA)))] + \
            [(f"D{int(np.log10(rc))}", (e.query(ge.X, rows).astype(np.float64), e.query(ge.Y, rows).astype(np.float64), e.get(ge.SIGMA))) for rc, e in devs.items()]:
        out.append(f"{name} {sampled_product_rel(x, y, xr, yr, m=50000, seed=a):.1e}/{sigma_rel(s, sr):.0e}")
    x8, y8 = ors[1e8].get(ref.X), ors[1e8].get(ref.Y)
    xd, yd = devs[1e8].query(ge.X, rows).astype(np.float64), devs[1e8].query(ge.Y, rows).astype(np.float64)
    out.append(f"D8vsO8 {sampled_product_rel(xd, yd, x8, y8, m=50000, seed=a):.1e}")
    out.append(f"cond D8 {devs[1e8].diag()['cond_estimate']:.1e} O8 {ors[1e8].stat(1):.1e} reb O8 {int(ors[1e8].stat(7))} O2 {int(ref.stat(7))}")
    print(b, " | ".join(out), flush=True)
