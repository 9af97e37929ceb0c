"""Dev diagnostic at full config 5: device vs compact oracles with rebase_cond
1e8 (the reference default) and 1e2, and the two oracles against each other."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from helpers import sampled_product_rel, sigma_rel
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
from test_gpu_configs import cfg5_like

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
m = int(sys.argv[2]) if len(sys.argv) > 2 else 600
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 50
d = 128
e, su, sv = cfg5_like(scale, d, m, seed=4)
rng = np.random.default_rng(5)
rows = np.unique(np.concatenate([su, sv, rng.integers(0, e.n, 1024)]))
fac = (e.query64(ge.XB, rows), e.query64(ge.YB, rows), e.get(ge.PX), e.get(ge.PY), e.get(ge.SIGMA))
g = oracle.Graph(len(rows), np.zeros(0, np.int64), np.zeros(0, np.int64), None, True)
ors = {rc: oracle.OracleEngine(g, d=d, alpha=1.0, rebase_cond=rc, factors=fac) for rc in (1e8, 1e4, 1e2)}
lu, lv = np.searchsorted(rows, su), np.searchsorted(rows, sv)
reb = 0
for a in range(0, m, chunk):
    b = min(m, a + chunk)
    for o in ors.values():
        o.apply(W.EventList.edges(1, lu[a:b], lv[a:b]))
    reb += e.apply(W.EventList.edges(1, su[a:b], sv[a:b]))["rebases"]
    ref = ors[1e2]
    xr, yr, sr = ref.get(ref.X), ref.get(ref.Y), ref.get(ref.SIGMA)
    xd, yd = e.query(ge.X, rows).astype(np.float64), e.query(ge.Y, rows).astype(np.float64)
    out = [f"{b:5d} D {sampled_product_rel(xd, yd, xr, yr, m=100000, seed=a):.1e}/{sigma_rel(e.get(ge.SIGMA), sr):.0e} reb {reb}"]
    for rc in (1e8, 1e4):
        o = ors[rc]
        out.append(f"O{int(np.log10(rc))} {sampled_product_rel(o.get(o.X), o.get(o.Y), xr, yr, m=100000, seed=a):.1e}/{sigma_rel(o.get(o.SIGMA), sr):.0e} reb {int(o.stat(7))}")
    print(" | ".join(out), flush=True)
