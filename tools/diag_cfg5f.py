"""Dev diagnostic at config 5: the device vs the oracle in the device's
storage model (fp32 base rows at every fold, rebases at the device's events)
and vs the fp64 oracle."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from helpers import sampled_product_rel, sigma_rel
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
from test_gpu_configs import cfg5_like

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
m = int(sys.argv[2]) if len(sys.argv) > 2 else 400
d = 128
e, su, sv = cfg5_like(scale, d, m, seed=4)
rng = np.random.default_rng(5)
rows = np.unique(np.concatenate([su, sv, rng.integers(0, e.n, 1024)]))
fac = (e.query64(ge.XB, rows), e.query64(ge.YB, rows), e.get(ge.PX), e.get(ge.PY), e.get(ge.SIGMA))
g = oracle.Graph(len(rows), np.zeros(0, np.int64), np.zeros(0, np.int64), None, True)
o32 = oracle.OracleEngine(g, d=d, alpha=1.0, rebase_cond=1e300, rebase_every=1 << 60, factors=fac)
o32.set_fp32_base(True)
o64 = oracle.OracleEngine(g, d=d, alpha=1.0, rebase_cond=1e2, factors=fac)
lu, lv = np.searchsorted(rows, su), np.searchsorted(rows, sv)
reb = 0
for i in range(m):
    st = e.apply(W.EventList.edges(1, su[i:i + 1], sv[i:i + 1]))
    ev = W.EventList.edges(1, lu[i:i + 1], lv[i:i + 1])
    o32.apply(ev)
    o64.apply(ev)
    if st["rebases"]:
        reb += 1
        o32.rebase()
    if (i + 1) % 25 == 0:
        xd, yd = e.query(ge.X, rows).astype(np.float64), e.query(ge.Y, rows).astype(np.float64)
        a = sampled_product_rel(xd, yd, o32.get(o32.X), o32.get(o32.Y), m=100000, seed=i)
        b = sampled_product_rel(xd, yd, o64.get(o64.X), o64.get(o64.Y), m=100000, seed=i)
        c = sampled_product_rel(o32.get(o32.X), o32.get(o32.Y), o64.get(o64.X), o64.get(o64.Y), m=100000, seed=i)
        print(f"{i + 1:5d} dev-vs-o32 {a:.1e} sig {sigma_rel(e.get(ge.SIGMA), o32.get(o32.SIGMA)):.0e} | "
              f"dev-vs-o64 {b:.1e} | o32-vs-o64 {c:.1e} | dev rebases {reb} o32 folds {int(o32.stat(6))}", flush=True)
