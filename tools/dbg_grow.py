import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from helpers import gpu_from_oracle, product
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200.workloads import EventList
g = oracle.Graph(6, [1], [0], None, False)
oe = oracle.OracleEngine(g, d=4, alpha=0.4, eps=1e-7, seed=3)
e = gpu_from_oracle(g, oe, d=4, alpha=0.4, eps=1e-7, node_capacity=8)
np.set_printoptions(precision=4, suppress=True, linewidth=150)
for u, v in ((2, 3), (4, 5), (0, 1), (3, 4)):
    ev = oracle.Events.edges(1, [u], [v])
    oe.apply(ev)
    st = e.apply(EventList(*(getattr(ev, f) for f in ("kind", "u", "v", "w", "in_off", "in_ids", "in_w", "out_off", "out_ids", "out_w"))))
    print("event", u, v, "k", e.k, oe.dims()[1], "folds", st["eager_folds"], "pushes", st["pushes"])
    print(" XY dev\n", product(e.get(ge.X), e.get(ge.Y)))
    print(" XY ora\n", product(oe.get(oe.X), oe.get(oe.Y)))
    print(" ZY dev\n", product(e.get(ge.Z), e.get(ge.Y)))
    print(" ZY ora\n", product(oe.get(oe.Z), oe.get(oe.Y)))
