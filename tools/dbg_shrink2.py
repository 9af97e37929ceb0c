import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from helpers import gpu_from_oracle, product
from paper_2306_08967_b200 import engine as ge
from test_gpu_parity import star_and_edge, to_dev, defect_of
np.set_printoptions(precision=5, suppress=False, linewidth=160)
g, d = star_and_edge(True)
oe = oracle.OracleEngine(g, d=d, alpha=0.3, eps=1e-6, seed=1)
e = gpu_from_oracle(g, oe, d=d, alpha=0.3, eps=1e-6, node_capacity=16)
print("init defect dev", defect_of(e, 0.3), "ora", oe.defect_bound())
for kind, u, v in [(2, 0, 1)]:
    ev = oracle.Events.edges(kind, [u], [v])
    oe.apply(ev)
    st = e.apply(to_dev(ev))
    print(st)
    print("defect dev", defect_of(e, 0.3), "ora", oe.defect_bound())
    print("X dev\n", e.get(ge.X), "\nZ dev\n", e.get(ge.Z), "\nrb dev\n", e.get(ge.RB))
    print("P_X dev\n", e.get(ge.PX))
    st = e.ppr_push()
    print("after extra push", st, "defect", defect_of(e, 0.3))
