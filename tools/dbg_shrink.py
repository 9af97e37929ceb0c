import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from helpers import gpu_from_oracle, product
from paper_2306_08967_b200 import engine as ge
from test_gpu_parity import star_and_edge, to_dev
np.set_printoptions(precision=5, suppress=False, linewidth=160)
for und in (False, True):
    g, d = star_and_edge(und)
    oe = oracle.OracleEngine(g, d=d, alpha=1.0, eps=1e-6, seed=1)
    e = gpu_from_oracle(g, oe, d=d, alpha=1.0, eps=1e-6, node_capacity=16)
    print("undirected", und, "X_b oracle\n", oe.get(oe.XB), "\nY_b\n", oe.get(oe.YB))
    for kind, u, v in [(2, 0, 1), (1, 0, 1)]:
        ev = oracle.Events.edges(kind, [u], [v])
        oe.row_log_enable(); oe.apply(ev)
        st = e.apply(to_dev(ev), mode=ge.APPLY_LOG_ROWS)
        print(kind, u, v, "k dev/ora", e.k, oe.dims()[1], "sig dev", e.get(ge.SIGMA), "ora", oe.get(oe.SIGMA))
        print("  log dev", e.row_log().tolist(), "ora", oe.row_log().tolist(), "folds", st["eager_folds"])
        print("  X dev\n", e.get(ge.X), "\n  X ora\n", oe.get(oe.X))
