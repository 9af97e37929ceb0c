import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_2306_08967_b200 import engine as ge, workloads as W
import test_gpu_configs as T
e, su, sv = T.cfg5_like(16, 128, 24, seed=7)
for i in range(24):
    e.apply(W.EventList.edges(ge.ADD_EDGE, [int(su[i])], [int(sv[i])]))
    P, Q = e.get(ge.PX), e.get(ge.QX)
    Py, Qy = e.get(ge.PY), e.get(ge.QY)
    I = np.eye(len(P))
    print(i, "QP-I", np.abs(Q @ P - I).max(), "PQ-I", np.abs(P @ Q - I).max(), "QT P-I", np.abs(Q.T @ P - I).max(),
          "Y:", np.abs(Qy @ Py - I).max(), "cond", e.diag()["cond_estimate"], "|P|", np.abs(P).max(), "|Q|", np.abs(Q).max(),
          "true cond", np.linalg.cond(P), "condY", np.linalg.cond(Py))
