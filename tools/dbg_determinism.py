import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
from paper_2306_08967_b200 import engine as ge, workloads as W
import test_gpu_configs as T
scale = int(sys.argv[1])
res = []
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    e, su, sv = T.cfg5_like(scale, 128, 8, seed=4)
    out = []
    for i in range(8):
        e.apply(W.EventList.edges(ge.ADD_EDGE, [int(su[i])], [int(sv[i])]))
        out.append((e.get(ge.SIGMA).copy(), e.get(ge.PX).copy(), e.get(ge.PY).copy(),
                    e.query(ge.XB, [int(su[i]), int(sv[i])]), e.diag()["cond_estimate"]))
    res.append(out)
    print("rep", rep, "sigma0", [float(o[0][0]) for o in out])
    e.close(); del e; torch.cuda.empty_cache()
for i in range(8):
    if len(res) < 3: break
    a, b, c = res[0][i], res[1][i], res[2][i]
    print(i, "sigma", np.abs(a[0] - b[0]).max(), np.abs(a[0] - c[0]).max(), "PX", np.abs(a[1] - b[1]).max(),
          "PY", np.abs(a[2] - b[2]).max(), "rows", np.abs(a[3] - b[3]).max(), np.abs(a[3] - c[3]).max(), "cond", a[4], b[4], c[4])
