"""Dev driver: Engine(g, cfg) (device randomized t-SVD) on an R-MAT graph, for
wall time and `ncu --metrics` launch lists of the init-path kernels:
  python tools/prof_init.py [scale] [d]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 21
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
u, v = W.rmat_edges(scale, 16, 3, device="cuda")
n = 1 << scale
off, tgt = W.undirected_csr(n, u.cpu().numpy(), v.cpu().numpy())
torch.cuda.synchronize(); t0 = time.perf_counter()
e = ge.Engine.from_graph(n, off, tgt, None, d, alpha=1.0, undirected=True, seed=0)
torch.cuda.synchronize(); print("init_s", round(time.perf_counter() - t0, 3), "arcs", len(tgt), "sigma[:3]", e.get(ge.SIGMA)[:3])
