"""Dev driver: launch one hot kernel in isolation for ncu captures.
  mat128 : Z = X F, n = 2^23, d = 128 (tcgen05 path)
  ppr    : init_propagate on R-MAT scale 20, ef 24, d = 128
  events : 200 cfg-2 stream events (one cluster-kernel launch)"""
import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
mode = sys.argv[1]
if mode == "mat128":
    n, d = 1 << 23, 128
    X = torch.randn(n, d, device="cuda") / math.sqrt(d); Z = torch.empty_like(X)
    F = W.cfg4_F(d, 3)
    for _ in range(3):
        print("ms", ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr()))
elif mode == "ppr":
    scale = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    u, v = W.rmat_edges(scale, 24, 3, device="cuda")
    n = 1 << scale
    off, tgt = W.undirected_csr(n, u.cpu().numpy(), v.cpu().numpy())
    X = (np.random.default_rng(0).standard_normal((n, 128)) / math.sqrt(128)).astype(np.float32)
    e = ge.Engine(n, off, tgt, None, 128, 128, X, X, W.cfg4_F(128, 3), np.eye(128), np.ones(128),
                  alpha=0.15, eps=1e-5, undirected=True)
    print(e.ppr_init())
elif mode == "events":
    import bench
    dd = bench.build_cfg2(); w = dd["w"]
    e = ge.Engine.from_graph(dd["n"], dd["off"], dd["tgt"], None, 128, alpha=0.15, eps=1e-5,
                             undirected=True, seed=0, node_capacity=4096)
    e.apply(w["stream"].slice(0, 50))
    print(e.apply(w["stream"].slice(50, 250)))
