"""Dev driver for ncu captures (round 2): one hot kernel family per mode.
  cfg5ev  : config-5-like state (R-MAT scale 20, orthonormal U/V,
            sigma_i = i^-1/2, d = 128), then one
            damf_event_kernel<16,0> launch over 50 insertions after 200 (past the
            rebase transient)
  cfg2ev  : config-2 stream, split mode: 20 events = 20 damf_event_kernel<16,0>
            + 20 damf_ppr_kernel<16> launches after 200 warm-up events
  mat5    : Z = X F at the config-5 shape (n = 2^26, d = 128)"""
import math
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W

mode = sys.argv[1]
if mode == "cfg5ev":
    from test_gpu_configs import cfg5_like
    e, su, sv = cfg5_like(20, 128, 250, seed=4)
    st = e.apply(W.EventList.edges(1, su[:200], sv[:200]))  # past the rebase transient
    torch.cuda.synchronize()
    # one event-kernel launch per launch group: a rebase ends a group
    print("event-kernel launches before the captured one:", st["rebases"] + 1)
    print(e.apply(W.EventList.edges(1, su[200:250], sv[200:250])))
elif mode == "cfg2ev":
    w = W.cfg2()
    off, tgt = W.undirected_csr(w["n"], *w["init"])
    e = ge.Engine.from_graph(w["n"], off, tgt, None, 128, alpha=0.15, eps=1e-5, undirected=True,
                             seed=0, node_capacity=4096)
    e.apply(w["stream"].slice(0, 200))
    print(e.apply(w["stream"].slice(200, 220)))
elif mode == "mat5":
    n, d = 1 << 26, 128
    X = torch.randn(n, d, device="cuda") / math.sqrt(d)
    Z = torch.empty_like(X)
    F = W.cfg4_F(d, 3)
    for _ in range(2):
        print("ms", ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr()))
