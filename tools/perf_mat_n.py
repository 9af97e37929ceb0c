"""Dev timing of Z = X F at d = 128 for growing n (efficiency vs footprint)."""
import sys, os, math, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
for sc in (22, 23, 24, 25, 26):
    n = 1 << sc
    X = torch.empty(n, d, device="cuda").normal_() ; X /= math.sqrt(d); Z = torch.empty_like(X)
    F = W.cfg4_F(d, 3); st = torch.cuda.current_stream().cuda_stream
    for _ in range(2): ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr(), st)
    ms = [ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr(), st) for _ in range(5)]
    t = float(np.median(ms)); gbs = 8.0 * n * d / (t * 1e-3) / 1e9
    print(json.dumps({"d": d, "log2n": sc, "ms": round(t, 4), "GBps": round(gbs, 1), "frac": round(gbs / 6545.6, 3)}), flush=True)
    del X, Z; torch.cuda.empty_cache()
