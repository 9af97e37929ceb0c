"""Dev timing of Z = X F at the cfg-4 shape (n = 2^23)."""
import sys, os, math, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
n = 1 << 23
for d in (32, 64, 128, 256):
    X = torch.randn(n, d, device="cuda") / math.sqrt(d); Z = torch.empty_like(X)
    F = W.cfg4_F(d, 3); st = torch.cuda.current_stream().cuda_stream
    for _ in range(3): ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr(), st)
    ms = [ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr(), st) for _ in range(10)]
    t = float(np.median(ms)); gbs = 8.0 * n * d / (t * 1e-3) / 1e9
    print(json.dumps({"d": d, "ms": round(t, 4), "GBps": round(gbs, 1), "frac": round(gbs / 6535.7, 3)}), flush=True)
    del X, Z; torch.cuda.empty_cache()
