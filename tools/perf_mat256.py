"""Dev: d = 256 materialisation, bf16x3 (default) vs tf32x3 (DAMF_MAT256_TF32), accuracy + timing."""
import sys, os, math, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
d = 256
rng = np.random.default_rng(3)
for n in (20000, 1000, 129, 1):
    x = (rng.standard_normal((n, d)) / np.sqrt(d)).astype(np.float32)
    F = W.cfg4_F(d, 3)
    X = torch.from_numpy(x).cuda(); Z = torch.empty_like(X)
    ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr())
    torch.cuda.synchronize()
    ref = x.astype(np.float64) @ F
    err = np.linalg.norm(Z.cpu().numpy() - ref) / np.linalg.norm(ref)
    print(json.dumps({"n": n, "rel_frob": float(err)}), flush=True)
n = 1 << 23
X = torch.randn(n, d, device="cuda") / math.sqrt(d); Z = torch.empty_like(X)
F = W.cfg4_F(d, 3); st = torch.cuda.current_stream().cuda_stream
for _ in range(3): ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr(), st)
ms = [ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr(), st) for _ in range(10)]
t = float(np.median(ms)); gbs = 8.0 * n * d / (t * 1e-3) / 1e9
print(json.dumps({"d": d, "tf32": bool(os.environ.get("DAMF_MAT256_TF32")), "ms": round(t, 4),
                  "GBps": round(gbs, 1), "frac": round(gbs / 6537.3, 3)}), flush=True)
