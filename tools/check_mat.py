"""Dev check of Z = X F on the device (tcgen05 path for d in {32,64,128})."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_08967_b200 import engine as ge
rng = np.random.default_rng(0)
for d in (32, 64, 128, 256):
    for n in (1, 127, 128, 1000, 20000):
        x = (rng.standard_normal((n, d)) / np.sqrt(d)).astype(np.float32)
        q, _ = np.linalg.qr(rng.standard_normal((d, d)))
        F = q * rng.uniform(0.5, 2.0, d)[None, :]
        X = torch.from_numpy(x).cuda(); Z = torch.full_like(X, float('nan'))
        ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr()); torch.cuda.synchronize()
        ref = x.astype(np.float64) @ F
        z = Z.cpu().numpy().astype(np.float64)
        err = np.linalg.norm(z - ref) / np.linalg.norm(ref)
        print(d, n, "rel err %.3g" % err, "nan" if np.isnan(z).any() else "", flush=True)
