"""Dev driver: one Z = X F launch at n = 2^23 for a given d (ncu target)."""
import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
d = int(sys.argv[1])
n = 1 << 23
X = torch.randn(n, d, device="cuda") / math.sqrt(d)
Z = torch.empty_like(X)
F = W.cfg4_F(d, 3)
for _ in range(3):
    print("ms", ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr()))
