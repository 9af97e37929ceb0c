"""Dump pre/post device state around the events of the cfg5-like stream."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
from paper_2306_08967_b200 import engine as ge, workloads as W
scale, d = 12, 128
n = 1 << scale
keys = W.rmat_keys_device(scale, 16, 7)
off, tgt = W.csr_from_keys_device(n, keys)
su, sv = W.degree_proportional_inserts(keys, tgt, 12, seed=7)
rng = np.random.default_rng(1)
Q, _ = np.linalg.qr(rng.standard_normal((n, d))); Q2, _ = np.linalg.qr(rng.standard_normal((n, d)))
sig = np.arange(1, d + 1) ** -0.5
xb, yb = Q * np.sqrt(sig), Q2 * np.sqrt(sig)
e = ge.Engine(n, off.cpu().numpy(), tgt.cpu().numpy(), None, d, d, xb.astype(np.float32), yb.astype(np.float32), np.eye(d), np.eye(d), sig, alpha=1.0, undirected=True)
dump = {}
for t in range(9):
    a, b = int(su[t]), int(sv[t])
    rows = np.array([a, b])
    pre = dict(px=e.get(ge.PX), py=e.get(ge.PY), qx=e.get(ge.QX), qy=e.get(ge.QY), s=e.get(ge.SIGMA),
               xb=e.query(ge.XB, rows), yb=e.query(ge.YB, rows))
    e.apply(W.EventList.edges(1, [a], [b]))
    post = dict(px=e.get(ge.PX), py=e.get(ge.PY), s=e.get(ge.SIGMA), xb=e.query(ge.XB, rows), yb=e.query(ge.YB, rows),
                x=e.query(ge.X, rows), y=e.query(ge.Y, rows))
    for kk, vv in pre.items(): dump[f"{t}_pre_{kk}"] = vv
    for kk, vv in post.items(): dump[f"{t}_post_{kk}"] = vv
    dump[f"{t}_uv"] = rows
    dump[f"{t}_diag"] = np.array([e.diag()["cond_estimate"]])
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/rl_dump.npz", **dump)
print("ok")
