"""Dev A/B: the whole-GPU PPR push after 1,000 structure-only insertions with
scatter rounds (float reductions, key bounds) vs every round forced into the
atomics-free pull form (DAMF_PPR_FORCE_PULL=1, read once per process):
  python tools/ab_push_pull.py [scale] [d]
prints the push time, rounds, pushes and a hash of Z_b (run twice per mode:
equal hashes mean the mode is bit-reproducible run to run)."""
import hashlib, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 23
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
u, v = W.rmat_edges(scale, 24, 3, device="cuda")
n = 1 << scale
src = torch.cat([u, v]); dst = torch.cat([v, u])
order = torch.argsort(src * n + dst); src, dst = src[order], dst[order]
cnt = torch.bincount(src, minlength=n)
off = torch.zeros(n + 1, dtype=torch.int64, device="cuda"); off[1:] = torch.cumsum(cnt, 0)
off_h = off.cpu().numpy(); tgt_h = dst.to(torch.int32).cpu().numpy()
del src, dst, order, cnt, off, u, v
gen = torch.Generator(device="cuda"); gen.manual_seed(3)
X = (torch.randn(n, d, device="cuda", generator=gen) / math.sqrt(d)).cpu().numpy()
e = ge.Engine(n, off_h, tgt_h, None, d, d, X, X, W.cfg4_F(d, 3), np.eye(d), np.ones(d),
              alpha=0.15, eps=1e-5, undirected=True, node_capacity=1024)
e.ppr_init()
rng = np.random.default_rng(4)
us, vs = rng.integers(0, n, 1500), rng.integers(0, n, 1500)
eu, ev, seen = [], [], set()
for a, b in zip(us.tolist(), vs.tolist()):
    if a == b or (a, b) in seen or np.any(tgt_h[off_h[a]:off_h[a + 1]] == b): continue
    seen.add((a, b)); seen.add((b, a)); eu.append(a); ev.append(b)
    if len(eu) == 1000: break
e.apply(W.EventList.edges(ge.ADD_EDGE, eu, ev), mode=ge.APPLY_GRAPH_AND_PPR_ONLY | ge.APPLY_DEFER_PUSH)
torch.cuda.synchronize(); t0 = time.perf_counter()
st = e.ppr_push(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
h = hashlib.sha1(e.get(ge.ZB).tobytes()).hexdigest()[:16] if scale <= 20 else "-"
print(f"force_pull={os.environ.get('DAMF_PPR_FORCE_PULL', '0')} scale={scale} d={d} push {dt*1e3:.2f} ms "
      f"rounds {st['push_rounds']} pushes {st['pushes']} Z_b sha1 {h}")
e.close()
