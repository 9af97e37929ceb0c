"""Dev driver: per-phase wall time of the whole-GPU PPR push (ctl->prof[24..28])
for init_propagate and a push after 1,000 structure-only insertions.
Phase timers need the library built with `make EXTRA=-DDAMF_PROF=1`."""
import sys, os, math, time
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
names = {24: "P1 push+sync", 25: "big marks", 26: "P3 dense", 27: "P3 sparse", 28: "P3c+sync"}
def run(label, fn):
    p0 = e.profile_counters().copy(); t0 = time.perf_counter()
    st = fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    p1 = e.profile_counters()
    print(label, f"wall {dt*1e3:.2f} ms", st)
    import ctypes as C
    tr = np.zeros(4 * 1024, np.int64)
    r = ge.lib().damf_gpu_ppr_trace(e.h, tr.ctypes.data_as(C.c_void_p), 1024)
    tr = tr[:4 * max(r, 0)].reshape(-1, 4)
    print("   rounds (nF, dense, items, scatter items[, push us, round us]):")
    print("   " + ";".join(f"{a},{b & 1},{c},{d_ & 0xffffffff}" + (f",{(d_ >> 32) / 1e3:.1f},{(b >> 1) / 1e3:.1f}" if (b >> 1) else "")
                         for a, b, c, d_ in tr.tolist()))
    for s, nm in names.items():
        print(f"   {nm:14s} {(int(p1[s]) - int(p0[s]))/1e6:9.3f} ms")
run("init", e.ppr_init)
if len(sys.argv) > 3:
    run("init2", e.ppr_init)
rng = np.random.default_rng(4)
us, vs = rng.integers(0, n, 1500), rng.integers(0, n, 1500)
eu, ev, seen = [], [], set()
for a, b in zip(us.tolist(), vs.tolist()):
    if a == b or (a, b) in seen or np.any(tgt_h[off_h[a]:off_h[a + 1]] == b): continue
    seen.add((a, b)); seen.add((b, a)); eu.append(a); ev.append(b)
    if len(eu) == 1000: break
e.apply(W.EventList.edges(ge.ADD_EDGE, eu, ev), mode=ge.APPLY_GRAPH_AND_PPR_ONLY | ge.APPLY_DEFER_PUSH)
if os.environ.get("PROF_PUSH_ONLY"):  # ncu --profile-from-start off: capture only this push
    torch.cuda.synchronize(); torch.cuda.profiler.start()
    run("push", e.ppr_push)
    torch.cuda.synchronize(); torch.cuda.profiler.stop()
else:
    run("push", e.ppr_push)
e.close()
