"""Dev: weighted graphs, periodic rebases, tiny / rank-deficient shapes and
directed enhanced streams against the oracle (one case per process: a
sticky CUDA fault in one case cannot hide the others)."""
import sys, subprocess, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
F = ("kind", "u", "v", "w", "in_off", "in_ids", "in_w", "out_off", "out_ids", "out_w")


def run(case):
    import oracle
    from helpers import gpu_from_oracle, sampled_product_rel, sigma_rel, dense_defect
    from paper_2306_08967_b200 import engine as ge
    from paper_2306_08967_b200.workloads import EventList
    name, d, alpha, weighted, every, undirected = case
    rng = np.random.default_rng(d * 7 + int(alpha * 10) + every)
    n = 220
    m = 1400
    src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    key = np.unique(src * n + dst) if not undirected else np.unique(np.minimum(src, dst) * n + np.maximum(src, dst))
    a, b = key // n, key % n
    w = rng.uniform(0.5, 2.0, len(a)) if weighted else np.ones(len(a))
    if undirected:
        g = oracle.Graph(n, np.concatenate([a, b]), np.concatenate([b, a]), np.concatenate([w, w]), True)
    else:
        g = oracle.Graph(n, a, b, w, False)
    have = set(zip(a.tolist(), b.tolist()))
    kinds, us, vs, ws = [], [], [], []
    while len(us) < 150:
        x, y = (int(t) for t in rng.integers(0, n, 2))
        if x == y:
            continue
        k2 = (min(x, y), max(x, y)) if undirected else (x, y)
        if k2 in have:
            kinds.append(2); have.discard(k2)
        else:
            kinds.append(1); have.add(k2)
        us.append(x); vs.append(y); ws.append(float(rng.uniform(0.5, 2.0)) if weighted else 1.0)
    ev = oracle.Events.edges(np.array(kinds, np.int32), us, vs, ws)
    oe = oracle.OracleEngine(g, d=d, alpha=alpha, eps=1e-6, seed=d, rebase_every=every)
    e = gpu_from_oracle(g, oe, d=d, alpha=alpha, eps=1e-6, rebase_every=every)
    st = e.apply(EventList(*(getattr(ev, f) for f in F)))
    oe.apply(ev)
    p = sampled_product_rel(e.get(ge.X), e.get(ge.Y), oe.get(oe.X), oe.get(oe.Y))
    s = sigma_rel(e.get(ge.SIGMA), oe.get(oe.SIGMA))
    off, ids, deg = e.graph_sets()
    oo, io, do = oe.graph_sets()
    gsame = np.array_equal(off, oo) and np.array_equal(ids.astype(np.int64), io) and np.allclose(deg, do, rtol=0, atol=1e-12)
    dfc = 0.0
    if alpha < 1:
        wv = None
        dfc = dense_defect(e.n, off, ids, deg, e.get(ge.X), e.get(ge.Z), alpha) if not weighted else -1.0
    ok = p <= 1e-4 and s <= 1e-6 and gsame and dfc <= 1e-6 * (1 + 1e-6) + 2e-7
    print(name, "OK" if ok else "BAD", st["applied"], st["rebases"], f"prod {p:.2e} sigma {s:.2e} graph {gsame} defect {dfc:.2e}", flush=True)


CASES = [("weighted-undirected-a1", 16, 1.0, True, 50000, True),
         ("weighted-directed-a.3", 16, 0.3, True, 50000, False),
         ("rebase-every-40-a.3", 16, 0.3, False, 40, True),
         ("rebase-every-40-a1", 24, 1.0, False, 40, False),
         ("d2-a.3", 2, 0.3, False, 50000, True),
         ("d1-a1", 1, 1.0, False, 50000, False),
         ("d64-directed-a.2", 64, 0.2, False, 50000, False)]
if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(CASES[int(sys.argv[1])])
    else:
        for i in range(len(CASES)):
            r = subprocess.run([sys.executable, __file__, str(i)], capture_output=True, text=True, timeout=300)
            out = (r.stdout.strip().splitlines() or [""])[-1]
            print(out if r.returncode == 0 else f"{CASES[i][0]} ERROR {r.stderr.strip().splitlines()[-1][:300]}", flush=True)
