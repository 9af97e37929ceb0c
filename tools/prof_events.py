"""Dev profiling helper: per-event latency of the cfg2 stream with and
without the PPR enhancer (alpha = 1 bypasses it), for kernel breakdowns.
Phase counters need the library built with `make EXTRA=-DDAMF_PROF=1`."""
import sys, os, time, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W

nev = int(sys.argv[1]) if len(sys.argv) > 1 else 300
alphas = [float(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1.0, 0.15]
w = W.cfg2()
off_, tgt_ = W.undirected_csr(w["n"], *w["init"])
d = {"n": w["n"], "off": off_, "tgt": tgt_}
for alpha in alphas:
    e = ge.Engine.from_graph(d["n"], d["off"], d["tgt"], None, w["d"], alpha=alpha, eps=w["eps"],
                             undirected=True, seed=0, node_capacity=4096)
    s = w["stream"]
    e.apply(s.slice(0, 50))
    t0 = time.perf_counter()
    st = e.apply(s.slice(50, 50 + nev), mode=ge.APPLY_TIME_EVENTS)
    t1 = time.perf_counter()
    lat = e.latencies_us()
    kinds = s.kind[50:50 + nev]
    out = {"alpha": alpha, "events": nev, "wall_ms": (t1 - t0) * 1e3, "p50_us": float(np.median(lat)),
           "mean_us": float(lat.mean()), "stats": st}
    for kk, nm in ((0, "node"), (1, "add"), (2, "remove")):
        if np.any(kinds == kk):
            out[nm + "_p50_us"] = float(np.median(lat[kinds == kk]))
    pc = e.profile_counters().astype(np.float64)
    # slot i accumulates the phase ENDING at PROF_MARK(i)
    names = ["gather+w", "B1+prep", "eigA", "z2+B4", "eigB", "E-gemm", "cols", "B7-reduce",
             "rowfix+inv-rows", "gemms(4)", "B8", "tail", "graph"]
    out["phase_us_per_event"] = {nm: round(pc[i] / 1.965e3 / (nev + 50), 2) for i, nm in enumerate(names)}
    en = ["eig.prep", "eig.roots", "eig.sync1", "eig.zhat", "eig.sync2", "eig.order", "eig.vecs"]
    out["eig_us_per_event"] = {nm: round(pc[16 + i] / 1.965e3 / (nev + 50), 2) for i, nm in enumerate(en)}
    pn = ["ppr.absorb", "ppr.smax", "ppr.cand0", "ppr.P1", "ppr.B1", "ppr.P2", "ppr.B2", "ppr.compact"]
    out["ppr_us_per_event"] = {nm: round(pc[23 + i] / 1.965e3 / (nev + 50), 2) for i, nm in enumerate(pn)}
    out["staged_gemm_us_per_event"] = {nm: round(pc[28 + i] / 1.965e3 / (nev + 50), 2)
                                       for i, nm in enumerate(["wait", "dmma", "whole_call"])}
    out["root_iters_mean"] = float(pc[13] / max(pc[14], 1))
    out["root_iters_max"] = int(pc[15])
    print(json.dumps(out))
    e.close()
