"""Dev profiling helper: per-phase cycles of the event kernel on a config-5-
like state (R-MAT scale 20, orthonormal U/V, sigma_i = i^-1/2, d = 128)
after the rebase transient. Needs the DAMF_PROF build:
DAMF_GPU_LIB=paper_2306_08967_b200/libdamf_gpu_prof.so python tools/prof_cfg5.py"""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
from test_gpu_configs import cfg5_like

nev = int(sys.argv[1]) if len(sys.argv) > 1 else 300
e, su, sv = cfg5_like(20, 128, 200 + nev, seed=4)
e.apply(W.EventList.edges(1, su[:200], sv[:200]))
if os.environ.get("DAMF_DUMP"):
    import ctypes as C
    ge.lib().damf_gpu_debug_dump.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    ge.lib().damf_gpu_debug_dump(e.h, None, -1)
p0 = e.profile_counters().astype(np.float64)
st = e.apply(W.EventList.edges(1, su[200:200 + nev], sv[200:200 + nev]), mode=ge.APPLY_TIME_EVENTS)
lat = e.latencies_us()
pc = e.profile_counters().astype(np.float64) - p0
clk = 1.965e3
out = {"events": nev, "p50_us": float(np.median(lat)), "mean_us": float(lat.mean()), "rebases": st["rebases"]}
names = ["gather+w", "B1+prep", "eigA", "z2+B4", "eigB", "E-gemm", "cols", "B7-reduce",
         "rowfix+inv-rows", "gemms(4)", "B8", "tail", "graph"]
out["phase_us_per_event"] = {nm: round(pc[i] / clk / nev, 2) for i, nm in enumerate(names)}
en = ["eig.prep", "eig.roots", "eig.sync1", "eig.zhat", "eig.sync2", "eig.order", "eig.vecs"]
out["eig_us_per_event"] = {nm: round(pc[16 + i] / clk / nev, 2) for i, nm in enumerate(en)}
out["staged_gemm_us_per_event"] = {nm: round(pc[28 + i] / clk / nev, 2)
                                   for i, nm in enumerate(["wait", "dmma", "whole_call"])}
gn = ["prologue", "bar_after_dmma", "issue_next", "epilogue", "tail"]
out["staged_gemm_detail_us_per_event"] = {nm: round(pc[99 + i] / clk / nev, 2) for i, nm in enumerate(gn)}
out["roots_us_per_event_by_rank"] = [round(pc[32 + r] / clk / nev, 1) for r in range(16)]
out["sync1_us_per_event_by_rank"] = [round(pc[48 + r] / clk / nev, 1) for r in range(16)]
out["root_iters_per_event_by_rank"] = [round(pc[64 + r] / nev, 1) for r in range(16)]
out["root_iters_mean"] = float(pc[13] / max(pc[14], 1))
out["root_iters_max"] = int(e.profile_counters()[15])
out["roots_with_10plus_iters_per_event"] = float(pc[31] / nev)
out["roots_per_event_rank0"] = float(pc[14] / nev)
print(json.dumps(out, indent=1))

if os.environ.get("DAMF_DUMP"):
    import ctypes as C
    buf = np.zeros(8 + 8 * 800)
    ge.lib().damf_gpu_debug_dump.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    ge.lib().damf_gpu_debug_dump(e.h, buf.ctypes.data, len(buf))
    np.save(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "slow_roots.npy"), buf)
    print("dumped", int(buf[0]))

if os.environ.get("DAMF_TLOG"):
    import ctypes as C
    n = 8 + 8 * 800 + 16 * 260
    buf = np.zeros(n)
    ge.lib().damf_gpu_debug_dump.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    ge.lib().damf_gpu_debug_dump(e.h, buf.ctypes.data, n)
    T = buf[8 + 8 * 800:].reshape(16, 260)
    m = int(T[:, 0].min())
    L = T[:, 4:4 + 4 * m].reshape(16, m, 4)
    print("solve: [last CTA arrival - first roots begin] [release - last arrival] (us); slowest rank; its group-0 time")
    for s in (13, 19, 23):
        t0 = L[:, s, 0].min()
        print("solve", s, "per rank [begin, group0 done, cta done, release] us")
        for r in range(16):
            print("  rank", r, [round((x - t0) / 1e3, 2) for x in L[r, s]])
    for s in range(8, min(m, 24)):
        t0 = L[:, s, 0].min()
        arr = L[:, s, 2]
        rel = L[:, s, 3]
        print(s, round((arr.max() - t0) / 1e3, 2), round((rel.min() - arr.max()) / 1e3, 2), int(arr.argmax()),
              [round((x - t0) / 1e3, 1) for x in arr])
