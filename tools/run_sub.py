"""Dev driver: run one bench.py sub-benchmark (cfg3 / cfg5 / ppr / mat) alone."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
ap = argparse.ArgumentParser()
ap.add_argument("which")
ap.add_argument("--cfg3-events", type=int, default=4096)
ap.add_argument("--cfg5-events", type=int, default=10000)
ap.add_argument("--ppr-scale", type=int, default=23)
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
hbm, kind = bench.peaks()
t0 = time.time()
if a.which == "cfg3":
    r = bench.bench_cfg3(a)
elif a.which == "cfg5":
    r = bench.bench_cfg5(a, hbm)
elif a.which == "ppr":
    r = bench.bench_ppr(a, hbm, kind)
else:
    r = dict(zip(("sweep", "roofline"), bench.bench_materialize(a, hbm, kind)))
r["wall_s"] = round(time.time() - t0, 1)
print(json.dumps(r))
