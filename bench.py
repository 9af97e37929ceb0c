#!/usr/bin/env python
"""Benchmark of the B200 DAMF hot path (BASELINE.json metric:
"edge updates/s & p50 us/update; Z=X.F and PPR-push GB/s vs HBM peak").

Headline workload (N = 1, the largest BASELINE configuration that fits one
GPU): config 5 -- R-MAT scale 26, ef 16 (seed 4; 67.1 M nodes, 2.10 B arcs,
int64 offsets), d = 128, U / V random orthonormal with sigma_i = i^-1/2
(34 GB fp32 each, generated on the device), the 10,000 degree-proportional
single-edge insertions of the config, plus its one full materialisation.
A "step" is one damf_gpu_apply call over the next 10,000 / (steps + warmup)
insertions, applied sequentially exactly as `for (e : batch) Engine::apply(e)`.

  value    insertions/s over the device span of the timed calls (CUDA events
           from each call's first launch, event descriptors already in HBM,
           to the end of its last kernel -- rebases included)
  e2e      insertions/s through the public call (damf_gpu_apply) with the
           events in host memory: descriptor build, H2D copy, the kernels and
           the D2H status read, wall clock per call
  latency  per-insertion device latency (%globaltimer stamps in the kernel)
  roofline the config's full materialisation X = X_b P_X (n = 2^26, d = 128,
           68.7 GB algorithmic), CUDA events on the engine stream
  cpu_baseline  the fp64 oracle port (oracle/, 1 thread) applying the same
           first insertions from the same initial factors (see cfg5_oracle)

Sub-benchmarks (`sub`): the config-2 SBM stream with its own CPU ratio,
config-3 batches 1 / 64 / 1024, the config-4 materialisation sweep and PPR
push, and CPU legs for query_all and init_propagate.

`--impl reference` times the reference's CPU implementation (the oracle port;
the reference itself cannot be built here) on the same
config-5 insertions with the same output line.

Multi-GPU: the update chain does not shard: N ranks run N
independent replicas ("replicas only", weak scaling); value = total
insertions / max-over-ranks device time. `--gpus N` without torchrun
re-launches itself under torch.distributed.run with N ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "edge updates/s & p50 us/update; Z=X.F and PPR-push GB/s vs HBM peak"
WORKLOAD = ("cfg5: R-MAT scale 26 ef 16 seed 4 (67.1M nodes, 2.10B arcs), d=128, U/V orthonormal "
            "sigma_i=i^-1/2, 10,000 degree-proportional single-edge insertions, alpha=1")
CFG5_EVENTS = 10_000


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_info():
    cpu = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu": cpu, "oracle_build": ORACLE_BUILD["flags"]}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu_index=0):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        self.gpu = gpu_index

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        try:
            rows = [l.split(",") for l in open(self.path).read().strip().splitlines() if l.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for nm, val in zip(names, r[4:8]):
                if "Active" in val and "Not" not in val:
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


def job_max(values, device="cpu"):
    """Max over ranks of per-rank timings (the contract's max-over-ranks
    clock); identity when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def replica_value(events_per_rank, world_size, seconds_max):
    """Whole-job throughput of N independent replicas (weak scaling): all
    ranks' events over the slowest rank's time."""
    return events_per_rank * world_size / seconds_max


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def descriptor_bytes(batch, undirected=True):
    """Host->device bytes damf_gpu_apply copies for a batch (EventDesc 112 B,
    StepDesc 56 B, sparse rows 16 B/nnz, AddNode lists 16 B/entry, touched 8 B)."""
    kinds = batch.kind
    ne = len(kinds)
    nin = int(batch.in_off[-1])
    edges = int(np.sum(kinds != 0))
    nodes = ne - edges
    steps = 2 * ne
    return ne * 112 + steps * 56 + (2 * edges + 2 * nin) * 16 + 2 * nin * 16 + (2 * edges + nin + nodes) * 8


def split_steps(n_events, steps, warmup):
    total = steps + warmup
    per = max(1, n_events // total)
    return per


def timed_stream(eng, stream, per, steps, warmup, ws, local):
    """Warm-up calls, then `steps` timed calls of `per` events each (one
    damf_gpu_apply per step). Returns device seconds (sum of the calls'
    device spans), wall seconds of the public calls, per-event latencies,
    rebases, launches and the clocks summary."""
    import torch
    from paper_2306_08967_b200 import engine as ge
    for s in range(warmup):
        eng.apply(stream.slice(s * per, (s + 1) * per), mode=ge.APPLY_TIME_EVENTS)
    dev_ms, wall_s, lat, h2d = 0.0, 0.0, [], []
    rebases = 0
    launches0 = eng.diag()["kernel_launches"]
    with ClockSampler(local) as clk:
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        for s in range(warmup, warmup + steps):
            batch = stream.slice(s * per, (s + 1) * per)
            t0 = time.perf_counter()
            st = eng.apply(batch, mode=ge.APPLY_TIME_EVENTS)
            wall_s += time.perf_counter() - t0
            dev_ms += st["device_ms"]
            rebases += st["rebases"]
            lat.extend(eng.latencies_us().tolist())  # read back outside the timed call
            h2d.append(descriptor_bytes(batch))
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
    launches = eng.diag()["kernel_launches"] - launches0
    return dict(dev_s=dev_ms * 1e-3, wall_s=wall_s, lat=np.array(lat), rebases=rebases,
                launches=launches, h2d=int(np.mean(h2d)), clocks=clk.summary())


def pct(lat):
    return {"p50": round(float(np.percentile(lat, 50)), 2),
            "p90": round(float(np.percentile(lat, 90)), 2),
            "p99": round(float(np.percentile(lat, 99)), 2),
            "mean": round(float(lat.mean()), 2), "events": int(len(lat))}


# ------------------------------------------------------------------ cfg 5
def build_cfg5(n_events):
    """Device engine at config 5 and the stream (host arrays)."""
    import torch
    from paper_2306_08967_b200 import engine as ge
    from paper_2306_08967_b200 import workloads as W
    t0 = time.time()
    d, n = 128, 1 << 26
    keys, off, tgt, su, sv = W.cfg5_inputs(n_events)
    edges = int(keys.numel())
    del keys
    torch.cuda.empty_cache()
    sig = np.arange(1, d + 1, dtype=np.float64) ** -0.5
    eng = ge.Engine(n, off, tgt, None, d, d, None, None, np.eye(d), np.eye(d), sig, alpha=1.0,
                    undirected=True, node_capacity=1024, arc_capacity=1 << 24)
    arcs = int(tgt.numel())
    del off, tgt
    torch.cuda.empty_cache()
    W.orthonormal_rows_into(eng, ge.XB, n, d, sig, seed=40)
    W.orthonormal_rows_into(eng, ge.YB, n, d, sig, seed=41)
    stream = W.EventList.edges(ge.ADD_EDGE, su, sv)
    return dict(eng=eng, stream=stream, su=su, sv=sv, n=n, d=d, sig=sig, edges=edges, arcs=arcs,
                setup_s=time.time() - t0)


def cfg5_materialize(eng, n, d, hbm, peak_kind):
    """One full materialisation X = X_b P_X (query_all, factor_state.cpp:
    120-123) into device memory; CUDA events on the engine stream."""
    import torch
    from paper_2306_08967_b200 import engine as ge
    out = torch.empty(n, d, dtype=torch.float32, device="cuda")
    es = torch.cuda.ExternalStream(eng.stream_ptr())
    ms, call_ms = [], []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(es)
        eng.materialize(ge.X, out.data_ptr(), on_device=True)
        e1.record(es)
        e1.synchronize()
        call_ms.append(e0.elapsed_time(e1))
        # the X F kernels alone (F split + tcgen05 kernel), CUDA events recorded by the
        # engine on its stream around their launch; the call adds a control-block round
        # trip and the fp64 patch of the side-table rows
        ms.append(eng.diag()["last_materialize_ms"])
    del out
    torch.cuda.empty_cache()
    t = float(np.median(ms))
    bytes_ = 8.0 * n * d + 8.0 * d * d
    gbs = bytes_ / (t * 1e-3) / 1e9
    return {"kernel": "materialize_tc128 (X = X_b P_X, n = 67,108,864, d = 128, 3 x TF32)",
            "bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(gbs / hbm, 4),
            "traffic": ncu_metric_traffic("r2_mat_cfg5_launches.csv", "materialize_tc128"),
            "traffic_source": "profiles/r2_mat_cfg5_launches.csv (ncu --metrics dram__bytes_read.sum,"
                              "dram__bytes_write.sum on the same kernel at the same shape, "
                              "tools/prof_r2.py mat5)",
            "peak_kind": peak_kind, "algorithmic_bytes_per_launch": int(bytes_),
            "launch_ms": round(t, 4), "launch_ms_all": [round(x, 4) for x in ms],
            "api_call_ms_all": [round(x, 4) for x in call_ms]}


ORACLE_BUILD = {"flags": "-O3 (portable build from make)"}


def oracle_module():
    """The CPU oracle for the baseline legs, compiled once per bench run with
    -O3 -march=native on the host that is about to be timed;
    falls back to the portable in-tree build if the compiler is missing."""
    if "oracle" not in sys.modules and not os.environ.get("DAMF_ORACLE_LIB"):
        import subprocess
        import tempfile
        out = os.path.join(tempfile.mkdtemp(prefix="damf_oracle_"), "libdamf_oracle_native.so")
        cmd = ["g++", "-O3", "-march=native", "-std=c++17", "-fPIC", "-shared", "-o", out,
               os.path.join(ROOT, "oracle", "damf_oracle.cpp"),
               os.path.join(ROOT, "oracle", "oracle_capi.cpp")]
        try:
            subprocess.run(cmd, check=True, capture_output=True, timeout=300)
            os.environ["DAMF_ORACLE_LIB"] = out
            ORACLE_BUILD["flags"] = "g++ -O3 -march=native, built on this host for this run"
        except Exception as ex:  # noqa: BLE001
            print(f"[bench] native oracle build failed ({ex}); using the portable build", file=sys.stderr)
    import oracle
    return oracle


def cfg5_oracle(su, sv, n, d, sig, budget_s, max_events=None, first=0):
    """The fp64 oracle (1 thread) applying config 5's insertions in order
    from the same initial factors as the device (the fp32 rows
    orthonormal_rows_into loads, widened). The reference's per-insertion work
    reads and writes only the endpoints' rows and the k x k state
    (update_engine.cpp:144-204, factor_state.cpp:158-213; alpha = 1 bypasses
    the enhancer, enhancer.cpp:34-38), so the oracle Engine holds exactly the
    stream's endpoints (their rows, the graph among them); Engine::apply --
    graph mutation, two rank-1 updates, cond_estimate, the rebase policy -- is
    timed per event with steady_clock like damf_cli.cpp:145-151."""
    oracle = oracle_module()
    from paper_2306_08967_b200 import workloads as W
    m = len(su) if max_events is None else min(max_events, len(su))
    first = min(first, m)
    rows = np.unique(np.concatenate([su[:m], sv[:m]]))
    xb = W.orthonormal_rows_subset(n, d, sig, 40, rows).astype(np.float64)
    yb = W.orthonormal_rows_subset(n, d, sig, 41, rows).astype(np.float64)
    g = oracle.Graph(len(rows), np.zeros(0, np.int64), np.zeros(0, np.int64), None, True)
    oe = oracle.OracleEngine(g, d=d, alpha=1.0, factors=(xb, yb, np.eye(d), np.eye(d), sig))
    lu, lv = np.searchsorted(rows, su[:m]), np.searchsorted(rows, sv[:m])
    # the events before `first` (our arm's warm-up) are applied untimed, so
    # the timed sample is the same events as our arm's timed region
    t_warm = time.perf_counter()
    for a in range(0, first, 50):
        oe.apply(oracle.Events.edges(1, lu[a:min(first, a + 50)], lv[a:min(first, a + 50)]))
    t_warm = time.perf_counter() - t_warm
    total_s, done, lat = 0.0, first, []
    while done < m and total_s < budget_s:
        b = min(m, done + 25)
        ev = oracle.Events.edges(1, lu[done:b], lv[done:b])
        t0 = time.perf_counter()
        l = oe.apply(ev, lat=True)
        total_s += time.perf_counter() - t0
        lat.extend(l.tolist())
        done = b
    return {"value": round((done - first) / total_s, 3), "unit": "insertions/s", "cores": 1,
            "kind": "port",
            "sample": f"insertions {first}..{done} of the {len(su)} cfg5 insertions (the first of "
                      f"our arm's timed events onward; events 0..{first} replayed untimed in "
                      f"{t_warm:.1f} s), in order, from the device's initial factors; fp64 oracle "
                      f"Engine over the stream's endpoints (per-event work is independent of n), "
                      f"1 thread, {total_s:.1f} s timed",
            "p50_ms": round(float(np.percentile(lat, 50)), 3),
            "rebases": int(oe.stat(7)), "eager_folds": int(oe.stat(6))}


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    hbm, peak_kind = peaks()
    c5 = build_cfg5(CFG5_EVENTS)
    eng = c5["eng"]
    per = split_steps(len(c5["stream"]), args.steps, args.warmup)
    r = timed_stream(eng, c5["stream"], per, args.steps, args.warmup, ws, local)
    ev_total = per * args.steps
    dev_s, wall_s = job_max([r["dev_s"], r["wall_s"]], device="cuda")
    value = replica_value(ev_total, ws, dev_s)
    e2e_value = replica_value(ev_total, ws, wall_s)
    roofline = cfg5_materialize(eng, c5["n"], c5["d"], hbm, peak_kind) if rank == 0 else None
    dg = eng.diag()
    eng.close()
    del eng
    c5["eng"] = None
    torch.cuda.empty_cache()
    sub = {}
    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cfg5_oracle(c5["su"], c5["sv"], c5["n"], c5["d"], c5["sig"], args.cpu_seconds,
                          max_events=per * (args.warmup + args.steps), first=per * args.warmup)
        cpu["host"] = host_info()
    if rank == 0 and not args.no_sub:
        sub["cfg2"] = bench_cfg2(args)
        sub["materialize_sweep"] = bench_materialize(args, hbm)
        if not args.quick:
            sub["ppr_push"] = bench_ppr(args, hbm, peak_kind)
        if args.cfg3_events > 0:
            sub["cfg3"] = bench_cfg3(args)
        if not args.no_cpu and not args.quick:
            sub["cpu_legs"] = cpu_legs(args)
    if rank != 0:
        return
    out = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "insertions/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(dev_s * 1e3 / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64 (d x d state, small SVD) / f32 (base rows)",
        "data": "synthetic (seeded R-MAT scale 26 + random orthonormal factors, cfg 5)",
        "config": {"workload": WORKLOAD, "events_per_step": per,
                   "parallelism": "replicas" if ws > 1 else "single",
                   "l2": "no flush: the 80 GB state is far above L2; each event's working set "
                         "(P, P^-1, sigma, two rows) is L2-resident by design (latency-bound path)"},
        "latency_us": pct(r["lat"]),
        "e2e": {"value": round(e2e_value, 2), "unit": "insertions/s",
                "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": 8 * 8 + 400,
                "note": "damf_gpu_apply with the step's events in host memory (descriptor build, "
                        "H2D, kernels, control-block D2H), wall clock per call"},
        "gpu_launches": int(r["launches"]),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": r["clocks"],
        "engine": {"setup_s": round(c5["setup_s"], 1), "rebases_timed": int(r["rebases"]),
                   "edges": c5["edges"], "arcs": c5["arcs"], "k": dg["k"],
                   "device_bytes": dg["device_bytes"], "cond_end": dg["cond_estimate"]},
        "sub": sub,
    }
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ subs
def ncu_traffic(fname, kernel_substr):
    """dram__bytes_read.sum + dram__bytes_write.sum (bytes) of the first
    launch of `kernel_substr` in a committed `ncu --set full` raw capture under
    profiles/ (per launch, like roofline.achieved), or None."""
    import csv
    path = os.path.join(ROOT, "profiles", fname)
    if not os.path.exists(path):
        return None
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None
    head, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for row in rows[2:]:
        rec = dict(zip(head, row))
        if kernel_substr not in rec.get("Kernel Name", ""):
            continue
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = head.index(m)
            tot += float(row[i].replace(",", "")) * scale.get(units[i], 1.0)
        return int(tot)
    return None


def ncu_metric_traffic(fname, kernel_substr):
    """dram__bytes_read.sum + dram__bytes_write.sum of the first launch of
    `kernel_substr` in a committed `ncu --metrics ... --csv` launch list
    (one row per metric) under profiles/, or None."""
    import csv
    path = os.path.join(ROOT, "profiles", fname)
    if not os.path.exists(path):
        return None
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    head = rows[0]
    tot, seen = 0.0, None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[1:]:
        rec = dict(zip(head, r))
        if kernel_substr not in rec["Kernel Name"]:
            continue
        if seen is None:
            seen = rec["ID"]
        if rec["ID"] != seen:
            break
        if rec["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(rec["Metric Value"].replace(",", "")) * scale.get(rec["Metric Unit"], 1.0)
    return int(tot) if seen is not None else None


def bench_cfg2(args):
    """Config 2: SBM n = 100,000 (20 blocks), d = 128, alpha 0.15, eps 1e-5,
    the stream of inserts / deletions / node additions (device t-SVD init),
    plus its own CPU ratio: the oracle resumes from the device's saved state
    (DAMF v1 file, io.cpp:182-269) after the warm-up and applies the same
    timed events."""
    import tempfile
    import torch
    from paper_2306_08967_b200 import engine as ge
    from paper_2306_08967_b200 import workloads as W
    w = W.cfg2()
    n = w["n"]
    eu, ev = w["init"]
    off, tgt = W.undirected_csr(n, eu, ev)
    t0 = time.time()
    eng = ge.Engine.from_graph(n, off, tgt, None, w["d"], alpha=w["alpha"], eps=w["eps"],
                               undirected=True, seed=0, node_capacity=4096)
    init_s = time.time() - t0
    stream = w["stream"]
    warm = 500
    eng.apply(stream.slice(0, warm), mode=ge.APPLY_TIME_EVENTS)
    res = {"graph": "SBM n=100000 (20 x 5000), d=128, alpha=0.15, eps=1e-5", "init_s": round(init_s, 2)}
    state = None
    if not args.no_cpu:
        state = os.path.join(tempfile.mkdtemp(), "cfg2.damf")
        eng.save_state(state)
    m = len(stream) - warm
    dev_ms, wall_s, lat = 0.0, 0.0, []
    for a in range(warm, len(stream), 500):
        part = stream.slice(a, min(len(stream), a + 500))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        st = eng.apply(part, mode=ge.APPLY_TIME_EVENTS)
        wall_s += time.perf_counter() - t1
        dev_ms += st["device_ms"]
        lat.extend(eng.latencies_us().tolist())
    lat = np.array(lat)
    res.update({"events": m, "device_events_per_s": round(m / (dev_ms * 1e-3), 1),
                "e2e_events_per_s": round(m / wall_s, 1), "latency_us": pct(lat)})
    eng.close()
    del eng
    torch.cuda.empty_cache()
    if state:
        oracle = oracle_module()
        t2 = time.time()
        oe = oracle.OracleEngine.load_state(state)
        load_s = time.time() - t2
        done, total_s = 0, 0.0
        while done < m and total_s < args.cpu_seconds:
            b = min(m, done + 20)
            part = stream.slice(warm + done, warm + b)
            t3 = time.perf_counter()
            oe.apply(part)
            total_s += time.perf_counter() - t3
            done = b
        os.remove(state)
        cpu_v = done / total_s
        res["cpu_baseline"] = {"value": round(cpu_v, 3), "unit": "events/s", "cores": 1,
                               "kind": "port",
                               "sample": f"events {warm}..{warm + done} of the cfg2 stream, oracle "
                                         f"resumed from the device's DAMF v1 state ({load_s:.1f} s "
                                         f"load), fp64, 1 thread"}
        res["device_vs_cpu"] = round(res["device_events_per_s"] / cpu_v, 1)
        res["e2e_vs_cpu"] = round(res["e2e_events_per_s"] / cpu_v, 1)
    return res


def bench_materialize(args, hbm):
    """Z = X F on the cfg-4 shape (n = 2^23, X ~ N(0,1/d), F = Q diag(U[.5,2]))."""
    import torch
    from paper_2306_08967_b200 import engine as ge
    from paper_2306_08967_b200 import workloads as W
    n = 1 << 23
    res = {}
    for d in (32, 64, 128, 256):
        g = torch.Generator(device="cuda")
        g.manual_seed(3)
        X = torch.randn(n, d, device="cuda", generator=g) / math.sqrt(d)
        Z = torch.empty_like(X)
        F = W.cfg4_F(d, 3)
        st = torch.cuda.current_stream().cuda_stream
        for _ in range(3):
            ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr(), st)
        ms = [ge.materialize_dev(X.data_ptr(), n, d, F, Z.data_ptr(), st) for _ in range(5)]
        t = float(np.mean(ms))
        bytes_ = 8.0 * n * d + 8.0 * d * d
        gbs = bytes_ / (t * 1e-3) / 1e9
        res[f"d{d}"] = {"ms": round(t, 4), "GBps": round(gbs, 1), "frac": round(gbs / hbm, 4),
                        "TFLOPs": round(2.0 * n * d * d / (t * 1e-3) / 1e12, 2)}
        del X, Z
        torch.cuda.empty_cache()
    res["d256"]["traffic"] = ncu_traffic("r1_mat256_raw.csv", "materialize_bf16_256")
    return res


def rmat_engine(scale, ef, seed, d, alpha, eps):
    import torch
    from paper_2306_08967_b200 import engine as ge
    from paper_2306_08967_b200 import workloads as W
    n = 1 << scale
    keys = W.rmat_keys_device(scale, ef, seed)
    off, tgt = W.csr_from_keys_device(n, keys)
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    X = (torch.randn(n, d, device="cuda", generator=g) / math.sqrt(d)).contiguous()
    F = W.cfg4_F(d, seed)
    eng = ge.Engine(n, off, tgt, None, d, d, X, X, F, np.eye(d), np.ones(d), alpha=alpha,
                    eps=eps, undirected=True, node_capacity=1024)
    return eng, keys, off, tgt, X, F


def bench_ppr(args, hbm, peak_kind):
    """init_propagate + 1,000 structure-only insertions and a push on R-MAT
    (cfg 4 shape: scale 23, ef 24, d = 128, alpha 0.15, eps 1e-5)."""
    import torch
    from paper_2306_08967_b200 import engine as ge
    from paper_2306_08967_b200 import workloads as W
    scale, d = args.ppr_scale, 128
    n = 1 << scale
    t0 = time.time()
    eng, keys, off, tgt, X, F = rmat_engine(scale, 24, 3, d, 0.15, 1e-5)
    arcs = int(tgt.numel())
    del X
    gen_s = time.time() - t0
    es = torch.cuda.ExternalStream(eng.stream_ptr())

    def gbytes(a, b):
        F_ = b["frontier"] - a["frontier"]
        L_ = b["affected"] - a["affected"]
        arcsL = b["affected_arcs"] - a["affected_arcs"]
        pulled = b["pulled_arcs"] - a["pulled_arcs"]
        return 16.0 * d * F_ + 8.0 * L_ + 4.0 * arcsL + 8.0 * d * L_ + 4.0 * d * pulled

    c0 = eng.push_counters()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(es)
    st = eng.ppr_init()
    e1.record(es)
    e1.synchronize()
    ms_init = e0.elapsed_time(e1)
    c1 = eng.push_counters()
    b_init = gbytes(c0, c1)
    gbs_init = b_init / (ms_init * 1e-3) / 1e9
    rng = np.random.default_rng(4)
    us, vs = rng.integers(0, n, 3000), rng.integers(0, n, 3000)
    lo, hi = np.minimum(us, vs), np.maximum(us, vs)
    kk = torch.as_tensor((lo << 32) | hi, device="cuda")
    pos = torch.searchsorted(keys, kk).clamp(max=keys.numel() - 1)
    fresh = ((keys[pos] != kk).cpu().numpy()) & (lo != hi)
    _, first = np.unique((lo << 32) | hi, return_index=True)
    ok = np.zeros(len(us), bool)
    ok[first] = True
    ok &= fresh
    eu, evv = us[ok][:1000], vs[ok][:1000]
    eng.apply(W.EventList.edges(ge.ADD_EDGE, eu, evv),
              mode=ge.APPLY_GRAPH_AND_PPR_ONLY | ge.APPLY_DEFER_PUSH)
    c2 = eng.push_counters()
    e0.record(es)
    st2 = eng.ppr_push()
    e1.record(es)
    e1.synchronize()
    ms_push = e0.elapsed_time(e1)
    c3 = eng.push_counters()
    b_push = gbytes(c2, c3)
    eng.close()
    del eng, keys, off, tgt
    torch.cuda.empty_cache()
    return {"graph": f"R-MAT scale {scale} ef 24 (n={n}, arcs={arcs})", "gen_s": round(gen_s, 1),
            "init_propagate": {"ms": round(ms_init, 3), "rounds": st["push_rounds"],
                               "pushes": st["pushes"], "alg_GB": round(b_init / 1e9, 3),
                               "GBps": round(gbs_init, 1), "frac": round(gbs_init / hbm, 4)},
            "push_after_1000_inserts": {"ms": round(ms_push, 3), "rounds": st2["push_rounds"],
                                        "pushes": st2["pushes"],
                                        "alg_GB": round(b_push / 1e9, 4),
                                        "GBps": round(b_push / (ms_push * 1e-3) / 1e9, 1)},
            "roofline": {"kernel": "ppr_push_kernel + ppr_pull_kernel (init_propagate)",
                         "bound": "hbm", "achieved": round(gbs_init, 1), "peak": hbm,
                         "unit": "GB/s", "frac": round(gbs_init / hbm, 4),
                         "traffic": ppr_traffic(), "peak_kind": peak_kind}}


def ppr_traffic():
    path = os.path.join(ROOT, "profiles", "r1_ppr23_traffic.json")
    if not os.path.exists(path):
        return None
    return int(json.load(open(path))["dram_bytes_per_init"])


def stream_latencies(eng, ev, batch, max_events):
    """Apply ev[:max_events] in calls of `batch` events: per-event device
    latencies, device span and wall time of the calls."""
    import torch
    from paper_2306_08967_b200 import engine as ge
    lat = []
    t_wall = dev_ms = 0.0
    rebases = 0
    m = min(len(ev), max_events)
    torch.cuda.synchronize()
    if batch == 1:
        # single events through Engine::apply's one-event call
        for a in range(m):
            u, v = int(ev.u[a]), int(ev.v[a])
            t0 = time.perf_counter()
            st = eng.apply_edge(int(ev.kind[a]), u, v, 1.0, ge.APPLY_TIME_EVENTS)
            t_wall += time.perf_counter() - t0
            dev_ms += st.device_ms
            rebases += st.rebases
            lat.extend(eng.latencies_us().tolist())
    for a in range(0, m if batch > 1 else 0, batch):
        part = ev.slice(a, min(m, a + batch))
        t0 = time.perf_counter()
        st = eng.apply(part, mode=ge.APPLY_TIME_EVENTS)
        t_wall += time.perf_counter() - t0
        dev_ms += st["device_ms"]
        rebases += st["rebases"]
        lat.extend(eng.latencies_us().tolist())
    lat = np.array(lat)
    return {"events": int(m), "batch": batch, **{k + "_us": v for k, v in pct(lat).items()
                                                  if k in ("p50", "p90", "p99")},
            "device_events_per_s": round(m / (dev_ms * 1e-3), 1),
            "kernel_events_per_s": round(m / (lat.sum() * 1e-6), 1),
            "e2e_events_per_s": round(m / t_wall, 1), "rebases": int(rebases)}


def bench_cfg3(args):
    """Config 3: R-MAT scale 22, ef 16 (seed 2), d = 128, all but 100,000
    edges in the snapshot (randomized t-SVD on the device), held-out edges
    streamed as insertions in calls of 1, 64 and 1024 events (alpha = 1)."""
    import torch
    from paper_2306_08967_b200 import engine as ge
    from paper_2306_08967_b200 import workloads as W
    t0 = time.time()
    scale, d = 22, 128
    n = 1 << scale
    keys = W.rmat_keys_device(scale, 16, 2)
    g = torch.Generator(device="cuda")
    g.manual_seed(2)
    held = torch.randperm(keys.numel(), generator=g, device="cuda")[:100_000]
    drop = torch.zeros(keys.numel(), dtype=torch.bool, device="cuda")
    drop[held] = True
    off, tgt = W.csr_from_keys_device(n, keys, drop)
    hk = keys[held]
    su, sv = (hk >> 32).cpu().numpy(), (hk & 0xFFFFFFFF).cpu().numpy()
    edges = int(keys.numel())
    del keys, drop, hk, held
    off_h, tgt_h = off.cpu().numpy(), tgt.cpu().numpy()
    del off, tgt
    torch.cuda.empty_cache()
    gen_s = time.time() - t0
    t1 = time.time()
    eng = ge.Engine.from_graph(n, off_h, tgt_h, None, d, alpha=1.0, undirected=True, seed=2,
                               node_capacity=1024, arc_capacity=1 << 22)
    init_s = time.time() - t1
    del off_h, tgt_h
    ev = W.EventList.edges(ge.ADD_EDGE, su, sv)
    res = {"graph": f"R-MAT scale 22 ef 16 (n={n}, edges={edges}), d=128, alpha=1",
           "setup_s": round(gen_s, 1), "init_s": round(init_s, 1),
           "init": "damf_gpu_create: device randomized t-SVD (l = d + 10, 4 power iterations)"}
    a = 0
    for batch, m in ((1, args.cfg3_events // 4), (64, args.cfg3_events // 2),
                     (1024, args.cfg3_events)):
        r = stream_latencies(eng, ev.slice(a, len(ev)), batch, m)
        a += r["events"]
        res[f"batch{batch}"] = r
    eng.close()
    del eng
    torch.cuda.empty_cache()
    return res


def cpu_legs(args):
    """CPU legs beside the GPU for the two bulk paths (oracle port, fp64,
    1 thread): query_all (X_b P_X, factor_state.cpp:120-123) on a 2^20-row
    slice of the cfg-4 shape at d = 128, and init_propagate
    (enhancer.cpp:26-47) on an R-MAT scale-16 ef-24 graph at d = 128 with the
    device's init_propagate on the same graph and signal."""
    import torch
    oracle = oracle_module()
    from paper_2306_08967_b200 import engine as ge
    from paper_2306_08967_b200 import workloads as W
    out = {}
    d, rows = 128, 1 << 20
    rng = np.random.default_rng(3)
    x = rng.standard_normal((rows, d)) / math.sqrt(d)
    F = W.cfg4_F(d, 3)
    _, ms = oracle.materialize_time_ms(x, F)
    gbs = 8.0 * rows * d / (ms * 1e-3) / 1e9
    out["query_all"] = {"rows": rows, "d": d, "cpu_ms": round(ms, 1), "cpu_GBps_fp32_equiv": round(gbs, 3),
                        "cores": 1, "kind": "port"}
    scale = 16
    eng, keys, off, tgt, X, F4 = rmat_engine(scale, 24, 5, d, 0.15, 1e-5)
    es = torch.cuda.ExternalStream(eng.stream_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(es)
    st = eng.ppr_init()
    e1.record(es)
    e1.synchronize()
    gms = e0.elapsed_time(e1)
    n = 1 << scale
    off_h, tgt_h = off.cpu().numpy(), tgt.cpu().numpy().astype(np.int64)
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(off_h))
    xh = X.cpu().numpy().astype(np.float64)
    eng.close()
    del eng, keys, off, tgt, X
    torch.cuda.empty_cache()
    g = oracle.Graph(n, src, tgt_h, None, True)
    t0 = time.perf_counter()
    oe = oracle.OracleEngine(g, d=d, alpha=0.15, eps=1e-5,
                             factors=(xh, xh, F4, np.eye(d), np.ones(d)))
    cms = (time.perf_counter() - t0) * 1e3
    out["init_propagate"] = {"graph": f"R-MAT scale {scale} ef 24 (arcs={len(tgt_h)}), d={d}, "
                                      "alpha 0.15, eps 1e-5",
                             "gpu_ms": round(gms, 3), "gpu_pushes": st["pushes"],
                             "cpu_ms_incl_engine_build": round(cms, 1),
                             "cpu_pushes": int(oe.stat(5)), "speedup": round(cms / gms, 1),
                             "cores": 1, "kind": "port"}
    return out


# ------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    import torch
    torch.cuda.set_device(local)
    from paper_2306_08967_b200 import workloads as W
    # inputs of the same workload: the cfg-5 graph and insertions (device
    # generation through torch, input preparation only)
    keys, off, tgt, su, sv = W.cfg5_inputs(CFG5_EVENTS)
    del keys, off, tgt
    torch.cuda.empty_cache()
    d, n = 128, 1 << 26
    sig = np.arange(1, d + 1, dtype=np.float64) ** -0.5
    per = split_steps(len(su), args.steps, args.warmup)
    # the same timed insertions as our arm (after its warm-up), bounded by time
    a = per * args.warmup
    res = cfg5_oracle(su, sv, n, d, sig, budget_s=args.cpu_seconds,
                      max_events=min(len(su), a + per * args.steps), first=a)
    res["host"] = host_info()
    out = {"metric": METRIC, "value": res["value"], "unit": "insertions/s", "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
           "data": "synthetic (seeded R-MAT scale 26 + random orthonormal factors, cfg 5)",
           "config": {"workload": WORKLOAD, "events_per_step": per, "parallelism": "single"},
           "cpu_baseline": res,
           "e2e": {"value": res["value"], "unit": "insertions/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "note": "reference arm = fp64 C++ restatement of the reference (oracle/), 1 thread, "
                   "the reference being single-threaded (SPEC.md:285); the reference itself "
                   "needs Eigen3 (absent) and cannot be built here"}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-sub", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ppr-scale", type=int, default=23)
    ap.add_argument("--cfg3-events", type=int, default=4096,
                    help="events per batch-size leg of config 3 (0 = skip)")
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if ws == 0 and args.gpus > 1:
        # not under torchrun: launch N ranks (one process per GPU)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={29500 + os.getpid() % 1000}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if ws and ws != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
