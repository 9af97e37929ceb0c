"""Generates the committed golden fixtures under tests/golden/ (run from the
repo root: `python tests/golden/make_golden.py`).

The reference (proj/, C++17 + Eigen3) cannot be built here (SURVEY.md 8(c):
no Eigen3, no vendored CLI11/doctest), so the expected outputs come from the
fp64 restatement in oracle/, which is pinned to the reference's own
known-answer tests (tests/oracle_kat.cpp: the doctest suite's cases, seeds and
tolerances). Each fixture holds the INPUTS the device path needs (graph, the
oracle's initial factors, the event stream) and the oracle's OUTPUTS, so the
GPU tests (tests/test_gpu_golden.py) need neither the oracle nor the
reference at run time, and tests/test_golden.py checks that the oracle still
reproduces them.

Fixtures
  stream_directed.npz   eval.cpp:648-705 mixed stream (directed; node adds,
                        edge adds, removals), d = 12, alpha = 0.3, eps 1e-6;
                        stream fixtures also hold `rowlog`, the (step, side,
                        row) triples of every ProjectionUpdate's dX / dY
                        (types.hpp:101-116)
  stream_undirected.npz random undirected graph (eval.cpp:616-631) + edge
                        insertions / removals, d = 16, alpha = 0.15, eps 1e-5
  init_tsvd.npz         FactorState::init_from_graph (svd.cpp:47-96) sigma and
                        6,000 sampled entries of X Y^T on a 400-node random
                        graph, d = 24
  materialize.npz       Z = X F (factor_state.cpp:120-123), d = 32 and 256
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def events_dict(ev, prefix="ev_"):
    return {prefix + f: getattr(ev, f) for f in ("kind", "u", "v", "w", "in_off", "in_ids", "in_w",
                                                 "out_off", "out_ids", "out_w")}


def stream_fixture(name, g, ev, d, alpha, eps, seed):
    oe = oracle.OracleEngine(g, d=d, alpha=alpha, eps=eps, seed=seed)
    off, tgt, w = g.csr()
    init = {"xb0": oe.get(oe.XB), "yb0": oe.get(oe.YB), "px0": oe.get(oe.PX), "py0": oe.get(oe.PY),
            "sigma0": oe.get(oe.SIGMA)}
    oe.row_log_enable()  # the dX / dY row sets of every rank-1 step
    oe.apply(ev)
    off1, ids1, deg1 = oe.graph_sets()
    np.savez_compressed(
        os.path.join(OUT, name), n=g.n, off=off, tgt=tgt, w=w, undirected=int(g.undirected), d=d,
        alpha=alpha, eps=eps, seed=seed, **init, **events_dict(ev),
        x=oe.get(oe.X), y=oe.get(oe.Y), z=oe.get(oe.Z), sigma=oe.get(oe.SIGMA),
        g_off=off1, g_ids=ids1, g_deg=deg1, rowlog=oe.row_log())


def main():
    g, ev = oracle.gen_mixed_stream(220, 160, 900, 160, 7)
    stream_fixture("stream_directed.npz", g, ev, 12, 0.3, 1e-6, 7)

    g = oracle.gen_random_graph(300, 1800, 11, undirected=True)
    rng = np.random.default_rng(11)
    off, tgt, _ = g.csr()
    us, vs, kinds, have = [], [], [], set(zip(g.src.tolist(), g.dst.tolist()))
    while len(us) < 120:
        a, b = (int(x) for x in rng.integers(0, g.n, 2))
        if a == b:
            continue
        if (a, b) in have:
            kinds.append(2)  # REMOVE_EDGE
            have.discard((a, b))
            have.discard((b, a))
        else:
            kinds.append(1)  # ADD_EDGE
            have.add((a, b))
            have.add((b, a))
        us.append(a)
        vs.append(b)
    ev = oracle.Events.edges(np.array(kinds, np.int32), us, vs)
    stream_fixture("stream_undirected.npz", g, ev, 16, 0.15, 1e-5, 11)

    g = oracle.gen_random_graph(400, 3000, 5, undirected=True)
    oe = oracle.OracleEngine(g, d=24, alpha=1.0, eps=1e-5, seed=5)
    off, tgt, w = g.csr()
    pr = np.random.default_rng(5)
    pi, pj = pr.integers(0, g.n, 6000), pr.integers(0, g.n, 6000)
    x, y = oe.get(oe.X), oe.get(oe.Y)
    np.savez_compressed(os.path.join(OUT, "init_tsvd.npz"), n=g.n, off=off, tgt=tgt, d=24, seed=5,
                        sigma=oe.get(oe.SIGMA), pi=pi, pj=pj,
                        prod=np.einsum("ij,ij->i", x[pi], y[pj]))

    rng = np.random.default_rng(3)
    mats = {}
    for d, n in ((32, 400), (256, 130)):
        x = (rng.standard_normal((n, d)) / np.sqrt(d)).astype(np.float32)
        q, _ = np.linalg.qr(rng.standard_normal((d, d)))
        f = q * rng.uniform(0.5, 2.0, d)[None, :]
        mats[f"x{d}"], mats[f"f{d}"], mats[f"z{d}"] = x, f, x.astype(np.float64) @ f
    np.savez_compressed(os.path.join(OUT, "materialize.npz"), **mats)


if __name__ == "__main__":
    main()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)), "bytes")
