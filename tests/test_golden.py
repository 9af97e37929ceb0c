"""The committed golden fixtures (tests/golden/, made by make_golden.py) are
reproduced by the fp64 oracle: pins the fixtures the GPU parity tests
(test_gpu_golden.py) compare against to the oracle, itself pinned to the
reference's known-answer tests (test_oracle_kat.py)."""
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name)))


def events(f):
    return oracle.Events(*(f["ev_" + k] for k in ("kind", "u", "v", "w", "in_off", "in_ids", "in_w",
                                                  "out_off", "out_ids", "out_w")))


def graph(f):
    n, off, tgt = int(f["n"]), f["off"], f["tgt"]
    src = np.repeat(np.arange(n), np.diff(off))
    w = f["w"] if "w" in f else None
    return oracle.Graph(n, src, tgt.astype(np.int64), w, bool(int(f.get("undirected", 1))))


@pytest.mark.parametrize("name", ["stream_directed.npz", "stream_undirected.npz"])
def test_oracle_reproduces_stream_fixture(name):
    f = load(name)
    oe = oracle.OracleEngine(graph(f), d=int(f["d"]), alpha=float(f["alpha"]), eps=float(f["eps"]),
                             seed=int(f["seed"]))
    assert np.allclose(oe.get(oe.SIGMA), f["sigma0"], rtol=1e-12, atol=0)
    oe.row_log_enable()
    oe.apply(events(f))
    assert np.array_equal(oe.row_log(), f["rowlog"])
    for key, which in (("x", oe.X), ("y", oe.Y), ("z", oe.Z), ("sigma", oe.SIGMA)):
        got = oe.get(which)
        assert np.abs(got - f[key]).max() <= 1e-12 * max(1.0, np.abs(f[key]).max()), key
    off, ids, deg = oe.graph_sets()
    assert np.array_equal(off, f["g_off"]) and np.array_equal(ids, f["g_ids"])
    assert np.array_equal(deg, f["g_deg"])


def test_oracle_reproduces_init_fixture():
    f = load("init_tsvd.npz")
    n, off, tgt = int(f["n"]), f["off"], f["tgt"]
    g = oracle.Graph(n, np.repeat(np.arange(n), np.diff(off)), tgt.astype(np.int64), None, True)
    oe = oracle.OracleEngine(g, d=int(f["d"]), alpha=1.0, eps=1e-5, seed=int(f["seed"]))
    assert np.allclose(oe.get(oe.SIGMA), f["sigma"], rtol=1e-12, atol=0)
    x, y = oe.get(oe.X), oe.get(oe.Y)
    prod = np.einsum("ij,ij->i", x[f["pi"]], y[f["pj"]])
    assert np.abs(prod - f["prod"]).max() <= 1e-12 * np.abs(f["prod"]).max()


def test_materialize_fixture_is_the_fp64_product():
    f = load("materialize.npz")
    for d in (32, 256):
        assert np.array_equal(f[f"x{d}"].astype(np.float64) @ f[f"f{d}"], f[f"z{d}"])
