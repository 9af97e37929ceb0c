"""State persistence in the reference's DAMF v1 format (io.cpp:182-264).

The format is parsed / written here independently from the library (the
layout of save_state: magic, version, RunConfig, counters, sigma, X_b, Y_b,
P_X, P_Y, Z_b, r_b as i64 rows, i64 cols and fp64 data in Eigen RowMajor order
-- DenseMatrix is RowMajor, types.hpp:17-18, and write_matrix dumps m.data(),
io.cpp:51-56 -- then the adjacency), so a file the device writes is readable
as the reference's, and a file laid out like the reference's resumes on the
device. The oracle restates save_state / load_state too: files cross between
the two in both directions bit-identically."""
import os
import struct

import numpy as np
import pytest

import oracle
from helpers import gpu_from_oracle, product, rel_frob, sigma_rel
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200.workloads import EventList

pytestmark = pytest.mark.gpu


def read_damf(path):
    b = open(path, "rb").read()
    pos = 0

    def take(fmt):
        nonlocal pos
        v = struct.unpack_from(fmt, b, pos)
        pos += struct.calcsize(fmt)
        return v

    assert b[:4] == b"DAMF"
    pos = 4
    (ver,) = take("<I")
    d, alpha, eps, seed, rc, re_, und, applied, since = take("<qddQdqBQq")
    (k,) = take("<q")
    sig = np.array(take(f"<{k}d"))

    def mat():
        r, c = take("<qq")
        return np.array(take(f"<{r * c}d")).reshape(r, c)  # row-major

    xb, yb, px, py, zb, rb = (mat() for _ in range(6))
    (n,) = take("<q")
    adj = []
    for _ in range(n):
        (c,) = take("<q")
        adj.append([take("<qd") for _ in range(c)])
    assert pos == len(b)
    return dict(ver=ver, d=d, alpha=alpha, eps=eps, undirected=und, applied=applied, since=since,
                sigma=sig, xb=xb, yb=yb, px=px, py=py, zb=zb, rb=rb, adj=adj)


def write_damf(path, st):
    with open(path, "wb") as f:
        f.write(b"DAMF")
        f.write(struct.pack("<I", 1))
        f.write(struct.pack("<qddQdqBQq", st["d"], st["alpha"], st["eps"], 0, 1e8, 50000,
                            st["undirected"], st["applied"], st["since"]))
        f.write(struct.pack("<q", len(st["sigma"])) + np.asarray(st["sigma"], "<f8").tobytes())
        for m in (st["xb"], st["yb"], st["px"], st["py"], st["zb"], st["rb"]):
            m = np.asarray(m, np.float64)
            f.write(struct.pack("<qq", *m.shape) + np.ascontiguousarray(m).tobytes(order="C"))
        f.write(struct.pack("<q", len(st["adj"])))
        for row in st["adj"]:
            f.write(struct.pack("<q", len(row)))
            for v, w in row:
                f.write(struct.pack("<qd", v, w))


def test_save_is_reference_layout_and_round_trips(tmp_path):
    g, ev = oracle.gen_mixed_stream(200, 150, 600, 120, 77)
    oe = oracle.OracleEngine(g, d=12, alpha=0.25, eps=1e-6, seed=77)
    e = gpu_from_oracle(g, oe, d=12, alpha=0.25, eps=1e-6)
    e.apply(ev.slice(0, 60))
    path = str(tmp_path / "state.damf")
    e.save_state(path)
    st = read_damf(path)
    assert st["ver"] == 1 and st["d"] == 12 and st["applied"] == 60
    # base rows exactly: fp32 rows widened, rows written through P^-1 at
    # their fp64 side-table values
    assert np.array_equal(st["xb"], e.get(ge.XB64))
    assert np.array_equal(st["yb"], e.get(ge.YB64))
    assert np.array_equal(st["xb"].astype(np.float32), e.get(ge.XB))
    assert np.array_equal(st["px"], e.get(ge.PX))
    assert np.array_equal(st["zb"], e.get(ge.ZB).astype(np.float64))
    off, ids, _ = e.graph_sets()
    for u in range(e.n):
        assert sorted(v for v, _ in st["adj"][u]) == sorted(ids[off[u]:off[u + 1]].tolist())
    # resume and continue: same results as the engine that never stopped
    e2 = ge.Engine.load_state(path)
    assert e2.diag()["events_applied"] == 60
    assert np.array_equal(e2.get(ge.Z), e.get(ge.Z))
    e.apply(ev.slice(60, 120))
    e2.apply(ev.slice(60, 120))
    wp = rel_frob(product(e2.get(ge.X), e2.get(ge.Y)), product(e.get(ge.X), e.get(ge.Y)))
    print("resumed vs uninterrupted product", wp)
    assert wp <= 1e-6 and sigma_rel(e2.get(ge.SIGMA), e.get(ge.SIGMA)) <= 1e-9


def test_reference_layout_file_resumes_on_device(tmp_path):
    # a file laid out like the reference's save_state, from the oracle's fp64
    # state, resumes on the device and answers the same queries
    g, ev = oracle.gen_mixed_stream(150, 120, 500, 60, 91)
    oe = oracle.OracleEngine(g, d=10, alpha=0.3, eps=1e-7, seed=91)
    oe.apply(ev.slice(0, 40))
    n = oe.dims()[0]
    off, ids, _ = oe.graph_sets()
    st = dict(d=10, alpha=0.3, eps=1e-7, undirected=0, applied=40, since=40,
              sigma=oe.get(oe.SIGMA), xb=oe.get(oe.XB), yb=oe.get(oe.YB), px=oe.get(oe.PX),
              py=oe.get(oe.PY), zb=oe.get(oe.ZB), rb=oe.get(oe.RB),
              adj=[[(int(v), 1.0) for v in ids[off[u]:off[u + 1]]] for u in range(n)])
    path = str(tmp_path / "ref.damf")
    write_damf(path, st)
    e = ge.Engine.load_state(path, node_capacity=64)
    assert e.n == n and e.k == len(st["sigma"])
    zr = rel_frob(e.get(ge.Z).astype(np.float64), oe.get(oe.Z))
    print("loaded Z vs oracle", zr)
    assert zr <= 1e-6
    e.apply(ev.slice(40, 60))
    oe.apply(ev.slice(40, 60))
    wp = rel_frob(product(e.get(ge.X), e.get(ge.Y)), product(oe.get(oe.X), oe.get(oe.Y)))
    print("after 20 more events: product vs oracle", wp)
    assert wp <= 1e-5


def test_non_square_layout_is_row_major(tmp_path):
    # n != k: a transposed or column-major file cannot pass this
    g, ev = oracle.gen_mixed_stream(90, 70, 300, 10, 5)
    oe = oracle.OracleEngine(g, d=6, alpha=0.3, eps=1e-6, seed=5)
    e = gpu_from_oracle(g, oe, d=6, alpha=0.3, eps=1e-6)
    path = str(tmp_path / "s.damf")
    e.save_state(path)
    raw = open(path, "rb").read()
    st = read_damf(path)
    xb = e.get(ge.XB).astype(np.float64)
    assert st["xb"].shape == xb.shape and xb.shape[0] != xb.shape[1]
    # the first row of X_b is the first k doubles of its payload
    i = raw.index(struct.pack("<qq", *xb.shape)) + 16
    assert np.array_equal(np.frombuffer(raw[i:i + 8 * xb.shape[1]], "<f8"), xb[0])


def test_oracle_file_resumes_on_device_bit_identically(tmp_path):
    # the oracle's restatement of save_state (io.cpp:182-219) writes the
    # reference's file; the device loads it: fp32 rows = fp64 rows rounded,
    # P / sigma and the adjacency exactly, and the device's own save_state
    # of that engine loads back into the oracle with the same state
    g, ev = oracle.gen_mixed_stream(160, 130, 520, 50, 13)
    oe = oracle.OracleEngine(g, d=9, alpha=0.2, eps=1e-7, seed=13)
    oe.apply(ev.slice(0, 30))
    path = str(tmp_path / "oracle.damf")
    oe.save_state(path)
    e = ge.Engine.load_state(path, node_capacity=64)
    for which, ow in ((ge.XB, oe.XB), (ge.YB, oe.YB), (ge.ZB, oe.ZB), (ge.RB, oe.RB)):
        assert np.array_equal(e.get(which), oe.get(ow).astype(np.float32)), which
    for which, ow in ((ge.PX, oe.PX), (ge.PY, oe.PY), (ge.SIGMA, oe.SIGMA)):
        assert np.array_equal(e.get(which), oe.get(ow)), which
    off_o, ids_o, deg_o = oe.graph_sets()
    off_g, ids_g, deg_g = e.graph_sets()
    assert np.array_equal(off_o, off_g) and np.array_equal(ids_o, ids_g.astype(np.int64))
    assert np.array_equal(deg_o, deg_g)
    dg = e.diag()
    assert dg["events_applied"] == 30 and dg["events_since_rebase"] == 30
    # device -> file -> oracle
    path2 = str(tmp_path / "device.damf")
    e.save_state(path2)
    o2 = oracle.OracleEngine.load_state(path2)
    # X_b / Y_b round-trip in fp64 (rows fp32 cannot hold sit in the fp64
    # side table); Z_b / r_b are fp32 on the device
    for ow in (oe.XB, oe.YB):
        assert np.array_equal(o2.get(ow), oe.get(ow)), ow
    assert np.array_equal(e.get(ge.XB64), oe.get(oe.XB))
    for which, ow in ((ge.ZB, oe.ZB), (ge.RB, oe.RB)):
        assert np.array_equal(o2.get(ow), e.get(which).astype(np.float64)), which
    assert np.array_equal(o2.get(o2.PX), oe.get(oe.PX))
    off2, ids2, _ = o2.graph_sets()
    assert np.array_equal(off2, off_o) and np.array_equal(np.sort(ids2), np.sort(ids_o))
    # both continue the stream and agree
    e.apply(ev.slice(30, 50))
    oe.apply(ev.slice(30, 50))
    wp = rel_frob(product(e.get(ge.X), e.get(ge.Y)), product(oe.get(oe.X), oe.get(oe.Y)))
    assert wp <= 1e-5, wp
