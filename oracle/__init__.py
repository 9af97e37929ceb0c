"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes wrapper over oracle/build/libdamf_oracle.so, the CPU fp64 restatement
of the DAMF reference (/root/reference/proj/src/*.cpp). Imported only by
tests/, __graft_entry__.smoke() (as the checker) and bench.py's cpu_baseline
/ --impl reference leg. The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DAMF_ORACLE_LIB: another build of the same sources (bench.py's CPU legs compile
# one with -O3 -march=native on the host they time; tests use the portable one)
_LIB_PATH = os.environ.get("DAMF_ORACLE_LIB") or os.path.join(_HERE, "build", "libdamf_oracle.so")
_lib = None

i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"oracle library missing: {_LIB_PATH} (run make)")
        L = C.CDLL(_LIB_PATH)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_engine_create.argtypes = [C.c_int64, C.c_int, C.c_int64, i64p, i64p, f64p,
                                           C.c_int64, C.c_double, C.c_double, C.c_uint64,
                                           C.c_double, C.c_int64, C.POINTER(C.c_void_p)]
        L.oracle_engine_create_from_factors.argtypes = [
            C.c_int64, C.c_int, C.c_int64, i64p, i64p, f64p, C.c_int64, C.c_int64, f64p, f64p,
            f64p, f64p, f64p, C.c_double, C.c_double, C.c_double, C.c_int64,
            C.POINTER(C.c_void_p)]
        L.oracle_engine_destroy.argtypes = [C.c_void_p]
        L.oracle_engine_clone.argtypes = [C.c_void_p]
        L.oracle_engine_clone.restype = C.c_void_p
        L.oracle_engine_apply.argtypes = [C.c_void_p, C.c_int64, i32p, i64p, i64p, f64p, i64p,
                                          i64p, f64p, i64p, i64p, f64p, i64p, f64p]
        L.oracle_engine_dims.argtypes = [C.c_void_p, i64p, i64p, i64p, i64p]
        L.oracle_engine_get.argtypes = [C.c_void_p, C.c_int, f64p]
        L.oracle_engine_stat.argtypes = [C.c_void_p, C.c_int]
        L.oracle_engine_stat.restype = C.c_double
        L.oracle_engine_rebase.argtypes = [C.c_void_p]
        L.oracle_engine_graph.argtypes = [C.c_void_p, f64p, i64p, i64p]
        L.oracle_engine_query.argtypes = [C.c_void_p, C.c_int, C.c_int64, f64p]
        L.oracle_engine_score.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int]
        L.oracle_engine_score.restype = C.c_double
        L.oracle_materialize.argtypes = [f64p, C.c_int64, C.c_int64, f64p, f64p]
        L.oracle_materialize.restype = C.c_double
        L.oracle_edge_update_rowlocal.argtypes = [C.c_int64, C.c_int64, f64p, f64p, f64p, f64p,
                                                  f64p, C.c_double, C.c_int, f64p, f64p, f64p,
                                                  f64p, f64p, i64p]
        L.oracle_edge_update_rowlocal_p.argtypes = [C.c_int64, C.c_int64, f64p, f64p, f64p,
                                                    f64p, f64p, C.c_double, f64p, f64p, f64p,
                                                    f64p, f64p, f64p, f64p, i64p]
        L.oracle_engine_row_log_enable.argtypes = [C.c_void_p, C.c_int]
        L.oracle_engine_set_fp32_base.argtypes = [C.c_void_p, C.c_int]
        L.oracle_engine_row_log.argtypes = [C.c_void_p, i64p, C.c_int64]
        L.oracle_engine_row_log.restype = C.c_int64
        L.oracle_engine_save_state.argtypes = [C.c_void_p, C.c_char_p]
        L.oracle_engine_load_state.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        for fn in ("oracle_gen_mixed_stream", "oracle_gen_random_graph", "oracle_gen_sbm2"):
            getattr(L, fn).restype = C.c_void_p
        L.oracle_gen_mixed_stream.argtypes = [C.c_int64] * 4 + [C.c_uint64]
        L.oracle_gen_random_graph.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_int]
        L.oracle_gen_sbm2.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_uint64]
        L.oracle_stream_destroy.argtypes = [C.c_void_p]
        L.oracle_stream_sizes.argtypes = [C.c_void_p, i64p, i64p, i64p, i64p, i64p]
        L.oracle_stream_graph.argtypes = [C.c_void_p, i64p, i64p, f64p]
        L.oracle_stream_events.argtypes = [C.c_void_p, i32p, i64p, i64p, f64p, i64p, i64p, f64p,
                                           i64p, i64p, f64p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, status, msg, index=-1):
        super().__init__(f"oracle status {status}: {msg} (event {index})")
        self.status = status
        self.index = index


@dataclass
class Events:
    """Flat event batch (same layout as damf_event_batch)."""
    kind: np.ndarray
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray
    in_off: np.ndarray
    in_ids: np.ndarray
    in_w: np.ndarray
    out_off: np.ndarray
    out_ids: np.ndarray
    out_w: np.ndarray

    def __len__(self):
        return len(self.kind)

    def slice(self, a, b):
        io, oo = self.in_off, self.out_off
        return Events(self.kind[a:b].copy(), self.u[a:b].copy(), self.v[a:b].copy(),
                      self.w[a:b].copy(), io[a:b + 1] - io[a], self.in_ids[io[a]:io[b]].copy(),
                      self.in_w[io[a]:io[b]].copy(), oo[a:b + 1] - oo[a],
                      self.out_ids[oo[a]:oo[b]].copy(), self.out_w[oo[a]:oo[b]].copy())

    @staticmethod
    def edges(kind, u, v, w=None):
        m = len(u)
        kind = np.full(m, kind, np.int32) if np.isscalar(kind) else np.asarray(kind, np.int32)
        z = np.zeros(m + 1, np.int64)
        return Events(kind, np.asarray(u, np.int64), np.asarray(v, np.int64),
                      np.ones(m) if w is None else np.asarray(w, np.float64), z,
                      np.zeros(0, np.int64), np.zeros(0), z.copy(), np.zeros(0, np.int64),
                      np.zeros(0))


class Graph:
    """Arc list (src, dst, w) in per-source insertion order + node count."""

    def __init__(self, n, src, dst, w=None, undirected=False):
        self.n = int(n)
        self.src = np.ascontiguousarray(src, np.int64)
        self.dst = np.ascontiguousarray(dst, np.int64)
        self.w = np.ones(len(self.src)) if w is None else np.ascontiguousarray(w, np.float64)
        self.undirected = bool(undirected)

    def csr(self):
        order = np.argsort(self.src, kind="stable")
        off = np.zeros(self.n + 1, np.int64)
        np.add.at(off, self.src + 1, 1)
        return np.cumsum(off), self.dst[order].astype(np.int32), self.w[order]


def _take_stream(h):
    L = lib()
    n, a, e, ni, no = (C.c_int64() for _ in range(5))
    L.oracle_stream_sizes(h, C.byref(n), C.byref(a), C.byref(e), C.byref(ni), C.byref(no))
    src = np.zeros(a.value, np.int64)
    dst = np.zeros(a.value, np.int64)
    w = np.zeros(a.value)
    L.oracle_stream_graph(h, _p(src, i64p), _p(dst, i64p), _p(w, f64p))
    E = e.value
    ev = Events(np.zeros(E, np.int32), np.zeros(E, np.int64), np.zeros(E, np.int64), np.zeros(E),
                np.zeros(E + 1, np.int64), np.zeros(max(ni.value, 1), np.int64),
                np.zeros(max(ni.value, 1)), np.zeros(E + 1, np.int64),
                np.zeros(max(no.value, 1), np.int64), np.zeros(max(no.value, 1)))
    L.oracle_stream_events(h, _p(ev.kind, i32p), _p(ev.u, i64p), _p(ev.v, i64p), _p(ev.w, f64p),
                           _p(ev.in_off, i64p), _p(ev.in_ids, i64p), _p(ev.in_w, f64p),
                           _p(ev.out_off, i64p), _p(ev.out_ids, i64p), _p(ev.out_w, f64p))
    L.oracle_stream_destroy(h)
    return n.value, src, dst, w, ev


def gen_mixed_stream(n_total, n0, m0, n_events, seed):
    """eval.cpp:648-705 (directed graph + mixed event stream)."""
    n, src, dst, w, ev = _take_stream(lib().oracle_gen_mixed_stream(n_total, n0, m0, n_events, seed))
    return Graph(n, src, dst, w, False), ev


def gen_random_graph(n, arcs, seed, undirected=False):
    """eval.cpp:616-631."""
    n, src, dst, w, _ = _take_stream(lib().oracle_gen_random_graph(n, arcs, seed, int(undirected)))
    return Graph(n, src, dst, w, undirected)


class OracleEngine:
    """damf::Engine restated in fp64 (engine.hpp:26-61)."""

    def __init__(self, g: Graph, d, alpha=0.3, eps=1e-5, seed=0, rebase_cond=1e8,
                 rebase_every=50000, factors=None):
        L = lib()
        self.h = C.c_void_p()
        if factors is None:
            st = L.oracle_engine_create(g.n, int(g.undirected), len(g.src), _p(g.src, i64p),
                                        _p(g.dst, i64p), _p(g.w, f64p), d, alpha, eps, seed,
                                        rebase_cond, rebase_every, C.byref(self.h))
        else:
            xb, yb, px, py, sig = (np.ascontiguousarray(x, np.float64) for x in factors)
            k = len(sig)
            st = L.oracle_engine_create_from_factors(
                g.n, int(g.undirected), len(g.src), _p(g.src, i64p), _p(g.dst, i64p),
                _p(g.w, f64p), k, d, _p(xb, f64p), _p(yb, f64p), _p(px, f64p), _p(py, f64p),
                _p(sig, f64p), alpha, eps, rebase_cond, rebase_every, C.byref(self.h))
        if st:
            raise OracleError(st, L.oracle_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_engine_destroy(self.h)
            self.h = None

    def apply(self, ev: Events, lat=False):
        L = lib()
        failed = C.c_int64(-1)
        lat_ms = np.zeros(len(ev)) if lat else None
        st = L.oracle_engine_apply(self.h, len(ev), _p(ev.kind, i32p), _p(ev.u, i64p),
                                   _p(ev.v, i64p), _p(ev.w, f64p), _p(ev.in_off, i64p),
                                   _p(ev.in_ids, i64p), _p(ev.in_w, f64p), _p(ev.out_off, i64p),
                                   _p(ev.out_ids, i64p), _p(ev.out_w, f64p), C.byref(failed),
                                   _p(lat_ms, f64p))
        if st:
            raise OracleError(st, L.oracle_last_error().decode(), failed.value)
        return lat_ms

    def dims(self):
        n, k, a, d = (C.c_int64() for _ in range(4))
        lib().oracle_engine_dims(self.h, C.byref(n), C.byref(k), C.byref(a), C.byref(d))
        return n.value, k.value, a.value, d.value

    def get(self, which):
        n, k, _, _ = self.dims()
        shape = {0: (n, k), 1: (n, k), 2: (k, k), 3: (k, k), 4: (k,), 5: (n, k), 6: (n, k),
                 7: (n, k), 8: (n, k), 9: (n, k)}[which]
        out = np.zeros(shape)
        lib().oracle_engine_get(self.h, which, _p(out, f64p))
        return out

    XB, YB, PX, PY, SIGMA, ZB, RB, X, Y, Z = range(10)

    def stat(self, which):
        return lib().oracle_engine_stat(self.h, which)

    def defect_bound(self):
        return self.stat(0)

    def graph_sets(self):
        n, _, arcs, _ = self.dims()
        deg = np.zeros(n)
        off = np.zeros(n + 1, np.int64)
        ids = np.zeros(max(arcs, 1), np.int64)
        lib().oracle_engine_graph(self.h, _p(deg, f64p), _p(off, i64p), _p(ids, i64p))
        return off, ids[:arcs], deg

    def rebase(self):
        lib().oracle_engine_rebase(self.h)

    def set_fp32_base(self, on=True):
        """The device's storage model: base rows rounded to fp32 at every
        fold (rebase / eager fold), lazily solved rows fp64 until then."""
        lib().oracle_engine_set_fp32_base(self.h, int(on))

    def row_log_enable(self, on=True):
        """Record the row sets of every ProjectionUpdate's dX / dY from now on
        (steps counted from 0 at enable)."""
        lib().oracle_engine_row_log_enable(self.h, int(on))

    def row_log(self):
        n = lib().oracle_engine_row_log(self.h, None, 0)
        out = np.zeros((n, 3), np.int64)
        lib().oracle_engine_row_log(self.h, _p(out, i64p), n)
        return out

    def save_state(self, path):
        """save_state (io.cpp:182-219), restated."""
        st = lib().oracle_engine_save_state(self.h, str(path).encode())
        if st:
            raise OracleError(st, lib().oracle_last_error().decode())

    @classmethod
    def load_state(cls, path):
        """load_state (io.cpp:221-269), restated."""
        self = cls.__new__(cls)
        self.h = C.c_void_p()
        st = lib().oracle_engine_load_state(str(path).encode(), C.byref(self.h))
        if st:
            self.h = None
            raise OracleError(st, lib().oracle_last_error().decode())
        return self

    def score(self, u, v, enhanced=True):
        return lib().oracle_engine_score(self.h, u, v, int(enhanced))


def materialize_time_ms(x, t):
    x = np.ascontiguousarray(x, np.float64)
    t = np.ascontiguousarray(t, np.float64)
    out = np.zeros((x.shape[0], t.shape[1]))
    ms = lib().oracle_materialize(_p(x, f64p), x.shape[0], x.shape[1], _p(t, f64p), _p(out, f64p))
    return out, ms


def edge_update_rowlocal(k, d, xu, yv, px, py, sigma, w):
    """Row-local fp64 oracle for one rank-1 edge update."""
    xu, yv, px, py, sigma = (np.ascontiguousarray(a, np.float64) for a in (xu, yv, px, py, sigma))
    s2 = np.zeros(k + 1)
    F = np.zeros((k + 1) * (k + 1))
    G = np.zeros((k + 1) * (k + 1))
    xn = np.zeros(k + 1)
    yn = np.zeros(k + 1)
    k2 = C.c_int64()
    st = lib().oracle_edge_update_rowlocal(k, d, _p(xu, f64p), _p(yv, f64p), _p(px, f64p),
                                           _p(py, f64p), _p(sigma, f64p), w, 0, _p(s2, f64p),
                                           _p(F, f64p), _p(G, f64p), _p(xn, f64p), _p(yn, f64p),
                                           C.byref(k2))
    if st:
        raise OracleError(st, lib().oracle_last_error().decode())
    k2 = k2.value
    return dict(sigma2=s2[:k2], F=F[:k * k2].reshape(k, k2), G=G[:k * k2].reshape(k, k2),
                xu=xn[:k2], yv=yn[:k2])


def edge_update_rowlocal_p(k, d, xu, yv, px, py, sigma, w):
    """edge_update_rowlocal, also returning the projections after
    apply_update (eager fold possible): current rows = xu @ px, yv @ py."""
    xu, yv, px, py, sigma = (np.ascontiguousarray(a, np.float64) for a in (xu, yv, px, py, sigma))
    s2 = np.zeros(k + 1)
    F = np.zeros((k + 1) * (k + 1))
    G = np.zeros((k + 1) * (k + 1))
    xn = np.zeros(k + 1)
    yn = np.zeros(k + 1)
    pxn = np.zeros((k + 1) * (k + 1))
    pyn = np.zeros((k + 1) * (k + 1))
    k2 = C.c_int64()
    st = lib().oracle_edge_update_rowlocal_p(k, d, _p(xu, f64p), _p(yv, f64p), _p(px, f64p),
                                             _p(py, f64p), _p(sigma, f64p), w, _p(s2, f64p),
                                             _p(F, f64p), _p(G, f64p), _p(xn, f64p), _p(yn, f64p),
                                             _p(pxn, f64p), _p(pyn, f64p), C.byref(k2))
    if st:
        raise OracleError(st, lib().oracle_last_error().decode())
    k2 = k2.value
    return dict(sigma2=s2[:k2], F=F[:k * k2].reshape(k, k2), G=G[:k * k2].reshape(k, k2),
                xu=xn[:k2], yv=yn[:k2], px=pxn[:k2 * k2].reshape(k2, k2),
                py=pyn[:k2 * k2].reshape(k2, k2))
