"""Python binding of the B200 DAMF hot path (ctypes over include/damf_gpu.h).

`Engine` mirrors damf::Engine (/root/reference/proj/include/damf/engine.hpp:
26-61): apply(events), context/content/enhanced(u), score(u, v), rebase(),
plus query_all-style materialisation and the PPR entry points. Everything
runs in libdamf_gpu.so on the GPU; there is no CPU fallback — importing this
module on a machine without the built library or without a GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdamf_gpu.so")

i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)
f32p = C.POINTER(C.c_float)

# status codes: damf::Error::Kind ordinal + 1 (types.hpp:21-41)
ERROR_KINDS = ["ParseError", "UnknownNode", "DuplicateEdge", "MissingEdge", "ShapeMismatch",
               "ZeroMatrix", "NonFinite", "SingularProjection", "NonConvergence",
               "DegenerateLabels", "KTooLarge", "GraphTooSmall", "TooLarge", "IoError"]
ADD_NODE, ADD_EDGE, REMOVE_EDGE = 0, 1, 2
XB, YB, PX, PY, SIGMA, ZB, RB, X, Y, Z, QX, QY, XB64, YB64 = range(14)
APPLY_GRAPH_AND_PPR_ONLY, APPLY_DEFER_PUSH, APPLY_TIME_EVENTS, APPLY_LOG_ROWS = 1, 2, 4, 8


class DamfError(RuntimeError):
    """Carries the reference's Error::Kind (types.hpp:21-41)."""

    def __init__(self, status, msg, index=-1):
        kind = ERROR_KINDS[status - 1] if 1 <= status <= len(ERROR_KINDS) else (
            "CudaError" if status == 100 else "Unsupported" if status == 101 else str(status))
        super().__init__(f"{kind}: {msg}" + (f" (event {index})" if index >= 0 else ""))
        self.status = status
        self.kind = kind
        self.index = index


class Config(C.Structure):
    _fields_ = [("d", C.c_int64), ("alpha", C.c_double), ("eps", C.c_double),
                ("seed", C.c_uint64), ("rebase_cond", C.c_double), ("rebase_every", C.c_int64),
                ("undirected", C.c_int32), ("flags", C.c_int32), ("node_capacity", C.c_int64),
                ("arc_capacity", C.c_int64)]


class Csr(C.Structure):
    _fields_ = [("n", C.c_int64), ("arcs", C.c_int64), ("offsets", i64p), ("targets", i32p),
                ("weights", f64p)]


class EventBatch(C.Structure):
    # pointer fields as void*: set from integer addresses (cheaper per call
    # than typed ctypes pointers)
    _fields_ = [("count", C.c_int64)] + [(f, C.c_void_p) for f in (
        "kind", "u", "v", "w", "in_off", "in_ids", "in_w", "out_off", "out_ids", "out_w")]


class ApplyStats(C.Structure):
    _fields_ = [("applied", C.c_int64), ("failed_index", C.c_int64),
                ("rank1_updates", C.c_int64), ("rebases", C.c_int64), ("eager_folds", C.c_int64),
                ("push_rounds", C.c_int64), ("pushes", C.c_int64), ("device_ms", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Diag(C.Structure):
    _fields_ = [("n", C.c_int64), ("k", C.c_int64), ("d", C.c_int64), ("arcs", C.c_int64),
                ("events_applied", C.c_int64), ("events_since_rebase", C.c_int64),
                ("cond_estimate", C.c_double), ("proj_row_bound", C.c_double),
                ("total_pushes", C.c_int64), ("device_bytes", C.c_int64),
                ("kernel_launches", C.c_int64), ("last_materialize_ms", C.c_double)]


_lib = None


def lib():
    """Load libdamf_gpu.so; fails loudly when it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built (run `make` or __graft_entry__.build())")
        # DAMF_GPU_LIB: load another build of the same library (A/B timing of kernel variants)
        L = C.CDLL(os.environ.get("DAMF_GPU_LIB", LIB_PATH))
        vp = C.c_void_p
        L.damf_gpu_last_error.restype = C.c_char_p
        L.damf_gpu_last_error.argtypes = [vp]
        L.damf_gpu_version.restype = C.c_char_p
        L.damf_gpu_create_from_factors.argtypes = [C.POINTER(Csr), C.POINTER(Config), C.c_int64,
                                                   f32p, f32p, f64p, f64p, f64p, C.POINTER(vp)]
        L.damf_gpu_create.argtypes = [C.POINTER(Csr), C.POINTER(Config), C.POINTER(vp)]
        L.damf_gpu_destroy.argtypes = [vp]
        L.damf_gpu_sync.argtypes = [vp]
        L.damf_gpu_apply.argtypes = [vp, C.POINTER(EventBatch), C.c_int32, C.POINTER(ApplyStats)]
        L.damf_gpu_apply_edge.argtypes = [vp, C.c_int32, C.c_int64, C.c_int64, C.c_double, C.c_int32,
                                          C.POINTER(ApplyStats)]
        L.damf_gpu_event_latencies.argtypes = [vp, f64p, C.c_int64]
        L.damf_gpu_event_latencies.restype = C.c_int64
        L.damf_gpu_row_log.argtypes = [vp, i64p, C.c_int64]
        L.damf_gpu_row_log.restype = C.c_int64
        L.damf_gpu_query_rows.argtypes = [vp, C.c_int32, i64p, C.c_int64, f32p]
        L.damf_gpu_query_rows64.argtypes = [vp, C.c_int32, i64p, C.c_int64, f64p]
        L.damf_gpu_load_rows.argtypes = [vp, C.c_int32, C.c_int64, C.c_int64, vp]
        L.damf_gpu_score_pairs.argtypes = [vp, i64p, i64p, C.c_int64, C.c_int32, f64p]
        L.damf_gpu_save_state.argtypes = [vp, C.c_char_p]
        L.damf_gpu_load_state.argtypes = [C.c_char_p, C.POINTER(Config), C.POINTER(vp)]
        L.damf_gpu_topk_pairs.argtypes = [vp, i64p, i64p, C.c_int64, C.c_int32, C.c_int64, i64p,
                                          f64p]
        L.damf_gpu_ppr_trace.argtypes = [vp, vp, C.c_int]
        L.damf_gpu_score.argtypes = [vp, C.c_int64, C.c_int64, C.c_int32, f64p]
        L.damf_gpu_materialize.argtypes = [vp, C.c_int32, vp, C.c_int32]
        L.damf_gpu_get_state.argtypes = [vp, C.c_int32, vp]
        L.damf_gpu_get_graph.argtypes = [vp, i64p, i32p, f64p]
        L.damf_gpu_ppr_init.argtypes = [vp, C.POINTER(ApplyStats)]
        L.damf_gpu_ppr_push.argtypes = [vp, C.POINTER(ApplyStats)]
        L.damf_gpu_rebase.argtypes = [vp]
        L.damf_gpu_diagnostics.argtypes = [vp, C.POINTER(Diag)]
        L.damf_gpu_stream.argtypes = [vp]
        L.damf_gpu_stream.restype = C.c_void_p
        L.damf_gpu_push_counters.argtypes = [vp, i64p]
        L.damf_gpu_profile_counters.argtypes = [vp, C.POINTER(C.c_uint64)]
        L.damf_materialize_dev.argtypes = [vp, C.c_int64, C.c_int64, f64p, vp, vp, f32p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


_BATCH_FIELDS = (("kind", np.int32), ("u", np.int64), ("v", np.int64), ("w", np.float64),
                 ("in_off", np.int64), ("in_ids", np.int64), ("in_w", np.float64),
                 ("out_off", np.int64), ("out_ids", np.int64), ("out_w", np.float64))


def make_batch(ev):
    """Build a damf_event_batch from an object with kind/u/v/w/in_*/out_* arrays."""
    arrs = {f: np.ascontiguousarray(getattr(ev, f), t) for f, t in _BATCH_FIELDS}
    b = EventBatch(len(arrs["kind"]), *(arrs[f].__array_interface__["data"][0]
                                        for f, _ in _BATCH_FIELDS))
    return b, arrs  # keep arrs alive while b is used


class Engine:
    """damf::Engine on one B200. Construct from explicit factors
    (FactorState(xb, yb, px, py, sigma, d), factor_state.hpp:22-23)."""

    def __init__(self, n, offsets, targets, weights, d, k, xb, yb, px, py, sigma, alpha=0.3,
                 eps=1e-5, undirected=False, rebase_cond=1e8, rebase_every=50000, seed=0,
                 node_capacity=0, arc_capacity=0):
        L = lib()
        # arrays may be numpy (host) or torch tensors (host or CUDA; device
        # arrays are consumed in place by the library); xb / yb may be None
        keep = []

        def arg(a, np_dtype, ctype, torch_dtype):
            if a is None:
                return ctype()
            if hasattr(a, "data_ptr"):
                import torch
                assert a.is_contiguous() and a.dtype == getattr(torch, torch_dtype), \
                    f"expected contiguous {torch_dtype} tensor"
                keep.append(a)
                return C.cast(C.c_void_p(a.data_ptr()), ctype)
            arr = np.ascontiguousarray(a, np_dtype)
            keep.append(arr)
            return _p(arr, ctype)

        arcs = int(targets.numel() if hasattr(targets, "numel") else len(targets))
        csr = Csr(n, arcs, arg(offsets, np.int64, i64p, "int64"),
                  arg(targets, np.int32, i32p, "int32"),
                  arg(weights, np.float64, f64p, "float64"))
        cfg = Config(d, alpha, eps, seed, rebase_cond, rebase_every, int(undirected), 0,
                     node_capacity, arc_capacity)
        xb_p = arg(xb, np.float32, f32p, "float32")
        yb_p = arg(yb, np.float32, f32p, "float32")
        px = np.ascontiguousarray(px, np.float64)
        py = np.ascontiguousarray(py, np.float64)
        sigma = np.ascontiguousarray(sigma, np.float64)
        self.h = C.c_void_p()
        st = L.damf_gpu_create_from_factors(C.byref(csr), C.byref(cfg), k, xb_p, yb_p,
                                            _p(px, f64p), _p(py, f64p), _p(sigma, f64p),
                                            C.byref(self.h))
        del keep
        if st:
            raise DamfError(st, "create_from_factors failed")
        self.d = d
        self.alpha = alpha

    @classmethod
    def from_graph(cls, n, offsets, targets, weights, d, alpha=0.3, eps=1e-5, undirected=False,
                   rebase_cond=1e8, rebase_every=50000, seed=0, node_capacity=0, arc_capacity=0):
        """Engine(g, cfg) (engine.cpp:5-10): factors from the device randomized
        t-SVD of the snapshot (damf_gpu_create, FactorState::init_from_graph)."""
        L = lib()
        offsets = np.ascontiguousarray(offsets, np.int64)
        targets = np.ascontiguousarray(targets, np.int32)
        weights = None if weights is None else np.ascontiguousarray(weights, np.float64)
        csr = Csr(n, len(targets), _p(offsets, i64p), _p(targets, i32p), _p(weights, f64p))
        cfg = Config(d, alpha, eps, seed, rebase_cond, rebase_every, int(undirected), 0,
                     node_capacity, arc_capacity)
        self = cls.__new__(cls)
        self.h = C.c_void_p()
        st = L.damf_gpu_create(C.byref(csr), C.byref(cfg), C.byref(self.h))
        if st:
            self.h = None
            raise DamfError(st, "damf_gpu_create failed")
        self.d = d
        self.alpha = alpha
        return self

    def save_state(self, path):
        """save_state (io.cpp:182-222): the reference's DAMF v1 binary."""
        self._check(lib().damf_gpu_save_state(self.h, str(path).encode()))

    @classmethod
    def load_state(cls, path, node_capacity=0, arc_capacity=0):
        """load_state (io.cpp:224-264): resume from a DAMF v1 file (ours or the
        reference's)."""
        L = lib()
        sizing = Config(0, 0.0, 0.0, 0, 0.0, 0, 0, 0, node_capacity, arc_capacity)
        self = cls.__new__(cls)
        self.h = C.c_void_p()
        st = L.damf_gpu_load_state(str(path).encode(), C.byref(sizing), C.byref(self.h))
        if st:
            self.h = None
            raise DamfError(st, f"damf_gpu_load_state({path}) failed")
        dg = self.diag()
        self.d = dg["d"]
        return self

    def close(self):
        if getattr(self, "h", None):
            lib().damf_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: module globals already torn down
            pass

    def _check(self, st, index=-1):
        if st:
            raise DamfError(st, lib().damf_gpu_last_error(self.h).decode(), index)

    def apply(self, ev, mode=0):
        b, keep = make_batch(ev)
        s = ApplyStats()
        st = lib().damf_gpu_apply(self.h, C.byref(b), mode, C.byref(s))
        del keep
        self._check(st, s.failed_index)
        return s.as_dict()

    def apply_edge(self, kind, u, v, w=1.0, mode=0):
        """Engine::apply(GraphEvent::add_edge(u, v, w) / remove_edge(u, v)) for
        one event (damf_gpu_apply_edge): no batch arrays to marshal."""
        s = ApplyStats()
        st = lib().damf_gpu_apply_edge(self.h, kind, u, v, w, mode, C.byref(s))
        self._check(st, s.failed_index)
        return s

    def latencies_us(self):
        n = lib().damf_gpu_event_latencies(self.h, None, 0)
        out = np.zeros(n)
        lib().damf_gpu_event_latencies(self.h, _p(out, f64p), n)
        return out

    def row_log(self):
        """(step, side, row) triples of the last apply with APPLY_LOG_ROWS:
        the base rows each rank-1 step modified (side 0 = X_b, 1 = Y_b)."""
        n = lib().damf_gpu_row_log(self.h, None, 0)
        out = np.zeros((n, 3), np.int64)
        lib().damf_gpu_row_log(self.h, _p(out, i64p), n)
        return out

    def diag(self):
        o = Diag()
        self._check(lib().damf_gpu_diagnostics(self.h, C.byref(o)))
        return {f: getattr(o, f) for f, _ in o._fields_}

    @property
    def k(self):
        return self.diag()["k"]

    @property
    def n(self):
        return self.diag()["n"]

    def get(self, which):
        dg = self.diag()
        n, k = dg["n"], dg["k"]
        if which in (XB, YB, ZB, RB, X, Y, Z):
            out = np.zeros((n, k), np.float32)
        elif which in (XB64, YB64):
            out = np.zeros((n, k), np.float64)
        elif which in (PX, PY, QX, QY):
            out = np.zeros((k, k), np.float64)
        else:
            out = np.zeros(k, np.float64)
        self._check(lib().damf_gpu_get_state(self.h, which, out.ctypes.data_as(C.c_void_p)))
        return out

    def load_rows(self, which, row0, rows):
        """Copy rows (m x k fp32; numpy or torch, host or CUDA) into X_b / Y_b
        at row0 (damf_gpu_load_rows)."""
        if hasattr(rows, "data_ptr"):
            assert rows.is_contiguous()
            m, ptr, keep = rows.shape[0], rows.data_ptr(), rows
        else:
            keep = np.ascontiguousarray(rows, np.float32)
            m, ptr = keep.shape[0], keep.ctypes.data
        self._check(lib().damf_gpu_load_rows(self.h, which, row0, m, C.c_void_p(ptr)))
        del keep

    def score_pairs(self, u, v, enhanced=True, symmetric_max=False):
        """pair_score over a batch (eval.cpp:211-215), fp64 scores."""
        u = np.ascontiguousarray(u, np.int64)
        v = np.ascontiguousarray(v, np.int64)
        out = np.zeros(len(u))
        flags = (1 if enhanced else 0) | (2 if symmetric_max else 0)
        self._check(lib().damf_gpu_score_pairs(self.h, _p(u, i64p), _p(v, i64p), len(u), flags,
                                               _p(out, f64p)))
        return out

    def topk_pairs(self, u, v, K, enhanced=True, symmetric_max=False):
        """Indices and scores of the K best pairs (score desc, index asc),
        run_graph_reconstruction's order (eval.cpp:336-371)."""
        u = np.ascontiguousarray(u, np.int64)
        v = np.ascontiguousarray(v, np.int64)
        kk = min(K, len(u))
        idx = np.zeros(kk, np.int64)
        sc = np.zeros(kk)
        flags = (1 if enhanced else 0) | (2 if symmetric_max else 0)
        self._check(lib().damf_gpu_topk_pairs(self.h, _p(u, i64p), _p(v, i64p), len(u), flags, K,
                                              _p(idx, i64p), _p(sc, f64p)))
        return idx, sc

    def query(self, which, ids):
        ids = np.ascontiguousarray(ids, np.int64)
        out = np.zeros((len(ids), self.k), np.float32)
        self._check(lib().damf_gpu_query_rows(self.h, which, _p(ids, i64p), len(ids), _p(out, f32p)))
        return out

    def query64(self, which, ids):
        """Exact base rows (XB or YB) in fp64, side-table aware."""
        ids = np.ascontiguousarray(ids, np.int64)
        out = np.zeros((len(ids), self.k), np.float64)
        self._check(lib().damf_gpu_query_rows64(self.h, which, _p(ids, i64p), len(ids), _p(out, f64p)))
        return out

    def context(self, u):
        return self.query(X, [u])[0]

    def content(self, u):
        return self.query(Y, [u])[0]

    def enhanced(self, u):
        return self.query(Z, [u])[0]

    def score(self, u, v, enhanced=True):
        out = C.c_double()
        self._check(lib().damf_gpu_score(self.h, u, v, int(enhanced), C.byref(out)))
        return out.value

    def materialize(self, which=X, dst_ptr=None, on_device=False):
        """FactorState::query_all (factor_state.cpp:120-123). Without dst_ptr
        returns a host array; with dst_ptr (int, n x k fp32) writes there
        (device memory when on_device)."""
        if dst_ptr is None:
            return self.get(which)
        self._check(lib().damf_gpu_materialize(self.h, which, C.c_void_p(dst_ptr), int(on_device)))

    def graph_sets(self):
        n = self.n
        arcs = self.diag()["arcs"]
        off = np.zeros(n + 1, np.int64)
        ids = np.zeros(max(arcs, 1), np.int32)
        deg = np.zeros(n)
        self._check(lib().damf_gpu_get_graph(self.h, _p(off, i64p), _p(ids, i32p), _p(deg, f64p)))
        return off, ids[:arcs], deg

    def ppr_init(self):
        s = ApplyStats()
        self._check(lib().damf_gpu_ppr_init(self.h, C.byref(s)))
        return s.as_dict()

    def ppr_push(self):
        s = ApplyStats()
        self._check(lib().damf_gpu_ppr_push(self.h, C.byref(s)))
        return s.as_dict()

    def rebase(self):
        self._check(lib().damf_gpu_rebase(self.h))

    def push_counters(self):
        out = np.zeros(4, np.int64)
        self._check(lib().damf_gpu_push_counters(self.h, _p(out, i64p)))
        return dict(frontier=int(out[0]), affected=int(out[1]), affected_arcs=int(out[2]),
                    pulled_arcs=int(out[3]))

    def profile_counters(self):
        out = np.zeros(128, np.uint64)
        self._check(lib().damf_gpu_profile_counters(self.h, out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out

    def stream_ptr(self):
        return lib().damf_gpu_stream(self.h)

    def sync(self):
        self._check(lib().damf_gpu_sync(self.h))


def materialize_dev(x_ptr, n, d, F, z_ptr, stream=None):
    """Standalone Z = X F on device buffers (pointers as ints). Returns ms."""
    F = np.ascontiguousarray(F, np.float64)
    ms = C.c_float()
    st = lib().damf_materialize_dev(C.c_void_p(x_ptr), n, d, _p(F, f64p), C.c_void_p(z_ptr),
                                    C.c_void_p(stream) if stream else None, C.byref(ms))
    if st:
        raise DamfError(st, "damf_materialize_dev failed")
    return ms.value
