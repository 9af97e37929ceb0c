"""Shared test helpers: build GPU engines from the same inputs the oracle
gets, and sign-invariant comparison metrics (SURVEY.md 8(d) tolerances)."""
import numpy as np

import oracle
from paper_2306_08967_b200 import engine as ge


def graph_csr(g: "oracle.Graph"):
    off, tgt, w = g.csr()
    return off, tgt, (None if np.all(w == 1.0) else w)


def gpu_from_oracle(g, oe, d, alpha, eps, **kw):
    """GPU engine started from the oracle's (fp64) state cast to fp32
    (SURVEY hard part 4: start from the oracle's factors)."""
    off, tgt, w = graph_csr(g)
    k = oe.dims()[1]
    return ge.Engine(g.n, off, tgt, w, d, k, oe.get(oe.XB).astype(np.float32),
                     oe.get(oe.YB).astype(np.float32), oe.get(oe.PX), oe.get(oe.PY),
                     oe.get(oe.SIGMA), alpha=alpha, eps=eps, undirected=g.undirected, **kw)


def gpu_from_factors(n, off, tgt, d, xb, yb, px, py, sig, alpha=1.0, eps=1e-5, undirected=False,
                     **kw):
    k = len(sig)
    return ge.Engine(n, off, tgt, None, d, k, np.asarray(xb, np.float32),
                     np.asarray(yb, np.float32), px, py, sig, alpha=alpha, eps=eps,
                     undirected=undirected, **kw)


def rel_frob(a, b):
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / den if den else np.linalg.norm(a)


def product(x, y):
    return np.asarray(x, np.float64) @ np.asarray(y, np.float64).T


def sampled_product_rel(xa, ya, xb, yb, m=20000, seed=0):
    """Relative Frobenius distance of X Y^T on sampled entries (sign-invariant)."""
    rng = np.random.default_rng(seed)
    n = xa.shape[0]
    i = rng.integers(0, n, m)
    j = rng.integers(0, n, m)
    pa = np.einsum("ij,ij->i", np.asarray(xa[i], np.float64), np.asarray(ya[j], np.float64))
    pb = np.einsum("ij,ij->i", np.asarray(xb[i], np.float64), np.asarray(yb[j], np.float64))
    return np.linalg.norm(pa - pb) / max(np.linalg.norm(pb), 1e-300)


def sigma_rel(a, b):
    k = max(len(a), len(b))
    aa = np.zeros(k)
    bb = np.zeros(k)
    aa[:len(a)] = a
    bb[:len(b)] = b
    return np.linalg.norm(aa - bb) / np.linalg.norm(bb)


def dense_defect(n, off, tgt, deg, x, z, alpha):
    """max_u |alpha X + (1-alpha) D^-1 A Z - Z|_inf[u] / max(deg u, 1)
    (eval.cpp:591-610) in fp64, current coordinates."""
    x = np.asarray(x, np.float64)
    z = np.asarray(z, np.float64)
    worst = 0.0
    for u in range(n):
        dfc = alpha * x[u] - z[u]
        if deg[u] > 0:
            nb = z[tgt[off[u]:off[u + 1]]].sum(0)
            dfc = dfc + (1 - alpha) / deg[u] * nb
        worst = max(worst, np.abs(dfc).max() / max(deg[u], 1.0))
    return worst


def sorted_rowlog(log):
    """(step, side, row) triples in lexicographic order: the per-step dX / dY
    row SETS (the write order inside a step is not part of the contract)."""
    log = np.asarray(log, np.int64).reshape(-1, 3)
    return log[np.lexsort((log[:, 2], log[:, 1], log[:, 0]))]


def assert_rowlog_equal(dev, ora, what=""):
    a, b = sorted_rowlog(dev), sorted_rowlog(ora)
    if not np.array_equal(a, b):
        sa = {tuple(r) for r in a.tolist()}
        sb = {tuple(r) for r in b.tolist()}
        raise AssertionError(f"{what} modified-row sets differ: device-only {sorted(sa - sb)[:8]}, "
                             f"oracle-only {sorted(sb - sa)[:8]} ({len(a)} vs {len(b)} rows)")


def weighted_defect(n, off, tgt, w, deg, x, z, alpha):
    """dense_defect_bound (eval.cpp:591-610) with arc weights: per row
    |alpha X + (1-alpha)/deg sum_v w_uv Z[v] - Z|_inf / max(deg, 1), fp64."""
    import scipy.sparse as sp
    x = np.asarray(x, np.float64)
    z = np.asarray(z, np.float64)
    src = np.repeat(np.arange(n), np.diff(off))
    A = sp.csr_matrix((np.ones(len(tgt)) if w is None else np.asarray(w, np.float64),
                       (src, np.asarray(tgt, np.int64))), shape=(n, n))
    dfc = alpha * x - z
    nz = deg > 0
    dfc[nz] += ((1 - alpha) / deg[nz])[:, None] * (A @ z)[nz]
    return (np.abs(dfc).max(1) / np.maximum(deg, 1.0)).max()
