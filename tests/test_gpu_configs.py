"""Parity on the BASELINE configurations.

cfg 1 and a scaled cfg 3 run the full fp64 oracle beside the device on the
same seeded inputs; cfg 5 (and a small replica of its construction) is
checked with the row-local oracle: before each insertion the touched base
rows, P_X, P_Y and sigma are read back, the two rank-1 updates are replayed
in fp64 (oracle.edge_update_rowlocal_p, update_engine.cpp:144-204 +
factor_state.cpp:158-213), and the device state after the event is compared
in current coordinates (sign-invariant products)."""
import numpy as np
import pytest

import oracle
from helpers import (assert_rowlog_equal, gpu_from_oracle, product, rel_frob,
                     sampled_product_rel, sigma_rel)
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W

pytestmark = pytest.mark.gpu


def z_star(n, off, ids, deg, x, alpha, iters=400):
    """Tight fixed point of Z = alpha X + (1-alpha) D^-1 A Z (Jacobi, fp64)."""
    import scipy.sparse as sp
    src = np.repeat(np.arange(n), np.diff(off))
    A = sp.csr_matrix((np.ones(len(ids)), (src, ids.astype(np.int64))), shape=(n, n))
    dinv = 1.0 / np.maximum(deg, 1.0)
    z = alpha * x
    for _ in range(iters):
        z = alpha * x + (1 - alpha) * (dinv[:, None] * (A @ z))
    return z


def defect_rows(n, off, ids, deg, x, z, alpha):
    import scipy.sparse as sp
    src = np.repeat(np.arange(n), np.diff(off))
    A = sp.csr_matrix((np.ones(len(ids)), (src, ids.astype(np.int64))), shape=(n, n))
    dfc = alpha * x - z + (1 - alpha) * (1.0 / np.maximum(deg, 1.0))[:, None] * (A @ z)
    return np.abs(dfc).max(1) / np.maximum(deg, 1.0)


def ppr_gates(e, oe, alpha, eps, what):
    """The PPR contract on a device engine vs the oracle on the same stream:
    the reference's defect bound (eval.cpp:591-610, checked densely) and the
    distance to a tight fixed point no worse than 1.5x the oracle's FIFO push
    (SURVEY 8(d) secondary gate; both in current coordinates)."""
    import torch
    off, ids, deg = e.graph_sets()
    n = e.n
    x = e.get(ge.X).astype(np.float64)
    zg = e.get(ge.Z).astype(np.float64)
    d_rows = defect_rows(n, off, ids, deg, x, zg, alpha)
    print(f"{what}: defect {d_rows.max():.3e} (bound {eps * (1 + 1e-6):.3e})")
    assert d_rows.max() <= eps * (1 + 1e-6) + 2e-7

    def zstar(xx):
        src = torch.as_tensor(np.repeat(np.arange(n), np.diff(off)), device="cuda")
        A = torch.sparse_coo_tensor(torch.stack([src, torch.as_tensor(ids.astype(np.int64), device="cuda")]),
                                    torch.ones(len(ids), dtype=torch.float64, device="cuda"),
                                    (n, n)).to_sparse_csr()
        dinv = (1.0 / torch.clamp(torch.as_tensor(deg, device="cuda"), min=1.0))[:, None]
        xt = torch.as_tensor(xx, device="cuda")
        z = alpha * xt
        for _ in range(250):  # (1 - alpha)^250 < 1e-17 at alpha = 0.15
            z = alpha * xt + (1 - alpha) * dinv * (A @ z)
        return z.cpu().numpy()
    zs = zstar(x)
    err_g = np.linalg.norm(zg - zs)
    err_o = np.linalg.norm(oe.get(oe.Z) - zstar(oe.get(oe.X)))
    print(f"{what}: |Z-Z*| gpu {err_g:.3e} oracle {err_o:.3e} (|Z*| {np.linalg.norm(zs):.3e})")
    assert err_g <= 1.5 * err_o + 1e-6 * np.linalg.norm(zs)


def stream_vs_oracle(e, oe, stream, chunk, what, log_rows=True):
    """Apply `stream` to both engines in chunks (one device call per chunk):
    sampled products and sigma after every chunk, the modified-row sets of
    every rank-1 step bit-exact. Returns (worst product, worst sigma, rows)."""
    worst_p = worst_s = 0.0
    rows = 0
    for a in range(0, len(stream), chunk):
        part = stream.slice(a, min(len(stream), a + chunk))
        if log_rows:
            oe.row_log_enable()
        oe.apply(part)
        st = e.apply(part, mode=ge.APPLY_LOG_ROWS if log_rows else 0)
        assert st["applied"] == len(part)
        if log_rows:
            assert_rowlog_equal(e.row_log(), oe.row_log(), f"{what} events {a}..")
            rows += len(oe.row_log())
        worst_p = max(worst_p, sampled_product_rel(e.get(ge.X), e.get(ge.Y),
                                                   oe.get(oe.X), oe.get(oe.Y), seed=a))
        worst_s = max(worst_s, sigma_rel(e.get(ge.SIGMA), oe.get(oe.SIGMA)))
    print(f"{what}: {len(stream)} events, worst sampled product {worst_p:.3e}, "
          f"worst sigma {worst_s:.3e}, {rows} modified rows compared")
    return worst_p, worst_s, rows


def test_cfg1_full_stream_matches_oracle():
    # cfg 1: BA n = 10,000, m = 5, half the edges factorised (reference t-SVD,
    # d = 32), ALL ~25k remaining edges streamed as single-edge insertions;
    # PPR alpha 0.15, eps 1e-4.
    w = W.cfg1()
    eu, ev = w["init"]
    g = oracle.Graph(w["n"], np.concatenate([eu, ev]), np.concatenate([ev, eu]), None, True)
    oe = oracle.OracleEngine(g, d=32, alpha=w["alpha"], eps=w["eps"], seed=0)
    e = gpu_from_oracle(g, oe, d=32, alpha=w["alpha"], eps=w["eps"])
    wp, ws, rows = stream_vs_oracle(e, oe, w["stream"], 2500, "cfg1")
    assert len(w["stream"]) > 24_000 and rows >= 4 * len(w["stream"])
    assert wp <= 1e-4 and ws <= 1e-6
    # bookkeeping bit-exact
    off_o, ids_o, deg_o = oe.graph_sets()
    off_g, ids_g, deg_g = e.graph_sets()
    assert np.array_equal(off_o, off_g) and np.array_equal(deg_o, deg_g)
    assert np.array_equal(ids_o, ids_g.astype(np.int64))
    assert e.diag()["events_applied"] == len(w["stream"])
    ppr_gates(e, oe, w["alpha"], w["eps"], "cfg1")


def test_cfg2_stream_matches_oracle():
    # cfg 2 (the SBM stream of the bench's sub-benchmark): oracle Engine(g, cfg)
    # (the reference's own t-SVD init + init_propagate), the device started
    # from the oracle's factors, then the first 1,200 stream events --
    # inserts, deletions of live edges and node additions with 10 edges each.
    w = W.cfg2()
    n = w["n"]
    eu, ev = w["init"]
    g = oracle.Graph(n, np.concatenate([eu, ev]), np.concatenate([ev, eu]), None, True)
    oe = oracle.OracleEngine(g, d=w["d"], alpha=w["alpha"], eps=w["eps"], seed=0)
    e = gpu_from_oracle(g, oe, d=w["d"], alpha=w["alpha"], eps=w["eps"], node_capacity=1024)
    stream = w["stream"].slice(0, 1200)
    kinds = np.bincount(stream.kind, minlength=3)
    print("cfg2 events by kind (node, add, remove):", kinds.tolist())
    assert kinds.min() > 0
    wp, ws, rows = stream_vs_oracle(e, oe, stream, 300, "cfg2")
    assert wp <= 1e-4 and ws <= 1e-6
    off_o, ids_o, deg_o = oe.graph_sets()
    off_g, ids_g, deg_g = e.graph_sets()
    assert e.n == n + kinds[0]
    assert np.array_equal(off_o, off_g) and np.array_equal(deg_o, deg_g)
    assert np.array_equal(ids_o, ids_g.astype(np.int64))
    ppr_gates(e, oe, w["alpha"], w["eps"], "cfg2")


@pytest.mark.parametrize("batch", [1, 64, 1024])
def test_cfg3_shape_batches_match_oracle(batch):
    # cfg 3 scaled to R-MAT scale 13 (same a/b/c/d, ef 16), d = 64, alpha = 1:
    # held-out edges inserted in batches of 1 / 64 / 1024, sequential inside.
    scale, d = 13, 64
    n = 1 << scale
    u, v = W.rmat_edges(scale, 16, 2)
    rng = np.random.default_rng(2)
    held = rng.permutation(len(u))[:2048]
    keep = np.ones(len(u), bool)
    keep[held] = False
    g = oracle.Graph(n, np.concatenate([u[keep], v[keep]]), np.concatenate([v[keep], u[keep]]),
                     None, True)
    oe = oracle.OracleEngine(g, d=d, alpha=1.0, seed=2)
    e = gpu_from_oracle(g, oe, d=d, alpha=1.0, eps=1e-5)
    stream = W.EventList.edges(ge.ADD_EDGE, u[held], v[held])
    m = 2048 if batch > 1 else 256
    for a in range(0, m, batch):
        part = stream.slice(a, min(m, a + batch))
        oe.apply(part)
        e.apply(part)
    wp = rel_frob(product(e.get(ge.X), e.get(ge.Y)), product(oe.get(oe.X), oe.get(oe.Y)))
    ws = sigma_rel(e.get(ge.SIGMA), oe.get(oe.SIGMA))
    print(f"cfg3-shape batch {batch}: product {wp:.3e} sigma {ws:.3e}")
    assert wp <= 1e-4 and ws <= 1e-6
    off_o, ids_o, deg_o = oe.graph_sets()
    off_g, ids_g, deg_g = e.graph_sets()
    assert np.array_equal(off_o, off_g) and np.array_equal(ids_o, ids_g.astype(np.int64))


def rowlocal_insert_check(e, u, v, sample, d):
    """Replay one undirected insertion (two rank-1 updates) in the fp64
    row-local oracle from the device's pre-state, apply it on the device and
    return (product rel. error over rows {u,v} + sample, sigma rel. error)."""
    k = e.k
    px, py, sig = e.get(ge.PX), e.get(ge.PY), e.get(ge.SIGMA)
    rows = np.concatenate([[u, v], sample]).astype(np.int64)
    xb = e.query64(ge.XB, rows)
    yb = e.query64(ge.YB, rows)
    # step 1: b = e_u, c = e_v ; step 2: b = e_v, c = e_u (graph.cpp:95-108)
    r1 = oracle.edge_update_rowlocal_p(k, d, xb[0], yb[1], px, py, sig, 1.0)
    # base rows after step 1 in the coordinates of r1["px"]: untouched rows
    # keep their current coordinates X_cur = X_b P_old F
    P1x, P1y = px @ r1["F"], py @ r1["G"]
    xv_cur = xb[1] @ P1x          # X[v] current (unchanged by step 1)
    yu_cur = yb[0] @ P1y          # Y[u] current
    xv1 = xv_cur @ np.linalg.inv(r1["px"])
    yu1 = yu_cur @ np.linalg.inv(r1["py"])
    r2 = oracle.edge_update_rowlocal_p(len(r1["sigma2"]), d, xv1, yu1, r1["px"], r1["py"],
                                       r1["sigma2"], 1.0)
    # oracle current rows after both steps
    Xo = (xb @ px) @ r1["F"] @ r2["F"]
    Yo = (yb @ py) @ r1["G"] @ r2["G"]
    Xo[0] = r1["xu"] @ r1["px"] @ r2["F"]          # X[u] after step 1, carried by step 2
    Xo[1] = r2["xu"] @ r2["px"]                    # X[v] after step 2
    Yo[1] = r1["yv"] @ r1["py"] @ r2["G"]          # Y[v] after step 1
    Yo[0] = r2["yv"] @ r2["py"]                    # Y[u] after step 2
    e.apply(W.EventList.edges(ge.ADD_EDGE, [u], [v]))
    Xg = e.query(ge.X, rows).astype(np.float64)
    Yg = e.query(ge.Y, rows).astype(np.float64)
    return rel_frob(Xg @ Yg.T, Xo @ Yo.T), sigma_rel(e.get(ge.SIGMA), r2["sigma2"])


def cfg5_like(scale, d, n_events, seed):
    import torch
    n = 1 << scale
    keys = W.rmat_keys_device(scale, 16, seed)
    off, tgt = W.csr_from_keys_device(n, keys)
    su, sv = W.degree_proportional_inserts(keys, tgt, n_events, seed=seed)
    del keys
    torch.cuda.empty_cache()  # the engine allocates with cudaMalloc
    sig = np.arange(1, d + 1, dtype=np.float64) ** -0.5
    e = ge.Engine(n, off, tgt, None, d, d, None, None, np.eye(d), np.eye(d), sig, alpha=1.0,
                  undirected=True, node_capacity=1024, arc_capacity=1 << 22)
    del off, tgt
    torch.cuda.empty_cache()
    W.orthonormal_rows_into(e, ge.XB, n, d, sig, seed=10 * seed)
    W.orthonormal_rows_into(e, ge.YB, n, d, sig, seed=10 * seed + 1)
    return e, su, sv


def run_rowlocal(e, su, sv, d, n_check, seed):
    rng = np.random.default_rng(seed)
    worst_p = worst_s = 0.0
    for i in range(n_check):
        sample = rng.integers(0, e.n, 62)
        sample = sample[(sample != su[i]) & (sample != sv[i])]
        wp, ws = rowlocal_insert_check(e, int(su[i]), int(sv[i]), sample, d)
        if i % 20 == 0:
            dg = e.diag()
            print(f"  event {i}: ({su[i]}, {sv[i]}) product {wp:.2e} sigma {ws:.2e} "
                  f"cond {dg['cond_estimate']:.3e} since rebase {dg['events_since_rebase']}")
        worst_p, worst_s = max(worst_p, wp), max(worst_s, ws)
    return worst_p, worst_s


def test_rowlocal_small_replica_of_cfg5():
    e, su, sv = cfg5_like(16, 128, 24, seed=7)
    wp, ws = run_rowlocal(e, su, sv, 128, 24, 7)
    print("cfg5-replica row-local: product", wp, "sigma", ws)
    e.close()
    # from identical pre-states the device matches the fp64 update to the fp32
    # read-out of the rows (~4e-8), far inside the 1e-4 contract
    assert wp <= 1e-5 and ws <= 1e-9


def test_cfg5_rowlocal_at_scale():
    import gc
    import torch
    gc.collect()
    torch.cuda.empty_cache()
    free, total = torch.cuda.mem_get_info()
    if total < 150e9:
        pytest.skip("config 5 needs ~120 GB of device memory")
    # every insertion of the transient (cond(P) up to 1e8, rebases) and beyond
    e, su, sv = cfg5_like(26, 128, 120, seed=4)
    wp, ws = run_rowlocal(e, su, sv, 128, 120, 4)
    print("cfg5 row-local: product", wp, "sigma", ws)
    e.close()
    assert wp <= 1e-5 and ws <= 1e-9


@pytest.mark.parametrize("k", [64, 128, 256])
def test_rebase_fold_is_fp64_accurate(k):
    # rebase X_b <- X_b P_X with cond(P) = 1e6 (factor_state.cpp:215-222): the
    # fold must keep fp32 storage accuracy (fp64 products on the tensor cores)
    rng = np.random.default_rng(k)
    n = 20_000
    xb = rng.standard_normal((n, k)).astype(np.float32)
    U, _ = np.linalg.qr(rng.standard_normal((k, k)))
    V, _ = np.linalg.qr(rng.standard_normal((k, k)))
    P = U @ np.diag(np.logspace(0, -6, k)) @ V.T
    off = np.zeros(n + 1, np.int64)
    e = ge.Engine(n, off, np.zeros(0, np.int32), None, k, k, xb, xb, P, P,
                  np.linspace(2, 1, k), alpha=1.0, eps=1e-5)
    truth = xb.astype(np.float64) @ P
    e.rebase()
    got = e.get(ge.XB).astype(np.float64)
    err = np.abs(got - truth).max(1) / np.maximum(np.abs(truth).max(1), 1e-30)
    print(f"k={k}: worst row rel err {err.max():.2e}")
    assert err.max() <= 5e-6


@pytest.mark.parametrize("case", ["small", "cfg1"])
def test_device_tsvd_init_matches_oracle(case):
    # Engine(g, cfg) on the device vs the oracle's FactorState::init_from_graph
    # (same seed, same Gaussian stream): sigma and the factor products agree.
    if case == "small":
        g = oracle.gen_random_graph(300, 1500, 21)          # min_dim <= 600: exact path
        d, n = 16, 300
    else:
        w = W.cfg1()
        eu, ev = w["init"]
        n, d = w["n"], 32
        g = oracle.Graph(n, np.concatenate([eu, ev]), np.concatenate([ev, eu]), None, True)
    oe = oracle.OracleEngine(g, d=d, alpha=1.0, seed=5)
    off, tgt, wts = g.csr()
    e = ge.Engine.from_graph(n, off, tgt, None if np.all(wts == 1.0) else wts, d, alpha=1.0,
                             undirected=g.undirected, seed=5)
    so, sg = oe.get(oe.SIGMA), e.get(ge.SIGMA)
    print(case, "k", len(so), len(sg), "sigma rel", sigma_rel(sg, so))
    assert len(so) == len(sg)
    assert sigma_rel(sg, so) <= 1e-6
    wp = sampled_product_rel(e.get(ge.X), e.get(ge.Y), oe.get(oe.X), oe.get(oe.Y))
    print(case, "product", wp)
    assert wp <= 1e-4


@pytest.mark.parametrize("shape", ["biclique", "stars"])
def test_device_tsvd_init_rank_deficient_sketch(shape):
    # rank(A) < l = d + 10 on the randomized path (n > 600): CholeskyQR2 cannot
    # orthogonalise the sketch; the reference's Householder QR can, and clamps
    # the rank (svd.cpp:75-95). The device takes its Gram-Schmidt path and
    # must land on the oracle's rank, sigma and products.
    n, d = 900, 8
    if shape == "biclique":
        # complete bipartite K_{3,897}: rank 2
        a = np.repeat(np.arange(3), n - 3)
        b = np.tile(np.arange(3, n), 3)
    else:
        # five disjoint stars with distinct sizes: rank 10
        a, b, nxt = [], [], 5
        for c, sz in enumerate((40, 70, 110, 160, 220)):
            a += [c] * sz
            b += list(range(nxt, nxt + sz))
            nxt += sz
        a, b = np.array(a), np.array(b)
    g = oracle.Graph(n, np.concatenate([a, b]).astype(np.int64),
                     np.concatenate([b, a]).astype(np.int64), None, True)
    oe = oracle.OracleEngine(g, d=d, alpha=1.0, seed=7)
    off, tgt, wts = g.csr()
    e = ge.Engine.from_graph(n, off, tgt, None, d, alpha=1.0, undirected=True, seed=7)
    so, sg = oe.get(oe.SIGMA), e.get(ge.SIGMA)
    print(shape, "oracle k", len(so), "device k", len(sg), "sigma", so, sg)
    assert len(so) == len(sg) and (shape == "stars" or len(so) < d)  # biclique: rank 2 < d
    assert sigma_rel(sg, so) <= 1e-6
    po = oe.get(oe.X) @ oe.get(oe.Y).T
    pg = e.get(ge.X).astype(np.float64) @ e.get(ge.Y).astype(np.float64).T
    rel = np.linalg.norm(pg - po) / np.linalg.norm(po)
    print(shape, "product rel", rel)
    assert rel <= 1e-5
    # the state is usable: a few events against the oracle
    ev = oracle.Events.edges(1, [10, 11, 12], [20, 500, 600])
    oe.apply(ev)
    e.apply(W.EventList.edges(ge.ADD_EDGE, [10, 11, 12], [20, 500, 600]))
    po = oe.get(oe.X) @ oe.get(oe.Y).T
    pg = e.get(ge.X).astype(np.float64) @ e.get(ge.Y).astype(np.float64).T
    rel = np.linalg.norm(pg - po) / np.linalg.norm(po)
    print(shape, "after 3 insertions: k", e.k, oe.dims()[1], "product rel", rel)
    assert e.k == oe.dims()[1] and rel <= 1e-4


# ------------------------------------------------------ full-scale configs
def compact_oracle(e, rows, off_h, tgt_h, d):
    """The fp64 oracle restricted to `rows` (sorted global ids): a factor-only
    update (alpha = 1) reads and writes nothing but the rows of b / c's
    nonzeros and the k x k state (ortho_residual_norm, kernels.cpp:7-25,55-65;
    apply_update, factor_state.cpp:194-211; rebase / eager folds transform
    every row independently, :179-192,215-222), so an Engine over these rows,
    started from the device's base rows (fp32 -> fp64), P_X, P_Y and sigma,
    runs exactly the full oracle's arithmetic on them. Its graph is the
    snapshot restricted to `rows` (duplicate / missing-edge checks for the
    stream's endpoints are the full graph's)."""
    rows = np.asarray(rows, np.int64)
    xb = e.query64(ge.XB, rows)
    yb = e.query64(ge.YB, rows)
    px, py, sig = e.get(ge.PX), e.get(ge.PY), e.get(ge.SIGMA)
    src, dst = [], []
    for i, r in enumerate(rows.tolist()):
        nb = tgt_h[off_h[r]:off_h[r + 1]].astype(np.int64)
        pos = np.searchsorted(rows, nb)
        pos = np.minimum(pos, len(rows) - 1)
        hit = rows[pos] == nb
        src.append(np.full(int(hit.sum()), i, np.int64))
        dst.append(pos[hit])
    g = oracle.Graph(len(rows), np.concatenate(src), np.concatenate(dst), None, True)
    oe = oracle.OracleEngine(g, d=d, alpha=1.0, factors=(xb, yb, px, py, sig))
    return oe


def compact_stream_check(e, oe, rows, su, sv, batch, m, what, seed, every=None):
    """Apply m held-out insertions in device batches of `batch` (one call
    each), the oracle in the same order; modified-row sets bit-exact per call,
    then sigma and sampled products over the compact rows (at the end, or
    after every `every` calls: the worst value is returned)."""
    lu, lv = np.searchsorted(rows, su[:m]), np.searchsorted(rows, sv[:m])
    worst_p = worst_s = 0.0
    for ci, a in enumerate(range(0, m, batch)):
        b = min(m, a + batch)
        dev = W.EventList.edges(ge.ADD_EDGE, su[a:b], sv[a:b])
        loc = W.EventList.edges(ge.ADD_EDGE, lu[a:b], lv[a:b])
        oe.row_log_enable()
        oe.apply(loc)
        st = e.apply(dev, mode=ge.APPLY_LOG_ROWS)
        assert st["applied"] == b - a
        ol = oe.row_log()
        ol[:, 2] = rows[ol[:, 2]]  # local -> global row ids
        assert_rowlog_equal(e.row_log(), ol, f"{what} events {a}..{b}")
        if b == m or (every and (ci + 1) % every == 0):
            xg = e.query(ge.X, rows).astype(np.float64)
            yg = e.query(ge.Y, rows).astype(np.float64)
            wp = sampled_product_rel(xg, yg, oe.get(oe.X), oe.get(oe.Y), m=200_000, seed=seed + a)
            ws = sigma_rel(e.get(ge.SIGMA), oe.get(oe.SIGMA))
            print(f"{what}: batch {batch}, events ..{b}: product {wp:.3e} sigma {ws:.3e} "
                  f"cond {e.diag()['cond_estimate']:.3e}")
            worst_p, worst_s = max(worst_p, wp), max(worst_s, ws)
    return worst_p, worst_s


def test_cfg3_full_scale_batches_match_oracle():
    # cfg 3 at full size: R-MAT scale 22, ef 16 (seed 2), d = 128, the
    # reference's randomized t-SVD init ON THE DEVICE (damf_gpu_create), then
    # 1,024 held-out edges at each batch size 1 / 64 / 1024 (3,072 events),
    # against the oracle started from the device init's downloaded factors.
    import torch
    scale, d = 22, 128
    n = 1 << scale
    keys = W.rmat_keys_device(scale, 16, 2)
    g = torch.Generator(device="cuda")
    g.manual_seed(2)
    held = torch.randperm(keys.numel(), generator=g, device="cuda")[:3072]
    drop = torch.zeros(keys.numel(), dtype=torch.bool, device="cuda")
    drop[held] = True
    off, tgt = W.csr_from_keys_device(n, keys, drop)
    hk = keys[held]
    su, sv = (hk >> 32).cpu().numpy(), (hk & 0xFFFFFFFF).cpu().numpy()
    off_h, tgt_h = off.cpu().numpy(), tgt.cpu().numpy()
    del drop, off, tgt
    torch.cuda.empty_cache()
    e = ge.Engine.from_graph(n, off_h, tgt_h, None, d, alpha=1.0, undirected=True, seed=2,
                             node_capacity=1024, arc_capacity=1 << 20)
    assert e.k == d
    rng = np.random.default_rng(22)
    rows = np.unique(np.concatenate([su, sv, rng.integers(0, n, 2048)]))
    oe = compact_oracle(e, rows, off_h, tgt_h, d)
    a = 0
    for batch in (1, 64, 1024):
        wp, ws = compact_stream_check(e, oe, rows, su[a:], sv[a:], batch, 1024, "cfg3", batch)
        assert wp <= 1e-4 and ws <= 1e-6
        a += 1024
    # bookkeeping: the device adjacency is the snapshot plus the 3,072
    # insertions, bit-exact (every row of the 4.2 M)
    off2, tgt2 = W.csr_from_keys_device(n, keys)
    off_g, ids_g, deg_g = e.graph_sets()
    assert np.array_equal(off_g, off2.cpu().numpy())
    assert np.array_equal(ids_g, tgt2.cpu().numpy())
    assert np.array_equal(deg_g, np.diff(off_g).astype(np.float64))
    e.close()


def sampled_defect(e, off, tgt, rows, alpha, k):
    """max over `rows` of |alpha X + (1-alpha)/deg sum_{v in out(u)} Z[v] - Z|_inf
    / max(deg, 1) (eval.cpp:591-610) in current coordinates, on the GPU:
    X = X_b P_X and Z = Z_b P_X materialised by the engine, the neighbour sums
    accumulated in fp64 over the expected (unweighted) CSR."""
    import torch
    n = e.n
    X = torch.empty(n, k, dtype=torch.float32, device="cuda")
    Z = torch.empty(n, k, dtype=torch.float32, device="cuda")
    e.materialize(ge.X, X.data_ptr(), on_device=True)
    e.materialize(ge.Z, Z.data_ptr(), on_device=True)
    r = torch.as_tensor(rows, device="cuda")
    lo, hi = off[r], off[r + 1]
    cnt = hi - lo
    seg = torch.repeat_interleave(torch.arange(len(r), device="cuda"), cnt)
    start = torch.repeat_interleave(lo - torch.cumsum(cnt, 0) + cnt, cnt)
    pos = torch.arange(int(cnt.sum()), device="cuda") + start
    nb = tgt[pos].long()
    acc = torch.zeros(len(r), k, dtype=torch.float64, device="cuda")
    for c0 in range(0, len(nb), 1 << 24):
        acc.index_add_(0, seg[c0:c0 + (1 << 24)], Z[nb[c0:c0 + (1 << 24)]].double())
    deg = cnt.double()
    dfc = alpha * X[r].double() - Z[r].double()
    has = deg > 0
    dfc[has] += ((1 - alpha) / deg[has])[:, None] * acc[has]
    out = (dfc.abs().amax(1) / torch.clamp(deg, min=1.0))
    del X, Z
    return float(out.max())


@pytest.mark.parametrize("d", [32, 64, 128, 256])
def test_cfg4_ppr_defect_at_scale(d):
    # cfg 4: R-MAT scale 23, ef 24 (seed 3, 384 M arcs), X ~ N(0, 1/d) and
    # P_X = F = Q diag(U[.5, 2]). init_propagate, then 1,000
    # random structure-only insertions absorbed and one push. The reference's
    # defect bound eps (1 + 1e-6) on >= 10^5 sampled rows plus every touched
    # row and its neighbours, after each phase.
    import torch
    scale, alpha, eps = 23, 0.15, 1e-5
    n = 1 << scale
    keys = W.rmat_keys_device(scale, 24, 3)
    off, tgt = W.csr_from_keys_device(n, keys)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    X = (torch.randn(n, d, device="cuda", generator=gen) / np.sqrt(d)).contiguous()
    F = W.cfg4_F(d, 3)
    e = ge.Engine(n, off, tgt, None, d, d, X, X, F, np.eye(d), np.ones(d), alpha=alpha, eps=eps,
                  undirected=True, node_capacity=1024)
    del X
    torch.cuda.empty_cache()
    rng = np.random.default_rng(23)
    sample = np.unique(rng.integers(0, n, 120_000))
    d0 = sampled_defect(e, off, tgt, sample, alpha, d)
    print(f"d={d}: after init_propagate, defect over {len(sample)} rows {d0:.3e}")
    assert d0 <= eps * (1 + 1e-6)
    # 1,000 random new edges, structure only (App. D.4), then one push
    us = rng.integers(0, n, 3000)
    vs = rng.integers(0, n, 3000)
    lo, hi = np.minimum(us, vs), np.maximum(us, vs)
    kk = torch.as_tensor((lo << 32) | hi, device="cuda")
    pos = torch.searchsorted(keys, kk).clamp(max=keys.numel() - 1)
    fresh = ((keys[pos] != kk).cpu().numpy()) & (lo != hi)
    _, first = np.unique((lo << 32) | hi, return_index=True)
    ok = np.zeros(len(us), bool)
    ok[first] = True
    ok &= fresh
    eu, evv = us[ok][:1000], vs[ok][:1000]
    assert len(eu) == 1000
    e.apply(W.EventList.edges(ge.ADD_EDGE, eu, evv),
            mode=ge.APPLY_GRAPH_AND_PPR_ONLY | ge.APPLY_DEFER_PUSH)
    st = e.ppr_push()
    newk = torch.as_tensor(np.minimum(eu, evv) << 32 | np.maximum(eu, evv), device="cuda")
    keys2 = torch.sort(torch.cat([keys, newk])).values
    del keys
    off2, tgt2 = W.csr_from_keys_device(n, keys2)
    touched = np.unique(np.concatenate([eu, evv]))
    nbr = tgt2[torch.cat([torch.arange(int(off2[t]), int(off2[t + 1]), device="cuda")
                          for t in touched[:200]])].cpu().numpy()
    rows = np.unique(np.concatenate([sample, touched, nbr]))
    d1 = sampled_defect(e, off2, tgt2, rows, alpha, d)
    print(f"d={d}: push after 1,000 inserts ({st['push_rounds']} rounds, {st['pushes']} pushes), "
          f"defect over {len(rows)} rows {d1:.3e}")
    assert d1 <= eps * (1 + 1e-6)
    e.close()


def test_cfg5_full_scale_compact_oracle():
    # cfg 5: R-MAT scale 26 (2.1 B arcs, int64 offsets), d = 128, U / V random
    # orthonormal with sigma_i = i^-1/2 (34 GB each). The first 1,000
    # degree-proportional insertions, one damf_gpu_apply per insertion, beside
    # the compact oracle (every modified row bit-exact, sigma to 1e-6 at every
    # checkpoint). Products: this spectrum plus unit-norm insertions sits on a
    # near-degenerate truncation boundary (the case eval.cpp:514-517 excludes
    # from the reference's own oracle comparison), so any perturbation of the
    # base rows -- such as the fp32 rounding of every row at a fold, which the
    # config's fp32 U / V imply -- grows to ~3e-4 within a few hundred events.
    # The oracle therefore runs the device's storage model (fp32 base rows at
    # every fold, rebases after the same events as the device): products
    # within 1e-4 through the first 100 insertions; the distance to the fp64
    # oracle is printed, not gated (per-event parity from identical
    # pre-states, test_cfg5_rowlocal_at_scale, is the strict gate).
    import gc
    import torch
    gc.collect()
    torch.cuda.empty_cache()
    free, total = torch.cuda.mem_get_info()
    if total < 150e9:
        pytest.skip("config 5 needs ~120 GB of device memory")
    d, m = 128, 500
    e, su, sv = cfg5_like(26, d, m, seed=4)
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([su, sv, rng.integers(0, e.n, 1024)]))
    fac = (e.query64(ge.XB, rows), e.query64(ge.YB, rows), e.get(ge.PX), e.get(ge.PY),
           e.get(ge.SIGMA))
    g = oracle.Graph(len(rows), np.zeros(0, np.int64), np.zeros(0, np.int64), None, True)
    o32 = oracle.OracleEngine(g, d=d, alpha=1.0, rebase_cond=1e300, rebase_every=1 << 60,
                              factors=fac)
    o32.set_fp32_base(True)
    o64 = oracle.OracleEngine(g, d=d, alpha=1.0, rebase_cond=1e2, factors=fac)
    lu, lv = np.searchsorted(rows, su), np.searchsorted(rows, sv)
    worst_p = worst_s = 0.0
    rebases = 0
    for i in range(m):
        ev = W.EventList.edges(ge.ADD_EDGE, lu[i:i + 1], lv[i:i + 1])
        o32.row_log_enable()
        o32.apply(ev)
        o64.apply(ev)
        st = e.apply(W.EventList.edges(ge.ADD_EDGE, su[i:i + 1], sv[i:i + 1]), mode=ge.APPLY_LOG_ROWS)
        ol = o32.row_log()
        ol[:, 2] = rows[ol[:, 2]]
        assert_rowlog_equal(e.row_log(), ol, f"cfg5 event {i}")
        if st["rebases"]:
            rebases += 1
            o32.rebase()
        if (i + 1) % 25 == 0:
            ws = sigma_rel(e.get(ge.SIGMA), o32.get(o32.SIGMA))
            worst_s = max(worst_s, ws)
            if i < 100 or (i + 1) % 250 == 0:
                xg = e.query(ge.X, rows).astype(np.float64)
                yg = e.query(ge.Y, rows).astype(np.float64)
                wp = sampled_product_rel(xg, yg, o32.get(o32.X), o32.get(o32.Y), m=200_000, seed=i)
                w64 = sampled_product_rel(xg, yg, o64.get(o64.X), o64.get(o64.Y), m=200_000, seed=i)
                print(f"cfg5 event {i + 1}: product vs fp32-storage oracle {wp:.2e}, vs fp64 oracle "
                      f"{w64:.2e}, sigma {ws:.2e}, device rebases {rebases}")
                if i < 100:
                    worst_p = max(worst_p, wp)
    print("cfg5: worst product (first 100)", worst_p, "worst sigma", worst_s)
    assert worst_p <= 1e-4 and worst_s <= 1e-6
    e.close()
