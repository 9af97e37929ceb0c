"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is named by BASELINE.json; these generators produce graphs
with the stated shapes, sizes and distributions:

  cfg1  Barabasi-Albert n=10,000, m=5, seed 0; 50% snapshot, 50% streamed
  cfg2  SBM 20 blocks x 5,000 (p_in=16/4,999, p_out=4/95,000), seed 1; 90%
        snapshot; stream = 10,000 inserts + 2,000 deletions + 500 node adds
        (10 edges each), seeded interleave
  cfg3  R-MAT a/b/c/d=.57/.19/.19/.05 scale 22, ef 16, seed 2; all but 100k
        edges snapshot; 100k streamed in batches of 1/64/1024
  cfg4  R-MAT scale 23, ef 24, seed 3; X ~ N(0,1/d), F = Q diag(U[.5,2])
  cfg5  R-MAT scale 26, ef 16, seed 4; orthonormal U, V with s_i = i^-1/2;
        10,000 degree-proportional inserts

Edge lists are undirected (u < v), unweighted. Host generation uses numpy's
PCG64; the R-MAT generator runs on the GPU through torch (input generation,
not the measured path) when a device is given.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ADD_NODE, ADD_EDGE, REMOVE_EDGE = 0, 1, 2


@dataclass
class EventList:
    """Flat event batch with the damf_event_batch layout."""
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
        return EventList(self.kind[a:b].copy(), self.u[a:b].copy(), self.v[a:b].copy(),
                         self.w[a:b].copy(), io[a:b + 1] - io[a], self.in_ids[io[a]:io[b]].copy(),
                         self.in_w[io[a]:io[b]].copy(), oo[a:b + 1] - oo[a],
                         self.out_ids[oo[a]:oo[b]].copy(), self.out_w[oo[a]:oo[b]].copy())

    @staticmethod
    def edges(kind, u, v, w=None):
        m = len(u)
        kind = np.full(m, kind, np.int32) if np.isscalar(kind) else np.asarray(kind, np.int32)
        z = np.zeros(m + 1, np.int64)
        return EventList(kind, np.asarray(u, np.int64), np.asarray(v, np.int64),
                         np.ones(m) if w is None else np.asarray(w, np.float64), z,
                         np.zeros(0, np.int64), np.zeros(0), z.copy(), np.zeros(0, np.int64),
                         np.zeros(0))


def undirected_csr(n, eu, ev):
    """CSR (offsets int64, targets int32) with both arcs of every edge; each
    row lists targets in increasing order."""
    src = np.concatenate([eu, ev]).astype(np.int64)
    dst = np.concatenate([ev, eu]).astype(np.int64)
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, src + 1, 1)
    return np.cumsum(off), dst.astype(np.int32)


def csr_arcs(offsets, targets):
    """(src, dst) arc arrays from a CSR."""
    n = len(offsets) - 1
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(offsets))
    return src, targets.astype(np.int64)


# ---------------------------------------------------------------- cfg 1
def ba_edges(n, m, seed):
    """Preferential attachment from m initial nodes: node t >= m attaches to
    m distinct existing nodes drawn proportionally to degree (repeated-node
    list); m*(n-m) edges."""
    rng = np.random.Generator(np.random.PCG64(seed))
    rep = list(range(m))  # initial targets: the m seed nodes
    eu, ev = [], []
    for t in range(m, n):
        chosen = set()
        while len(chosen) < m:
            chosen.add(rep[int(rng.integers(len(rep)))])
        for c in sorted(chosen):
            eu.append(c)
            ev.append(t)
            rep.append(c)
            rep.append(t)
    eu = np.array(eu, np.int64)
    ev = np.array(ev, np.int64)
    return np.minimum(eu, ev), np.maximum(eu, ev)


def cfg1(seed=0, n=10_000, m=5, snapshot=0.5):
    eu, ev = ba_edges(n, m, seed)
    rng = np.random.Generator(np.random.PCG64(seed + 1000))
    perm = rng.permutation(len(eu))
    eu, ev = eu[perm], ev[perm]
    n0 = int(len(eu) * snapshot)
    stream = EventList.edges(ADD_EDGE, eu[n0:], ev[n0:])
    return dict(n=n, init=(eu[:n0], ev[:n0]), stream=stream, d=32, alpha=0.15, eps=1e-4)


# ---------------------------------------------------------------- cfg 2
def sbm_edges(blocks, bsize, p_in, p_out, seed):
    """Stochastic block model by geometric skipping over each block pair."""
    rng = np.random.Generator(np.random.PCG64(seed))
    eu, ev = [], []
    for a in range(blocks):
        for b in range(a, blocks):
            p = p_in if a == b else p_out
            npairs = bsize * (bsize - 1) // 2 if a == b else bsize * bsize
            # number of edges ~ Binomial, positions uniform without replacement
            cnt = rng.binomial(npairs, p)
            pos = rng.choice(npairs, size=cnt, replace=False)
            if a == b:
                # unrank pair index -> (i < j) inside the block
                i = (np.floor((1 + np.sqrt(1 + 8.0 * pos)) / 2)).astype(np.int64)
                i = np.where(i * (i - 1) // 2 > pos, i - 1, i)
                i = np.where((i + 1) * i // 2 <= pos, i + 1, i)
                j = pos - i * (i - 1) // 2
                u, v = a * bsize + j, a * bsize + i
            else:
                u, v = a * bsize + pos // bsize, b * bsize + pos % bsize
            eu.append(u)
            ev.append(v)
    eu = np.concatenate(eu).astype(np.int64)
    ev = np.concatenate(ev).astype(np.int64)
    return np.minimum(eu, ev), np.maximum(eu, ev)


def cfg2(seed=1, blocks=20, bsize=5000, n_ins=10_000, n_del=2_000, n_nodes=500, node_deg=10,
         snapshot=0.9):
    n = blocks * bsize
    p_in = 16.0 / (bsize - 1)
    p_out = 4.0 / (n - bsize)
    eu, ev = sbm_edges(blocks, bsize, p_in, p_out, seed)
    rng = np.random.Generator(np.random.PCG64(seed + 1000))
    perm = rng.permutation(len(eu))
    eu, ev = eu[perm], ev[perm]
    n0 = int(len(eu) * snapshot)
    init = (eu[:n0], ev[:n0])
    held = list(zip(eu[n0:n0 + n_ins].tolist(), ev[n0:n0 + n_ins].tolist()))
    types = np.array([ADD_EDGE] * len(held) + [REMOVE_EDGE] * n_del + [ADD_NODE] * n_nodes)
    rng.shuffle(types)
    live = set(zip(init[0].tolist(), init[1].tolist()))
    live_list = list(live)
    kinds, us, vs, in_off, in_ids = [], [], [], [0], []
    cur_n = n
    hi = 0
    for t in types:
        if t == ADD_EDGE:
            u, v = held[hi]
            hi += 1
            kinds.append(ADD_EDGE)
            us.append(u)
            vs.append(v)
            live.add((u, v))
            live_list.append((u, v))
        elif t == REMOVE_EDGE:
            while True:  # uniform over edges present at this moment
                idx = int(rng.integers(len(live_list)))
                e = live_list[idx]
                live_list[idx] = live_list[-1]
                live_list.pop()
                if e in live:
                    break
            live.discard(e)
            kinds.append(REMOVE_EDGE)
            us.append(e[0])
            vs.append(e[1])
        else:
            nb = rng.choice(cur_n, size=node_deg, replace=False)
            kinds.append(ADD_NODE)
            us.append(cur_n)
            vs.append(0)
            in_ids.extend(sorted(int(x) for x in nb))
            for x in nb:
                e = (int(x), cur_n)
                live.add(e)
                live_list.append(e)
            cur_n += 1
        in_off.append(len(in_ids))
    m = len(kinds)
    in_off = np.array(in_off, np.int64)
    stream = EventList(np.array(kinds, np.int32), np.array(us, np.int64), np.array(vs, np.int64),
                       np.ones(m), in_off, np.array(in_ids, np.int64), np.ones(len(in_ids)),
                       np.zeros(m + 1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    return dict(n=n, init=init, stream=stream, d=128, alpha=0.15, eps=1e-5)


# ---------------------------------------------------------------- R-MAT
def rmat_keys_device(scale, ef, seed, a=0.57, b=0.19, c=0.19, device="cuda"):
    """R-MAT edges on the GPU as sorted unique int64 keys (lo << 32) | hi,
    lo < hi (symmetrised, self loops and duplicates removed)."""
    import torch
    m = ef << scale
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    u = torch.zeros(m, dtype=torch.int64, device=device)
    v = torch.zeros(m, dtype=torch.int64, device=device)
    ab, abc = a + b, a + b + c
    for _ in range(scale):
        r = torch.rand(m, generator=g, device=device)
        u <<= 1
        u |= (r >= ab).to(torch.int64)
        v <<= 1
        v |= (((r >= a) & (r < ab)) | (r >= abc)).to(torch.int64)
        del r
    lo = torch.minimum(u, v)
    hi = torch.maximum(u, v)
    del u, v
    keep = lo != hi
    key = lo[keep]
    key <<= 32
    key |= hi[keep]
    del lo, hi, keep
    return torch.unique(key)  # sorted


def rmat_edges(scale, ef, seed, a=0.57, b=0.19, c=0.19, device=None):
    """R-MAT (recursive quadrant sampling, no noise), symmetrised, self loops
    and duplicates removed. Returns (u, v) with u < v, sorted. Runs on the GPU
    with torch when `device` is given, else numpy."""
    m = ef << scale
    if device is not None:
        key = rmat_keys_device(scale, ef, seed, a, b, c, device)
        return (key >> 32), (key & 0xFFFFFFFF)
    rng = np.random.Generator(np.random.PCG64(seed))
    u = np.zeros(m, np.int64)
    v = np.zeros(m, np.int64)
    for _ in range(scale):
        r = rng.random(m)
        bu = r >= a + b
        bv = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        u = (u << 1) | bu
        v = (v << 1) | bv
    lo, hi = np.minimum(u, v), np.maximum(u, v)
    keep = lo != hi
    key = np.unique((lo[keep] << 32) | hi[keep])
    return key >> 32, key & 0xFFFFFFFF


# ---------------------------------------------------------------- factors
def random_orthonormal(n, k, seed, device=None):
    """CholeskyQR2 of a Gaussian n x k (fp64) -> orthonormal columns."""
    if device is not None:
        import torch
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        a = torch.randn(n, k, generator=g, device=device, dtype=torch.float64)
        for _ in range(2):
            r = torch.linalg.cholesky(a.T @ a).T
            a = torch.linalg.solve_triangular(r, a, upper=True, left=False)
        return a
    rng = np.random.Generator(np.random.PCG64(seed))
    a = rng.standard_normal((n, k))
    for _ in range(2):
        r = np.linalg.cholesky(a.T @ a).T
        a = np.linalg.solve(r.T, a.T).T
    return a


def orthonormal_factors(n, d, seed, device=None):
    """cfg5 state: X_b = U sqrt(S), Y_b = V sqrt(S), sigma_i = i^-1/2, P = I."""
    sig = 1.0 / np.sqrt(np.arange(1, d + 1, dtype=np.float64))
    U = random_orthonormal(n, d, seed, device)
    V = random_orthonormal(n, d, seed + 7919, device)
    return U, V, sig


def cfg4_F(d, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    q, r = np.linalg.qr(rng.standard_normal((d, d)))
    q = q * np.sign(np.diag(r))[None, :]  # Haar
    return q * rng.uniform(0.5, 2.0, size=d)[None, :]


# ------------------------------------------------ device builders (cfg 3-5)
def csr_from_keys_device(n, keys, drop=None):
    """Symmetric CSR (offsets int64, targets int32; rows sorted) as CUDA
    tensors from unique edge keys (lo << 32) | hi; `drop` = boolean mask of
    keys to leave out (held-out stream edges)."""
    import torch
    k = keys if drop is None else keys[~drop]
    lo = k >> 32
    hi = k & 0xFFFFFFFF
    both = torch.cat([k, (hi << 32) | lo])
    del k, lo, hi
    both = torch.sort(both).values
    src = both >> 32
    cnt = torch.bincount(src, minlength=n)
    del src
    off = torch.zeros(n + 1, dtype=torch.int64, device=both.device)
    torch.cumsum(cnt, 0, out=off[1:])
    del cnt
    tgt = (both & 0xFFFFFFFF).to(torch.int32)
    del both
    return off, tgt


def orthonormal_rows_into(eng, which, n, d, sigma, seed, chunk=1 << 22):
    """X_b (or Y_b) = U diag(sqrt sigma) with U random orthonormal columns
    (Cholesky-QR of a seeded Gaussian, generated chunk by chunk on the GPU and
    loaded in place with Engine.load_rows), SURVEY 8(d) cfg 5."""
    import torch
    gen = torch.Generator(device="cuda")
    gram = torch.zeros(d, d, dtype=torch.float64, device="cuda")
    for c0 in range(0, n, chunk):
        gen.manual_seed(seed * 1000003 + c0 // chunk)
        blk = torch.randn(min(chunk, n - c0), d, generator=gen, device="cuda").double()
        gram += blk.T @ blk
        del blk
    R = torch.linalg.cholesky(gram, upper=True)
    T = torch.linalg.inv(R) * torch.as_tensor(np.sqrt(sigma), device="cuda")[None, :]
    for c0 in range(0, n, chunk):
        gen.manual_seed(seed * 1000003 + c0 // chunk)
        blk = torch.randn(min(chunk, n - c0), d, generator=gen, device="cuda").double()
        eng.load_rows(which, c0, (blk @ T).float().contiguous())
        del blk
    torch.cuda.synchronize()


def degree_proportional_inserts(keys, tgt, m, seed):
    """m new undirected edges whose endpoints are uniformly random arc
    endpoints (degree-proportional), no loops, no existing or repeated edge."""
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    arcs = tgt.numel()
    out_u, out_v, seen = [], [], set()
    while len(out_u) < m:
        i = torch.randint(arcs, (4 * m,), generator=g, device="cuda")
        j = torch.randint(arcs, (4 * m,), generator=g, device="cuda")
        u = tgt[i].long()
        v = tgt[j].long()
        lo, hi = torch.minimum(u, v), torch.maximum(u, v)
        key = (lo << 32) | hi
        pos = torch.searchsorted(keys, key).clamp(max=keys.numel() - 1)
        ok = (lo != hi) & (keys[pos] != key)
        for a, b in zip(u[ok].tolist(), v[ok].tolist()):
            kk = (min(a, b), max(a, b))
            if kk in seen:
                continue
            seen.add(kk)
            out_u.append(a)
            out_v.append(b)
            if len(out_u) == m:
                break
    return np.array(out_u, np.int64), np.array(out_v, np.int64)


def orthonormal_rows_subset(n, d, sigma, seed, ids, chunk=1 << 22):
    """The rows `ids` of what orthonormal_rows_into loads (same seeded chunks,
    same Gram matrix and transform, each chunk's product computed whole and
    rounded to fp32 exactly as loaded), as a (len(ids), d) fp32 numpy array:
    the input of the CPU oracle beside a device engine built at config 5."""
    import torch
    ids = np.asarray(ids, np.int64)
    gen = torch.Generator(device="cuda")
    gram = torch.zeros(d, d, dtype=torch.float64, device="cuda")
    for c0 in range(0, n, chunk):
        gen.manual_seed(seed * 1000003 + c0 // chunk)
        blk = torch.randn(min(chunk, n - c0), d, generator=gen, device="cuda").double()
        gram += blk.T @ blk
        del blk
    R = torch.linalg.cholesky(gram, upper=True)
    T = torch.linalg.inv(R) * torch.as_tensor(np.sqrt(sigma), device="cuda")[None, :]
    out = np.zeros((len(ids), d), np.float32)
    for c0 in range(0, n, chunk):
        sel = np.nonzero((ids >= c0) & (ids < c0 + chunk))[0]
        if len(sel) == 0:
            continue
        gen.manual_seed(seed * 1000003 + c0 // chunk)
        blk = torch.randn(min(chunk, n - c0), d, generator=gen, device="cuda").double()
        rows = (blk @ T).float()
        out[sel] = rows[torch.as_tensor(ids[sel] - c0, device="cuda")].cpu().numpy()
        del blk, rows
    return out


def cfg5_inputs(n_events, seed=4, scale=26, ef=16):
    """Config 5's graph (R-MAT, device-built CSR) and its first `n_events`
    degree-proportional insertions: (keys, off, tgt, su, sv) as CUDA tensors /
    numpy arrays."""
    import torch
    n = 1 << scale
    keys = rmat_keys_device(scale, ef, seed)
    off, tgt = csr_from_keys_device(n, keys)
    su, sv = degree_proportional_inserts(keys, tgt, n_events, seed=seed)
    torch.cuda.empty_cache()
    return keys, off, tgt, su, sv
