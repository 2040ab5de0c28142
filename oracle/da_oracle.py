"""CPU ORACLE for the DA hot path -- test infrastructure, NOT product code.

A numpy restatement of the reference algorithm (annq, /root/reference/pkg/src/
annq) used only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
/ reference arm, as the checker.  The product path (paper_1509_05194_b200)
never imports this module.

Pinning: tests/golden/*.npz were produced by the reference itself
(oracle/make_golden.py imports /root/reference/pkg/src in the build
container); tests/test_oracle_golden.py requires this oracle to reproduce
them bit-for-bit.  Every numpy call below keeps the reference's evaluation
order, so on the same machine the oracle and the reference agree exactly.

Each function cites the reference lines it restates (paths relative to
pkg/src/annq/).
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# ---------------------------------------------------------------------------
# codebook side (codebook.py)


def sq_norms(cw64: np.ndarray) -> np.ndarray:
    """||c_mk||^2 (M, K) -- codebook.py:129, 237, 260 (einsum)."""
    return np.einsum("mkd,mkd->mk", cw64, cw64)


def cross_table(cw32: np.ndarray):
    """(P (M,M,K,K), sq (M,K)) -- codebook.py:231-238."""
    cw64 = cw32.astype(np.float64)
    M, K, d = cw64.shape
    flat = cw64.reshape(M * K, d)
    full = flat @ flat.T
    P = np.ascontiguousarray(full.reshape(M, K, M, K).transpose(0, 2, 1, 3))
    return P, sq_norms(cw64)


def cross_refresh(P: np.ndarray, sq: np.ndarray, cw32: np.ndarray, m: int):
    """Copy of (P, sq) with dictionary m's rows/cols rebuilt -- codebook.py:241-252."""
    cw64 = cw32.astype(np.float64)
    M, K, d = cw64.shape
    P2, sq2 = P.copy(), sq.copy()
    blk = (cw64[m] @ cw64.reshape(M * K, d).T).reshape(K, M, K).transpose(1, 0, 2)
    P2[m] = blk
    P2[:, m] = blk.transpose(0, 2, 1)
    sq2[m] = (cw64[m] * cw64[m]).sum(axis=1)
    return P2, sq2


def reconstruct_rows(cw64: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """sum_m C[m][codes[:, m]] accumulated in m order from zero -- codebook.py:181-188."""
    acc = np.zeros((codes.shape[0], cw64.shape[2]))
    for m in range(codes.shape[1]):
        acc += cw64[m][codes[:, m]]
    return acc


def row_errors(cw64, X64, codes) -> np.ndarray:
    """||x - recon||^2 per row -- annealing.py:135-137, codebook.py:299-300."""
    r = X64 - reconstruct_rows(cw64, codes)
    return (r * r).sum(axis=1)


def beam_encode(cw64: np.ndarray, P: np.ndarray, X64: np.ndarray, L: int):
    """Beam search with stable (value, flat index) selection -- codebook.py:255-300.

    Returns (codes int64 (n, M), exact errors (n,)).
    """
    n = X64.shape[0]
    M, K, d = cw64.shape
    t = np.einsum("mkd,mkd->mk", cw64, cw64).reshape(1, M, K) - 2.0 * (
        X64 @ cw64.reshape(M * K, d).T
    ).reshape(n, M, K)
    keep = min(L, K)
    pick = np.sort(np.argsort(t[:, 0, :], axis=1, kind="stable")[:, :keep], axis=1)
    paths = pick[:, :, None].astype(np.int64)
    score = np.take_along_axis(t[:, 0, :], pick, axis=1)
    for m in range(1, M):
        live = paths.shape[1]
        cross = np.zeros((n, live, K))
        for j in range(m):
            cross += P[j, m][paths[:, :, j], :]
        cand = (score[:, :, None] + t[:, m, :][:, None, :] + 2.0 * cross).reshape(n, live * K)
        keep = min(L, live * K)
        pick = np.sort(np.argsort(cand, axis=1, kind="stable")[:, :keep], axis=1)
        paths = np.concatenate(
            [np.take_along_axis(paths, (pick // K)[:, :, None], axis=1), (pick % K)[:, :, None].astype(np.int64)],
            axis=2,
        )
        score = np.take_along_axis(cand, pick, axis=1)
    win = paths[np.arange(n), np.argmin(score, axis=1)]
    return win, row_errors(cw64, X64, win)


def encode_chunked(cw32, P, X32, L, n_jobs=1):
    """encode_dataset's chunking + thread pool (codebook.py:338-353); int64 codes."""
    X64 = X32.astype(np.float64)
    cw64 = cw32.astype(np.float64)
    n = X64.shape[0]
    step = max(64, min(n, int(4e6) // max(L * cw32.shape[1], 1)))
    starts = list(range(0, n, step))
    work = lambda s: beam_encode(cw64, P, X64[s:s + step], L)[0]  # noqa: E731
    if n_jobs > 1 and len(starts) > 1:
        with ThreadPoolExecutor(max_workers=n_jobs) as ex:
            parts = list(ex.map(work, starts))
    else:
        parts = [work(s) for s in starts]
    return np.vstack(parts) if parts else np.empty((0, cw32.shape[0]), dtype=np.int64)


def adc_lut(cw32: np.ndarray, q: np.ndarray):
    """(values (M,K) clipped at 0, ||q||^2) -- codebook.py:361-369 with :123-132."""
    cw64 = cw32.astype(np.float64)
    M, K, d = cw64.shape
    qq = float(q @ q)
    v = qq - 2.0 * (q @ cw64.reshape(M * K, d).T).reshape(M, K) + sq_norms(cw64)
    np.maximum(v, 0.0, out=v)
    return v, qq


def pair_terms(P: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """2 * sum_{a<b} P[a,b][i_a, i_b] -- codebook.py:388-396."""
    n, M = codes.shape
    acc = np.zeros(n)
    for a in range(M):
        for b in range(a + 1, M):
            acc += P[a, b][codes[:, a], codes[:, b]]
    return 2.0 * acc


def adc_topr(values, qq, codes, pair, r):
    """Top-r by (distance, position) -- codebook.py:419-429.  Returns (positions, dists)."""
    M = values.shape[0]
    dist = pair - (M - 1) * qq
    for m in range(M):
        dist = dist + values[m][codes[:, m]]
    kth = np.partition(dist, r - 1)[r - 1]
    cand = np.flatnonzero(dist <= kth)
    sel = cand[np.lexsort((cand, dist[cand]))[:r]]
    return sel.astype(np.int64), dist[sel]


def variance_order(cw32: np.ndarray) -> np.ndarray:
    """Permutation to non-increasing dictionary variance -- codebook.py:211-228."""
    cw = cw32.astype(np.float64)
    c = cw - cw.mean(axis=1, keepdims=True)
    var = (c * c).sum(axis=2).mean(axis=1)
    return np.argsort(-var, kind="stable").astype(np.int64)


# ---------------------------------------------------------------------------
# clustering side (clustering.py)


def schedule(d: int, stages: int = 10) -> list:
    """clustering.py:116-131."""
    out: list = []
    for i in range(1, stages + 1):
        v = min(d, math.ceil(d ** (i / stages)))
        if not out or v > out[-1]:
            out.append(v)
    if out[-1] != d:
        out.append(d)
    return out


def nearest(Xa: np.ndarray, Ca: np.ndarray):
    """First-min nearest centroid on the given columns -- clustering.py:139-148."""
    d2 = (Xa * Xa).sum(axis=1)[:, None] - 2.0 * (Xa @ Ca.T) + (Ca * Ca).sum(axis=1)[None, :]
    np.maximum(d2, 0.0, out=d2)
    lab = np.argmin(d2, axis=1)
    return lab, d2[np.arange(Xa.shape[0]), lab]


def segment_means(X: np.ndarray, lab: np.ndarray, k: int):
    """Means over all columns via stable sort + reduceat -- clustering.py:151-162."""
    perm = np.argsort(lab, kind="stable")
    cnt = np.bincount(lab, minlength=k)
    tot = np.zeros((k, X.shape[1]))
    live = np.flatnonzero(cnt)
    if live.size:
        starts = np.concatenate([[0], np.cumsum(cnt[live])[:-1]])
        tot[live] = np.add.reduceat(X[perm], starts, axis=0)
    return tot / np.maximum(cnt, 1)[:, None], cnt


def lloyd(X: np.ndarray, C_init: np.ndarray, active: int, iters: int):
    """clustering.py:165-203.  Returns (C, labels, trace)."""
    C = np.array(C_init, dtype=np.float64, copy=True)
    k = C.shape[0]
    Xa = X[:, :active]
    lab, err = nearest(Xa, C[:, :active])
    trace = [float(err.mean())]
    for _ in range(iters):
        mu, cnt = segment_means(X, lab, k)
        full = np.flatnonzero(cnt > 0)
        C[full] = mu[full]
        holes = np.flatnonzero(cnt == 0)
        if holes.size:
            C[holes] = X[np.argsort(err, kind="stable")[::-1][: holes.size]]
        nxt, err = nearest(Xa, C[:, :active])
        trace.append(float(err.mean()))
        done = np.array_equal(nxt, lab)
        lab = nxt
        if done:
            break
    return C, lab.astype(np.int64), trace


def _fill_basis(rows_in: np.ndarray, d: int) -> np.ndarray:
    """clustering.py:63-79."""
    rows = list(rows_in)
    for j in range(d):
        if len(rows) == d:
            break
        v = np.zeros(d)
        v[j] = 1.0
        for _ in range(2):
            for u in rows:
                v -= (v @ u) * u
        nv = np.linalg.norm(v)
        if nv > 1e-8:
            rows.append(v / nv)
    return np.vstack(rows)


def pca(X: np.ndarray):
    """(rotation (d,d), mean (d,)) -- clustering.py:82-113 (X float64)."""
    n, d = X.shape
    mu = X.mean(axis=0)
    Xc = X - mu
    if n > d:
        w, V = np.linalg.eigh((Xc.T @ Xc) / (n - 1))
        idx = np.argsort(w, kind="stable")[::-1]
        return V[:, idx].T, mu
    w, U = np.linalg.eigh(Xc @ Xc.T)
    idx = np.argsort(w, kind="stable")[::-1]
    w = np.maximum(w[idx], 0.0)
    U = U[:, idx]
    tol = max(w[0], 1.0) * 1e-10 if w.size else 0.0
    ok = w > tol
    comps = (Xc.T @ U[:, ok]) / np.sqrt(w[ok])[None, :]
    return _fill_basis(comps.T, d), mu


def staged_kmeans(X64: np.ndarray, C0: np.ndarray, sched, iters: int):
    """clustering.py:215-250.  Returns (points, labels, trace)."""
    R, mu = pca(X64)
    Xr = (X64 - mu) @ R.T
    Cr = (np.asarray(C0, dtype=np.float64) - mu) @ R.T
    tr: list = []
    for dims in sched:
        Cr, _, tr = lloyd(Xr, Cr, dims, iters)
    C = Cr @ R + mu
    fl, fe = nearest(X64, C)
    il, ie = nearest(X64, C0)
    if fe.mean() <= ie.mean():
        return C, fl.astype(np.int64), tr
    return np.array(C0, copy=True), il.astype(np.int64), [float(ie.mean())]


# ---------------------------------------------------------------------------
# annealing side (annealing.py)


def heat_up(X32, cw32, codes, m):
    """annealing.py:97-112 -> float32."""
    X64 = X32.astype(np.float64)
    cw64 = cw32.astype(np.float64)
    return (X64 - reconstruct_rows(cw64, codes) + cw64[m][codes[:, m]]).astype(np.float32)


def cool_down(inter32, cw32, m, stages, iters):
    """annealing.py:115-126 -> (dictionary float32, labels int64)."""
    pts, lab, _ = staged_kmeans(inter32.astype(np.float64), cw32[m].astype(np.float64),
                                schedule(cw32.shape[2], stages), iters)
    return pts.astype(np.float32), lab


def sweep(X32, cw32, codes, P, sq, L, stages, iters, steps=None, sweep_index=1):
    """annealing.py:140-181 on plain arrays; returns (cw32, codes, P, sq)."""
    X64 = X32.astype(np.float64)
    cw32 = cw32.copy()
    codes = codes.copy()
    for m in range(cw32.shape[0]):
        inter = heat_up(X32, cw32, codes, m)
        new, lab = cool_down(inter, cw32, m, stages, iters)
        cw32[m] = new
        P, sq = cross_refresh(P, sq, cw32, m)
        inc = codes.copy()
        inc[:, m] = lab
        cw64 = cw32.astype(np.float64)
        bc, be = beam_encode(cw64, P, X64, L)
        ie = row_errors(cw64, X64, inc)
        take = be <= ie
        codes = np.where(take[:, None], bc, inc)
        if steps is not None:
            steps.append((sweep_index, m, float(np.where(take, be, ie).mean())))
    return cw32, codes, P, sq


def growth(X32, M, K, stages, iters, steps=None):
    """annealing.py:184-205."""
    n, d = X32.shape
    cw32 = np.zeros((M, K, d), dtype=np.float32)
    codes = np.zeros((n, M), dtype=np.int64)
    X64 = X32.astype(np.float64)
    for m in range(M):
        inter = heat_up(X32, cw32, codes, m)
        cw32[m], codes[:, m] = cool_down(inter, cw32, m, stages, iters)
        if steps is not None:
            steps.append((0, m, float(row_errors(cw32.astype(np.float64), X64, codes).mean())))
    return cw32, codes


def anneal(X32, cw32, codes, L, stages, iters, sweeps, rel_tol, steps):
    """annealing.py:208-222."""
    P, sq = cross_table(cw32)
    prev = float(row_errors(cw32.astype(np.float64), X32.astype(np.float64), codes).mean())
    for s in range(1, sweeps + 1):
        cw32, codes, P, sq = sweep(X32, cw32, codes, P, sq, L, stages, iters, steps, s)
        cur = steps[-1][2] if steps else prev
        if prev > 0 and (prev - cur) / prev < rel_tol:
            break
        prev = cur
    return cw32, codes


def train_from_scratch(X32, M, K, L=10, stages=10, sweeps=3, rel_tol=1e-3, iters=30):
    """annealing.py:225-245 -> (codewords float32 reordered, codes, steps, order)."""
    steps: list = []
    cw32, codes = growth(X32, M, K, stages, iters, steps)
    cw32, codes = anneal(X32, cw32, codes, L, stages, iters, sweeps, rel_tol, steps)
    perm = variance_order(cw32)
    return cw32[perm].copy(), codes[:, perm], steps, perm


def train_online(cw32, X32, L=10, stages=10, sweeps=3, rel_tol=1e-3, iters=30):
    """annealing.py:248-262 -> (codewords float32, steps)."""
    steps: list = []
    P, _ = cross_table(cw32)
    codes = encode_chunked(cw32, P, X32, L)
    cw32, _ = anneal(X32, cw32, codes, L, stages, iters, sweeps, rel_tol, steps)
    return cw32, steps


def beam_min_gap(cw64: np.ndarray, P: np.ndarray, X64: np.ndarray, L: int) -> np.ndarray:
    """Per vector, the smallest relative decision gap the beam faces: at every
    stage the gap between the kept L-th and the first dropped candidate, and at
    the end between the best and second-best beam, each divided by
    (score + ||x||^2), i.e. by the squared distance.  Vectors
    whose gap is < 1e-6 are oracle near-ties, exempt from code bit-parity."""
    n = X64.shape[0]
    M, K, d = cw64.shape
    xx = (X64 * X64).sum(axis=1)
    t = np.einsum("mkd,mkd->mk", cw64, cw64).reshape(1, M, K) - 2.0 * (
        X64 @ cw64.reshape(M * K, d).T).reshape(n, M, K)
    gap = np.full(n, np.inf)

    def boundary(cand, keep):
        if cand.shape[1] > keep:
            srt = np.sort(cand, axis=1)
            g = (srt[:, keep] - srt[:, keep - 1]) / np.maximum(np.abs(srt[:, keep - 1] + xx), 1e-300)
            np.minimum(gap, g, out=gap)

    keep = min(L, K)
    boundary(t[:, 0, :], keep)
    pick = np.sort(np.argsort(t[:, 0, :], axis=1, kind="stable")[:, :keep], axis=1)
    paths = pick[:, :, None].astype(np.int64)
    score = np.take_along_axis(t[:, 0, :], pick, axis=1)
    for m in range(1, M):
        live = paths.shape[1]
        cross = np.zeros((n, live, K))
        for j in range(m):
            cross += P[j, m][paths[:, :, j], :]
        cand = (score[:, :, None] + t[:, m, :][:, None, :] + 2.0 * cross).reshape(n, live * K)
        keep = min(L, live * K)
        boundary(cand, keep)
        pick = np.sort(np.argsort(cand, axis=1, kind="stable")[:, :keep], axis=1)
        paths = np.concatenate(
            [np.take_along_axis(paths, (pick // K)[:, :, None], axis=1), (pick % K)[:, :, None].astype(np.int64)],
            axis=2)
        score = np.take_along_axis(cand, pick, axis=1)
    if score.shape[1] > 1:
        boundary(score, 1)
    return gap


# ---------------------------------------------------------------------------
# A-Tree traversal (atree.py:336-475; compiled form _traverse.py:52-255)


def _keep_first_smallest(vals: np.ndarray, count: int) -> np.ndarray:
    """Mask of the `count` smallest; among values equal to the count-th
    smallest the earliest positions win (_traverse.py:26-48)."""
    n = vals.size
    if n <= count:
        return np.ones(n, dtype=bool)
    kth = np.partition(vals, count - 1)[count - 1]
    keep = vals < kth
    need = count - int(keep.sum())
    eq = np.flatnonzero(vals == kth)[:need]
    keep[eq] = True
    return keep


def atree_traverse(ts, q_sq, tree, budgets, r):
    """Per-query layered search -> (ids, dists, nodes_visited, table_lookups,
    per_layer).  `ts` = adc values - ||q||^2 (M, K); `tree` has the ATree
    arrays (atree.py:91-117).  Distances accumulate as in the compiled kernel:
    internal steps (d + ts) + 2 eps, suffix steps d + (ts + 2 eps)."""
    M = ts.shape[0]
    code, eps = tree.code, tree.eps.astype(np.float64)
    s_code, s_eps = tree.suffix_code, tree.suffix_eps.astype(np.float64)
    visited = lookups = 0
    per_layer = []
    nodes = np.arange(tree.n_root_children, dtype=np.int64)
    nd = np.array([(q_sq + ts[0, code[v]]) + 2.0 * eps[v] for v in nodes])
    internal = np.empty(0, dtype=np.int64)
    idist = np.empty(0)
    leaves = np.empty(0, dtype=np.int64)
    lpos = np.empty(0, dtype=np.int64)
    ldist = np.empty(0)
    for layer in range(M):
        if layer > 0:
            if internal.size == 0 and leaves.size <= int(np.min(budgets[layer:])):
                rem = M - layer
                for j in range(leaves.size):
                    acc = ldist[j]
                    for t in range(rem):
                        acc += ts[layer + t, s_code[lpos[j] + t]] + 2.0 * s_eps[lpos[j] + t]
                    ldist[j] = acc
                lookups += leaves.size * rem
                per_layer += [leaves.size] * rem
                break
            nn, dd = [], []
            for v, pdv in zip(internal, idist):
                for c in range(tree.child_lo[v], tree.child_hi[v]):
                    nn.append(c)
                    dd.append((pdv + ts[layer, code[c]]) + 2.0 * eps[c])
            nodes = np.array(nn, dtype=np.int64)
            nd = np.array(dd)
            for j in range(leaves.size):
                p = lpos[j]
                ldist[j] += ts[layer, s_code[p]] + 2.0 * s_eps[p]
            lpos = lpos + 1
            lookups += leaves.size
        visited += nodes.size
        lookups += nodes.size
        b = int(budgets[layer])
        size = nodes.size + leaves.size
        per_layer.append(min(size, b))
        if size > b:
            keep = _keep_first_smallest(np.concatenate([nd, ldist]), b)
            kn, kl = keep[:nodes.size], keep[nodes.size:]
            nodes, nd = nodes[kn], nd[kn]
            leaves, lpos, ldist = leaves[kl], lpos[kl], ldist[kl]
        is_leaf = tree.leaf_ref[nodes] >= 0
        enter = tree.leaf_ref[nodes[is_leaf]]
        leaves = np.concatenate([enter, leaves])
        lpos = np.concatenate([tree.suffix_lo[enter], lpos])
        ldist = np.concatenate([nd[is_leaf], ldist])
        internal, idist = nodes[~is_leaf], nd[~is_leaf]
    out_ids, out_d = [], []
    for j, lf in enumerate(leaves):
        for p in range(tree.ids_lo[lf], tree.ids_hi[lf]):
            out_ids.append(tree.leaf_ids[p])
            out_d.append(ldist[j])
    out_ids = np.array(out_ids, dtype=np.int64)
    out_d = np.array(out_d)
    order = np.lexsort((out_ids, out_d))[:r]
    return out_ids[order], out_d[order], visited, lookups, per_layer
