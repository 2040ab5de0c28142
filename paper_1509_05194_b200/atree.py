"""A-Tree: prefix tree over the DA codes, searched on the GPU.

Same data structure and public API as the reference (`annq/atree.py`):

* `build_atree(encoded, codebook, cross)` -> `ATree` (flat arrays; node ids
  level by level in code order, children contiguous, leaf-suffix compression;
  `atree.py:158-324`).  Built on the host: it is a one-off sort-and-scan over
  the codes, not part of the per-query hot path.
* `atree_search(tree, codebook, q, params)` -> (ids, distances, SearchStats)
  (`atree.py:336-475`, `_traverse.py:52-255`) and the batched
  `atree_search_batch(tree, codebook, Q, params)`.  One CTA per query walks the
  layers: expand the surviving internal nodes, advance the in-suffix leaves,
  keep the layer budget by distance (boundary ties keep the earliest entries),
  split into internals and entering leaves, and finally take the r best ids by
  (distance, id).  Tables come from the ADC LUT kernel (`da_adc_lut`).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _engine as E
from ._engine import P
from ._native import native
from .validation import FormatError, check_query

__all__ = ["SearchParams", "SearchStats", "ATree", "build_atree", "atree_search", "atree_search_batch",
           "node_distance"]


@dataclass(frozen=True)
class SearchParams:
    """Per-layer candidate budgets, explicit or geometric (l0 * ls ** i) (atree.py:50-72)."""

    l0: int = 8
    ls: float = 2.0
    r: int = 10
    budgets: tuple | None = None

    def __post_init__(self):
        if self.r < 1:
            raise ValueError("r must be >= 1")
        if self.budgets is None and (self.l0 < 1 or self.ls <= 0):
            raise ValueError("l0 must be >= 1 and ls > 0")

    def layer_budgets(self, m_count: int) -> np.ndarray:
        if self.budgets is not None:
            b = np.asarray(self.budgets, dtype=np.int64)
            if b.shape != (m_count,) or (b < 1).any():
                raise ValueError(f"budgets must be {m_count} positive ints")
            return b
        i = np.arange(1, m_count + 1, dtype=np.float64)
        return np.maximum(np.floor(self.l0 * self.ls ** i + 0.5), 1.0).astype(np.int64)


@dataclass
class SearchStats:
    nodes_visited: int = 0
    table_lookups: int = 0
    per_layer_sizes: list = field(default_factory=list)
    table_seconds: float = 0.0
    traversal_seconds: float = 0.0


@dataclass
class ATree:
    """Flat-array tree (atree.py:91-133); children of a node occupy a contiguous id range."""

    codebook_hash: bytes
    m_count: int
    k_count: int
    n_root_children: int
    code: np.ndarray
    eps: np.ndarray
    child_lo: np.ndarray
    child_hi: np.ndarray
    leaf_ref: np.ndarray
    suffix_lo: np.ndarray
    suffix_hi: np.ndarray
    suffix_code: np.ndarray
    suffix_eps: np.ndarray
    ids_lo: np.ndarray
    ids_hi: np.ndarray
    leaf_ids: np.ndarray

    @property
    def leaf_count(self) -> int:
        return self.suffix_lo.shape[0]

    @property
    def internal_count(self) -> int:
        return self.code.shape[0] - self.leaf_count

    @property
    def node_count(self) -> int:
        return self.code.shape[0]

    @property
    def n_ids(self) -> int:
        return self.leaf_ids.shape[0]


def _eps_of(products, U_rows: np.ndarray, depth: int) -> np.ndarray:
    """epsilon = sum_{i<depth} c_i . c_depth over code rows, accumulated from 0
    in i order in float64, stored as float32 (atree.py:150-155)."""
    return _eps_cols(products, [U_rows[:, i] for i in range(depth + 1)], depth)


def _eps_cols(products, cols, depth: int) -> np.ndarray:
    """_eps_of on per-depth code columns (1-D arrays, cols[i] = codes at depth i)."""
    acc = np.zeros(cols[depth].shape[0])
    for i in range(depth):
        acc = acc + products[i, depth][cols[i], cols[depth]]
    return acc.astype(np.float32)


def build_atree(encoded, codebook, cross=None) -> ATree:
    """Prefix tree with leaf-suffix compression, identical arrays to atree.py:158-324."""
    from .codebook import cross_products

    h = codebook.content_hash()
    if encoded.codebook_hash is not None and encoded.codebook_hash != h:
        raise FormatError("encoded dataset was produced by a different codebook", exit_code=2)
    if encoded.m_count != codebook.m_count or encoded.k_count != codebook.k_count:
        raise ValueError("encoded shape does not match the codebook")
    if cross is None:
        cross = cross_products(codebook)
    M, n = codebook.m_count, encoded.n
    i64, i32, f32 = np.int64, np.int32, np.float32
    if n == 0:
        e = np.empty(0, dtype=i64)
        return ATree(h, M, codebook.k_count, 0, np.empty(0, i32), np.empty(0, f32), e, e, e, e, e,
                     np.empty(0, i32), np.empty(0, f32), e, e, e)
    ids = np.arange(n, dtype=i64) if encoded.id_map is None else np.asarray(encoded.id_map, dtype=i64)
    codes = np.asarray(encoded.codes).astype(i64)
    # rows in lexicographic code order (stable), then distinct full codes
    bits = max(1, int(codebook.k_count - 1).bit_length())
    if bits * M <= 64:
        # one packed key (code 0 most significant): a single stable radix sort
        key = np.zeros(n, dtype=np.uint64)
        for m in range(M):
            key = (key << np.uint64(bits)) | codes[:, m].astype(np.uint64)
        order = np.argsort(key, kind="stable")
    else:
        order = np.lexsort([codes[:, m] for m in range(M - 1, -1, -1)])
    S = codes[order]
    ids_sorted = ids[order]
    first = np.ones(n, dtype=bool)
    if n > 1:
        first[1:] = np.any(S[1:] != S[:-1], axis=1)
    U = S[first]
    g = U.shape[0]
    gstart = np.flatnonzero(first)
    gend = np.append(gstart[1:], n)
    # differs[m, i]: prefix U[i, :m+1] differs from U[i-1, :m+1] (row 0 starts one)
    differs = np.ones((M, g), dtype=bool)
    if g > 1:
        running = np.zeros(g - 1, dtype=bool)
        for m in range(M):
            running |= U[1:, m] != U[:-1, m]
            differs[m, 1:] = running
    products = cross.products

    # level by level: a depth-m prefix is a node iff its parent node is internal;
    # it is a leaf iff exactly one distinct code lies under it
    levels = []
    parent_internal = None   # per depth-(m-1) prefix index: parent node is internal (materialised)
    for m in range(M):
        starts = np.flatnonzero(differs[m])
        width = np.append(starts[1:], g) - starts
        if m == 0:
            exists = np.ones(starts.size, dtype=bool)
        else:
            prev_prefix_of_row = np.cumsum(differs[m - 1]) - 1
            exists = parent_internal[prev_prefix_of_row[starts]]
        leaf = width == 1
        rows = starts[exists]
        levels.append({"rows": rows, "leaf": leaf[exists],
                       "parent_prefix": (np.cumsum(differs[m - 1]) - 1)[rows] if m else None})
        # internal & existing, per depth-m prefix (for the next level)
        parent_internal = exists & ~leaf

    # global ids: level m occupies [base_m, base_m + count_m)
    counts = [lv["rows"].size for lv in levels]
    bases = np.concatenate([[0], np.cumsum(counts)]).astype(i64)
    total = int(bases[-1])
    code_a = np.empty(total, dtype=i32)
    eps_a = np.empty(total, dtype=f32)
    child_lo = np.zeros(total, dtype=i64)
    child_hi = np.zeros(total, dtype=i64)
    leaf_ref = np.full(total, -1, dtype=i64)
    leaf_row, leaf_depth = [], []
    n_leaf = 0
    Uc = np.ascontiguousarray(U.T)          # code columns: 1-D gathers below
    for m, lv in enumerate(levels):
        rows, base = lv["rows"], int(bases[m])
        cols = [Uc[i][rows] for i in range(m + 1)]
        code_a[base:base + rows.size] = cols[m]
        eps_a[base:base + rows.size] = _eps_cols(products, cols, m)
        if m > 0 and rows.size:
            # parent of each node = the position of its depth-(m-1) prefix among the
            # previous level's nodes; children are contiguous in code order
            prev = levels[m - 1]
            prev_prefix_ids = (np.cumsum(differs[m - 1]) - 1)[prev["rows"]]
            slot = np.searchsorted(prev_prefix_ids, lv["parent_prefix"])
            cnt = np.bincount(slot, minlength=prev["rows"].size)
            off = np.concatenate([[0], np.cumsum(cnt)])
            pb = int(bases[m - 1])
            child_lo[pb:pb + cnt.size] = base + off[:-1]
            child_hi[pb:pb + cnt.size] = base + off[1:]
        lf = np.flatnonzero(lv["leaf"])
        leaf_ref[base + lf] = n_leaf + np.arange(lf.size)
        n_leaf += lf.size
        leaf_row.append(rows[lf])
        leaf_depth.append(np.full(lf.size, m, dtype=i64))
    child_lo[leaf_ref >= 0] = 0
    child_hi[leaf_ref >= 0] = 0
    leaf_row = np.concatenate(leaf_row)
    leaf_depth = np.concatenate(leaf_depth)

    # compressed suffixes: depths depth+1 .. M-1 of the leaf's single code
    slen = (M - 1) - leaf_depth
    suffix_lo = np.concatenate([[0], np.cumsum(slen)[:-1]]).astype(i64)
    suffix_hi = suffix_lo + slen
    suffix_code = np.empty(int(slen.sum()), dtype=i32)
    suffix_eps = np.empty(int(slen.sum()), dtype=f32)
    Lc = [Uc[i][leaf_row] for i in range(M)]   # code columns of the leaves' rows
    for t in range(1, M):
        sel = np.flatnonzero(leaf_depth < t)
        if sel.size:
            at = suffix_lo[sel] + (t - 1 - leaf_depth[sel])
            cols = [Lc[i][sel] for i in range(t + 1)]
            suffix_code[at] = cols[t]
            suffix_eps[at] = _eps_cols(products, cols, t)

    # vector ids of each leaf, ascending
    cnt = gend[leaf_row] - gstart[leaf_row]
    ids_lo = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(i64)
    ids_hi = ids_lo + cnt
    if encoded.id_map is None:
        ids_g = ids_sorted            # the stable sort kept row order inside each group
    else:
        gid = np.cumsum(first) - 1    # ids ascending inside each group: sort by (group, id)
        ids_g = ids_sorted[np.lexsort((ids_sorted, gid))]
    total_ids = int(cnt.sum())
    pos = np.repeat(gstart[leaf_row] - ids_lo, cnt) + np.arange(total_ids, dtype=i64)
    leaf_ids = ids_g[pos]
    return ATree(h, M, codebook.k_count, int(counts[0]), code_a, eps_a, child_lo, child_hi, leaf_ref,
                 suffix_lo, suffix_hi, suffix_code, suffix_eps, ids_lo, ids_hi, leaf_ids)


def node_distance(parent_dist: float, table, code: int, epsilon: float, layer: int, q_sq_norm: float) -> float:
    """One path step (atree.py:327-333)."""
    return parent_dist + table[layer, code] - q_sq_norm + 2.0 * epsilon


_TREE_FIELDS = ("code", "eps", "child_lo", "child_hi", "leaf_ref", "suffix_lo", "suffix_hi", "suffix_code",
                "suffix_eps", "ids_lo", "ids_hi", "leaf_ids")


def _tree_dev(tree):
    """Device copies of the tree arrays (cached on the tree object)."""
    dev = E.device()
    cache = getattr(tree, "__dict__", {}).get("_dev_cache")
    if cache is not None and cache[0] == dev and cache[1] is tree.code:
        return cache[2]
    want = {"code": np.int32, "eps": np.float32, "suffix_code": np.int32, "suffix_eps": np.float32}
    arrs = {}
    for f in _TREE_FIELDS:
        a = np.ascontiguousarray(getattr(tree, f), dtype=want.get(f, np.int64))
        arrs[f] = E.to_dev(a if a.size else np.zeros(1, dtype=a.dtype))
    lens = np.asarray(tree.child_hi) - np.asarray(tree.child_lo)
    arrs["max_children"] = int(max(int(lens.max()) if lens.size else 0, int(tree.n_root_children)))
    try:
        tree.__dict__["_dev_cache"] = (dev, tree.code, arrs)
    except (AttributeError, TypeError):
        pass
    return arrs


def atree_search_batch(tree, codebook, Q, params: SearchParams):
    """Batched search -> (ids (nq, r) int64 padded with -1, dists (nq, r) padded with nan,
    counts (nq,), stats (nq, 2 + M): nodes_visited, table_lookups, per-layer sizes)."""
    from .codebook import _codebook_dev

    if tree.codebook_hash != codebook.content_hash():
        raise FormatError("tree was built against a different codebook", exit_code=2)
    Q = np.asarray(Q, dtype=np.float64)
    if Q.ndim != 2 or Q.shape[1] != codebook.dim:
        raise ValueError(f"queries must be (nq, {codebook.dim})")
    if not np.isfinite(Q).all():
        raise ValueError("queries contain non-finite values")
    M, r, nq = tree.m_count, int(params.r), Q.shape[0]
    budgets = params.layer_budgets(M)
    if tree.node_count == 0 or nq == 0:
        return (np.full((nq, r), -1, dtype=np.int64), np.full((nq, r), np.nan), np.zeros(nq, dtype=np.int64),
                np.zeros((nq, 2 + M), dtype=np.int64))
    cw, sq = _codebook_dev(codebook)
    lut, qsq = E.adc_lut(E.to_dev(Q), cw, sq)
    return _search_tables(tree, lut, qsq, budgets, r)


def _search_tables(tree, lut: torch.Tensor, qsq: torch.Tensor, budgets: np.ndarray, r: int):
    """Traversal on given device tables lut (nq, M, K) and qsq (nq,)."""
    nq, M = lut.shape[0], tree.m_count
    t = _tree_dev(tree)
    dev = lut.device
    b_h = np.ascontiguousarray(budgets, dtype=np.int64)
    ids = torch.empty((nq, r), dtype=torch.int64, device=dev)
    dists = torch.empty((nq, r), dtype=torch.float64, device=dev)
    cnt = torch.empty(nq, dtype=torch.int64, device=dev)
    stats = torch.empty((nq, 2 + M), dtype=torch.int64, device=dev)
    native.da_atree_search(P(lut), P(qsq), nq, M, lut.shape[2],
                           P(t["code"]), P(t["eps"]), P(t["child_lo"]), P(t["child_hi"]), P(t["leaf_ref"]),
                           P(t["suffix_lo"]), P(t["suffix_code"]), P(t["suffix_eps"]), P(t["ids_lo"]),
                           P(t["ids_hi"]), P(t["leaf_ids"]), tree.node_count, tree.leaf_count,
                           int(tree.n_root_children), t["max_children"], b_h.ctypes.data, r,
                           P(ids), P(dists), P(cnt), P(stats), E.stream())
    return ids.cpu().numpy(), dists.cpu().numpy(), cnt.cpu().numpy(), stats.cpu().numpy()


def atree_search(tree, codebook, q, params: SearchParams, use_kernel=None):
    """Non-exhaustive top-r search for one query (atree.py:336-475)."""
    import time

    q = check_query(q, codebook.dim)
    t0 = time.perf_counter()
    ids, d, cnt, st = atree_search_batch(tree, codebook, q.reshape(1, -1), params)
    k = int(cnt[0])
    M = tree.m_count
    stats = SearchStats(nodes_visited=int(st[0, 0]), table_lookups=int(st[0, 1]),
                        per_layer_sizes=[int(v) for v in st[0, 2:2 + M] if v >= 0])
    stats.traversal_seconds = time.perf_counter() - t0
    return ids[0, :k].copy(), d[0, :k].copy(), stats
