"""A-Tree: prefix tree over the DA codes, searched on the GPU.

Same data structure and public API as the reference (`annq/atree.py`):

* `build_atree(encoded, codebook, cross)` -> `ATree` (flat arrays; node ids
  level by level in code order, children contiguous, leaf-suffix compression;
  `atree.py:158-324`).  Built on the GPU: stable radix passes of the library's
  counting sort put the codes in lexicographic order, device scans find the
  prefix boundaries, epsilons come from the device cross tables.
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


def _eps_cols(Pt: torch.Tensor, cols, depth: int) -> torch.Tensor:
    """epsilon = sum_{i<depth} c_i . c_depth over per-depth code columns, accumulated
    from 0 in i order in float64 (the reference's order, atree.py:150-155), as
    float32.  Pt: device cross tables (M, M, K, K)."""
    acc = torch.zeros(cols[depth].shape[0], dtype=torch.float64, device=Pt.device)
    for i in range(depth):
        acc = acc + Pt[i, depth][cols[i], cols[depth]]
    return acc.to(torch.float32)


def _lex_order(codes: torch.Tensor, K: int) -> torch.Tensor:
    """Stable lexicographic order of the code rows (code 0 most significant): LSD
    radix passes of the library's stable counting sort (da_label_order), one per
    code column from the last to the first."""
    n, M = codes.shape
    order = torch.arange(n, dtype=torch.int64, device=codes.device)
    o = torch.empty(n, dtype=torch.int32, device=codes.device)
    cnt = torch.empty(K, dtype=torch.int32, device=codes.device)
    for m in range(M - 1, -1, -1):
        lab = codes[order, m].to(torch.int32).contiguous()
        native.da_label_order(P(lab), n, K, P(o), P(cnt), E.stream())
        order = order[o.long()]
    return order


def build_atree(encoded, codebook, cross=None) -> ATree:
    """Prefix tree with leaf-suffix compression, built on the GPU: identical
    arrays to the reference's build (atree.py:158-324).  Rows are put in
    lexicographic code order by stable radix passes (da_label_order), distinct
    codes and per-depth prefix boundaries come from device scans, and node
    epsilons are gathered from the device cross tables in the reference's
    addition order.  oracle/atree_build.py holds the host restatement the tests
    compare against."""
    from .codebook import _cross_dev, cross_products

    h = codebook.content_hash()
    if encoded.codebook_hash is not None and encoded.codebook_hash != h:
        raise FormatError("encoded dataset was produced by a different codebook", exit_code=2)
    if encoded.m_count != codebook.m_count or encoded.k_count != codebook.k_count:
        raise ValueError("encoded shape does not match the codebook")
    if cross is None:
        cross = cross_products(codebook)
    M, n, K = codebook.m_count, encoded.n, codebook.k_count
    i64, i32, f32 = np.int64, np.int32, np.float32
    if n == 0:
        e = np.empty(0, dtype=i64)
        return ATree(h, M, K, 0, np.empty(0, i32), np.empty(0, f32), e, e, e, e, e,
                     np.empty(0, i32), np.empty(0, f32), e, e, e)
    E.require_cuda()
    dev = E.device()
    Pt = _cross_dev(cross)[0] if hasattr(cross, "sq_norms") else E.to_dev(
        np.ascontiguousarray(cross.products, dtype=np.float64))
    T = torch
    codes = T.from_numpy(np.ascontiguousarray(encoded.codes).astype(i64)).to(dev)
    ids = (T.arange(n, dtype=T.int64, device=dev) if encoded.id_map is None
           else T.from_numpy(np.asarray(encoded.id_map, dtype=i64)).to(dev))
    order = _lex_order(codes, K)
    S = codes[order]
    ids_sorted = ids[order]
    first = T.ones(n, dtype=T.bool, device=dev)
    if n > 1:
        first[1:] = (S[1:] != S[:-1]).any(dim=1)
    U = S[first]
    g = U.shape[0]
    gstart = T.nonzero(first).flatten()
    gend = T.cat([gstart[1:], T.tensor([n], dtype=T.int64, device=dev)])
    # differs[m, i]: prefix U[i, :m+1] differs from U[i-1, :m+1] (row 0 starts one)
    differs = T.ones((M, g), dtype=T.bool, device=dev)
    if g > 1:
        neq = (U[1:] != U[:-1]).to(T.int32)
        differs[:, 1:] = neq.cummax(dim=1).values.T.bool()
    prefix_id = [T.cumsum(differs[m].to(T.int64), 0) - 1 for m in range(M)]

    levels = []
    parent_internal = None
    for m in range(M):
        starts = T.nonzero(differs[m]).flatten()
        width = T.cat([starts[1:], T.tensor([g], dtype=T.int64, device=dev)]) - starts
        exists = (T.ones(starts.numel(), dtype=T.bool, device=dev) if m == 0
                  else parent_internal[prefix_id[m - 1][starts]])
        leaf = width == 1
        rows = starts[exists]
        levels.append({"rows": rows, "leaf": leaf[exists],
                       "parent_prefix": prefix_id[m - 1][rows] if m else None})
        parent_internal = exists & ~leaf

    counts = [int(lv["rows"].numel()) for lv in levels]
    bases = np.concatenate([[0], np.cumsum(counts)]).astype(i64)
    total = int(bases[-1])
    code_a = T.empty(total, dtype=T.int32, device=dev)
    eps_a = T.empty(total, dtype=T.float32, device=dev)
    child_lo = T.zeros(total, dtype=T.int64, device=dev)
    child_hi = T.zeros(total, dtype=T.int64, device=dev)
    leaf_ref = T.full((total,), -1, dtype=T.int64, device=dev)
    leaf_row, leaf_depth = [], []
    n_leaf = 0
    Uc = U.T.contiguous()
    for m, lv in enumerate(levels):
        rows, base = lv["rows"], int(bases[m])
        R = rows.numel()
        cols = [Uc[i][rows] for i in range(m + 1)]
        code_a[base:base + R] = cols[m].to(T.int32)
        eps_a[base:base + R] = _eps_cols(Pt, cols, m)
        if m > 0 and R:
            prev = levels[m - 1]
            prev_prefix_ids = prefix_id[m - 1][prev["rows"]]
            slot = T.searchsorted(prev_prefix_ids, lv["parent_prefix"])
            cnt = T.bincount(slot, minlength=prev["rows"].numel())
            off = T.cat([T.zeros(1, dtype=T.int64, device=dev), T.cumsum(cnt, 0)])
            pb = int(bases[m - 1])
            child_lo[pb:pb + cnt.numel()] = base + off[:-1]
            child_hi[pb:pb + cnt.numel()] = base + off[1:]
        lf = T.nonzero(lv["leaf"]).flatten()
        leaf_ref[base + lf] = n_leaf + T.arange(lf.numel(), dtype=T.int64, device=dev)
        n_leaf += lf.numel()
        leaf_row.append(rows[lf])
        leaf_depth.append(T.full((lf.numel(),), m, dtype=T.int64, device=dev))
    is_leaf = leaf_ref >= 0
    child_lo[is_leaf] = 0
    child_hi[is_leaf] = 0
    leaf_row = T.cat(leaf_row)
    leaf_depth = T.cat(leaf_depth)

    # compressed suffixes: depths depth+1 .. M-1 of the leaf's single code
    slen = (M - 1) - leaf_depth
    csl = T.cumsum(slen, 0)
    suffix_lo = T.cat([T.zeros(1, dtype=T.int64, device=dev), csl[:-1]])
    suffix_hi = suffix_lo + slen
    ns = int(csl[-1].item()) if csl.numel() else 0
    suffix_code = T.empty(ns, dtype=T.int32, device=dev)
    suffix_eps = T.empty(ns, dtype=T.float32, device=dev)
    Lc = [Uc[i][leaf_row] for i in range(M)]
    for t in range(1, M):
        sel = T.nonzero(leaf_depth < t).flatten()
        if sel.numel():
            at = suffix_lo[sel] + (t - 1 - leaf_depth[sel])
            cols = [Lc[i][sel] for i in range(t + 1)]
            suffix_code[at] = cols[t].to(T.int32)
            suffix_eps[at] = _eps_cols(Pt, cols, t)

    # vector ids of each leaf, ascending
    cnt = gend[leaf_row] - gstart[leaf_row]
    ccnt = T.cumsum(cnt, 0)
    ids_lo = T.cat([T.zeros(1, dtype=T.int64, device=dev), ccnt[:-1]])
    ids_hi = ids_lo + cnt
    if encoded.id_map is None:
        ids_g = ids_sorted            # the stable sort kept row order inside each group
    else:
        gid = T.cumsum(first.to(T.int64), 0) - 1   # ids ascending inside each group
        o1 = T.sort(ids_sorted, stable=True).indices
        o2 = T.sort(gid[o1], stable=True).indices
        ids_g = ids_sorted[o1[o2]]
    total_ids = int(ccnt[-1].item()) if ccnt.numel() else 0
    pos = T.repeat_interleave(gstart[leaf_row] - ids_lo, cnt) + T.arange(total_ids, dtype=T.int64, device=dev)
    leaf_ids = ids_g[pos]
    host = lambda t: t.cpu().numpy()
    return ATree(h, M, K, int(counts[0]), host(code_a), host(eps_a), host(child_lo), host(child_hi), host(leaf_ref),
                 host(suffix_lo), host(suffix_hi), host(suffix_code), host(suffix_eps), host(ids_lo), host(ids_hi),
                 host(leaf_ids))


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
