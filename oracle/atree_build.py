"""Host (numpy) restatement of the reference's A-Tree build (annq/atree.py:
158-324) -- TEST INFRASTRUCTURE: it pins paper_1509_05194_b200.atree.build_atree
(the device build) to the reference's arrays (tests/golden/atree.npz, made by
the reference itself through oracle/make_golden_atree.py).  Nothing in the
package imports it."""

from __future__ import annotations

import numpy as np

from paper_1509_05194_b200.atree import ATree
from paper_1509_05194_b200.validation import FormatError


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


def build_atree_host(encoded, codebook, cross=None) -> ATree:
    """Prefix tree with leaf-suffix compression, identical arrays to atree.py:158-324."""
    from paper_1509_05194_b200.codebook import cross_products

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


