"""Generate tests/golden/atree.npz (A-Tree build + search) and tests/golden/knn.npz
(brute_force_knn) by running the REFERENCE.

Build container only (imports /root/reference/pkg/src):

    python oracle/make_golden_atree.py

Cases:
  * "small": the reference's own `trained_small` system (3000 x 16, M=4, K=16,
    two sweeps; pkg/tests/conftest.py:8-17), its tree, and searches for seeded
    queries under several budget settings (geometric l0/ls, explicit, unbounded);
  * "ties": hand-made codes with many duplicates over a codebook with duplicate
    codewords, so truncations cut through exact distance ties.
Searches use the reference's default traversal (the compiled kernel when numba
is present, `atree.py:360-373`), and the array path for comparison.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)
import annq  # noqa: E402
from annq import atree as rat  # noqa: E402

TREE_FIELDS = ("code", "eps", "child_lo", "child_hi", "leaf_ref", "suffix_lo", "suffix_hi", "suffix_code",
               "suffix_eps", "ids_lo", "ids_hi", "leaf_ids")
PARAMS = [  # (l0, ls, r, budgets or None)
    (1, 2.0, 15, None), (3, 2.0, 15, None), (8, 2.0, 15, None), (64, 2.0, 15, None),
    (4, 2.0, 10, None), (2, 1.0, 7, None), (None, None, 10, "b5000"), (None, None, 20, "bn"),
]


def params_for(p, m, n):
    l0, ls, r, b = p
    if b == "b5000":
        return rat.SearchParams(r=r, budgets=(5000,) * m)
    if b == "bn":
        return rat.SearchParams(r=r, budgets=(n,) * m)
    return rat.SearchParams(l0=l0, ls=ls, r=r)


def run_case(prefix, book, enc, Q, out):
    cross = annq.cross_products(book)
    tree = rat.build_atree(enc, book, cross)
    for f in TREE_FIELDS:
        out[f"{prefix}_tree_{f}"] = getattr(tree, f)
    out[f"{prefix}_tree_meta"] = np.array([tree.n_root_children, tree.m_count, tree.k_count], dtype=np.int64)
    out[f"{prefix}_codewords"] = book.codewords
    out[f"{prefix}_order"] = book.order
    out[f"{prefix}_codes"] = enc.codes
    out[f"{prefix}_queries"] = Q
    M = book.m_count
    for pi, p in enumerate(PARAMS):
        sp = params_for(p, M, enc.n)
        out[f"{prefix}_p{pi}_budgets"] = sp.layer_budgets(M)
        out[f"{prefix}_p{pi}_r"] = np.array([sp.r])
        ids_l, d_l, st_l, same = [], [], [], []
        for q in Q:
            ids, d, st = rat.atree_search(tree, book, q, sp)
            ia, da, _ = rat.atree_search(tree, book, q, sp, use_kernel=False)
            same.append(np.array_equal(ids, ia) and np.array_equal(d, da))
            k = len(ids)
            pad_i = np.full(sp.r, -1, dtype=np.int64)
            pad_d = np.full(sp.r, np.nan)
            pad_i[:k] = ids
            pad_d[:k] = d
            ids_l.append(pad_i)
            d_l.append(pad_d)
            st_l.append([st.nodes_visited, st.table_lookups] + list(st.per_layer_sizes)
                        + [-1] * (M - len(st.per_layer_sizes)))
        out[f"{prefix}_p{pi}_ids"] = np.array(ids_l)
        out[f"{prefix}_p{pi}_dists"] = np.array(d_l)
        out[f"{prefix}_p{pi}_stats"] = np.array(st_l, dtype=np.int64)
        print(prefix, pi, "kernel==array on", int(np.sum(same)), "of", len(Q))


def main():
    out = {}
    # the reference's shared small system (conftest.trained_small)
    X = annq.generate_synthetic(3000, 16, clusters=30, spread=0.1, seed=5)
    config = annq.TrainConfig(m_count=4, k_count=16, sweeps=2, beam_width=10, seed=5)
    book, enc, _ = annq.train_from_scratch(X, config)
    rng = np.random.default_rng(10)
    Q = np.vstack([rng.standard_normal((12, 16)), X[[0, 17, 999]], np.zeros((1, 16))])
    run_case("small", book, enc, Q, out)

    # exact ties: duplicate codewords and many duplicate / shared-prefix codes
    rng = np.random.default_rng(3)
    M, K, D = 3, 4, 6
    cw = rng.standard_normal((M, K, D)).astype(np.float32)
    cw[1, 3] = cw[1, 1]
    cw[2, 2] = cw[2, 0]
    tb = annq.Codebook(codewords=cw, order=np.arange(M, dtype=np.int64))
    codes = rng.integers(0, K, size=(300, M)).astype(np.uint8)
    codes[::7] = codes[3]
    te = annq.EncodedDataset(codes=codes, k_count=K)
    Qt = np.vstack([rng.standard_normal((8, D)), np.zeros((1, D))])
    run_case("ties", tb, te, Qt, out)

    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, "atree.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def knn_fixture():
    """brute_force_knn on a small base with duplicate rows (exact ties)."""
    rng = np.random.default_rng(21)
    base = annq.generate_synthetic(2000, 16, clusters=20, spread=0.2, seed=21)
    base[100:110] = base[5]
    queries = np.vstack([rng.standard_normal((30, 16)).astype(np.float32), base[[5, 7]]])
    out = {"base": base, "queries": queries}
    for r in (1, 10, 37):
        gt = annq.brute_force_knn(base, queries, r)
        out[f"r{r}_ids"] = gt.ids
        out[f"r{r}_dists"] = gt.distances
    path = os.path.join(OUT, "knn.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


if __name__ == "__main__":
    if not os.environ.get("KNN_ONLY"):
        main()
    knn_fixture()
