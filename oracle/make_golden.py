"""Generate tests/golden/*.npz by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    python oracle/make_golden.py [--skip-slow]

The fixtures pin both the CPU oracle (tests/test_oracle_golden.py, CPU) and
the CUDA path (tests/test_gpu_parity.py, GPU).  Inputs are regenerated from
seeds in tests (they are small); outputs are stored.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden")
sys.path.insert(0, os.path.join(HERE, ".."))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from paper_1509_05194_b200 import synthetic  # noqa: E402  (generators only)

sys.path.insert(0, REF)
import annq  # noqa: E402
from annq import clustering as rcl  # noqa: E402
from annq import codebook as rcb  # noqa: E402

sys.path.insert(0, os.path.join(HERE, "..", "tests"))
import cases  # noqa: E402  (seeded small inputs shared with the tests)


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def np_order():
    c = cases.np_order_inputs()
    segs = []
    for arr in c["seg_arrays"]:
        segs.append(np.add.reduceat(arr, [0], axis=0)[0])
    save("np_order.npz",
         pairwise=np.array([a.sum() for a in c["vectors"]]),
         rowsum=np.array([(a * a).sum() for a in c["vectors"]]),
         mean=np.array([a.mean() for a in c["vectors"]]),
         einsum=np.concatenate([np.einsum("kd,kd->k", m, m) for m in c["matrices"]]),
         reduceat=np.concatenate(segs))


def small_ops():
    out = {}
    c = cases.assign_case()
    lab, d2 = rcl._assign(c["X"][:, : c["active"]], c["C"][:, : c["active"]])
    out.update(assign_labels=lab, assign_d2=d2)
    c = cases.group_case()
    means, counts = rcl._group_means(c["X"], c["labels"], c["k"])
    out.update(group_means=means, group_counts=counts)
    c = cases.lloyd_case()
    fit = rcl.lloyd_kmeans(c["X"], c["C"], active_dims=c["active"], max_iters=c["iters"])
    out.update(lloyd_points=fit.points, lloyd_assign=fit.assignment, lloyd_trace=np.array(fit.objective_trace))
    c = cases.reseed_case()
    fit = rcl.lloyd_kmeans(c["X"], c["C"], max_iters=c["iters"])
    out.update(reseed_points=fit.points, reseed_assign=fit.assignment, reseed_trace=np.array(fit.objective_trace))
    c = cases.pca_case()
    pm = rcl.pca_fit(c["X"])
    out.update(pca_rotation=pm.rotation, pca_mean=pm.mean, pca_var=pm.explained_variance)
    pg = rcl.pca_fit(c["Xgram"])
    out.update(pcag_rotation=pg.rotation, pcag_mean=pg.mean, pcag_var=pg.explained_variance)
    c = cases.staged_case()
    fit = rcl.improved_kmeans(c["X"], c["C"], max_iters=c["iters"])
    out.update(staged_points=fit.points, staged_assign=fit.assignment, staged_trace=np.array(fit.objective_trace))
    c = cases.codebook_case()
    book = annq.Codebook(codewords=c["cw"], order=np.arange(c["cw"].shape[0]))
    cross = rcb.cross_products(book)
    out.update(cross_P=cross.products, cross_sq=cross.sq_norms)
    ref2 = rcb.refresh_cross_products(cross, annq.Codebook(codewords=c["cw2"], order=np.arange(c["cw"].shape[0])), 1)
    out.update(refresh_P=ref2.products, refresh_sq=ref2.sq_norms)
    for L in cases.BEAM_WIDTHS:
        codes, errs = rcb._beam_encode_chunk(c["cw"].astype(np.float64), cross, c["X"].astype(np.float64), L)
        out[f"beam_codes_L{L}"] = codes
        out[f"beam_errs_L{L}"] = errs
        enc = rcb.encode_dataset(book, c["X"], beam_width=L)
        out[f"enc_codes_L{L}"] = enc.codes
    code, err = rcb.encode_multipath(book, cross, c["q"], 4)
    out.update(multipath_code=code, multipath_err=np.array(err))
    t = rcb.adc_table(book, c["q"])
    out.update(adc_values=t.values, adc_qsq=np.array(t.q_sq_norm))
    enc = rcb.encode_dataset(book, c["X"], beam_width=8)
    pair = rcb.code_pair_sums(cross, enc.codes.astype(np.int64))
    ids, dists = rcb.exhaustive_adc_search(book, enc, c["q"], 10, cross=cross, pair_sums=pair)
    out.update(pair_sums=pair, search_ids=ids, search_dists=dists)
    out.update(distortion=np.array(rcb.distortion(book, c["X"], enc)))
    save("small_ops.npz", **out)


def small_training():
    out = {}
    c = cases.sweep_case()
    book = annq.Codebook(codewords=c["cw"], order=np.arange(c["cw"].shape[0]))
    enc = rcb.encode_dataset(book, c["X"], beam_width=8)
    inter = annq.heat_up(c["X"], book, enc, 1)
    out.update(sweep_init_codes=enc.codes, heat_up_1=inter)
    cfg = annq.TrainConfig(m_count=3, k_count=8, sweeps=1, beam_width=8)
    nd, asg = annq.cool_down(inter, book, 1, cfg)
    out.update(cool_dict=nd, cool_assign=asg)
    rep = annq.TrainReport(config=cfg)
    b2, e2, x2 = annq.da_sweep(c["X"], book, enc, cfg, report=rep)
    out.update(sweep_cw=b2.codewords, sweep_codes=e2.codes, sweep_dist=rep.distortions(), sweep_P=x2.products)
    c = cases.train_case()
    cfg = annq.TrainConfig(**c["config"])
    b, e, r = annq.train_from_scratch(c["X"], cfg)
    out.update(train_cw=b.codewords, train_order=b.order, train_codes=e.codes, train_dist=r.distortions())
    rb, re_ = annq.rvq_train(c["X"], cfg)
    out.update(rvq_cw=rb.codewords, rvq_codes=re_.codes)
    b3, r3 = annq.train_online(b, c["X2"], cfg)
    out.update(online_cw=b3.codewords, online_order=b3.order, online_dist=r3.distortions())
    save("small_training.npz", **out)


def config_a():
    X = synthetic.config_a()
    cfg = annq.TrainConfig(m_count=4, k_count=256, beam_width=10, sweeps=3, rel_tol=0.0, kmeans_iters=30,
                           schedule_stages=10)
    t0 = time.perf_counter()
    b, e, r = annq.train_from_scratch(X, cfg)
    dt = time.perf_counter() - t0
    mse = rcb.distortion(b, X, e)
    print(f"config A: {dt:.1f}s, MSE {mse:.10f}")
    save("config_a.npz", cw=b.codewords, order=b.order, codes=e.codes, dist=r.distortions(), mse=np.array(mse),
         seconds=np.array(dt))


def config_b_sub():
    X = synthetic.config_b(n=cases.B_TRAIN + cases.B_ENC)
    Xt, Xe = X[: cases.B_TRAIN], X[cases.B_TRAIN:]
    cfg = annq.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
    t0 = time.perf_counter()
    book, enc, rep = annq.train_from_scratch(Xt, cfg)
    print(f"config B growth on {len(Xt)}: {time.perf_counter() - t0:.1f}s")
    cross = rcb.cross_products(book)
    out = dict(cw=book.codewords, order=book.order, train_codes=enc.codes, train_dist=rep.distortions())
    for L in (1, 10):
        t0 = time.perf_counter()
        codes, errs = rcb._beam_encode_chunk(book.codewords.astype(np.float64), cross, Xe.astype(np.float64), L)
        print(f"config B encode L={L} on {len(Xe)}: {time.perf_counter() - t0:.1f}s")
        out[f"enc_codes_L{L}"] = codes.astype(np.uint8)
        out[f"enc_errs_L{L}"] = errs
    rep2 = annq.TrainReport(config=cfg)
    t0 = time.perf_counter()
    cfg1 = annq.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=1, rel_tol=0.0)
    b2, e2, _ = annq.da_sweep(Xt, book, enc, cfg1, report=rep2)
    print(f"config B da_sweep on {len(Xt)}: {time.perf_counter() - t0:.1f}s")
    out.update(sweep_cw=b2.codewords, sweep_codes=e2.codes, sweep_dist=rep2.distortions())
    # ADC: 16 queries against the encoded slice
    Q = synthetic.config_e_queries(16)
    encx = rcb.EncodedDataset(out["enc_codes_L10"], 256)
    pair = rcb.code_pair_sums(cross, encx.codes.astype(np.int64))
    ids, ds = [], []
    for q in Q.astype(np.float64):
        i, d = rcb.exhaustive_adc_search(book, encx, q, 100, cross=cross, pair_sums=pair)
        ids.append(i)
        ds.append(d)
    out.update(adc_pair=pair, adc_ids=np.array(ids), adc_dists=np.array(ds))
    save("config_b_sub.npz", **out)


def config_c_sub():
    X = synthetic.config_c(n=cases.C_TRAIN + cases.C_ENC)
    Xt, Xe = X[: cases.C_TRAIN], X[cases.C_TRAIN:]
    cfg = annq.TrainConfig(m_count=4, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
    t0 = time.perf_counter()
    book, enc, rep = annq.train_from_scratch(Xt, cfg)
    print(f"config C growth on {len(Xt)}: {time.perf_counter() - t0:.1f}s")
    cross = rcb.cross_products(book)
    codes, errs = rcb._beam_encode_chunk(book.codewords.astype(np.float64), cross, Xe.astype(np.float64), 10)
    save("config_c_sub.npz", cw=book.codewords, order=book.order, train_codes=enc.codes,
         train_dist=rep.distortions(), enc_codes=codes.astype(np.uint8), enc_errs=errs)


def meta():
    import json

    import numpy

    info = {"numpy": numpy.__version__}
    try:
        from threadpoolctl import threadpool_info

        info["blas"] = [{k: v for k, v in d.items() if k in ("internal_api", "version", "architecture")}
                        for d in threadpool_info()]
    except Exception:
        pass
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "meta.json"), "w") as f:
        json.dump(info, f, indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-slow", action="store_true")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    jobs = [meta, np_order, small_ops, small_training]
    if not a.skip_slow:
        jobs += [config_b_sub, config_c_sub, config_a]
    for j in jobs:
        if a.only and j.__name__ != a.only:
            continue
        j()
