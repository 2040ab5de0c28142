"""Benchmark of the DA hot path on BASELINE.json config B (configs[1]).

Workload: N=1,000,000 vectors per GPU, D=128, fp32 holding integers in
[0,255] (seeded synthetic stand-in for SIFT1M, see paper_1509_05194_b200/
synthetic.py), M=8 dictionaries x K=256 codewords, beam width L=10.
One step = one beam encode of the GPU's 1M resident vectors.  Each rank
encodes its own shard (weak scaling, no data-path collective).  The codebook
is trained on the device first (growth pass on a 100k subsample, untimed).
Also reported: L=1 encode rate, one full anneal pass (da_sweep) at N=1M in
seconds, the end-to-end rate through the public API (host arrays in, host
codes out), the CPU reference timed on this host, and the dominant kernel's
roofline from live CUDA-event timing.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DA encode vectors/s (D=128,M=8,K=256) & anneal-pass sec; % of roofline"
N_PER_GPU = 1_000_000
D, M, K, L = 128, 8, 256, 10
TRAIN_SUB = 100_000


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=N_PER_GPU, help="vectors per GPU")
    ap.add_argument("--no-anneal", action="store_true", help="skip the full anneal-pass timing")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--no-adc", action="store_true", help="skip the config-E ADC scan timing")
    ap.add_argument("--no-atree", action="store_true", help="skip the A-Tree build + search timing")
    ap.add_argument("--adc-n", type=int, default=1_000_000_000, help="encoded vectors for the ADC scan")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def rank_data(rank, n):
    """Each rank's own slice of the config-B stream (chunks 4*rank.. of seed 1)."""
    from paper_1509_05194_b200 import synthetic

    chunk = 250_000
    out = np.empty((n, D), dtype=np.float32)
    means = synthetic.mixture_b_params(1)
    for i, c0 in enumerate(range(0, n, chunk)):
        rng = synthetic.substream(1, f"b-chunk-{rank * 4 + i}")
        out[c0:c0 + chunk] = synthetic._draw_b(rng, means, min(chunk, n - c0))
    return out


class Clocks:
    """nvidia-smi sampler for the timed region (clocks + throttle reasons)."""

    def __init__(self, index=0):
        self.samples, self._stop, self.index = [], threading.Event(), index

    def __enter__(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver) + profiles/peaks_r01.jsonl (ours)."""
    out = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            out.update(json.load(f))
    except Exception:
        out["hbm_gbs"] = 6650.0  # B200_PROFILING.md fallback
        out["hbm_source"] = "fallback"
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_r01.jsonl")) as f:
            rows = [json.loads(x) for x in f if x.strip()]
        out["fp64_dfma_tflops"] = max(r["fp64_dfma_tflops"] for r in rows)
        out["fp32_ffma_tflops"] = max(r["fp32_ffma_tflops"] for r in rows)
    except Exception:
        out["fp64_dfma_tflops"], out["fp32_ffma_tflops"] = 34.0, 70.8
    # dense TF32 tensor peak: no measured figure on this pool; B200_PROFILING.md nominal
    out.setdefault("tf32_tflops", 1100.0)
    return out


def cpu_encode_rate(book_cw, X, L_, seconds_budget=15.0):
    """Oracle encode (reference algorithm, numpy + thread pool) on a bounded sample."""
    from oracle import da_oracle as O

    cores = os.cpu_count() or 1
    P, _ = O.cross_table(book_cw)
    n = 2000
    t0 = time.perf_counter()
    O.encode_chunked(book_cw, P, X[:n], L_, n_jobs=cores)
    dt = time.perf_counter() - t0
    # grow the sample to fill the budget (bounded)
    n2 = int(min(len(X), max(n, n * seconds_budget / max(dt, 1e-3) * 0.5)))
    if n2 > n:
        t0 = time.perf_counter()
        O.encode_chunked(book_cw, P, X[:n2], L_, n_jobs=cores)
        dt, n = time.perf_counter() - t0, n2
    return n / dt, cores, n


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1509_05194_b200 import synthetic
    from oracle import da_oracle as O

    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))
    X = rank_data(0, 60_000)
    # codebook: oracle growth pass on a small slice (untimed)
    cw, _ = O.growth(X[:4096], M, K, 10, 30)
    cores = os.cpu_count() or 1
    P, _ = O.cross_table(cw)
    sample = 4000
    for i in range(args.warmup):
        O.encode_chunked(cw, P, X[:500], L, n_jobs=cores)
    times = []
    for s in range(args.steps):
        lo = (s * sample) % (len(X) - sample)
        t0 = time.perf_counter()
        O.encode_chunked(cw, P, X[lo:lo + sample], L, n_jobs=cores)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    v = sample * args.steps / total
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "vectors/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config B encode (D=128,M=8,K=256,L=10)", "sample_per_step": sample,
                   "global_batch": sample, "parallelism": "cpu threads"},
        "cpu_baseline": {"value": v, "unit": "vectors/s", "cores": cores, "kind": "port",
                         "sample": f"{sample} config-B vectors per step, oracle encode_dataset restatement"},
        "e2e": {"value": v, "unit": "vectors/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1509_05194_b200 as da
    from paper_1509_05194_b200 import _engine as E
    from paper_1509_05194_b200 import _native

    n = args.n
    X_h = rank_data(rank, n)
    X = E.to_dev(X_h)
    # --- codebook (untimed): growth pass on a device-resident subsample
    cfg0 = da.TrainConfig(m_count=M, k_count=K, beam_width=L, sweeps=0, rel_tol=0.0)
    t0 = time.perf_counter()
    cw, codes0 = E.growth_pass(X[:TRAIN_SUB].contiguous(), cfg0)
    torch.cuda.synchronize()
    t_growth_sub = time.perf_counter() - t0
    sq = E.einsum_sq(cw)
    Pt, _ = E.cross_full(cw)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    def encode_once(Lw):
        return E.encode(X, cw, sq, Pt, Lw, out_dtype=torch.uint8, with_err=False)[0]

    # --- warmup
    for _ in range(args.warmup):
        encode_once(L)
    barrier()
    # --- timed region: K encode steps, CUDA events on the launching stream
    recheck = torch.zeros(1, dtype=torch.int64, device="cuda")
    E.encode_config(0, recheck)
    launches0 = _native.launch_count()
    _native.prof_enable(True)
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            encode_once(L)
        ev1.record(stream)
        barrier()
    _native.prof_enable(False)
    prof = _native.prof_collect()
    launches = _native.launch_count() - launches0
    E.encode_config(0)
    cand_per_vec = sum(min(L, K ** m) * K for m in range(0, M))
    recheck_frac = float(recheck.item()) / (n * args.steps * cand_per_vec)
    ms_local = ev0.elapsed_time(ev1)
    ms = ms_local
    if dist is not None:
        t = torch.tensor([ms_local], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = n * world / (ms_per_step / 1e3)

    # --- L=1 encode rate (same protocol, untimed for the headline)
    for _ in range(2):
        encode_once(1)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        encode_once(1)
    e1.record(stream)
    torch.cuda.synchronize()
    l1_rate = n * args.steps / (e0.elapsed_time(e1) / 1e3)

    # --- end to end through the public API: host f32 in, host uint8 codes out
    book = da.Codebook(codewords=cw.cpu().numpy(), order=np.arange(M))
    cross = da.cross_products(book)
    for _ in range(max(1, min(args.warmup, 2))):   # warm: same call, same size
        da.encode_dataset(book, X_h, beam_width=L, cross=cross)
    barrier()
    t0 = time.perf_counter()
    enc = da.encode_dataset(book, X_h, beam_width=L, cross=cross)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": n * world / e2e_s, "unit": "vectors/s", "h2d_bytes_per_step": int(X_h.nbytes),
           "d2h_bytes_per_step": int(enc.codes.nbytes), "seconds": e2e_s}

    # --- one full anneal pass at N (da_sweep over M dictionaries), seconds
    anneal = None
    if not args.no_anneal:
        cw_a = cw.clone()
        codes_a, _ = E.encode(X, cw_a, sq, Pt, L, out_dtype=torch.int32, with_err=False)
        Pt_a, sq_a = E.cross_full(cw_a)
        cfg1 = da.TrainConfig(m_count=M, k_count=K, beam_width=L, sweeps=1, rel_tol=0.0)
        rep = da.TrainReport(config=cfg1)
        comm = None
        if dist is not None:
            from paper_1509_05194_b200 import distributed as DD

            comm = DD.Comm()  # NCCL: per-iteration allreduce of K x D sums + counts
        # warm-up pass on copies (first-call scratch growth and kernel attribute setup
        # stay out of the timed pass); it also yields the per-kernel breakdown, so the
        # timed pass runs without the profiling events
        _native.prof_enable(True)
        if comm is None:
            E.da_sweep(X, cw_a.clone(), codes_a.clone(), Pt_a.clone(), sq_a.clone(), cfg1,
                       report=da.TrainReport(config=cfg1), comm=None)
        _native.prof_enable(False)
        aprof = _native.prof_collect()
        barrier()
        t0 = time.perf_counter()
        if comm is None:
            E.da_sweep(X, cw_a, codes_a, Pt_a, sq_a, cfg1, report=rep, comm=None)
        else:
            DD.da_sweep_sharded(X, cw_a, codes_a, Pt_a, sq_a, cfg1, comm, report=rep)
        torch.cuda.synchronize()
        anneal_s = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([anneal_s], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            anneal_s = float(t.item())
        anneal = {"seconds": anneal_s, "rows": n * world, "gpus": world,
                  "per_dictionary_s": [round(s.seconds, 4) for s in rep.steps],
                  "distortion_after": rep.steps[-1].distortion,
                  "kernels_ms": {k: round(v[1], 3) for k, v in aprof.items()}}
        # the Lloyd update's HBM-bound kernel at full width: leaf sums of 1M float64
        # rows (d=128) gathered through a label order, live CUDA-event time on the
        # launching stream (ProfScope), algorithmic N*(8*d + 4) bytes per call
        Xr = X.to(torch.float64)
        lab = torch.randint(0, K, (n,), dtype=torch.int32, device="cuda",
                            generator=torch.Generator(device="cuda").manual_seed(5))
        Cg = torch.empty((K, D), dtype=torch.float64, device="cuda")
        cg = torch.empty(K, dtype=torch.int32, device="cuda")

        def group_sums():
            E.native.da_group_sums(E.P(Xr), n, Xr.stride(0), D, E.P(lab), K, 0, E.P(Cg), D, E.P(cg), E.stream())

        for _ in range(3):
            group_sums()
        _native.prof_collect()
        _native.prof_enable(True)
        for _ in range(10):
            group_sums()
        torch.cuda.synchronize()
        _native.prof_enable(False)
        gprof = _native.prof_collect()
        leaf_ms = gprof["group_sums_leaf"][1] / gprof["group_sums_leaf"][0]
        upd_bytes = n * (8 * D + 4)
        hbm = float(peaks().get("hbm_gbs", 6550.4))
        anneal["update_roofline"] = {
            "kernel": "leaf_sum_narrow_kernel (Lloyd update, d=128)", "bound": "hbm",
            "achieved": upd_bytes / (leaf_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": upd_bytes / (leaf_ms * 1e-3) / 1e9 / hbm,
            "ms_per_call": leaf_ms, "whole_update_ms": gprof["group_sums"][1] / gprof["group_sums"][0],
            "algorithmic": "N*(8*d + 4) B per update (float64 rows + int32 label)"}
        del Xr

    # --- ADC candidate scan, config E shape: 10,000 queries x 100,000 uniform random
    # candidate ids over N_E encoded vectors (random codes stand in for the encoded
    # set: the scan cost does not depend on code values), top-100 per query
    adc = None
    if not args.no_adc:
        N_E, NQ_E, NC_E, R_E = args.adc_n, 10_000, 100_000, 100
        g = torch.Generator(device="cuda").manual_seed(4 + rank)
        codes_e = torch.randint(0, K, (N_E, M), dtype=torch.uint8, device="cuda", generator=g)
        pair_e = E.pair_sums(codes_e, Pt)
        rec_e = E.adc_pack(codes_e, pair_e)
        del codes_e, pair_e
        Qe = torch.randn((NQ_E, D), dtype=torch.float64, device="cuda", generator=g) * 20.0 + 30.0
        lut_e, qsq_e = E.adc_lut(Qe, cw, sq)
        cand_e = torch.randint(0, N_E, (NQ_E, NC_E), dtype=torch.int64, device="cuda", generator=g)
        E.adc_scan_packed(rec_e, lut_e[:64], qsq_e[:64], R_E, cand=cand_e[:64])
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        E.adc_scan_packed(rec_e, lut_e, qsq_e, R_E, cand=cand_e)
        a1.record(stream)
        barrier()
        adc_ms = a0.elapsed_time(a1)
        ncand_tot = NQ_E * NC_E
        ach = 40.0 * ncand_tot / (adc_ms / 1e3) / 1e9
        adc = {"workload": f"config E: {NQ_E} queries x {NC_E} random candidates over {N_E} codes, top-{R_E}",
               "ms": adc_ms, "candidates_per_s": ncand_tot / (adc_ms / 1e3),
               "roofline": {"bound": "hbm", "achieved": ach, "peak": peaks().get("hbm_gbs", 6550.4), "unit": "GB/s",
                            "frac": ach / peaks().get("hbm_gbs", 6550.4),
                            "algorithmic": "40 B per candidate (8-B id + one 32-B sector of the 16-B packed record)",
                            "traffic_note": "random 16-B records: ncu dram bytes ~129 B/candidate (sector overfetch), "
                                            "profiles/README.md"}}
        del rec_e, cand_e, lut_e, Qe

    # --- A-Tree: host build over this GPU's L=10 codes, GPU batched search
    atree = None
    if not args.no_atree:
        from paper_1509_05194_b200 import atree as AT

        book_t = da.Codebook(codewords=cw.cpu().numpy(), order=np.arange(M))
        cross_t = da.cross_products(book_t)
        codes_t = encode_once(L)
        enc_t = da.EncodedDataset(codes=codes_t.cpu().numpy(), k_count=K, codebook_hash=book_t.content_hash())
        t0 = time.perf_counter()
        tree = AT.build_atree(enc_t, book_t, cross_t)
        build_s = time.perf_counter() - t0
        Qa = rank_data(7 + rank, 10_000).astype(np.float64)
        params = AT.SearchParams(l0=8, ls=2.0, r=10)
        AT.atree_search_batch(tree, book_t, Qa, params)   # warm-up sizes the per-CTA scratch
        barrier()
        t0 = time.perf_counter()
        _, _, _, st = AT.atree_search_batch(tree, book_t, Qa, params)
        torch.cuda.synchronize()
        search_s = time.perf_counter() - t0
        ids_t, _, _, st = AT.atree_search_batch(tree, book_t, Qa[:1000], params)
        # recall@10 against the exact neighbours (GPU brute force)
        from paper_1509_05194_b200.groundtruth import brute_force_knn

        t0 = time.perf_counter()
        gt = brute_force_knn(X_h, Qa[:1000].astype(np.float32), 10)
        gt_s = time.perf_counter() - t0
        recall = float(np.mean([len(set(a_) & set(b_)) / 10.0 for a_, b_ in zip(ids_t, gt.ids)]))
        atree = {"workload": f"{n} codes per GPU, 10,000 queries, SearchParams(l0=8, ls=2, r=10)",
                 "build_s_host": build_s, "nodes": tree.node_count, "search_ms": search_s * 1e3,
                 "queries_per_s": 10_000 / search_s, "mean_nodes_visited": float(st[:, 0].mean()),
                 "recall_at_10": recall, "ground_truth_ms_1000_queries": gt_s * 1e3}
        del tree

    # --- roofline of the dominant kernel in the timed region
    pk = peaks()
    kernels = {k: {"launches": c, "ms_per_launch": round(t / max(c, 1), 4), "share": round(t / ms_local, 4)}
               for k, (c, t) in prof.items()}
    # the score-table GEMM is the nearest-codeword contraction: 2*M*K*D flop per vector
    for gname, peak_key, prec in (("encode_table_sgemm", "fp32_ffma_tflops", "fp32"),
                                  ("encode_table_tc", "tf32_tflops", "3xtf32"),
                                  ("encode_table_gemm", "fp64_dfma_tflops", "fp64"),
                                  ("encode_beam_tc", "tf32_tflops", "3xtf32")):
        if gname in prof:
            c, t = prof[gname]
            rows = n * args.steps / max(c, 1)
            tf = 2.0 * M * K * D * rows / (t / max(c, 1) / 1e3) / 1e12
            kernels[gname].update({"tflops": round(tf, 2), "precision": prec,
                                   "frac_of_peak": round(tf / pk[peak_key], 3), "peak_tflops": pk[peak_key]})
    name, (cnt, tot_ms) = max(prof.items(), key=lambda kv: kv[1][1])
    per_launch_ms = tot_ms / max(cnt, 1)
    rows_per_launch = n * args.steps / max(cnt, 1)
    if name in ("encode_table_sgemm", "encode_table_gemm", "encode_table_tc"):
        k = kernels[name]
        roof = {"kernel": name, "bound": "compute", "achieved": k["tflops"], "peak": k["peak_tflops"],
                "unit": "TFLOP/s", "frac": k["frac_of_peak"], "traffic": None,
                "algorithmic": "2*M*K*D flop per vector"}
    else:
        # beam selection: streams the fp32 score table (M*K*4 B per vector) and the
        # cross-term tables out of L2; algorithmic HBM bytes = table + codes
        tab_b = M * K * (4 if ("fast" in name or "pair" in name) else 8)
        achieved = rows_per_launch * (tab_b + M) / (per_launch_ms / 1e3) / 1e9
        roof = {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": pk.get("hbm_gbs", 6550.4),
                "unit": "GB/s", "frac": achieved / pk.get("hbm_gbs", 6550.4), "traffic": None,
                "algorithmic": f"{tab_b + M} B per vector (score table read + codes write)"}
    roof["peak_source"] = "MEASURED_PEAKS.json (HBM) / profiles/peaks_r01.jsonl (FFMA, DFMA: measured on this pool)"
    roof["share_of_step"] = tot_ms / ms_local
    # DRAM traffic of this kernel per launch, from the committed ncu --set full capture
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic_r01.json")) as f:
            tr = json.load(f).get(name)
        if tr:
            roof["traffic"] = tr["bytes_per_vector"] * rows_per_launch
            roof["traffic_source"] = "profiles/ncu_traffic_r01.json: " + tr["capture"]
    except (OSError, ValueError, KeyError):
        pass
    # the whole encode step against BASELINE's compute roofline (2*M*K*D flop per vector)
    step_tflops = 2.0 * M * K * D * value / world / 1e12
    roof["encode_step_compute"] = {"achieved": step_tflops, "peak": pk["fp32_ffma_tflops"], "unit": "TFLOP/s",
                                   "frac": step_tflops / pk["fp32_ffma_tflops"],
                                   "note": "2*M*K*D flop per vector at the step rate vs measured FP32 FFMA peak"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))
        v_cpu, cores, sample = cpu_encode_rate(cw.cpu().numpy(), X_h, L)
        cpu = {"value": v_cpu, "unit": "vectors/s", "cores": cores, "kind": "port",
               "sample": f"{sample} config-B vectors, L=10, oracle (numpy/OpenBLAS) encode with {cores} threads"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "vectors/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 filter + f64 exact", "data": "synthetic",
            "config": {"workload": "config B: beam encode L=10 of 1M resident vectors per GPU "
                                   "(D=128, M=8, K=256)", "vectors_per_gpu": n, "global_batch": n * world,
                       "beam_width": L, "parallelism": f"dp{world} (row shards, no collective)",
                       "l2_flush": "none needed: 512 MB input per step > 126 MB L2",
                       "codebook": f"device growth pass on {TRAIN_SUB} vectors ({t_growth_sub:.1f}s, untimed)"},
            "encode_L1_vectors_per_s": l1_rate,
            "exact_recheck_fraction": recheck_frac,
            "anneal_pass": anneal,
            "adc_scan": adc,
            "atree_search": atree,
            "roofline": roof,
            "kernels": kernels,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
