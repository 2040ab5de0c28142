"""Benchmark of the DA hot path on BASELINE.json config B (configs[1]).

Workload: N=1,000,000 vectors per GPU, D=128, fp32 holding integers in
[0,255] (seeded synthetic stand-in for SIFT1M, see paper_1509_05194_b200/
synthetic.py), M=8 dictionaries x K=256 codewords, beam width L=10.

  * headline (`value`): one step = one L=10 beam encode of the GPU's 1M
    resident vectors.  Each rank encodes its own rows (weak scaling, no
    data-path collective).  The codebook is trained once on rank 0 (device
    growth pass on a 100k subsample, untimed) and broadcast to every rank.
  * `anneal_pass`: one full anneal pass (da_sweep over the M dictionaries) of
    the first 1M config-B rows, STRONG-scaled: rank r holds rows
    shard_rows(1M, N, r); Lloyd statistics, PCA moments and reseeds go through
    NCCL.  T(1)/T(k) is the scaling the north star asks for.
  * `e2e`: the same L=10 encode through the public API (host f32 in, host
    uint8 codes out, copies inside the timed region).
  * `rooflines`: the SURVEY 8(d) figures for the encode (L=10 and L=1), the
    assign, the Lloyd update and the ADC scan, from live CUDA-event timing of
    each kernel on its launching stream; TF32 peak measured live (cuBLAS).
  * `cpu_baseline`: the unmodified reference (annq from baseline/_ref, all host
    threads) on a bounded sample of the same rows, codes compared with ours.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

With --gpus N > 1 and no torchrun environment the script re-launches itself
through torch.distributed.run with N ranks (one per GPU, NCCL).
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "baseline", "_ref")

METRIC = "DA encode vectors/s (D=128,M=8,K=256) & anneal-pass sec; % of roofline"
N_PER_GPU = 1_000_000
N_ANNEAL = 1_000_000
D, M, K, L = 128, 8, 256, 10
TRAIN_SUB = 100_000
B_CHUNK = 250_000
REF_CHUNK = max(64, min(10**9, 4_000_000 // (L * K)))   # encode_dataset's chunk (codebook.py:341)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=N_PER_GPU, help="vectors per GPU (encode)")
    ap.add_argument("--n-anneal", type=int, default=N_ANNEAL, help="total rows of the strong-scaled anneal pass")
    ap.add_argument("--no-anneal", action="store_true", help="skip the full anneal-pass timing")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--cpu-anneal", type=int, default=0,
                    help="also time the reference's da_sweep on this many rows (slow: ~66 s for 4096)")
    ap.add_argument("--no-adc", action="store_true", help="skip the config-E ADC scan timing")
    ap.add_argument("--no-atree", action="store_true", help="skip the A-Tree build + search timing")
    ap.add_argument("--no-configc", action="store_true", help="skip the config-C (D=960) encode timing")
    ap.add_argument("--configc-n", type=int, default=131_072, help="config-C vectors (D=960) for the L=1 encode")
    ap.add_argument("--adc-n", type=int, default=1_000_000_000, help="encoded vectors for the ADC scan")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher/collective plumbing only (gloo on CPU, no kernels): for CPU-box tests")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args) -> int:
    """--gpus N without a torchrun environment: run N ranks of this script."""
    env = dict(os.environ)
    if not args.dry_run:
        # NCCL's init lines (rank count, NVLS, transports) go to per-process logs
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        logdir = os.path.join(ROOT, "gpurun_out")
        os.makedirs(logdir, exist_ok=True)
        env.setdefault("NCCL_DEBUG_FILE", os.path.join(logdir, "nccl.%h.%p.log"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def config_b_rows(lo: int, hi: int, stream_base: int = 0):
    """Rows [lo, hi) of the config-B stream whose 250k-row chunks are seeded
    b-chunk-(stream_base + i): only the chunks that overlap are generated."""
    import numpy as np

    from paper_1509_05194_b200 import synthetic

    means = synthetic.mixture_b_params(1)
    out = np.empty((max(hi - lo, 0), D), dtype=np.float32)
    c = lo // B_CHUNK
    while c * B_CHUNK < hi:
        c0 = c * B_CHUNK
        rng = synthetic.substream(1, f"b-chunk-{stream_base + c}")
        block = synthetic._draw_b(rng, means, B_CHUNK)
        a, b = max(lo, c0), min(hi, c0 + B_CHUNK)
        out[a - lo:b - lo] = block[a - c0:b - c0]
        c += 1
    return out


def rank_data(rank: int, n: int):
    """Rank r's own encode rows: chunks 4r, 4r+1, ... of the seed-1 stream
    (rank 0's are the first 1M config-B rows)."""
    return config_b_rows(0, n, stream_base=4 * rank)


def host_info():
    cpu = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    cpu = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    ram = None
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal"):
                    ram = round(int(line.split()[1]) / 1024 / 1024, 1)
                    break
    except OSError:
        pass
    import numpy as np

    return {"cpu_model": cpu, "cpu_count": os.cpu_count(), "ram_gb": ram, "numpy": np.__version__}


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
                self._stop.wait(0.1)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        import numpy as np

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
    """Roofline denominators: MEASURED_PEAKS.json (driver) + profiles/peaks_r01.jsonl
    (FFMA / DFMA micro-benchmarks measured on this pool, tools/peaks.cu)."""
    out = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            out.update(json.load(f))
        out["hbm_source"] = "MEASURED_PEAKS.json"
    except Exception:
        out["hbm_gbs"] = 6650.0
        out["hbm_source"] = "B200_PROFILING.md fallback"
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_r01.jsonl")) as f:
            rows = [json.loads(x) for x in f if x.strip()]
        out["fp64_dfma_tflops"] = max(r["fp64_dfma_tflops"] for r in rows)
        out["fp32_ffma_tflops"] = max(r["fp32_ffma_tflops"] for r in rows)
    except Exception:
        out["fp64_dfma_tflops"], out["fp32_ffma_tflops"] = 34.0, 70.8
    return out


def measure_tf32_peak(torch):
    """Dense TF32 tensor-core throughput on this GPU: cuBLAS fp32 GEMM with TF32
    allowed, 8192^3, best of 5 (CUDA events)."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        c = a @ b
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b, c
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def reference_encoder():
    """(kind, encode(cw32, X32, L, n_jobs) -> codes): the unmodified reference
    (annq.encode_dataset from baseline/_ref) when shipped, else the oracle port."""
    import numpy as np

    if os.path.isdir(os.path.join(REF, "annq")):
        if REF not in sys.path:
            sys.path.insert(0, REF)
        import annq

        def enc(cw32, X32, Lw, n_jobs):
            book = annq.Codebook(codewords=cw32, order=np.arange(cw32.shape[0], dtype=np.int64))
            cross = annq.cross_products(book)
            return annq.encode_dataset(book, X32, beam_width=Lw, n_jobs=n_jobs, cross=cross).codes

        return "reference", enc
    from oracle import da_oracle as O

    def enc(cw32, X32, Lw, n_jobs):
        P, _ = O.cross_table(cw32)
        return O.encode_chunked(cw32, P, X32, Lw, n_jobs=n_jobs)

    return "port", enc


def cpu_sample_rows(cores: int) -> int:
    """Two full waves of the reference's encode chunks on every core (>= 32k rows)."""
    return max(32_768, 2 * cores * REF_CHUNK)


def cpu_codebook():
    """Codebook for the reference arm: seeded random codewords in the data's range
    (the encode's cost does not depend on how the codebook was trained)."""
    import numpy as np

    rng = np.random.default_rng(11)
    return (rng.uniform(0.0, 12.0, size=(M, K, D)) * (0.5 ** np.arange(M))[:, None, None]).astype(np.float32)


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cores))
    kind, enc = reference_encoder()
    sample = cpu_sample_rows(cores)
    X = rank_data(0, sample)
    cw = cpu_codebook()
    for _ in range(args.warmup):
        enc(cw, X[:2 * REF_CHUNK], L, cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        enc(cw, X, L, cores)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    v = sample * args.steps / total
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "vectors/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config B beam encode L=10 (D=128, M=8, K=256)", "sample_per_step": sample,
                   "global_batch": sample, "parallelism": f"{cores} host threads (encode_dataset n_jobs)"},
        "cpu_baseline": {"value": v, "unit": "vectors/s", "cores": cores, "kind": kind,
                         "sample": f"{sample} config-B rows per step through "
                                   + ("annq.encode_dataset (unmodified reference, baseline/_ref)"
                                      if kind == "reference" else "the oracle port of encode_dataset"),
                         "host": host_info()},
        "e2e": {"value": v, "unit": "vectors/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def dry_run(args):
    """Plumbing only (CPU, gloo): rank count, codebook broadcast, max-over-ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    cw = torch.from_numpy(cpu_codebook()) if rank == 0 else torch.zeros((M, K, D))
    if world > 1:
        dist.broadcast(cw, 0)
        dist.barrier()
    t = torch.tensor([float(rank + 1)])
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    same = bool(np.array_equal(cw.numpy(), cpu_codebook()))
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "value": None,
                          "codebook_broadcast_equal": same, "max_over_ranks": float(t.item())}))
    if world > 1:
        dist.destroy_process_group()


def _adc_traffic() -> float:
    """DRAM bytes per ADC candidate from the committed ncu capture (72 B: the 64-B L2 granule + the id)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")) as f:
            return float(json.load(f)["adc_scan_packed"]["bytes_per_candidate"])
    except (OSError, KeyError, ValueError):
        return float("nan")


def anneal_flop(log, N, Dd, Mm, Kk):
    """sum_m [2ND^2 (Gram) + 2ND^2 (rotate) + sum_s (I+1) 2NKd_s
    + 2*2NKD (final/init assigns) + 2NMKD (encode)], I from the Lloyd log."""
    f = Mm * (4.0 * N * Dd * Dd + 4.0 * N * Kk * Dd + 2.0 * N * Mm * Kk * Dd)
    f += sum((it + 1) * 2.0 * N * k * d for (d, _, k, it) in log)
    return f


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.dry_run:
        return dry_run(args)
    import numpy as np
    import torch

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1509_05194_b200 as da
    from paper_1509_05194_b200 import _engine as E
    from paper_1509_05194_b200 import _native
    from paper_1509_05194_b200 import distributed as DD

    pk = peaks()
    tf32_peak = measure_tf32_peak(torch)
    n = args.n
    X_h = rank_data(rank, n)
    X = E.to_dev(X_h)
    # --- codebook (untimed): growth pass on rank 0, broadcast to every rank
    cfg0 = da.TrainConfig(m_count=M, k_count=K, beam_width=L, sweeps=0, rel_tol=0.0)
    t0 = time.perf_counter()
    if rank == 0:
        cw, _ = E.growth_pass(X[:TRAIN_SUB].contiguous(), cfg0)
    else:
        cw = torch.empty((M, K, D), dtype=torch.float32, device="cuda")
    if dist is not None:
        dist.broadcast(cw, 0)
    torch.cuda.synchronize()
    t_growth_sub = time.perf_counter() - t0
    sq = E.einsum_sq(cw)
    Pt, _ = E.cross_full(cw)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def encode_once(Lw, out=None):
        return E.encode(X, cw, sq, Pt, Lw, out_dtype=torch.uint8, with_err=False)[0]

    # --- warmup
    for _ in range(args.warmup):
        codes_dev = encode_once(L)
    barrier()
    # --- timed region: K encode steps, CUDA events on the launching stream
    recheck = torch.zeros(1, dtype=torch.int64, device="cuda")
    E.encode_config(0, recheck)
    launches0 = _native.launch_count()
    _native.prof_enable(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            codes_dev = encode_once(L)
        ev1.record(stream)
        barrier()
    _native.prof_enable(False)
    prof = _native.prof_collect()
    launches = _native.launch_count() - launches0
    E.encode_config(0)
    cand_per_vec = sum(min(L, K ** m) * K for m in range(0, M))
    recheck_frac = float(recheck.item()) / (n * args.steps * cand_per_vec)
    ms_local = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms_local)
    ms_per_step = ms / args.steps
    value = n * world / (ms_per_step / 1e3)

    # --- L=1 encode (nearest codeword per stage), same protocol
    for _ in range(2):
        encode_once(1)
    barrier()
    _native.prof_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        encode_once(1)
    e1.record(stream)
    torch.cuda.synchronize()
    _native.prof_enable(False)
    prof1 = _native.prof_collect()
    l1_ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    l1_rate = n * world / (l1_ms / 1e3)

    # --- end to end through the public API: host f32 in, host uint8 codes out
    book = da.Codebook(codewords=cw.cpu().numpy(), order=np.arange(M))
    cross = da.cross_products(book)
    for _ in range(max(1, min(args.warmup, 2))):   # warm: same call, same size
        da.encode_dataset(book, X_h, beam_width=L, cross=cross)
    barrier()
    t0 = time.perf_counter()
    enc = da.encode_dataset(book, X_h, beam_width=L, cross=cross)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": n * world / e2e_s, "unit": "vectors/s", "h2d_bytes_per_step": int(X_h.nbytes),
           "d2h_bytes_per_step": int(enc.codes.nbytes), "seconds": e2e_s,
           "path": "paper_1509_05194_b200.encode_dataset (host float32 -> pinned slots -> device -> host uint8)"}
    e2e_codes_equal = bool(np.array_equal(enc.codes, codes_dev.cpu().numpy()))
    del enc

    rooflines = {}
    ffma = pk["fp32_ffma_tflops"]

    def compute_roof(name, flop, sec, extra=None):
        a = flop / sec / 1e12
        r = {"bound": "compute", "achieved": a, "unit": "TFLOP/s", "peak_ffma": ffma, "frac_ffma": a / ffma,
             "peak_3xtf32": tf32_peak / 3.0, "frac_3xtf32": a / (tf32_peak / 3.0),
             # /2 when x is exact in tf32 (integer config-B rows): the score table then runs two
             # tf32 MMAs per k step (table_tc_stream_kernel<true>), so this is the tensor-core roof of the encode table
             "peak_2xtf32": tf32_peak / 2.0, "frac_2xtf32": a / (tf32_peak / 2.0)}
        if extra:
            r.update(extra)
        rooflines[name] = r

    mkd = 2.0 * M * K * D
    compute_roof("encode_L10_step", mkd * n, ms_per_step / 1e3,
                 {"algorithmic": "2*M*K*D = 524,288 flop per vector at the whole L=10 step rate (beam bookkeeping "
                                 "not credited, SURVEY 8d)"})
    compute_roof("encode_L1_step", mkd * n, l1_ms / 1e3,
                 {"algorithmic": "2*M*K*D flop per vector at the whole L=1 step rate (the nearest-codeword "
                                 "kernel of SURVEY 8d)", "kernels_ms_per_step": {
                     k: round(t / args.steps, 4) for k, (c, t) in prof1.items()}})

    # --- one full anneal pass, strong-scaled over the ranks
    anneal = None
    if not args.no_anneal:
        NA = args.n_anneal
        sl = DD.shard_rows(NA, world, rank)
        if world == 1 and NA == n:
            XA = X
        else:
            XA = E.to_dev(config_b_rows(sl.start, sl.stop))
        cw_a = cw.clone()
        codes_a, _ = E.encode(XA, cw_a, sq, Pt, L, out_dtype=torch.int32, with_err=False)
        Pt_a, sq_a = E.cross_full(cw_a)
        cfg1 = da.TrainConfig(m_count=M, k_count=K, beam_width=L, sweeps=1, rel_tol=0.0)
        comm = DD.Comm().bind_rows(XA.shape[0]) if dist is not None else None

        def sweep(state, rep):
            if comm is None:
                E.da_sweep(XA, *state, cfg1, report=rep, comm=None)
            else:
                DD.da_sweep_sharded(XA, *state, cfg1, comm, report=rep)

        # warm-up pass on copies (first-call scratch growth stays out of the timed
        # pass); it also yields the per-kernel breakdown, so the timed pass runs
        # without the profiling events
        _native.prof_enable(True)
        sweep([cw_a.clone(), codes_a.clone(), Pt_a.clone(), sq_a.clone()], da.TrainReport(config=cfg1))
        torch.cuda.synchronize()
        _native.prof_enable(False)
        aprof = _native.prof_collect()
        rep = da.TrainReport(config=cfg1)
        E.LLOYD_LOG = []
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a0.record(stream)
        sweep([cw_a, codes_a, Pt_a, sq_a], rep)
        a1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        anneal_s = max_over_ranks(a0.elapsed_time(a1) / 1e3)
        log, E.LLOYD_LOG = E.LLOYD_LOG, None
        flop = anneal_flop(log, NA, D, M, K)
        iters = [[it for (d_, _, _, it) in log[m * 10:(m + 1) * 10]] for m in range(M)]
        gs_ms = aprof.get("group_sums", (0, 0.0))
        upd_bytes = sum(NA * (4 * d_ + 4) * it for (d_, _, _, it) in log)
        anneal = {"seconds": anneal_s, "wall_seconds_rank0": wall, "rows_total": NA,
                  "rows_per_gpu": XA.shape[0], "gpus": world, "scaling": "strong",
                  "timing": "CUDA events around the pass on the launching stream, max over ranks",
                  "per_dictionary_s": [round(s.seconds, 4) for s in rep.steps],
                  "distortion_after": rep.steps[-1].distortion,
                  "lloyd_iters_per_stage": iters, "lloyd_iters_total": int(sum(map(sum, iters))),
                  "flop": flop, "tflops": flop / anneal_s / 1e12,
                  "frac_ffma": flop / anneal_s / 1e12 / ffma,
                  "flop_formula": "SURVEY 8(d): sum_m [4ND^2 + sum_s (I_ms+1) 2NK d_s + 4NKD + 2NMKD]",
                  "kernels_ms": {k: round(v[1], 3) for k, v in aprof.items()},
                  "kernel_launches": {k: v[0] for k, v in aprof.items()}}
        if gs_ms[0]:
            # pass average of the Lloyd update against SURVEY 8(d)'s N*(4*d+4) B
            # (float32-width rows + int32 label; our rows are float64 for parity)
            ach = upd_bytes / (gs_ms[1] * 1e-3) / 1e9
            rooflines["lloyd_update_pass_avg"] = {
                "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": ach / pk["hbm_gbs"],
                "updates": gs_ms[0], "ms_total": gs_ms[1],
                "algorithmic": "N*(4*d_active + 4) B per update (SURVEY 8d), summed over the pass's updates; "
                               "rows are float64 (8*d B read) for bit parity"}
        # the assigns of the pass against 2*K*d flop per point
        a_ms = sum(v[1] for k, v in aprof.items() if k.startswith("assign_") and k != "assign_image")
        a_flop = sum((it + 1) * 2.0 * NA * k_ * d_ for (d_, _, k_, it) in log) + M * 2 * 2.0 * NA * K * D
        if a_ms:
            compute_roof("assign_pass_avg", a_flop / world, a_ms / 1e3,
                         {"algorithmic": "2*K*d_active flop per point per assign, all assigns of the pass "
                                         "(per GPU)", "ms_total": a_ms})
        # the Lloyd update's HBM-bound kernel at full width: leaf sums of 1M float64
        # rows (d=128) gathered through a label order (best single call)
        if world == 1:
            Xr = XA.to(torch.float64)
            nn = Xr.shape[0]
            lab = torch.randint(0, K, (nn,), dtype=torch.int32, device="cuda",
                                generator=torch.Generator(device="cuda").manual_seed(5))
            Cg = torch.empty((K, D), dtype=torch.float64, device="cuda")
            cg = torch.empty(K, dtype=torch.int32, device="cuda")

            def group_sums():
                E.native.da_group_sums(E.P(Xr), nn, Xr.stride(0), D, E.P(lab), K, 0, E.P(Cg), D, E.P(cg),
                                       E.stream())

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
            whole_ms = gprof["group_sums"][1] / gprof["group_sums"][0]
            b32 = nn * (4 * D + 4)
            b64 = nn * (8 * D + 4)
            rooflines["lloyd_update_d128"] = {
                "bound": "hbm", "kernel": "leaf_sum_narrow_kernel", "unit": "GB/s", "peak": pk["hbm_gbs"],
                "achieved": b32 / (whole_ms * 1e-3) / 1e9, "frac": b32 / (whole_ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                "algorithmic": "N*(4*D + 4) B per update (SURVEY 8d) over the whole update incl. the sort",
                "ms_whole_update": whole_ms, "ms_leaf_kernel": leaf_ms,
                "leaf_kernel_bytes_moved_frac": b64 / (leaf_ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                "note": "rows are float64 for bit parity: the leaf kernel moves N*(8*D+4) B"}
            del Xr
            # scaling projection: the pass over one rank's share at 8 GPUs
            # (1/8 of the rows) on this GPU.  Its device time bounds T(8) from below
            # (collective latency excluded), so T(1M) / T(1M/8) bounds the 8-GPU
            # strong-scaling factor from above.
            n8 = NA // 8
            X8 = XA[:n8].contiguous()
            cw8 = cw.clone()
            codes8, _ = E.encode(X8, cw8, sq, Pt, L, out_dtype=torch.int32, with_err=False)
            P8, s8 = E.cross_full(cw8)
            for _ in range(2):   # warm-up: the second pass captures the Lloyd graphs, later ones replay them
                E.da_sweep(X8, cw8.clone(), codes8.clone(), P8.clone(), s8.clone(), cfg1)
            torch.cuda.synchronize()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(stream)
            E.da_sweep(X8, cw8, codes8, P8, s8, cfg1)
            b1.record(stream)
            torch.cuda.synchronize()
            t8 = b0.elapsed_time(b1) / 1e3
            anneal["projection_8gpu"] = {
                "rows_per_gpu": n8, "seconds_one_share": t8, "speedup_bound": anneal_s / t8,
                "note": "anneal pass over 1/8 of the rows on one GPU: a lower bound of T(8) (no collective "
                        "latency), so anneal_pass.seconds / seconds_one_share bounds the 8-GPU strong scaling"}
            del X8, codes8, P8, s8
        del XA

    # --- ADC candidate scan, config E shape: 10,000 queries (sharded over the
    # ranks) x 100,000 uniform random candidate ids over N_E encoded vectors
    # (random codes stand in for the encoded set: the scan's cost does not depend
    # on code values), top-100 per query
    adc = None
    cpu_adc = None
    if not args.no_adc:
        N_E, NQ_E, NC_E, R_E = args.adc_n, 10_000, 100_000, 100
        q_sl = DD.shard_rows(NQ_E, world, rank)
        nq = q_sl.stop - q_sl.start
        g = torch.Generator(device="cuda").manual_seed(4)
        codes_e = torch.randint(0, K, (N_E, M), dtype=torch.uint8, device="cuda", generator=g)
        pair_e = E.pair_sums(codes_e, Pt)
        Qe = torch.randn((NQ_E, D), dtype=torch.float64, device="cuda", generator=g) * 20.0 + 30.0
        cand_e = torch.randint(0, N_E, (NQ_E, NC_E), dtype=torch.int64, device="cuda", generator=g)
        if rank == 0 and world == 1 and not args.no_cpu:
            # reference exhaustive_adc_search on EncodedDataset(codes[cand], id_map=cand)
            # for 100 queries (BASELINE CPU plan), candidates/s
            nqc = 100
            cc = cand_e[:nqc].cpu().numpy()
            sub_codes = codes_e[cand_e[:nqc].reshape(-1)].cpu().numpy().reshape(nqc, NC_E, M)
            sub_pair = pair_e[cand_e[:nqc].reshape(-1)].cpu().numpy().reshape(nqc, NC_E)
            qh = Qe[:nqc].cpu().numpy()
            kind, _ = reference_encoder()
            if kind == "reference":
                import annq

                rbook = annq.Codebook(codewords=cw.cpu().numpy(), order=np.arange(M, dtype=np.int64))
                rcross = annq.cross_products(rbook)
                t0 = time.perf_counter()
                for i in range(nqc):
                    ed = annq.EncodedDataset(codes=sub_codes[i], k_count=K, codebook_hash=rbook.content_hash(),
                                             id_map=cc[i])
                    annq.exhaustive_adc_search(rbook, ed, qh[i], R_E, cross=rcross, pair_sums=sub_pair[i])
                dt = time.perf_counter() - t0
                cpu_adc = {"value": nqc * NC_E / dt, "unit": "candidates/s", "cores": os.cpu_count(),
                           "kind": "reference", "sample": f"{nqc} queries x {NC_E} candidates, "
                                                         "annq.exhaustive_adc_search (numpy, one query at a time)"}
            del sub_codes, sub_pair
        rec_e = E.adc_pack(codes_e, pair_e)
        del codes_e, pair_e
        lut_e, qsq_e = E.adc_lut(Qe[q_sl], cw, sq)
        cand_r = cand_e[q_sl].contiguous()
        del cand_e
        E.adc_scan_packed(rec_e, lut_e[:64], qsq_e[:64], R_E, cand=cand_r[:64])
        barrier()
        _native.prof_enable(True)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        E.adc_scan_packed(rec_e, lut_e, qsq_e, R_E, cand=cand_r)
        a1.record(stream)
        barrier()
        _native.prof_enable(False)
        _native.prof_collect()
        adc_ms = max_over_ranks(a0.elapsed_time(a1))
        ncand_tot = NQ_E * NC_E
        ach = 40.0 * ncand_tot / (adc_ms / 1e3) / 1e9
        adc = {"workload": f"config E: {NQ_E} queries (sharded over {world} GPU) x {NC_E} random candidates over "
                           f"{N_E} codes, top-{R_E}",
               "ms": adc_ms, "candidates_per_s": ncand_tot / (adc_ms / 1e3), "cpu_baseline": cpu_adc}
        rooflines["adc_scan"] = {"bound": "hbm", "kernel": "adc_scan_packed_kernel", "achieved": ach,
                                 "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": ach / pk["hbm_gbs"],
                                 "algorithmic": "40 B per candidate (8-B id + one 32-B sector of the 16-B record)",
                                 "traffic": _adc_traffic() * ncand_tot,
                                 "traffic_unit": "bytes per launch (DRAM read + write, ncu)",
                                 "traffic_source": "profiles/ncu_traffic_r02.json: adc_scan_packed bytes per candidate"}
        del rec_e, cand_r, lut_e, Qe

    # --- config C (D = 960): the D-tiled tcgen05 score table + greedy L=1 encode on a
    # bounded sample (the 1M-vector config does not change per-vector cost: the encode
    # runs in 131k-row chunks), and the L=10 encode (chunked FFMA table) for reference
    configc = None
    if not args.no_configc and rank == 0:
        from paper_1509_05194_b200 import synthetic as SY

        nc_ = args.configc_n
        Dc = 960
        Xc = E.to_dev(np.ascontiguousarray(SY.config_c(n=nc_), dtype=np.float32))
        cwc, _ = E.growth_pass(Xc[:20_000].contiguous(), cfg0)
        Pc, _ = E.cross_full(cwc)
        sqc = E.einsum_sq(cwc)
        cc_out = {"workload": f"config C: {nc_} vectors, D=960, M=8, K=256 (codebook: growth pass on 20,000 rows)"}
        for Lw, reps in ((1, 3), (10, 1)):
            E.encode(Xc, cwc, sqc, Pc, Lw, out_dtype=torch.uint8, with_err=False)
            torch.cuda.synchronize()
            _native.prof_collect()
            _native.prof_enable(True)
            c0e, c1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0e.record(stream)
            for _ in range(reps):
                E.encode(Xc, cwc, sqc, Pc, Lw, out_dtype=torch.uint8, with_err=False)
            c1e.record(stream)
            torch.cuda.synchronize()
            _native.prof_enable(False)
            cprof = _native.prof_collect()
            c_ms = c0e.elapsed_time(c1e) / reps
            cc_out[f"L{Lw}_vectors_per_s"] = nc_ / (c_ms / 1e3)
            cc_out[f"L{Lw}_ms"] = c_ms
            cc_out[f"L{Lw}_kernels_ms"] = {k: round(t / reps, 4) for k, (c, t) in cprof.items()}
            if Lw == 1 and "encode_table_tc" in cprof:
                t_tab = cprof["encode_table_tc"][1] / reps / 1e3
                # issued tensor work: 3 tf32 MMAs per 8 columns over D+1 columns padded to 16
                kpad = ((Dc + 1 + 15) // 16) * 16
                issued = 3 * 2.0 * M * K * kpad * nc_
                rooflines["configC_table_tc_stream"] = {
                    "bound": "tensor", "kernel": "table_tc_stream_kernel (+ image and codeword preps)",
                    "achieved": issued / t_tab / 1e12, "peak": tf32_peak, "unit": "TFLOP/s",
                    "frac": issued / t_tab / 1e12 / tf32_peak,
                    "algorithmic_tflops": 2.0 * M * K * Dc * nc_ / t_tab / 1e12,
                    "frac_3xtf32": 2.0 * M * K * Dc * nc_ / t_tab / 1e12 / (tf32_peak / 3.0),
                    "peak_nominal": 1125.0, "frac_nominal": issued / t_tab / 1e12 / 1125.0,
                    "algorithmic": "2*M*K*D flop per vector (SURVEY 8d) against the 3xTF32 roof; `achieved` counts "
                                   "the three tf32 MMAs issued per k step against the dense TF32 peak measured with "
                                   "a cuBLAS TF32 GEMM in this run (a conservative denominator: this kernel can "
                                   "exceed it; peak_nominal = half the nominal dense bf16 rate)",
                    "ms": t_tab * 1e3}
        configc = cc_out
        del Xc, Pc

    # --- A-Tree: GPU build over this GPU's L=10 codes, GPU batched search
    atree = None
    if not args.no_atree:
        from paper_1509_05194_b200 import atree as AT

        enc_t = da.EncodedDataset(codes=codes_dev.cpu().numpy(), k_count=K, codebook_hash=book.content_hash())
        AT.build_atree(enc_t, book, cross)           # warm-up (scratch growth)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tree = AT.build_atree(enc_t, book, cross)
        build_s = time.perf_counter() - t0
        Qa = rank_data(7 + rank, 10_000).astype(np.float64)
        params = AT.SearchParams(l0=8, ls=2.0, r=10)
        AT.atree_search_batch(tree, book, Qa, params)   # warm-up sizes the per-CTA scratch
        barrier()
        t0 = time.perf_counter()
        _, _, _, st = AT.atree_search_batch(tree, book, Qa, params)
        torch.cuda.synchronize()
        search_s = time.perf_counter() - t0
        ids_t, _, _, st = AT.atree_search_batch(tree, book, Qa[:1000], params)
        from paper_1509_05194_b200.groundtruth import brute_force_knn

        t0 = time.perf_counter()
        gt = brute_force_knn(X_h, Qa[:1000].astype(np.float32), 10)
        gt_s = time.perf_counter() - t0
        recall = float(np.mean([len(set(a_) & set(b_)) / 10.0 for a_, b_ in zip(ids_t, gt.ids)]))
        atree = {"workload": f"{n} codes per GPU, 10,000 queries, SearchParams(l0=8, ls=2, r=10)",
                 "build_s_gpu": build_s, "nodes": tree.node_count, "search_ms": search_s * 1e3,
                 "queries_per_s": 10_000 / search_s, "mean_nodes_visited": float(st[:, 0].mean()),
                 "recall_at_10": recall, "ground_truth_ms_1000_queries": gt_s * 1e3}
        del tree

    # --- roofline of the dominant kernel of the timed region.  SURVEY 8(d): the
    # encode is compute-bound, 2*M*K*D flop per encoded vector against the
    # measured FP32 FFMA peak, whichever kernel of the step dominates
    kernels = {k: {"launches": c, "ms_per_launch": round(t / max(c, 1), 4), "share": round(t / ms_local, 4)}
               for k, (c, t) in prof.items()}
    name, (cnt, tot_ms) = max(prof.items(), key=lambda kv: kv[1][1])
    per_launch_ms = tot_ms / max(cnt, 1)
    rows_per_launch = n * args.steps / max(cnt, 1)
    achieved = mkd * rows_per_launch / (per_launch_ms / 1e3) / 1e12
    roof = {"kernel": name, "bound": "compute", "achieved": achieved, "peak": ffma, "unit": "TFLOP/s",
            "frac": achieved / ffma, "traffic": None,
            "algorithmic": f"2*M*K*D = {int(mkd)} flop per vector x {int(rows_per_launch)} vectors per launch "
                           "(SURVEY 8d), over this kernel's average launch time",
            "peak_source": "profiles/peaks_r01.jsonl (FP32 FFMA micro-benchmark on this pool)",
            "share_of_step": tot_ms / ms_local}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")) as f:
            tr = json.load(f).get(name)
        if tr:
            roof["traffic"] = tr["bytes_per_vector"] * rows_per_launch
            roof["traffic_source"] = "profiles/ncu_traffic_r02.json: " + tr["capture"]
    except (OSError, ValueError, KeyError):
        pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        kind, enc_ref = reference_encoder()
        sample = min(cpu_sample_rows(cores), n)
        t0 = time.perf_counter()
        ref_codes = enc_ref(cw.cpu().numpy(), X_h[:sample], L, cores)
        dt = time.perf_counter() - t0
        ours = codes_dev[:sample].cpu().numpy()
        equal_rows = int((ref_codes.astype(np.int64) == ours.astype(np.int64)).all(axis=1).sum())
        cpu = {"value": sample / dt, "unit": "vectors/s", "cores": cores, "kind": kind,
               "sample": f"first {sample} of this GPU's config-B rows, L=10, "
                         + ("annq.encode_dataset (unmodified reference, baseline/_ref)" if kind == "reference"
                            else "oracle port") + f" with n_jobs={cores}",
               "codes_equal_rows": equal_rows, "codes_compared_rows": sample, "host": host_info()}
        if args.cpu_anneal:
            # one reference da_sweep on a slice (slow; opt-in), extrapolated linearly
            if kind == "reference":
                import annq
                from annq import annealing as RA

                na = args.cpu_anneal
                rbook = annq.Codebook(codewords=cw.cpu().numpy(), order=np.arange(M, dtype=np.int64))
                renc = annq.encode_dataset(rbook, X_h[:na], beam_width=L, n_jobs=cores)
                t0 = time.perf_counter()
                RA.da_sweep(X_h[:na], rbook, renc, cfg0)
                dt = time.perf_counter() - t0
                cpu["anneal_pass"] = {"rows": na, "seconds": dt, "extrapolated_1M_seconds": dt * 1e6 / na,
                                      "note": "reference da_sweep on a slice, linear extrapolation to 1M rows"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "vectors/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 filter + f64 exact", "data": "synthetic",
            "config": {"workload": "config B: beam encode L=10 of 1M resident vectors per GPU "
                                   "(D=128, M=8, K=256)", "vectors_per_gpu": n, "global_batch": n * world,
                       "beam_width": L, "parallelism": f"dp{world} (row shards, no collective)",
                       "l2_flush": "none needed: 512 MB input per step > 126 MB L2",
                       "codebook": f"device growth pass on {TRAIN_SUB} vectors on rank 0, broadcast "
                                   f"({t_growth_sub:.1f}s, untimed)"},
            "encode_L1_vectors_per_s": l1_rate,
            "exact_recheck_fraction": recheck_frac,
            "anneal_pass": anneal,
            "adc_scan": adc,
            "atree_search": atree,
            "config_c": configc,
            "roofline": roof,
            "rooflines": rooflines,
            "peaks": {"fp32_ffma_tflops": ffma, "tf32_dense_tflops_measured": tf32_peak,
                      "hbm_gbs": pk["hbm_gbs"], "hbm_source": pk.get("hbm_source")},
            "kernels": kernels,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_codes_equal_device_codes": e2e_codes_equal,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
