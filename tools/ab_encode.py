"""A/B timing of the config-B encode across library builds.
usage: python tools/ab_encode.py [n] [L,...] -- name1 name2 ... (tools/ab/NAME/libda_b200.so; 'cur' = in-tree)
Each variant runs in its own process (the library is loaded once per process)."""
import os, sys, json, subprocess, hashlib
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if "--child" in sys.argv:
    sys.path.insert(0, ROOT)
    import time, torch
    import paper_1509_05194_b200 as da
    from paper_1509_05194_b200 import _engine as E
    import bench
    n = int(sys.argv[2]); Ls = [int(x) for x in sys.argv[3].split(",")]
    X = E.to_dev(bench.rank_data(0, n))
    cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
    cw, _ = E.growth_pass(X[:100000].contiguous(), cfg0)
    Pt, sq = E.cross_full(cw)
    sqe = E.einsum_sq(cw)
    out = {}
    for L in Ls:
        codes, _ = E.encode(X, cw, sqe, Pt, L, with_err=False)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); E.encode(X, cw, sqe, Pt, L, with_err=False); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out[L] = (min(ts), hashlib.sha1(codes.cpu().numpy().tobytes()).hexdigest()[:12])
    print(json.dumps(out))
    sys.exit(0)
args = sys.argv[1:]
sep = args.index("--") if "--" in args else len(args)
n = args[0] if sep > 0 else "1000000"
Ls = args[1] if sep > 1 else "1,10"
for name in args[sep + 1:]:
    env = dict(os.environ)
    if name != "cur":
        env["DA_LIB_PATH"] = os.path.join(ROOT, "tools", "ab", name, "libda_b200.so")
    r = subprocess.run([sys.executable, __file__, "--child", n, Ls], env=env, capture_output=True, text=True)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    print(f"{name:16s}", line[-1] if line else r.stderr[-800:], flush=True)
