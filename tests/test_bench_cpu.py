"""bench.py's launcher contract on CPU: --gpus N without torchrun re-launches
N ranks (gloo in --dry-run), broadcasts rank 0's codebook and reports n_gpus."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_self_launches_two_ranks():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2
    assert out["codebook_broadcast_equal"] is True
    assert out["max_over_ranks"] == 2.0


def test_bench_anneal_flop_formula():
    sys.path.insert(0, ROOT)
    import bench

    # one dictionary, one stage of d=128 with 2 iterations: 4ND^2 + 4NKD + 2NMKD + 3*2NKd
    N, D, M, K = 1000, 128, 1, 256
    f = bench.anneal_flop([(128, N, K, 2)], N, D, M, K)
    assert f == 4.0 * N * D * D + 4.0 * N * K * D + 2.0 * N * M * K * D + 3 * 2.0 * N * K * 128
