"""Streamed file encode rate: a synthetic config-B bvecs file (n vectors, D=128)
is written to /tmp, then encode_vecs streams it (raw records through pinned
slots, device unpack, L=10 beam encode, codes to an HCLE file).
usage: python tools/bench_ingest.py [n] [L]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, synthetic
from paper_1509_05194_b200.data import encode_vecs
import bench

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
L = int(sys.argv[2]) if len(sys.argv) > 2 else 10
path, out = "/tmp/ingest.bvecs", "/tmp/ingest.hcle"
t0 = time.perf_counter()
with open(path, "wb") as f:
    step = 1_000_000
    for r0 in range(0, n, step):
        X = synthetic.mixture_b_chunk(4, r0 // step, n=min(step, n - r0)).astype(np.uint8)
        rec = np.empty((X.shape[0], 132), dtype=np.uint8)
        rec[:, :4] = np.frombuffer(np.int32(128).tobytes(), dtype=np.uint8)
        rec[:, 4:] = X
        f.write(rec.tobytes())
gen_s = time.perf_counter() - t0
Xd = E.to_dev(bench.rank_data(0, 100_000))
cw, _ = E.growth_pass(Xd, da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0))
book = da.Codebook(codewords=cw.cpu().numpy(), order=np.arange(8))
cross = da.cross_products(book)
encode_vecs(book, path, L, cross=cross, chunk_rows=1 << 18) if n <= 2_000_000 else None
torch.cuda.synchronize()
t0 = time.perf_counter()
enc = encode_vecs(book, path, L, out_path=out, cross=cross)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(json.dumps({"n": n, "L": L, "file_GB": os.path.getsize(path) / 1e9, "generate_s": round(gen_s, 1),
                  "encode_vecs_s": dt, "vectors_per_s": n / dt, "hcle_bytes": os.path.getsize(out)}))
os.remove(path); os.remove(out)
