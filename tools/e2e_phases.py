"""Phases of the end-to-end encode (encode_dataset on host float32 rows, config B)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, codebook as cbm
import bench
n = 1000000
X = bench.rank_data(0, n)
Xd = E.to_dev(X)
cw, _ = E.growth_pass(Xd[:100000].contiguous(), da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0))
book = da.Codebook(codewords=cw.cpu().numpy(), order=np.arange(8))
cross = da.cross_products(book)
cwd, sqd = cbm._codebook_dev(book); Pt, _ = cbm._cross_dev(cross)
def t(f, label, rep=3):
    best = 1e9
    for _ in range(rep):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    print(f"{label:44s} {best*1e3:8.2f} ms", flush=True)
t(lambda: E.encode(Xd, cwd, sqd, Pt, 10, out_dtype=torch.uint8, with_err=False), "device encode (resident)")
for ch in (32768, 65536, 131072, 262144):
    t(lambda: E.encode_host(X, cwd, sqd, Pt, 10, out_dtype=torch.uint8, chunk=ch), f"encode_host chunk {ch}")
codes = E.encode_host(X, cwd, sqd, Pt, 10, out_dtype=torch.uint8)
t(lambda: codes.cpu(), "codes D2H 8 MB")
h = codes.cpu().numpy()
t(lambda: da.EncodedDataset(codes=h, k_count=256, codebook_hash=book.content_hash()), "EncodedDataset (checks)")
t(lambda: book.content_hash(), "content_hash")
t(lambda: da.encode_dataset(book, X, beam_width=10, cross=cross), "encode_dataset (public API)")
# isolate: pipeline without the host copy (slot contents stale), and without H2D
D = 128
def fill_nop(slot, r0, rows):
    pass
def to_rows_f32(raw, rows, buf):
    return raw.view(torch.float32).view(rows, D)
t(lambda: E._encode_stream(n, D, 4 * D, fill_nop, to_rows_f32, cwd, sqd, Pt, 10, torch.uint8, 131072), "stream: no host copy (H2D + encode)")
def to_rows_dev(raw, rows, buf, _c=[0]):
    return Xd[:rows]
t(lambda: E._encode_stream(n, D, 4 * D, fill_nop, to_rows_dev, cwd, sqd, Pt, 10, torch.uint8, 131072), "stream: no copy, device rows (H2D unused)")
t(lambda: [E.encode(Xd[i:i + 131072], cwd, sqd, Pt, 10, out_dtype=torch.uint8, with_err=False) for i in range(0, n, 131072)], "8 device encode calls of 131072")
