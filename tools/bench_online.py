"""Online DA (config D shape) on one GPU: stream 1M-vector uint8 chunks of the
config-B mixture (seed 3, substream per chunk) through the public
`train_online(codebook, chunk, TrainConfig(sweeps=1, rel_tol=0))`: per chunk
host uint8 -> float32, upload, beam encode, one anneal pass, codebook back to
the host.  Chunks are generated before the timed loop.

usage: python tools/bench_online.py [chunks] [chunk_rows]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import synthetic

chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
data = [synthetic.mixture_b_chunk(3, c, n=rows).astype(np.uint8) for c in range(chunks + 1)]
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
book, _, _ = da.train_from_scratch(data[0][:100_000].astype(np.float32), cfg0)
cfg = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=1, rel_tol=0.0)
book, _ = da.train_online(book, data[0].astype(np.float32), cfg)  # warm-up chunk (untimed)
torch.cuda.synchronize()
per_chunk = []
for c in range(1, chunks + 1):
    t0 = time.perf_counter()
    book, rep = da.train_online(book, data[c].astype(np.float32), cfg)
    per_chunk.append(time.perf_counter() - t0)
print(json.dumps({"workload": f"config D shape on 1 GPU: {chunks} chunks x {rows} uint8 vectors, train_online sweeps=1",
                  "seconds_per_chunk": [round(t, 3) for t in per_chunk],
                  "vectors_per_s": rows * chunks / sum(per_chunk),
                  "distortion_last": rep.steps[-1].distortion}))
