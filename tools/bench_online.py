"""Online DA (config D shape): stream 1M-vector uint8 chunks of the config-B
mixture (seed 3, substream per chunk).  Two paths are timed on the same chunks:

  * public: the one-GPU `train_online(codebook, chunk, TrainConfig(sweeps=1,
    rel_tol=0))` per chunk (host uint8 -> float32, synchronous upload);
  * stream: `distributed.train_online_stream` -- each rank's 1/world slice of
    every chunk uploaded as bytes through pinned buffers one chunk ahead
    (ChunkFeeder), trained with the exact shard reductions, an HCLB checkpoint
    written by rank 0 after every chunk.  Launch with torch.distributed.run for
    world > 1 (NCCL); without a launcher it runs as world 1.

The two paths must produce the same codebook (checked at world 1).
usage: [torchrun ...] python tools/bench_online.py [chunks] [chunk_rows]"""
import os, sys, time, json, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import synthetic, codebook as cb, distributed as DD

chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
if "RANK" not in os.environ:
    os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(29600 + os.getpid() % 1000))
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
dist.init_process_group("nccl")
comm = DD.Comm()
data = [synthetic.mixture_b_chunk(3, c, n=rows).astype(np.uint8) for c in range(chunks + 1)]
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
book0, _, _ = da.train_from_scratch(data[0][:100_000].astype(np.float32), cfg0)
cfg = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=1, rel_tol=0.0)
cw0, _ = cb._codebook_dev(book0)
mine = [ch[DD.shard_rows(len(ch), world, rank)] for ch in data[1:]]
ckdir = tempfile.mkdtemp()


def checkpoint(c, cw):
    if rank == 0:
        cb.write_codebook(os.path.join(ckdir, f"chunk{c}.hclb"),
                          da.Codebook(codewords=cw.cpu().numpy(), order=book0.order))


DD.train_online_stream(cw0, [m[: max(1, len(m) // 10)] for m in mine[:1]], cfg, comm)   # warm-up (untimed)
torch.cuda.synchronize()
dist.barrier()
t0 = time.perf_counter()
cw_s, reps = DD.train_online_stream(cw0, mine, cfg, comm, checkpoint=checkpoint)
torch.cuda.synchronize()
t_stream = time.perf_counter() - t0
out = {"workload": f"config D shape: {chunks} chunks x {rows} uint8 vectors over {world} GPU(s), sweeps=1",
       "stream_seconds_per_chunk": t_stream / chunks, "stream_vectors_per_s": rows * chunks / t_stream,
       "distortion_last": reps[-1].steps[-1].distortion, "checkpoints": sorted(os.listdir(ckdir))}
if world == 1:
    book = book0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for c in range(1, chunks + 1):
        book, rep = da.train_online(book, data[c].astype(np.float32), cfg)
    torch.cuda.synchronize()
    t_pub = time.perf_counter() - t0
    out.update({"public_seconds_per_chunk": t_pub / chunks, "public_vectors_per_s": rows * chunks / t_pub,
                "same_codebook": bool(np.array_equal(book.codewords, cw_s.cpu().numpy()))})
if rank == 0:
    print(json.dumps(out))
dist.destroy_process_group()
