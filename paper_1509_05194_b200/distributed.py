"""Row-sharded DA across the GPUs of one box (one process per GPU, NCCL).

The dataset is split by rows; every GPU keeps its shard, its codes and a
replica of the codebook + cross tables in HBM.  The only exchange steps are
the ones the algorithm has:

  * Lloyd update      allreduce of the K x D float64 per-codeword sums and
                      the K counts (plus the changed-row count);
  * PCA               a rank-ordered ring: each shard continues the column-sum
                      chains and the covariance's OpenBLAS block chains where
                      the previous shard stopped, so mean and covariance are
                      bit-identical to the unsharded reference (exact_pca_moments);
  * empty reseed      allgather of each shard's local worst (err, row id, row)
                      candidates, merged with the reference's order
                      (descending error, ties -> higher global row id);
  * distortions       allreduce of per-shard error sums.

Encoding and ADC shard with no collective at all.  The merge rules below are
plain functions of local partials so they are tested on CPU with gloo
(tests/test_distributed_cpu.py) and run on NCCL device tensors in production.
"""

from __future__ import annotations

import numpy as np
import torch

__all__ = ["Comm", "merge_worst", "shard_rows", "train_from_scratch_sharded", "da_sweep_sharded",
           "train_online_sharded", "ChunkFeeder", "train_online_stream",
           "blas_block_starts", "cov_segments", "exact_pca_moments"]


class Comm:
    """Thin torch.distributed wrapper used by the engine (`comm=` argument)."""

    def __init__(self, group=None, exact: bool = True):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        # exact=True: Lloyd sums in the reference's order across shards
        # (bit-identical to one GPU; W-1 neighbour rounds + a leaf-sum allreduce
        # per update).  exact=False: one allreduce of shard partial sums per
        # update (same algorithm, float64 sums in another order).
        self.exact = exact
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._bound = None
        self.row_offset = 0

    @property
    def _host_staged(self) -> bool:
        # gloo reduces on the host; NCCL works on device memory directly
        return self.dist.get_backend(self.group) != "nccl"

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        if self._host_staged and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, op=self.dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
            return t
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def allgather(self, t: torch.Tensor) -> torch.Tensor:
        src = t.contiguous().cpu() if (self._host_staged and t.is_cuda) else t.contiguous()
        parts = [torch.empty_like(src) for _ in range(self.world)]
        self.dist.all_gather(parts, src, group=self.group)
        out = torch.cat(parts, dim=0)
        return out.to(t.device) if t.is_cuda else out

    def _staged(self, t: torch.Tensor) -> torch.Tensor:
        return t.cpu() if (self._host_staged and t.is_cuda) else t

    def send_(self, t: torch.Tensor, dst: int) -> None:
        self.dist.send(self._staged(t.contiguous()), dst, group=self.group)

    def recv_(self, t: torch.Tensor, src: int) -> torch.Tensor:
        buf = self._staged(t)
        self.dist.recv(buf, src, group=self.group)
        if buf is not t:
            t.copy_(buf)
        return t

    def broadcast_(self, t: torch.Tensor, src: int) -> torch.Tensor:
        buf = self._staged(t)
        self.dist.broadcast(buf, src, group=self.group)
        if buf is not t:
            t.copy_(buf)
        return t

    def shift_(self, send: torch.Tensor, recv: torch.Tensor) -> torch.Tensor:
        """send -> rank + 1 and recv <- rank - 1 at once (the ends skip theirs)."""
        ops = []
        sb, rb = self._staged(send.contiguous()), self._staged(recv)
        if self.rank + 1 < self.world:
            ops.append(self.dist.P2POp(self.dist.isend, sb, self.rank + 1, group=self.group))
        if self.rank > 0:
            ops.append(self.dist.P2POp(self.dist.irecv, rb, self.rank - 1, group=self.group))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        if rb is not recv and self.rank > 0:
            recv.copy_(rb)
        return recv

    def sizes(self, n_local: int) -> list:
        """Every rank's shard size.  The allgather runs unless bind_rows() already
        recorded the sizes for this n_local; bind_rows is itself collective, so
        whether a call communicates is decided identically on every rank."""
        if self._bound is not None and self._bound[0] == n_local:
            return self._bound[1]
        dev = "cpu" if self._host_staged else "cuda"
        t = torch.tensor([n_local], dtype=torch.int64, device=dev)
        return [int(x) for x in self.allgather(t).cpu().tolist()]

    def total(self, n_local: int) -> int:
        return int(sum(self.sizes(n_local)))

    def bind_rows(self, n_local: int) -> "Comm":
        """Collective: record every shard's size and this shard's first global
        row id (shards are rank-ordered).  Later sizes()/total() calls with the
        same n_local read the record instead of communicating."""
        self._bound = None
        s = self.sizes(n_local)
        self._bound = (n_local, s)
        self.row_offset = int(sum(s[: self.rank]))
        return self


def shard_rows(n: int, world: int, rank: int) -> slice:
    """Contiguous, rank-ordered, near-equal row shards."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return slice(lo, lo + base + (1 if rank < extra else 0))


def blas_block_starts(n: int) -> list:
    """Row offsets of OpenBLAS's GEMM_Q blocks over an n-long contraction (the
    dsyrk behind Xc.T @ Xc, clustering.py:96): 384 rows, the last two balanced
    (common.cuh: blas_block_len)."""
    q = 384
    starts = [0]
    while starts[-1] < n:
        rest = n - starts[-1]
        step = q if rest >= 2 * q else (((rest // 2 + 1) // 2) * 2 if rest > q else rest)
        starts.append(starts[-1] + step)
    return starts


def cov_segments(n_total: int, lo: int, hi: int):
    """This shard's pieces of the global blocks: (segments as local row offsets
    [(r0, r1), ...], cont_first, open_last, total_valid_in).  cont_first: the
    first piece continues a block begun on an earlier shard; open_last: the
    last piece's block ends on a later shard; total_valid_in: some block
    completed before this shard (the incoming running total is live)."""
    st = blas_block_starts(n_total)
    segs, blocks = [], []
    for a, b in zip(st[:-1], st[1:]):
        if a < hi and b > lo:
            segs.append((max(a, lo) - lo, min(b, hi) - lo))
            blocks.append((a, b))
    cont_first = bool(blocks) and blocks[0][0] < lo
    open_last = bool(blocks) and blocks[-1][1] > hi
    total_valid_in = len(st) > 1 and st[1] <= lo
    return segs, cont_first, open_last, total_valid_in


def exact_pca_moments(X, comm: "Comm", ops):
    """Mean (D,) and covariance (D, D) of the row-sharded X (clustering.py:93-96),
    bit-identical to the unsharded computation.

    Both reductions of the reference are sequential in row order: X.mean(axis=0)
    is one add chain per column, and OpenBLAS's dsyrk cuts the n-long contraction
    into GEMM_Q blocks (each an FMA chain from zero) added into C in order.  So
    shards run a rank-ordered ring: rank r receives the running column sums,
    continues them over its rows and forwards them; then it receives the
    running covariance total and the carried chain of a block cut at the shard
    boundary, finishes that chain, adds its own blocks in order (their chains
    were computed before the receive, in parallel with the other ranks) and
    forwards the total plus its own cut chain.  The last rank divides and
    broadcasts.  `ops` supplies the arithmetic (device kernels in production,
    numpy in the CPU ring tests): zeros(shape), col_sums(X, init|None),
    div(t, d), cov_chains(X, mean, starts, init|None) -> (nseg, D, D),
    fold(total|None, parts) -> total."""
    n, D = X.shape
    sizes = comm.sizes(n)
    N = int(sum(sizes))
    lo = int(sum(sizes[: comm.rank]))
    hi = lo + n
    last = comm.world - 1
    prev, nxt = comm.rank - 1, comm.rank + 1
    # ---- column sums: one chain per column across the shards
    S = ops.zeros((D,))
    if prev >= 0:
        comm.recv_(S, prev)
    if n:
        S = ops.col_sums(X, S if lo > 0 else None)
    if nxt <= last:
        comm.send_(S, nxt)
    mean = ops.div(S, N) if comm.rank == last else ops.zeros((D,))
    comm.broadcast_(mean, last)
    if N <= D:
        return mean, None
    # ---- covariance: block chains, block totals added in global order
    segs, cont_first, open_last, t_valid = cov_segments(N, lo, hi)
    first = 1 if cont_first else 0
    parts = None
    if len(segs) > first:
        st = [segs[first][0]] + [b for _, b in segs[first:]]
        parts = ops.cov_chains(X, mean, st, None)      # before the receive: in parallel
    state = ops.zeros((2, D, D))
    if prev >= 0:
        comm.recv_(state, prev)
    T, C = state[0], state[1]
    if not segs:
        out = state                                   # empty shard: pass everything on
    else:
        chains = list(parts) if parts is not None else []
        if cont_first:
            chain0 = ops.cov_chains(X, mean, [segs[0][0], segs[0][1]], C)[0]
            chains = [chain0] + chains
        ncomplete = len(chains) - (1 if open_last else 0)
        out = ops.zeros((2, D, D))
        total = T if t_valid else None
        if cont_first and ncomplete >= 1:
            total = ops.fold(total, chain0.reshape(1, D, D))
        k = ncomplete - (1 if cont_first else 0)
        if k > 0:
            total = ops.fold(total, parts[:k])
        if total is not None:
            out[0] = total
        if open_last:
            out[1] = chains[-1]                       # the block continues on the next shard
    if nxt <= last:
        comm.send_(out, nxt)
    cov = ops.div(out[0], N - 1) if comm.rank == last else ops.zeros((D, D))
    comm.broadcast_(cov, last)
    return mean, cov


def merge_worst(all_err: np.ndarray, all_gid: np.ndarray, e: int) -> np.ndarray:
    """Indices (into the gathered candidate arrays) of the e globally worst
    points: descending error, ties broken towards the higher global row id --
    the order of argsort(errs, stable)[::-1] over the unsharded dataset
    (annq/clustering.py:195).  Padding entries carry err=-inf, gid=-1."""
    order = np.lexsort((-all_gid, -all_err))
    return order[:e]


def train_from_scratch_sharded(X_local: torch.Tensor, config, comm: Comm):
    """Growth pass + sweeps over row shards; returns (cw, local codes, report).

    Every rank ends with the same codebook (replicated state updated from
    allreduced statistics)."""
    from . import _engine as E
    from .annealing import TrainReport

    comm.bind_rows(X_local.shape[0])
    if comm.total(X_local.shape[0]) < config.k_count:
        raise ValueError(f"need at least k_count={config.k_count} vectors")
    report = TrainReport(config=config)
    cw, codes = E.growth_pass(X_local, config, report, comm=comm)
    E.sweep_until_converged(X_local, cw, codes, config, report, comm=comm)
    return cw, codes, report


def da_sweep_sharded(X_local, cw, codes, Pt, sq, config, comm: Comm, sweep_index=1, report=None):
    """One anneal pass over row shards (state mutated in place on every rank)."""
    from . import _engine as E

    comm.bind_rows(X_local.shape[0])
    E.da_sweep(X_local, cw, codes, Pt, sq, config, sweep_index=sweep_index, report=report, comm=comm)


def train_online_sharded(cw: torch.Tensor, X_local: torch.Tensor, config, comm: Comm, report=None):
    """annealing.py:248-262 over row shards (config D: each GPU holds 1/world of
    the batch): encode this shard's rows with the current codebook, then
    config.sweeps annealing passes with the exact shard reductions.  Every rank
    returns the same new codebook (float32 (M, K, D) on the device) -- the
    codebook the one-GPU train_online returns for the whole batch."""
    from . import _engine as E
    from .annealing import TrainReport

    comm.bind_rows(X_local.shape[0])
    report = report if report is not None else TrainReport(config=config)
    cw = cw.clone()
    Pt, sq = E.cross_full(cw)
    codes, _ = E.encode(X_local, cw, sq, Pt, config.beam_width, out_dtype=torch.int32, with_err=False)
    E.sweep_until_converged(X_local, cw, codes, config, report, comm=comm)
    return cw, report


class ChunkFeeder:
    """Host chunks (this rank's rows, numpy uint8 or float32) -> device float32,
    uploaded through page-locked buffers on a side stream one chunk ahead: while
    chunk c trains, chunk c+1 is copied into pinned memory (a worker thread) and
    sent to the device asynchronously (config D's pinned async copies).  uint8
    rows travel as bytes (128 B per config-D row) and widen on the device."""

    def __init__(self, chunks, device=None):
        import threading

        self.chunks = list(chunks)
        self.dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.side = torch.cuda.Stream(device=self.dev)
        self._threading = threading

    def _stage(self, i):
        a = np.ascontiguousarray(self.chunks[i])
        dt = torch.uint8 if a.dtype == np.uint8 else torch.float32
        if a.dtype not in (np.uint8, np.float32):
            a = a.astype(np.float32)
        pin = torch.empty(a.shape, dtype=dt, pin_memory=True)
        pin.numpy()[...] = a
        dev = torch.empty(a.shape, dtype=dt, device=self.dev)
        with torch.cuda.stream(self.side):
            dev.copy_(pin, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.side)
        return pin, dev, ev

    def __iter__(self):
        if not self.chunks:
            return
        nxt = self._stage(0)
        for i in range(len(self.chunks)):
            pin, dev, ev = nxt
            holder = {}
            th = None
            if i + 1 < len(self.chunks):
                # next chunk: host copy into pinned memory + async upload, off the critical path
                th = self._threading.Thread(target=lambda: holder.setdefault("v", self._stage(i + 1)))
                th.start()
            main = torch.cuda.current_stream(self.dev)
            main.wait_event(ev)
            dev.record_stream(main)                   # read on the main stream: no early reuse
            X = dev.float() if dev.dtype == torch.uint8 else dev
            yield X
            if th is not None:
                th.join()
                nxt = holder["v"]
            del pin


def train_online_stream(cw: torch.Tensor, chunks, config, comm: Comm, checkpoint=None):
    """Online DA over a stream of chunks (config D): this rank's slice of each
    chunk is uploaded one chunk ahead (ChunkFeeder) and trained with
    train_online_sharded.  checkpoint(c, cw) is called after every chunk (rank 0
    writes an HCLB checkpoint in tools/bench_online.py).  Returns (cw, reports)."""
    reports = []
    for c, X in enumerate(ChunkFeeder(chunks)):
        cw, rep = train_online_sharded(cw, X, config, comm)
        reports.append(rep)
        if checkpoint is not None:
            checkpoint(c, cw)
    return cw, reports
