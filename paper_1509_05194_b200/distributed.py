"""Row-sharded DA across the GPUs of one box (one process per GPU, NCCL).

The dataset is split by rows; every GPU keeps its shard, its codes and a
replica of the codebook + cross tables in HBM.  The only exchange steps are
the ones the algorithm has:

  * Lloyd update      allreduce of the K x D float64 per-codeword sums and
                      the K counts (plus the changed-row count);
  * PCA               allreduce of the column sums, then of the centred Gram;
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

__all__ = ["Comm", "merge_worst", "shard_rows", "train_from_scratch_sharded", "da_sweep_sharded"]


class Comm:
    """Thin torch.distributed wrapper used by the engine (`comm=` argument)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
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
