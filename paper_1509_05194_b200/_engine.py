"""Device-resident DA engine: torch tensors in HBM, kernels through the C-ABI.

Everything here works on CUDA tensors and never round-trips data to the host
except (a) the few scalars the reference's control flow branches on
(empty-cluster counts, the Lloyd stable test, the keep-staged-or-init test,
the sweep's convergence test) and (b) the D x D covariance handed to LAPACK's
eigh, exactly as the reference computes it on the CPU
(annq/clustering.py:97).  Public, reference-shaped functions live in
codebook.py / clustering.py / annealing.py and call into this module.

`comm` (see distributed.py) is None for one GPU; with a communicator the rows
of X are a shard of the dataset and every reduction the reference performs
over rows is completed with an NCCL allreduce.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from ._native import load_library as native_lib, native

F32, F64, I32, I64 = torch.float32, torch.float64, torch.int32, torch.int64


# ---------------------------------------------------------------------------
# plumbing


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1509_05194_b200 runs on a CUDA device only (no CPU fallback); "
            "no GPU is visible"
        )


def device() -> torch.device:
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def P(t) -> ctypes.c_void_p | None:
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def is_f32(t: torch.Tensor) -> int:
    if t.dtype == F32:
        return 1
    if t.dtype == F64:
        return 0
    raise TypeError(f"expected float32/float64 tensor, got {t.dtype}")


def code_bytes(t: torch.Tensor) -> int:
    return {torch.uint8: 1, torch.uint16: 2, torch.int32: 4}[t.dtype]


def to_dev(a, dtype=None) -> torch.Tensor:
    """Host array -> contiguous CUDA tensor (pinned staging for large arrays)."""
    if isinstance(a, torch.Tensor):
        t = a
    else:
        a = np.ascontiguousarray(a)
        t = torch.from_numpy(a)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.to(device(), non_blocking=False).contiguous()


def scalar(t: torch.Tensor) -> float:
    return float(t.item())


# ---------------------------------------------------------------------------
# reductions in numpy order


def true_div(t: torch.Tensor, d) -> torch.Tensor:
    """t / d as an IEEE division (numpy's true_divide).  torch turns a division
    by a Python scalar into a multiply by its reciprocal, which can differ in
    the last bit, so the divisor is passed as a tensor."""
    return t / torch.full_like(t, float(d))


def np_mean(a: torch.Tensor, comm=None) -> torch.Tensor:
    """Device scalar equal to numpy's a.mean() (pairwise) on one GPU.

    Sharded: per-shard pairwise sums, allreduced, divided by the global n.
    """
    out = torch.empty(1, dtype=F64, device=a.device)
    n = a.numel()
    if comm is None:
        native.da_np_sum(P(a), n, 1, P(out), stream())
        return out
    if n:
        native.da_np_sum(P(a), n, 0, P(out), stream())
    else:
        out.zero_()
    comm.allreduce_(out)
    return true_div(out, comm.total(n))


def row_sqnorms(A: torch.Tensor, d: int) -> torch.Tensor:
    out = torch.empty(A.shape[0], dtype=F64, device=A.device)
    native.da_row_sqnorms(P(A), is_f32(A), A.shape[0], A.stride(0), d, P(out), stream())
    return out


def assign(X: torch.Tensor, d: int, C: torch.Tensor, cc: torch.Tensor | None = None,
           prev: torch.Tensor | None = None, changed: torch.Tensor | None = None, xx: torch.Tensor | None = None,
           want_d2: bool = True):
    """annq/clustering.py:139-148 on the first d columns; labels int32, d2 f64.
    `xx` = row_sqnorms(X, d) may be passed to reuse it across Lloyd iterations.
    want_d2=False returns (labels, None): rows whose nearest codeword the
    tensor-core filter decides alone skip the float64 recheck."""
    n, K = X.shape[0], C.shape[0]
    if cc is None:
        cc = row_sqnorms(C, d)
    labels = torch.empty(n, dtype=I32, device=X.device)
    d2 = torch.empty(n, dtype=F64, device=X.device) if want_d2 else None
    native.da_assign(P(X), is_f32(X), n, X.stride(0), d, P(C), C.stride(0), K, P(cc), P(xx), P(labels), P(d2),
                     P(prev), P(changed), stream())
    return labels, d2


class assign_image:
    """Context manager binding the tf32 row image of X[:, :d] for the assigns of
    one Lloyd call (da_assign_bind_image); the buffer is reused across calls."""

    _buf = None

    def __init__(self, X: torch.Tensor, d: int):
        self.X, self.d = X, d

    def __enter__(self):
        n = self.X.shape[0]
        nbytes = int(native_lib().da_assign_image_bytes(n, self.d)) if n else 0
        if nbytes:
            buf = assign_image._buf
            if buf is None or buf.numel() < nbytes or buf.device != self.X.device:
                assign_image._buf = buf = None
                buf = torch.empty(nbytes, dtype=torch.uint8, device=self.X.device)
                assign_image._buf = buf
            native.da_assign_bind_image(P(self.X), is_f32(self.X), n, self.X.stride(0), self.d, P(buf), stream())
        return self

    def __exit__(self, *exc):
        native.da_assign_bind_image(None, 0, 0, 0, 0, None, stream())
        return False


# ---------------------------------------------------------------------------
# Lloyd k-means with an active prefix (annq/clustering.py:165-203)


def _reseed_single(Xr, errs, empty_idx, C):
    """C[empty] = X[worst], worst = argsort(errs, stable)[::-1][:e] (clustering.py:192-196)."""
    e = len(empty_idx)
    errs_h = errs.cpu().numpy()
    worst = np.argsort(errs_h, kind="stable")[::-1][:e].copy()
    src = torch.from_numpy(worst.astype(np.int64)).to(Xr.device)
    dst = torch.from_numpy(np.asarray(empty_idx, dtype=np.int32)).to(Xr.device)
    native.da_gather_rows(P(Xr), Xr.stride(0), Xr.shape[1], P(src), P(dst), e, P(C), C.stride(0), stream())


def _reseed_sharded(Xr, errs, empty_idx, C, comm):
    """Global worst points across shards: each shard offers its local top-e
    (err, global row id) pairs, merged with the reference's order
    (descending error, ties to the higher row id)."""
    e = len(empty_idx)
    errs_h = errs.cpu().numpy()
    local = np.argsort(errs_h, kind="stable")[::-1][:e].copy()
    offset = comm.row_offset
    cand_err = torch.full((e,), -np.inf, dtype=F64)
    cand_gid = torch.full((e,), -1, dtype=I64)
    cand_err[: len(local)] = torch.from_numpy(errs_h[local])
    cand_gid[: len(local)] = torch.from_numpy(local.astype(np.int64) + offset)
    rows = torch.zeros((e, Xr.shape[1]), dtype=F64, device=Xr.device)
    if len(local):
        rows[: len(local)] = Xr[torch.from_numpy(local.astype(np.int64)).to(Xr.device)]
    all_err = comm.allgather(cand_err.to(Xr.device)).cpu().numpy().reshape(-1)
    all_gid = comm.allgather(cand_gid.to(Xr.device)).cpu().numpy().reshape(-1)
    all_rows = comm.allgather(rows).reshape(-1, Xr.shape[1])
    from .distributed import merge_worst

    pick = torch.from_numpy(merge_worst(all_err, all_gid, e).astype(np.int64)).to(Xr.device)
    C[torch.from_numpy(np.asarray(empty_idx, dtype=np.int64)).to(C.device)] = all_rows[pick]


def _sharded_update(red, K, d, C, comm):
    """red = [local (K, d) sums | local K counts] in one f64 buffer: one
    allreduce, then C[filled, :d] = sums / counts (the division of
    clustering.py:161); empty clusters keep their rows for the reseed.
    Returns the number of empty clusters as a device scalar."""
    comm.allreduce_(red)
    sums, cnt = red[: K * d].view(K, d), red[K * d:]
    C[:, :d] = torch.where(cnt.unsqueeze(1) > 0, sums / cnt.unsqueeze(1), C[:, :d])
    return (cnt == 0).sum()


_FLAGS_H: list = []


def _pinned_flags() -> list:
    """Two page-locked int64[2] flag buffers for the Lloyd loop (kept: pinning is slow)."""
    if not _FLAGS_H:
        _FLAGS_H.extend(torch.zeros(2, dtype=torch.int64, pin_memory=True) for _ in range(2))
    return _FLAGS_H


# When a list, every Lloyd call appends (active width, rows, K, iterations):
# the per-stage iteration counts I_{m,s} of SURVEY 8(d)'s anneal-pass FLOP formula.
LLOYD_LOG: list | None = None


def lloyd(Xr: torch.Tensor, C_init: torch.Tensor, active: int, max_iters: int, comm=None, want_trace: bool = True):
    """Returns (C f64 (K,D), labels int32 (n,), trace list[float]).

    want_trace=False (the cool-down inside DA, whose traces nobody reads): the
    trace is not computed (returned empty) and the assigns write labels only.
    The per-row errors are then needed only by an empty-cluster reseed
    (clustering.py:195, ~1% of updates); they are recomputed there against a
    snapshot of the centroids they belong to.  Centroids and labels are the
    same bits either way."""
    Xa = _active_prefix(Xr, active) if comm is None else None
    with assign_image(Xr if Xa is None else Xa, active):
        return _lloyd(Xr, C_init, active, max_iters, comm, not want_trace, Xa=Xa)


def _active_prefix(Xr: torch.Tensor, active: int):
    """A compact copy of the active columns for narrow prefixes (one-GPU loop).

    The iterations of a stage read only the first `active` columns of the rotated rows; at
    D = 128 those are 16-64 bytes out of every 1-KB row, one DRAM granule per row for every
    gather of the Lloyd update and every assign.  A (n, 8 or 16) float64 copy (64-128 MB at 1M
    rows, L2-sized below ~1M x 8) serves the whole stage: same values, same order, same bits."""
    n, D = Xr.shape
    if active > 16 or D < 64 or n < 32768 or Xr.dtype != F64:
        return None
    apad = 8 if active <= 8 else 16
    Xa = _arena("lloyd_xa", (n, apad), F64, Xr.device)
    Xa.copy_(Xr[:, :apad])
    return Xa


def _arena(name: str, shape, dtype, dev) -> torch.Tensor:
    """A persistent device buffer per (name, shape, dtype, device)."""
    key = (name, tuple(shape), dtype, dev)
    t = _ARENA.get(key)
    if t is None:
        t = _ARENA[key] = torch.empty(tuple(shape), dtype=dtype, device=dev)
    return t


_ARENA: dict = {}
_EVENTS: dict = {}


def _lloyd_events():
    dev = torch.cuda.current_device()
    if dev not in _EVENTS:
        evs = [torch.cuda.Event(), torch.cuda.Event()]
        for e in evs:
            e.record()                                # creates the handles da_lloyd_step records into
        _EVENTS[dev] = evs
    return _EVENTS[dev]


def _lloyd(Xr: torch.Tensor, C_init: torch.Tensor, active: int, max_iters: int, comm=None, lazy=False, Xa=None):
    if comm is not None and comm.world == 1 and not os.environ.get("DA_SHARD_LOOP"):
        comm = None   # one shard: nothing to exchange (DA_SHARD_LOOP=1 keeps the shard loop, for timing it)
    if Xa is None or comm is not None:
        Xa = Xr       # the rows the iterations read (a compact copy of the active columns, or Xr itself)
    n, D = Xr.shape
    K = C_init.shape[0]
    dev = Xr.device
    if comm is None:
        C = _arena("lloyd_C0", C_init.shape, F64, dev)
        C.copy_(C_init)
    else:
        C = C_init.clone().contiguous()
    trace_d = torch.empty(max_iters + 1, dtype=F64, device=dev)
    xx = None
    if n:
        xx = _arena("lloyd_xx", (n,), F64, dev) if comm is None else torch.empty(n, dtype=F64, device=dev)
        native.da_row_sqnorms(P(Xa), is_f32(Xa), n, Xa.stride(0), active, P(xx), stream())   # fixed for the stage
    labels, errs = assign(Xa, active, C, xx=xx, want_d2=not lazy)
    if comm is None and n:
        lab2 = _arena("lloyd_lab2", (n,), I32, dev)   # the ring slot iteration 0 reads (labels_prev)
        lab2.copy_(labels)
        labels = lab2
        if not lazy:
            d22 = _arena("lloyd_d22", (n,), F64, dev)
            d22.copy_(errs)
            errs = d22
    if not lazy:
        trace_d[0:1] = np_mean(errs, comm)
    iters = 0
    counts = torch.empty(K, dtype=I32, device=dev)
    if comm is None:
        # Only the active prefix feeds the assignments, so the iterations average the
        # active columns; the remaining columns are averaged once at the end over the
        # labels of the last update (per-column sums: identical bits).  Reseeds write
        # whole rows, as in the reference.
        #
        # Iteration i+1 is launched before the host looks at iteration i's flags
        # (rows changed, clusters emptied), so the device never idles on the
        # per-iteration sync.  It runs in the other of two centroid buffers and is
        # dropped when iteration i converged or emptied a cluster (the reseed
        # changes C_i, so i+1 is recomputed); accepted results are the
        # reference's, step for step.
        # Persistent buffers (same addresses every call of this shape): the
        # library replays a CUDA graph of an iteration whose arguments it has
        # seen before (da_lloyd_step), so slots, label and error rings and the
        # events are reused across Lloyd calls and dictionary steps.
        slots = [(C, _arena("lloyd_cnt0", (K,), I32, dev), _arena("lloyd_fl0", (2,), torch.int64, dev)),
                 (_arena("lloyd_C1", C.shape, F64, dev), _arena("lloyd_cnt1", (K,), I32, dev),
                  _arena("lloyd_fl1", (2,), torch.int64, dev))]
        flags_h = _pinned_flags()
        done_ev = _lloyd_events()
        snaps = [_arena("lloyd_snap0", C.shape, F64, dev), _arena("lloyd_snap1", C.shape, F64, dev)] if lazy else None
        lab_ring = [_arena(f"lloyd_lab{i}", (n,), I32, dev) for i in range(3)]
        d2_ring = None if lazy else [_arena(f"lloyd_d2{i}", (n,), F64, dev) for i in range(3)]
        nlaunch = [0]

        def launch(C_prev, labels_prev, slot):
            Cn, cn, fl = slots[slot]
            j = nlaunch[0]
            nlaunch[0] += 1
            nl = lab_ring[j % 3]
            if nl is labels_prev:                    # a reseed re-assign broke the rotation
                nl = lab_ring[(j + 1) % 3]
            ne = None if lazy else d2_ring[j % 3]
            # group means, #empty, assign, flags -> pinned host, event: one call
            native.da_lloyd_step(P(Xa), n, Xa.stride(0), active, K, P(C_prev), P(Cn), Cn.stride(0),
                                 P(snaps[slot]) if lazy else None, P(labels_prev), P(nl), P(ne), P(xx), P(cn), P(fl),
                                 P(flags_h[slot]), ctypes.c_void_p(done_ev[slot].cuda_event), stream())
            return [slot, labels_prev, nl, ne]

        gs_labels = None
        cur = launch(C, labels, 0) if max_iters > 0 else None
        while cur is not None:
            slot, labels_prev, new_labels, errs_new = cur
            Cn, cn, fl = slots[slot]
            spec = launch(Cn, new_labels, slot ^ 1) if iters + 1 < max_iters else None
            done_ev[slot].synchronize()
            fh = flags_h[slot].numpy().copy()
            if fh[1]:
                spec = None                          # computed from pre-reseed centroids
                empty = np.flatnonzero(cn.cpu().numpy() == 0)
                if lazy:
                    errs = assign(Xa, active, snaps[slot], xx=xx)[1]
                _reseed_single(Xr, errs, empty, Cn)
                fl.zero_()
                new_labels, errs_new = assign(Xa, active, Cn, prev=labels_prev, changed=fl[0:1], xx=xx,
                                              want_d2=not lazy)
                fh = fl.cpu().numpy()
            C = Cn
            gs_labels = labels_prev
            errs = errs_new
            iters += 1
            if not lazy:
                trace_d[iters:iters + 1] = np_mean(errs, comm)
            labels = new_labels
            if int(fh[0]) == 0 or iters >= max_iters:
                break
            cur = spec if spec is not None else launch(C, labels, slot ^ 1)
        if gs_labels is not None and active < D:
            native.da_group_sums(P(Xr), n, Xr.stride(0), D, P(gs_labels), K, 0, P(C), C.stride(0), P(counts),
                                 stream())
        trace = [] if lazy else trace_d[: iters + 1].cpu().tolist()
        if LLOYD_LOG is not None:
            LLOYD_LOG.append((active, n, K, iters))
        return C.clone(), labels.clone(), trace   # the loop's buffers are reused by the next call
    return _lloyd_sharded(Xr, C, labels, errs, xx, trace_d, active, max_iters, comm, lazy)


_FLAGS_SH: list = []


class _ShardSums:
    """Buffers + calls of the exact sharded Lloyd update (da_gs_shard_*): the
    one-GPU reduceat order across row shards (see groupsum.cu)."""

    def __init__(self, K, D, n_total, comm, dev):
        self.K, self.comm = K, comm
        self.cap = K + n_total // 64 + 2           # >= the global leaf count
        self.cnt_local = torch.empty(K, dtype=I32, device=dev)
        self.send = torch.zeros(K * 8 * D, dtype=F64, device=dev)
        self.recv = torch.zeros(K * 8 * D, dtype=F64, device=dev)

    def plan(self, Xr, d, labels, red, gcount, rounds=None, overflow=None):
        """Leaf sums + first rows of this shard into red (then allreduced by
        the caller); gcount = global label counts.  `rounds` neighbour
        exchanges (default: all world-1); the plan adds to `overflow` for cut
        leaves spanning more boundaries (the caller redoes the update)."""
        comm, K = self.comm, self.K
        n = Xr.shape[0]
        native.da_gs_shard_sort(P(Xr), n, Xr.stride(0), d, P(labels), K, P(self.cnt_local), stream())
        cnt_all = comm.allgather(self.cnt_local)
        send, recv = self.send[: K * 8 * d], self.recv[: K * 8 * d]
        rounds = comm.world - 1 if rounds is None else min(rounds, comm.world - 1)
        native.da_gs_shard_plan(P(Xr), n, Xr.stride(0), d, K, P(cnt_all), comm.world, comm.rank, self.cap, P(red),
                                P(send), P(gcount), rounds, P(overflow), stream())
        for _ in range(rounds):
            comm.shift_(send, recv)
            native.da_gs_shard_round(P(Xr), Xr.stride(0), d, K, P(recv), P(send), P(red), stream())

    def fold(self, d, red, gcount, mode, out):
        native.da_gs_shard_fold(d, self.K, P(red), self.cap, P(gcount), mode, P(out), out.stride(0), stream())


def _lloyd_sharded(Xr, C, labels, errs, xx, trace_d, active, max_iters, comm, lazy=False):
    """The Lloyd loop over row shards (clustering.py:165-203, statistics allreduced).

    Same restructuring as the one-GPU loop: the iterations sum only the active
    prefix and the remaining columns are summed once at the end; iteration i+1
    is launched before the host reads iteration i's flags.  ONE collective per
    iteration: the allreduce of [active sums | counts | rows changed | error
    sum], where the last two belong to the previous iteration's assign (so the
    stop decision for iteration i is read from iteration i+1's allreduce; when
    it says "converged", i+1 is dropped).  Every decision the host takes
    (converged, reseed) is a function of allreduced values, so all ranks launch
    the same collective sequence.
    """
    n, D = Xr.shape
    K = C.shape[0]
    dev = Xr.device
    da = active
    ntot = float(comm.total(n))
    if not _FLAGS_SH:
        _FLAGS_SH.extend(torch.zeros(4, dtype=F64, pin_memory=True) for _ in range(2))
    flags_h = _FLAGS_SH
    # neighbour rounds of the exact exchange: most cut leaves span one boundary;
    # an update whose leaves need more is redone with world - 1 rounds (flag)
    rounds = min(comm.world - 1, int(os.environ.get("DA_SHARD_ROUNDS", "2")))
    exact = getattr(comm, "exact", False)
    sh = _ShardSums(K, D, int(ntot), comm, dev) if exact else None
    # reduced buffer: [sums | counts] (fast) or [leaf sums | first rows] (exact),
    # then the stats of the assign before this update
    nst = sh.cap * da + K * da if exact else K * da + K

    def new_slot(Cbuf):
        nred = nst + 3
        return (Cbuf, torch.empty(nred, dtype=F64, device=dev), torch.empty(K, dtype=I32, device=dev),
                torch.zeros(1, dtype=torch.int64, device=dev), torch.zeros(4, dtype=F64, device=dev),
                torch.cuda.Event())

    slots = [new_slot(C), new_slot(torch.empty_like(C))]
    snaps = [torch.empty_like(C), torch.empty_like(C)]   # C before each update: reseed errors, exchange redo

    def put_stats(dst, chg, ne):
        """dst[0:2] = this shard's [rows changed, error sum] of one assign."""
        if chg is None:
            dst.zero_()
            return
        dst[0:1].copy_(chg)
        if n and ne is not None:
            native.da_np_sum(P(ne), n, 0, P(dst[1:2]), stream())
        else:
            dst[1:2].zero_()

    for sl in slots:
        sl[5].record()                               # creates the event handles da_lloyd_finish records into

    def launch(C_prev, labels_prev, slot, pchg, pne, nrounds=None):
        Cn, red, cn, chg, fl, ev = slots[slot]
        # C_out = C_prev (+ snapshot), previous assign's stats -> red[nst:]
        native.da_lloyd_prepare(P(C_prev), P(Cn), P(snaps[slot]) if C_prev is not snaps[slot] else None, C.numel(),
                                P(pchg), P(red[nst:]), stream())
        if pne is not None and n:
            native.da_np_sum(P(pne), n, 0, P(red[nst + 1:nst + 2]), stream())
        if exact:
            sh.plan(Xr, da, labels_prev, red, cn, rounds if nrounds is None else nrounds, red[nst + 2:nst + 3])
        else:
            if n:
                native.da_group_sums(P(Xr), n, Xr.stride(0), da, P(labels_prev), K, 1, P(red), da, P(cn), stream())
                red[K * da:nst].copy_(cn)
            else:
                red[:nst].zero_()
        comm.allreduce_(red)
        if exact:
            sh.fold(da, red, cn, 0, Cn)
        nl = torch.empty(n, dtype=I32, device=dev)
        ne = None if lazy else torch.empty(n, dtype=F64, device=dev)
        # means (fast mode), flags -> pinned host + event, then the assign
        native.da_lloyd_finish(0 if exact else 1, P(red), P(cn), K, da, P(Cn), Cn.stride(0), P(red[nst:]), P(fl),
                               P(flags_h[slot]), ctypes.c_void_p(ev.cuda_event), P(Xr), n, Xr.stride(0), P(xx),
                               P(labels_prev), P(nl) if n else None, P(ne), P(chg), stream())
        return [slot, labels_prev, nl, ne]

    iters = 0
    gs_labels = None
    cur = launch(C, labels, 0, None, None) if max_iters > 0 else None
    spec = None
    if cur is not None and max_iters > 1:
        spec = launch(slots[0][0], cur[2], 1, slots[0][3], cur[3])
    while cur is not None:
        slot, labels_prev, _, _ = cur
        Cn, red, cn, chg, fl, ev = slots[slot]
        ev.synchronize()
        if flags_h[slot][3].item():
            # a cut leaf spanned more shards than the exchange rounds: redo this update
            if os.environ.get("DA_DEBUG"):
                print(f"[da] shard exchange overflow at iteration {iters}: redo with {comm.world - 1} rounds", flush=True)
            spec = None
            cur = launch(snaps[slot], labels_prev, slot, None, None, comm.world - 1)
            ev.synchronize()
        if flags_h[slot][0].item():
            spec = None                              # computed from pre-reseed centroids
            gcnt = cn if exact else red[K * da:nst]
            empty = np.flatnonzero(gcnt.cpu().numpy() == 0)
            if lazy:
                errs = assign(Xr, active, snaps[slot], xx=xx)[1] if n else torch.empty(0, dtype=F64, device=dev)
            _reseed_sharded(Xr, errs, empty, Cn, comm)
            chg.zero_()
            cur[2], cur[3] = assign(Xr, active, Cn, prev=labels_prev, changed=chg, xx=xx, want_d2=not lazy)
        C = Cn
        gs_labels = labels_prev
        labels, errs = cur[2], cur[3]
        iters += 1
        if iters >= max_iters:
            if not lazy:                             # no next iteration carries the last assign's stats
                st = torch.zeros(2, dtype=F64, device=dev)
                put_stats(st, chg, errs)
                comm.allreduce_(st)
                trace_d[iters:iters + 1] = true_div(st[1:2], ntot)
            break
        if spec is None:
            spec = launch(C, labels, slot ^ 1, chg, errs)
        s2 = spec[0]
        slots[s2][5].synchronize()
        fh = flags_h[s2].numpy().copy()
        trace_d[iters] = fh[2] / ntot
        if int(fh[1]) == 0:
            break                                    # iteration `iters` changed no row: spec dropped
        cur, spec = spec, None
        if iters + 1 < max_iters:
            spec = launch(slots[s2][0], cur[2], s2 ^ 1, slots[s2][3], cur[3])
    if gs_labels is not None and active < D and exact:
        full = torch.empty(sh.cap * D + K * D, dtype=F64, device=dev)
        gcnt = torch.empty(K, dtype=I32, device=dev)
        sh.plan(Xr, D, gs_labels, full, gcnt)
        comm.allreduce_(full)
        sh.fold(D, full, gcnt, 0, C)
    elif gs_labels is not None and active < D:
        full = torch.empty(K * D + K, dtype=F64, device=dev)
        sums, cnt = full[: K * D].view(K, D), full[K * D:]
        counts = torch.empty(K, dtype=I32, device=dev)
        if n:
            native.da_group_sums(P(Xr), n, Xr.stride(0), D, P(gs_labels), K, 1, P(sums), D, P(counts), stream())
        else:
            full.zero_()
            counts.zero_()
        cnt.copy_(counts)
        _sharded_update(full, K, D, C, comm)
    trace = [] if lazy else trace_d[: iters + 1].cpu().tolist()
    if LLOYD_LOG is not None:
        LLOYD_LOG.append((active, n, K, iters))
    return C, labels, trace


# ---------------------------------------------------------------------------
# PCA (annq/clustering.py:82-113) and the staged k-means (clustering.py:215-250)


def _complete_basis(components: np.ndarray, d: int) -> np.ndarray:
    """Gram-Schmidt completion of an orthonormal row set (clustering.py:63-79)."""
    rows = [components[i] for i in range(components.shape[0])]
    for j in range(d):
        if len(rows) == d:
            break
        v = np.zeros(d)
        v[j] = 1.0
        for _ in range(2):
            for u in rows:
                v -= (v @ u) * u
        nv = np.linalg.norm(v)
        if nv > 1e-8:
            rows.append(v / nv)
    if len(rows) != d:
        raise RuntimeError("failed to complete an orthonormal basis")
    return np.vstack(rows)


class _DevicePcaOps:
    """Device arithmetic of distributed.exact_pca_moments (the sharded PCA ring)."""

    def __init__(self, dev):
        self.dev = dev

    def zeros(self, shape):
        return torch.zeros(shape, dtype=F64, device=self.dev)

    def div(self, t, d):
        return true_div(t, d)

    def col_sums(self, X, init):
        out = torch.empty(X.shape[1], dtype=F64, device=X.device)
        native.da_col_sums(P(X), is_f32(X), X.shape[0], X.stride(0), X.shape[1], P(init), P(out), stream())
        return out

    def cov_chains(self, X, mean, starts, init):
        D = X.shape[1]
        nseg = len(starts) - 1
        out = torch.empty((nseg, D, D), dtype=F64, device=X.device)
        for s0 in range(0, nseg, 65535):
            s1 = min(nseg, s0 + 65535)
            arr = (ctypes.c_int64 * (s1 - s0 + 1))(*starts[s0:s1 + 1])
            native.da_cov_chains(P(X), is_f32(X), X.shape[0], X.stride(0), D, P(mean), ctypes.cast(arr, ctypes.c_void_p),
                                 s1 - s0, P(init) if s0 == 0 else None, P(out[s0]), stream())
        return out

    def fold(self, total, parts):
        out = total if total is not None else torch.empty_like(parts[0])
        native.da_fold(P(parts), parts.shape[0], parts[0].numel(), 0 if total is None else 1, P(out), stream())
        return out


def pca(X: torch.Tensor, comm=None):
    """Returns (R dev f64 (D,D), mean dev f64 (D,), variances np, R host).

    Mean and covariance are reduced on the device; across shards they run the
    rank-ordered ring of distributed.exact_pca_moments (bit-identical);
    the D x D eigendecomposition runs in LAPACK on the host, like the reference.
    """
    n_local, D = X.shape
    if comm is not None and comm.world == 1:
        comm = None  # one shard: the allreduces are identities, keep the one-GPU rounding
    n = comm.total(n_local) if comm is not None else n_local
    if n < 2:
        raise ValueError(f"PCA needs at least 2 vectors, got {n}")
    if comm is None:
        mean = torch.empty(D, dtype=F64, device=X.device)
        native.da_col_mean(P(X), is_f32(X), n_local, X.stride(0), D, P(mean), stream())
        if n > D:
            cov = torch.empty((D, D), dtype=F64, device=X.device)
            native.da_pca_cov(P(X), is_f32(X), n_local, X.stride(0), D, P(mean), P(cov), 1, stream())
    else:
        if n <= D:
            raise ValueError("the Gram-matrix PCA route (n <= d) is not sharded")
        from .distributed import exact_pca_moments

        # rank-ordered ring: the same chains as one GPU, cut at the shard boundaries
        mean, cov = exact_pca_moments(X, comm, _DevicePcaOps(X.device))
    if n > D:
        cov_h = cov.cpu().numpy()
        w, V = np.linalg.eigh(cov_h)
        order = np.argsort(w, kind="stable")[::-1]
        R_h = np.ascontiguousarray(V[:, order].T)
        variances = np.maximum(w[order], 0.0)
    else:
        # Gram route (clustering.py:101-112): n <= d, so these products are tiny
        Xc = torch.empty((n, D), dtype=F64, device=X.device)
        ident = torch.eye(D, dtype=F64, device=X.device)
        native.da_rotate(P(X), is_f32(X), n, X.stride(0), D, P(ident), P(mean), P(Xc), 0, stream())
        gram = torch.empty((n, n), dtype=F64, device=X.device)
        native.da_gemm_strided(P(Xc), 0, D, 1, P(Xc), 0, 1, D, P(gram), n, 1, n, n, D, stream())
        w, U = np.linalg.eigh(gram.cpu().numpy())
        order = np.argsort(w, kind="stable")[::-1]
        w = np.maximum(w[order], 0.0)
        U = U[:, order]
        tol = max(w[0], 1.0) * 1e-10 if w.size else 0.0
        keep = w > tol
        Uk = to_dev(np.ascontiguousarray(U[:, keep]), F64)
        r = int(keep.sum())
        comps_d = torch.empty((D, max(r, 1)), dtype=F64, device=X.device)
        if r:
            native.da_gemm_strided(P(Xc), 0, 1, D, P(Uk), 0, r, 1, P(comps_d), r, 1, D, r, n, stream())
        comps = comps_d.cpu().numpy()[:, :r] / np.sqrt(w[keep])[None, :]
        R_h = np.ascontiguousarray(_complete_basis(comps.T, D))
        variances = np.zeros(D)
        variances[:r] = w[keep] / (n - 1)
    R = to_dev(R_h, F64)
    return R, mean, variances, R_h


def rotate(X: torch.Tensor, R: torch.Tensor, mean: torch.Tensor, inverse: bool = False) -> torch.Tensor:
    n, D = X.shape
    out = torch.empty((n, D), dtype=F64, device=X.device)
    native.da_rotate(P(X), is_f32(X), n, X.stride(0), D, P(R), P(mean), P(out), int(inverse), stream())
    return out


def improved_kmeans(X: torch.Tensor, C0: torch.Tensor, schedule, max_iters: int, comm=None, want_trace=True):
    """Staged k-means in PCA space.  Returns (points f64, labels int32, trace);
    the trace is the last stage's (empty when want_trace is False)."""
    D = X.shape[1]
    if schedule[-1] != D:
        raise ValueError(f"schedule must end at d={D}, got {schedule}")
    R, mean, _, _ = pca(X, comm)
    Xr = rotate(X, R, mean)
    Cr = rotate(C0, R, mean)
    trace = []
    for dims in schedule:
        Cr, _, trace = lloyd(Xr, Cr, dims, max_iters, comm, want_trace=want_trace and dims == schedule[-1])
    del Xr
    C = rotate(Cr, R, mean, inverse=True)
    final_labels, final_errs = assign(X, D, C)
    init_labels, init_errs = assign(X, D, C0)
    fm = np_mean(final_errs, comm)
    im = np_mean(init_errs, comm)
    both = torch.cat([fm, im]).cpu().numpy()
    if both[0] <= both[1]:
        return C, final_labels, trace
    return C0.clone(), init_labels, [float(both[1])]


def check_k(n: int, K: int):
    if K > n:
        raise ValueError(f"k={K} exceeds the number of points n={n}")


# ---------------------------------------------------------------------------
# codebook-side kernels


def einsum_sq(cw: torch.Tensor) -> torch.Tensor:
    M, K, D = cw.shape
    out = torch.empty((M, K), dtype=F64, device=cw.device)
    native.da_einsum_sq(P(cw), M * K, D, P(out), stream())
    return out


def cross_full(cw: torch.Tensor):
    M, K, D = cw.shape
    Pt = torch.empty((M, M, K, K), dtype=F64, device=cw.device)
    sq = torch.empty((M, K), dtype=F64, device=cw.device)
    native.da_cross_products(P(cw), M, K, D, -1, P(Pt), P(sq), stream())
    return Pt, sq


def cross_refresh(cw: torch.Tensor, m: int, Pt: torch.Tensor, sq: torch.Tensor):
    """In-place refresh of the rows/cols of dictionary m."""
    M, K, D = cw.shape
    native.da_cross_products(P(cw), M, K, D, m, P(Pt), P(sq), stream())


def heat_up(X: torch.Tensor, codes: torch.Tensor, cw: torch.Tensor, m: int) -> torch.Tensor:
    n, D = X.shape
    M, K, _ = cw.shape
    out = torch.empty((n, D), dtype=F32, device=X.device)
    native.da_heat_up(P(X), n, D, P(codes), P(cw), M, K, m, P(out), stream())
    return out


def vec_err(X: torch.Tensor, codes: torch.Tensor, cw: torch.Tensor) -> torch.Tensor:
    n, D = X.shape
    M, K, _ = cw.shape
    err = torch.empty(n, dtype=F64, device=X.device)
    native.da_vec_err(P(X), is_f32(X), n, X.stride(0), D, P(codes), code_bytes(codes), codes.stride(0), P(cw),
                      M, K, P(err), stream())
    return err


def reconstruct(codes: torch.Tensor, cw: torch.Tensor) -> torch.Tensor:
    n = codes.shape[0]
    M, K, D = cw.shape
    out = torch.empty((n, D), dtype=F64, device=cw.device)
    native.da_reconstruct(P(codes), code_bytes(codes), n, codes.stride(0), P(cw), M, K, D, P(out), stream())
    return out


def encode(X: torch.Tensor, cw: torch.Tensor, sq: torch.Tensor, Pt: torch.Tensor, L: int,
           out_dtype=I32, with_err: bool = True):
    """Beam encode (codebook.py:264-300).  Returns (codes (n,M), err f64 | None)."""
    n, D = X.shape
    M, K, _ = cw.shape
    codes = torch.empty((n, M), dtype=out_dtype, device=X.device)
    err = torch.empty(n, dtype=F64, device=X.device) if with_err else None
    native.da_encode(P(X), is_f32(X), n, X.stride(0), D, P(cw), M, K, int(L), P(sq), P(Pt), P(codes),
                     code_bytes(codes), codes.stride(0), P(err), stream())
    return codes, err


_PINNED: list = []


def _pinned_slots(nslot: int, nbytes: int) -> list:
    """Reusable page-locked byte staging buffers (allocation is slow; keep them)."""
    global _PINNED
    if len(_PINNED) < nslot or _PINNED[0].numel() < nbytes:
        size = max(nbytes, _PINNED[0].numel() if _PINNED else 0)
        _PINNED = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(nslot)]
    return _PINNED[:nslot]


def _encode_stream(n: int, D: int, row_bytes: int, fill, to_rows, cw: torch.Tensor, sq: torch.Tensor,
                   Pt: torch.Tensor, L: int, out_dtype, chunk: int) -> torch.Tensor:
    """Streamed beam encode of n host rows.  A worker thread runs fill(slot, r0, rows)
    to copy the raw bytes of rows [r0, r0+rows) into a pinned byte slot; the copy
    stream uploads a slot while the compute stream turns the previous upload into
    float32 rows (to_rows(raw_dev, rows, out_f32)) and encodes them.  Three pinned
    slots, two device buffers.  Returns the device codes (n, M)."""
    import threading

    M = cw.shape[0]
    dev = device()
    codes = torch.empty((n, M), dtype=out_dtype, device=dev)
    if n == 0:
        return codes
    chunk = max(1, min(chunk, n))
    nslot = 3
    pinned = [p_[: chunk * row_bytes] for p_ in _pinned_slots(nslot, chunk * row_bytes)]
    draw = [torch.empty(chunk * row_bytes, dtype=torch.uint8, device=dev) for _ in range(2)]
    drows = [torch.empty((chunk, D), dtype=torch.float32, device=dev) for _ in range(2)]
    # ramped chunk sizes: the device starts after a small first copy instead of a
    # full chunk's (host copy + upload of 64 MB is ~3 ms before any encode)
    starts, sizes, r0, size = [], [], 0, min(chunk, 16384)
    while r0 < n:
        starts.append(r0)
        sizes.append(min(size, n - r0))
        r0 += size
        size = min(chunk, 2 * size)
    filled = [threading.Semaphore(0) for _ in range(nslot)]
    free = [threading.Semaphore(1) for _ in range(nslot)]
    errors = []
    stop = threading.Event()

    def producer():
        try:
            for i, r0 in enumerate(starts):
                s = i % nslot
                free[s].acquire()
                if stop.is_set():                    # the consumer failed: stop filling
                    return
                fill(pinned[s], r0, sizes[i])
                filled[s].release()
        except BaseException as e:  # surfaced on the caller's thread
            errors.append(e)
            for f in filled:
                f.release()

    th = threading.Thread(target=producer, daemon=True)
    th.start()
    comp = torch.cuda.current_stream()
    cstream = torch.cuda.Stream()
    comp_done = [None, None]
    try:
        for i, r0 in enumerate(starts):
            s, b = i % nslot, i % 2
            rows = sizes[i]
            filled[s].acquire()
            if errors:
                raise errors[0]
            with torch.cuda.stream(cstream):
                if comp_done[b] is not None:
                    cstream.wait_event(comp_done[b])        # device buffers b are free again
                draw[b][: rows * row_bytes].copy_(pinned[s][: rows * row_bytes], non_blocking=True)
                up = torch.cuda.Event()
                up.record(cstream)
            comp.wait_event(up)
            x = to_rows(draw[b][: rows * row_bytes], rows, drows[b])
            native.da_encode(P(x), 1, rows, x.stride(0), D, P(cw), M, cw.shape[1], int(L), P(sq), P(Pt),
                             P(codes[r0:]), code_bytes(codes), codes.stride(0), None, stream())
            ev = torch.cuda.Event()
            ev.record(comp)
            comp_done[b] = ev
            up.synchronize()                                 # pinned slot s has been read
            free[s].release()
    except BaseException:
        # wake the producer wherever it waits so the join below cannot hang
        stop.set()
        for f in free:
            f.release()
        raise
    finally:
        th.join()
    if errors:
        raise errors[0]
    return codes


_COPY_POOL = None


def _parallel_copy(dst: np.ndarray, src: np.ndarray, parts: int = 4) -> None:
    """Row-split host copy on a small thread pool (numpy releases the GIL): one
    thread's memcpy into pinned memory is slower than the device encodes."""
    global _COPY_POOL
    rows = src.shape[0]
    if rows < 4096 or parts <= 1:
        np.copyto(dst, src)
        return
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _COPY_POOL = ThreadPoolExecutor(max_workers=parts, thread_name_prefix="da-copy")
    step = (rows + parts - 1) // parts
    futs = [_COPY_POOL.submit(np.copyto, dst[i:i + step], src[i:i + step]) for i in range(0, rows, step)]
    for f in futs:
        f.result()


def encode_host(X_np: np.ndarray, cw: torch.Tensor, sq: torch.Tensor, Pt: torch.Tensor, L: int,
                out_dtype=I32, chunk: int = 131072, name: str = "data") -> torch.Tensor:
    """Beam-encode a host float32 array through _encode_stream.  Non-finite input
    raises ValueError (checked on the device).  Returns the device codes (n, M)."""
    n, D = X_np.shape
    ok = torch.ones((), dtype=torch.bool, device=device())

    def fill(slot, r0, rows):
        dst = slot[: rows * D * 4].view(torch.float32).numpy().reshape(rows, D)
        _parallel_copy(dst, X_np[r0:r0 + rows])

    def to_rows(raw, rows, buf):
        x = raw.view(torch.float32).view(rows, D)
        ok.logical_and_(torch.isfinite(x).all())
        return x

    codes = _encode_stream(n, D, 4 * D, fill, to_rows, cw, sq, Pt, L, out_dtype, chunk)
    if n and not bool(ok.item()):
        raise ValueError(f"{name} contains non-finite values")
    return codes


def encode_records(fill, n: int, D: int, kind: int, cw: torch.Tensor, sq: torch.Tensor, Pt: torch.Tensor,
                   L: int, out_dtype=I32, chunk: int = 1 << 18) -> tuple[torch.Tensor, int]:
    """Beam-encode n texmex records (kind 0 = fvecs, 1 = bvecs) streamed as raw
    file bytes: fill(slot, r0, rows) copies the records; the device unpacks them
    (da_unpack_vecs).  Returns (device codes, count of non-finite payload values)."""
    rec = 4 + D * (1 if kind else 4)
    bad = torch.zeros(1, dtype=torch.int64, device=device())

    def to_rows(raw, rows, buf):
        x = buf[:rows]
        native.da_unpack_vecs(P(raw), rows, D, kind, P(x), x.stride(0), P(bad), stream())
        return x

    codes = _encode_stream(n, D, rec, fill, to_rows, cw, sq, Pt, L, out_dtype, chunk)
    return codes, int(bad.item())


def assign_config(mode: int, counter: torch.Tensor | None = None) -> None:
    """0 = tcgen05 3xTF32 filter with exact float64 recheck (default, K <= 256),
    1 = plain float64 kernel.  `counter` accumulates rechecked (row, codeword) pairs."""
    native.da_assign_config(int(mode), P(counter))


def encode_config(mode: int, counter: torch.Tensor | None = None) -> None:
    """0 = default (currently 2), 1 = plain float64 tables, 2 = fp32 score-table +
    cross-gather filter, 3 = tcgen05 residual-GEMM filter; every mode returns the
    same codes and errors.  `counter` accumulates exact rechecks."""
    native.da_encode_config(int(mode), P(counter))


def pair_sums(codes: torch.Tensor, Pt: torch.Tensor) -> torch.Tensor:
    n, M = codes.shape
    K = Pt.shape[2]
    out = torch.empty(n, dtype=F64, device=codes.device)
    native.da_pair_sums(P(codes), code_bytes(codes), n, codes.stride(0), P(Pt), M, K, P(out), stream())
    return out


def adc_lut(Q: torch.Tensor, cw: torch.Tensor, sq: torch.Tensor):
    nq, D = Q.shape
    M, K, _ = cw.shape
    lut = torch.empty((nq, M, K), dtype=F64, device=Q.device)
    qsq = torch.empty(nq, dtype=F64, device=Q.device)
    native.da_adc_lut(P(Q), nq, D, P(cw), M, K, P(sq), P(lut), P(qsq), stream())
    return lut, qsq


def adc_scan(codes: torch.Tensor, pair: torch.Tensor, lut: torch.Tensor, qsq: torch.Tensor, r: int,
             cand: torch.Tensor | None = None):
    nq, M, K = lut.shape
    ncand = cand.shape[1] if cand is not None else codes.shape[0]
    ids = torch.empty((nq, r), dtype=I64, device=lut.device)
    dists = torch.empty((nq, r), dtype=F64, device=lut.device)
    native.da_adc_scan(P(codes), code_bytes(codes), codes.stride(0), P(pair), P(cand), ncand, nq, P(lut),
                       P(qsq), M, K, int(r), P(ids), P(dists), stream())
    return ids, dists


def adc_pack(codes: torch.Tensor, pair: torch.Tensor) -> torch.Tensor | None:
    """(n, 16) uint8 packed records (codes + pair sum), or None when the codes do not
    fit (more than 8 dictionaries or codes wider than one byte)."""
    n, M = codes.shape
    if codes.dtype != torch.uint8 or M > 8:
        return None
    rec = torch.empty((n, 16), dtype=torch.uint8, device=codes.device)
    native.da_adc_pack(P(codes), 1, n, codes.stride(0), P(pair), M, P(rec), stream())
    return rec


def adc_scan_packed(rec: torch.Tensor, lut: torch.Tensor, qsq: torch.Tensor, r: int,
                    cand: torch.Tensor | None = None):
    nq, M, K = lut.shape
    ncand = cand.shape[1] if cand is not None else rec.shape[0]
    ids = torch.empty((nq, r), dtype=I64, device=lut.device)
    dists = torch.empty((nq, r), dtype=F64, device=lut.device)
    native.da_adc_scan_packed(P(rec), P(cand), ncand, nq, P(lut), P(qsq), M, K, int(r), P(ids), P(dists), stream())
    return ids, dists


# ---------------------------------------------------------------------------
# DA training on device (annq/annealing.py:115-262)


def dimension_schedule(d: int, i_count: int = 10) -> list[int]:
    """annq/clustering.py:116-131 (pure integer bookkeeping)."""
    import math

    if d < 1 or i_count < 1:
        raise ValueError("d and i_count must be >= 1")
    dims: list[int] = []
    for i in range(1, i_count + 1):
        v = min(d, math.ceil(d ** (i / i_count)))
        if not dims or v > dims[-1]:
            dims.append(v)
    if dims[-1] != d:
        dims.append(d)
    return dims


def cool_down(inter: torch.Tensor, C0_f32: torch.Tensor, config, comm=None):
    """annealing.py:115-126: (new dictionary f32 (K,D), assignment int32)."""
    D = inter.shape[1]
    schedule = dimension_schedule(D, config.schedule_stages)
    n_total = comm.total(inter.shape[0]) if comm is not None else inter.shape[0]
    check_k(n_total, C0_f32.shape[0])
    pts, labels, _ = improved_kmeans(inter, C0_f32.to(F64), schedule, config.kmeans_iters, comm, want_trace=False)
    return pts.to(F32), labels


class StepTimer:
    def __init__(self):
        import time

        self._t = time.perf_counter
        self.t0 = self._t()

    def seconds(self):
        return self._t() - self.t0


def dict_step(X, cw, codes, Pt, sq, m, config, comm=None):
    """One heat-up / cool-down / re-encode step of da_sweep (annealing.py:162-178).

    Updates cw, codes and the cross table (Pt, sq = its sq_norms) in place;
    returns the step distortion (float).
    """
    inter = heat_up(X, codes, cw, m)
    new_dict, assign_m = cool_down(inter, cw[m], config, comm)
    del inter
    cw[m] = new_dict
    cross_refresh(cw, m, Pt, sq)
    incumbent = codes.clone()
    native.da_set_column(P(incumbent), incumbent.shape[0], incumbent.shape[1], m, P(assign_m), stream())
    # beam tables use einsum norms of the current codebook (codebook.py:260)
    beam_codes, beam_err = encode(X, cw, einsum_sq(cw), Pt, config.beam_width)
    inc_err = vec_err(X, incumbent, cw)
    native.da_select_better(X.shape[0], codes.shape[1], P(beam_codes), P(beam_err), P(incumbent), P(inc_err),
                            stream())
    codes.copy_(incumbent)
    return float(np_mean(inc_err, comm).item())


def growth_pass(X, config, report=None, comm=None):
    """annealing.py:184-205 (all-zero start, greedy residual cool-downs)."""
    n, D = X.shape
    M, K = config.m_count, config.k_count
    cw = torch.zeros((M, K, D), dtype=F32, device=X.device)
    codes = torch.zeros((n, M), dtype=I32, device=X.device)
    for m in range(M):
        t = StepTimer()
        inter = heat_up(X, codes, cw, m)
        new_dict, assign_m = cool_down(inter, cw[m], config, comm)
        del inter
        cw[m] = new_dict
        native.da_set_column(P(codes), n, M, m, P(assign_m), stream())
        if report is not None:
            dist = float(np_mean(vec_err(X, codes, cw), comm).item())
            report.record(0, m, dist, t.seconds())
    return cw, codes


def da_sweep(X, cw, codes, Pt, sq, config, sweep_index=1, report=None, comm=None):
    """annealing.py:140-181 on device state (mutated in place)."""
    for m in range(cw.shape[0]):
        t = StepTimer()
        dist = dict_step(X, cw, codes, Pt, sq, m, config, comm)
        if report is not None:
            report.record(sweep_index, m, dist, t.seconds())


def sweep_until_converged(X, cw, codes, config, report, comm=None):
    """annealing.py:208-222."""
    Pt, sq = cross_full(cw)
    prev = float(np_mean(vec_err(X, codes, cw), comm).item())
    for s in range(1, config.sweeps + 1):
        da_sweep(X, cw, codes, Pt, sq, config, sweep_index=s, report=report, comm=comm)
        cur = report.steps[-1].distortion if report is not None and report.steps else prev
        if prev > 0 and (prev - cur) / prev < config.rel_tol:
            break
        prev = cur
    return Pt, sq
