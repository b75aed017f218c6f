"""Row-sharded pass over P GPUs: one process per GPU, NCCL collectives via torch.distributed.

Rank r owns the contiguous rows [row_offset_r, row_offset_r + l_r) of the global matrix (rank
order == row order, which makes the tie quota of E_top a rank-ordered prefix).  Every numerical
step runs in libavd's kernels through the stage entry points of include/avd.h; between them this
module all-reduces exactly the exchange buffers the header lists:

  stats   : row-sample column sums + #rows (SUM f64), max (MAX), min (MIN), |x| histogram
            level 1 (SUM i64)  -> identical quantiser centre / scale and candidate bin everywhere
  split   : column sums + sum x^2 + counts (SUM f64), column range about the quantiser centre (MAX)
  gram    : the exact int64 Gram partials — their upper 128-tiles, packed (GRAMP) — and integer
            column sums of the quantised operand (SUM i64)  -> identical exactly-centred G on
            every rank
  eig     : distributed: every G Q product of the subspace iteration is split by
            row blocks over the ranks and all-gathered (EIGZ / EIGY f64, SUM of zero-padded
            blocks) through a callback the library calls; the p x p work is replicated (same G,
            same seed -> identical V_k, sigma_k on every rank); may ask for a 3-digit Gram
            (AVD_EREPEAT) -> gram again, exchange GRAMP, QSUM, QERR, eig again
  project : elementwise energy sums + column sums of P (SUM f64)
  gram    : + candidate count / overflow flag (SUM i64) -> same candidate-vs-stream decision
  select  : radix histograms of |x| bits (SUM i64), per-rank sel/tie counts (SUM = all-gather)
  gather  : rho aggregates (SUM f64)

The exchange logic is written against a tiny `Comm` interface so the CPU tests can drive the
same orchestration with the gloo backend (tests/test_distributed_gloo.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib as L
from .api import Decomposer, Result

# (stage, buffer name, dtype, reduce op) in call order
EXCHANGES = {
    "stats": [("SAMPLE", torch.float64, "sum"), ("SMAX", torch.float32, "max"),
              ("SMIN", torch.float32, "min"), ("HIST1", torch.int64, "sum")],
    "split": [("STATS", torch.float64, "sum"), ("COLMAX", torch.float32, "max"), ("DIAG", torch.float64, "sum")],
    "gram": [("GRAMP", torch.int64, "sum"), ("CAND", torch.int64, "sum"), ("QSUM", torch.int64, "sum"),
             ("QERR", torch.float64, "sum")],
    "regram": [("GRAMP", torch.int64, "sum"), ("QSUM", torch.int64, "sum"), ("QERR", torch.float64, "sum")],
    # called back by the library from inside the distributed eigensolve
    "eig": [("EIGZ", torch.float64, "sum"), ("EIGY", torch.float64, "sum")],
    "project": [("ENERGY", torch.float64, "sum")],
    "select0": [("HIST0", torch.int64, "sum")],
    "select1": [("HIST2", torch.int64, "sum")],
    "select2": [("HIST3", torch.int64, "sum")],
    "select3": [("TIES", torch.int64, "sum")],
    "gather": [("AGG", torch.float64, "sum")],
}

_OPS = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}


def shard_rows(l_global: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous near-equal row shard of `rank`: (row_offset, l_local)."""
    r0 = l_global * rank // world
    r1 = l_global * (rank + 1) // world
    return r0, r1 - r0


class TorchComm:
    """all_reduce over a torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_reduce(self, t: torch.Tensor, op: str) -> None:
        dist.all_reduce(t, op=_OPS[op], group=self.group)


class StageFailed(RuntimeError):
    """A stage failed on some rank; every rank raises it (the first failing rank's message)."""


def run_stages(backend, comm, X) -> object:
    """The sharded pass: stage calls of `backend` interleaved with `comm` exchanges.  With
    world > 1 every stage is followed by a status all-reduce (MAX), so a stage that fails on one
    rank (a CUDA error, AVD_ESTATE, ...) makes every rank raise instead of leaving the others
    blocked in the next collective."""
    rank = comm.rank
    status = None
    if comm.world > 1:
        dev = X.device if torch.is_tensor(X) else torch.device("cpu")
        status = torch.zeros(1, dtype=torch.int64, device=dev)

    def guarded(fn, *a):
        if comm.world == 1:
            return fn(*a)
        err, res = None, None
        try:
            res = fn(*a)
        except Exception as e:  # noqa: BLE001 - re-raised below on every rank
            err = e
        status.fill_(0 if err is None else 1)
        comm.all_reduce(status, "max")
        if err is not None:
            raise err
        if int(status.item()) != 0:
            raise StageFailed(f"{getattr(fn, '__name__', 'stage')} failed on another rank")
        return res

    def exchange(stage):
        if comm.world == 1:
            return
        for name, dtype, op in EXCHANGES[stage]:
            comm.all_reduce(backend.exchange_buffer(name, dtype), op)

    guarded(backend.stage_stats, X)
    exchange("stats")
    guarded(backend.stage_split, X)
    exchange("split")
    guarded(backend.stage_gram, X)
    exchange("gram")

    def eig():
        if comm.world == 1:
            return backend.stage_eig()
        dtypes = {name: dt for name, dt, _ in EXCHANGES["eig"]}

        def eig_exchange(name):  # the library's all-gather of a row-split product
            comm.all_reduce(backend.exchange_buffer(name, dtypes[name]), "sum")
        return backend.stage_eig_dist(rank, eig_exchange)

    if guarded(eig) == L.AVD_EREPEAT:
        # automatic digits: the replicated precision bound raised the Gram operand to 3 digits
        # on every rank alike; redo the Gram (the candidate count is already global)
        guarded(backend.stage_gram, X)
        exchange("regram")
        guarded(eig)
    guarded(backend.stage_project, X)
    exchange("project")
    for lv in range(4):
        guarded(backend.stage_select, X, lv, rank)
        exchange(f"select{lv}")
    guarded(backend.stage_gather, X, rank)
    exchange("gather")
    return guarded(backend.stage_report)


class _LibBackend:
    """Stage calls into libavd (device pointers of torch tensors)."""

    def __init__(self, dec: Decomposer):
        self.dec = dec
        self.h = dec.h
        self.out = None
        self._views = {}

    def exchange_buffer(self, name, dtype):
        if name not in self._views:
            self._views[name] = self.dec.buffer(name, dtype)
        return self._views[name]

    def stage_stats(self, X):
        L.avd_stage_stats(self.h, X.data_ptr())

    def stage_split(self, X):
        L.avd_stage_split(self.h, X.data_ptr())

    def stage_gram(self, X):
        L.avd_stage_gram(self.h, X.data_ptr())

    def stage_eig(self):
        self.eig_status = L.avd_stage_eig(self.h)
        return self.eig_status

    def stage_eig_dist(self, rank, exchange):
        """exchange(name): all-reduce (SUM) the named exchange buffer over the ranks; the library
        calls it back (through an avd_exchange_fn) from inside the distributed eigensolve."""
        def cb(which, ptr, dtype, op, count, user):
            try:
                exchange(L.BUF_NAME[which])
                return 0
            except Exception:  # noqa: BLE001 - reported to the library as AVD_EEXCHANGE
                return 1
        fn = L.EXCHANGE_FN(cb)  # kept alive for the duration of the call
        self.eig_status = L.avd_stage_eig_dist(self.h, rank, fn, None)
        return self.eig_status

    def stage_project(self, X):
        L.avd_stage_project(self.h, X.data_ptr())

    def stage_select(self, X, level, rank):
        L.avd_stage_select(self.h, X.data_ptr(), level, rank)

    def stage_gather(self, X, rank):
        self.out = self.dec._outputs()
        L.avd_stage_gather(self.h, X.data_ptr(), rank, self.out)

    def stage_report(self) -> Result:
        L.avd_stage_report(self.h, self.out)
        return self.dec._result(self.out, self.eig_status)


class ShardedDecomposer:
    """Decomposer of a row-sharded matrix: call on this rank's [l_local, m] CUDA block."""

    def __init__(self, l_global: int, m: int, group=None, **kw):
        self.comm = TorchComm(group)
        self.row_offset, self.l_local = shard_rows(l_global, self.comm.world, self.comm.rank)
        self.dec = Decomposer(l_global, m, world=self.comm.world, l_local=self.l_local,
                              row_offset=self.row_offset, **kw)
        self.backend = _LibBackend(self.dec)

    def __call__(self, X_local: torch.Tensor) -> Result:
        self.dec._check_X(X_local)
        return run_stages(self.backend, self.comm, X_local)

    def launches(self) -> int:
        return self.dec.launches()

    def close(self):
        self.dec.close()
