"""World-size-2 test of the row-sharded orchestration on CPU (gloo).

`paper_2603_10444_b200.distributed.run_stages` drives the SAME exchange schedule it uses with the
CUDA library over NCCL, here with a numpy model of each stage's contract (tests-only: it mirrors
what the header says each stage computes into each exchange buffer) and the library's REAL
host-side tie-quota logic (`avd_tie_quota`).  The concatenated per-rank outputs must equal the
single-process fp64 oracle: mu, sigma_k, E_top (exact, including a tie block that straddles the
rank boundary) and rho.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth.gen import SynthSpec, generate


def _keys(X):
    return (X.view(np.uint32) & np.uint32(0x7FFFFFFF)).astype(np.int64)


class ModelBackend:
    """Numpy model of the stage contract of include/avd.h (test infrastructure only)."""

    def __init__(self, l, m, k, n_top, row0, world, rank):
        self.l, self.m, self.k, self.n_top, self.row0 = l, m, k, n_top, row0
        self.world, self.rank = world, rank
        self.buf = {}

    def exchange_buffer(self, name, dtype):
        return self.buf[name]

    def _sample_step(self):
        want = max(1, min(16, self.l // 4096))
        s = 1
        while s * 2 <= want:
            s *= 2
        return s

    def stage_stats(self, X):
        s = self._sample_step()
        rows = np.arange(X.shape[0]) + self.row0
        Xs = X[rows % s == 0]
        key = _keys(X[rows % (4 * s) == 0])
        self.buf["SAMPLE"] = torch.tensor(np.concatenate([Xs.astype(np.float64).sum(0), [len(Xs)]]))
        self.buf["SMAX"] = torch.tensor(Xs.max(0) if len(Xs) else np.full(self.m, -np.inf, np.float32))
        self.buf["SMIN"] = torch.tensor(Xs.min(0) if len(Xs) else np.full(self.m, np.inf, np.float32))
        h = np.bincount((key[key != 0] >> 19).ravel(), minlength=4096)
        self.buf["HIST1"] = torch.tensor(h.astype(np.int64))

    def stage_split(self, X):
        Xd = X.astype(np.float64)
        key = _keys(X)
        self.buf["STATS"] = torch.tensor(np.concatenate([Xd.sum(0), [np.sum(Xd * Xd), 0.0, np.count_nonzero(key), 0.0]]))
        self.buf["COLMAX"] = torch.tensor(np.abs(X).max(0))
        smp = self.buf["SAMPLE"].numpy()
        mu0 = (smp[: self.m] / max(smp[self.m], 1.0)).astype(np.float32).astype(np.float64)
        self.buf["DIAG"] = torch.tensor(((X.astype(np.float64) - mu0) ** 2).sum(0))  # exact diag of G
        s = self._sample_step()
        h = self.buf["HIST1"].numpy()
        cum, b0 = 0, 0
        for b in range(4095, -1, -1):
            cum += h[b] * s * 4
            if cum >= 2 * self.n_top + 256 * s * 4:
                b0 = b
                break
        li = np.arange(X.size).reshape(X.shape) + self.row0 * self.m
        sel = (key != 0) & ((key >> 19) >= b0)
        self.ckey, self.cidx = key[sel], li[sel]
        self.buf["CAND"] = torch.tensor([len(self.ckey), 0], dtype=torch.int64)
        self.X = X

    def stage_gram(self, X):
        st = self.buf["STATS"].numpy()
        self.mu = st[: self.m] / self.l
        self.n_eff = int(min(self.n_top, st[self.m + 2]))
        self.Xc = self.X.astype(np.float64) - self.mu
        self.buf["GRAMP"] = torch.tensor(self.Xc.T @ self.Xc)  # (the model keeps it unpacked)
        self.buf["QSUM"] = torch.zeros(2 * self.m, dtype=torch.int64)
        self.buf["QERR"] = torch.zeros(self.m, dtype=torch.float64)

    def stage_eig_dist(self, rank, exchange):
        """Model of avd_stage_eig_dist: block power iterations whose G Q products are split by
        row blocks over the ranks, each rank's rows written into a zero-padded m x p block that
        `exchange` all-reduces (EIGZ, EIGY in fp64, like the library), then Rayleigh-Ritz
        on the replicated orthonormal basis."""
        G = self.buf["GRAMP"].numpy()
        m, p = self.m, self.k + 6
        r0, r1 = m * rank // self.world, m * (rank + 1) // self.world
        Q = np.linalg.qr(np.random.default_rng(7).standard_normal((m, p)))[0]
        for _ in range(60):
            Z = np.zeros((m, p))
            Z[r0:r1] = G[r0:r1] @ Q
            self.buf["EIGZ"] = torch.tensor(Z)
            exchange("EIGZ")
            Z = self.buf["EIGZ"].numpy()
            Y = np.zeros((m, p))
            Y[r0:r1] = G[r0:r1] @ Z
            self.buf["EIGY"] = torch.tensor(Y)
            exchange("EIGY")
            Q = np.linalg.qr(self.buf["EIGY"].numpy())[0]
        Y = np.zeros((m, p))
        Y[r0:r1] = G[r0:r1] @ Q
        self.buf["EIGY"] = torch.tensor(Y)
        exchange("EIGY")
        H = Q.T @ self.buf["EIGY"].numpy()
        th, W = np.linalg.eigh(0.5 * (H + H.T))
        U = Q @ W[:, ::-1][:, : self.k]
        for r in range(self.k):
            j = np.argmax(np.abs(U[:, r]))
            if U[j, r] < 0:
                U[:, r] *= -1
        self.V, self.sigma = U, np.sqrt(np.maximum(th[::-1][: self.k], 0))
        return 0

    def stage_eig(self):
        lam, W = np.linalg.eigh(self.buf["GRAMP"].numpy())  # the exchanged (global) Gram
        lam, W = lam[::-1][: self.k], W[:, ::-1][:, : self.k]
        for r in range(self.k):
            j = np.argmax(np.abs(W[:, r]))
            if W[j, r] < 0:
                W[:, r] *= -1
        self.V, self.sigma = W, np.sqrt(np.maximum(lam, 0))

    def stage_project(self, X):
        self.P = self.Xc @ self.V
        S = self.P @ self.V.T
        T = self.Xc - S
        self.buf["ENERGY"] = torch.tensor(np.concatenate([[np.sum(S * S), np.sum(T * T), np.sum(S * T),
                                                           np.sum(self.Xc ** 2)], self.P.sum(0)]))

    def stage_select(self, X, level, rank):
        key, idx = self.ckey, self.cidx
        if level == 0:
            self.from_x = int(self.buf["CAND"][0]) < self.n_eff
            if self.from_x:
                k2 = _keys(X)
                self.ckey = key = k2[k2 != 0]
                self.cidx = idx = (np.arange(X.size).reshape(X.shape) + self.row0 * self.m)[k2 != 0]
            self.buf["HIST0"] = torch.tensor(np.bincount(key >> 19, minlength=4096).astype(np.int64))
        elif level == 1:
            self.b1, self.cnt = self._find(self.buf["HIST0"].numpy(), self.n_eff)
            sel = (key >> 19) == self.b1
            self.buf["HIST2"] = torch.tensor(np.bincount((key[sel] >> 7) & 0xFFF, minlength=4096).astype(np.int64))
        elif level == 2:
            self.b2, c = self._find(self.buf["HIST2"].numpy(), self.n_eff - self.cnt)
            self.cnt += c
            sel = (key >> 7) == ((self.b1 << 12) | self.b2)
            self.buf["HIST3"] = torch.tensor(np.bincount(key[sel] & 0x7F, minlength=128).astype(np.int64))
        else:
            b3, c = self._find(self.buf["HIST3"].numpy(), self.n_eff - self.cnt)
            self.T = (self.b1 << 19) | (self.b2 << 7) | b3
            self.q = self.n_eff - (self.cnt + c)
            t = np.zeros(2 * self.world, np.int64)
            t[rank] = np.sum(key > self.T)
            t[self.world + rank] = np.sum(key == self.T)
            self.buf["TIES"] = torch.tensor(t)

    @staticmethod
    def _find(h, need):
        cum = 0
        for b in range(len(h) - 1, -1, -1):
            if cum + h[b] >= need:
                return b, cum
            cum += h[b]
        raise AssertionError("rank beyond histogram")

    def stage_gather(self, X, rank):
        from paper_2603_10444_b200._lib import avd_tie_quota
        t = self.buf["TIES"].numpy()
        quota, self.offset = avd_tie_quota(t[: self.world], t[self.world:], rank, self.q)
        gt = np.sort(self.cidx[self.ckey > self.T])
        ties = np.sort(self.cidx[self.ckey == self.T])[:quota]
        self.top = np.sort(np.concatenate([gt, ties]))
        i = self.top // self.m - self.row0
        j = self.top % self.m
        x = X[i, j].astype(np.float64)
        M = self.mu[j]
        S = np.sum(self.P[i] * self.V[j], axis=1)
        Tt = self.Xc[i, j] - S
        rho = np.stack([M * M, S * S, Tt * Tt], 1) / (x * x)[:, None]
        self.rho = np.concatenate([rho, 1 - rho.sum(1, keepdims=True)], 1)
        self.buf["AGG"] = torch.tensor(np.concatenate([self.rho.sum(0), [np.sum(M * M), np.sum(S * S),
                                                                        np.sum(Tt * Tt), np.sum(x * x)]]))

    def stage_report(self):
        return dict(mu=self.mu, sigma=self.sigma, top=self.top, rho=self.rho, offset=self.offset,
                    energy=self.buf["ENERGY"].numpy()[:4].copy(), agg=self.buf["AGG"].numpy().copy())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, X, k, n_top, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_10444_b200.distributed import TorchComm, run_stages, shard_rows
    r0, lr = shard_rows(X.shape[0], world, rank)
    be = ModelBackend(X.shape[0], X.shape[1], k, n_top, r0, world, rank)
    res = run_stages(be, TorchComm(), X[r0:r0 + lr])
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


def _run(X, k, n_top, world=2):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), X, k, n_top, out), nprocs=world, join=True)
    return [out[r] for r in range(world)]


@pytest.mark.parametrize("n_top", [32, 300, 700])
def test_two_rank_matches_oracle(n_top):
    from oracle import oracle as O
    X = generate(SynthSpec(512, 64, seed=3, k_s=2, f_mean=0.8)).numpy()
    X[:, 5] = 40.0  # 512 tied maxima: the tie block straddles the rank boundary (rows 256+)
    k = 2
    res = _run(X, k, n_top)
    o = O.decompose(X, k=k, n_top=n_top)
    for r in res:
        np.testing.assert_allclose(r["mu"], o["mu"], rtol=1e-14, atol=1e-14)
        np.testing.assert_allclose(r["sigma"], o["sigma"], rtol=1e-10)
    assert res[0]["offset"] == 0 and res[1]["offset"] == len(res[0]["top"])
    top = np.concatenate([r["top"] for r in res])
    np.testing.assert_array_equal(top, o["top_idx"])
    rho = np.concatenate([r["rho"] for r in res])
    np.testing.assert_allclose(rho, o["rho"], atol=1e-9)
    # exchanged energies / aggregates are global sums
    np.testing.assert_allclose(res[0]["energy"], res[1]["energy"])
    np.testing.assert_allclose(res[0]["energy"][0], o["energy_el"][2], rtol=1e-9)
    np.testing.assert_allclose(res[0]["agg"][:4] / n_top, o["rho_mean_aggr"], atol=1e-9)


def _gram_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(rank)
    part = torch.tensor(rng.integers(-2**40, 2**40, size=(64, 64)), dtype=torch.int64)
    total = part.clone()
    dist.all_reduce(total)
    out[rank] = (part.numpy(), total.numpy())
    dist.destroy_process_group()


def test_gram_allreduce_is_exact():
    """The int64 Gram exchange is an exact integer sum: identical on every rank and equal to
    the sum of the partials regardless of order."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gram_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    p0, t0 = out[0]
    p1, t1 = out[1]
    np.testing.assert_array_equal(t0, t1)
    np.testing.assert_array_equal(t0, p0 + p1)


class _FailingBackend(ModelBackend):
    def stage_split(self, X):
        if self.rank == 1:
            raise RuntimeError("injected failure on rank 1")
        return super().stage_split(X)


def _fail_worker(rank, world, port, X, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_10444_b200.distributed import TorchComm, run_stages, shard_rows
    r0, lr = shard_rows(X.shape[0], world, rank)
    be = _FailingBackend(X.shape[0], X.shape[1], 2, 32, r0, world, rank)
    try:
        run_stages(be, TorchComm(), X[r0:r0 + lr])
        out[rank] = "no error"
    except Exception as e:  # noqa: BLE001
        out[rank] = type(e).__name__ + ": " + str(e)
    dist.destroy_process_group()


def test_stage_failure_reaches_every_rank():
    """a stage failing on one rank makes every rank raise (status all-reduce after each
    stage) instead of leaving the others blocked in the next collective."""
    X = generate(SynthSpec(512, 64, seed=3, k_s=2, f_mean=0.8)).numpy()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_fail_worker, args=(2, _free_port(), X, out), nprocs=2, join=True)
    assert out[1].startswith("RuntimeError: injected failure")
    assert out[0].startswith("StageFailed")
