"""Row-sharded pass on a real GPU: two processes share cuda:0 and exchange the stage buffers of
include/avd.h with torch.distributed (gloo, which all-reduces CUDA tensors through the host).
This runs the library's real stage kernels on each shard — the row sample, the fused pass with
the exchanged quantiser, the integer Gram partials, the replicated eigensolver, the radix
selection with a tie block straddling the rank boundary — and the concatenated per-rank outputs
must match the single-process fp64 oracle at the north-star tolerances.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth.gen import SynthSpec, generate

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec, col_fix, out, flags=0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2603_10444_b200.distributed import ShardedDecomposer, shard_rows
    r0, lr = shard_rows(spec.l, world, rank)
    X = generate(spec, r0, lr, device="cuda")
    if col_fix is not None:
        X[:, col_fix[0]] = col_fix[1]
    sd = ShardedDecomposer(spec.l, spec.m, flags=flags)
    r = sd(X)
    torch.cuda.synchronize()
    out[rank] = dict(mu=r.mu.cpu().numpy(), sigma=r.sigma.cpu().numpy(), top=r.top_idx.cpu().numpy(),
                     rho=r.rho.cpu().numpy(), offset=int(r.top_offset), n_top=int(r.n_top_global),
                     energy_cf=list(r.energy_cf), energy_el=list(r.energy_el), digits=int(r.digits_used))
    sd.close()
    dist.barrier()
    dist.destroy_process_group()


def _run(spec, col_fix=None, world=2, flags=0):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), spec, col_fix, out, flags), nprocs=world, join=True)
    return [out[r] for r in range(world)]


@pytest.mark.parametrize("l,m,col_fix,flags", [(4096, 256, (5, 40.0), 0), (65536, 128, None, 0),
                                               (4096, 256, None, 4)])
def test_two_ranks_match_oracle(cuda_device, l, m, col_fix, flags):
    """flags = 4 (AVD_FLAG_FORCE_ESCALATE): the AVD_EREPEAT re-Gram with its GRAM/QSUM/QERR
    re-exchange on both ranks."""
    from oracle import oracle as O
    spec = SynthSpec(l, m, seed=17, f_mean=0.8)
    res = _run(spec, col_fix, flags=flags)
    if flags:
        assert all(r["digits"] == 3 for r in res)
    X = generate(spec)
    if col_fix is not None:
        X[:, col_fix[0]] = col_fix[1]  # l tied maxima: the tie block straddles the rank boundary
    o = O.decompose(X.numpy())
    for r in res:
        assert np.max(np.abs(r["mu"] - o["mu"])) <= 1e-6 * np.max(np.abs(o["mu"]))
        np.testing.assert_allclose(r["sigma"], o["sigma"], rtol=1e-4)
        assert r["n_top"] == o["n_top"]
        s_g = np.array(r["energy_cf"][1:]) / r["energy_cf"][0]
        s_o = np.array(o["energy_cf"][1:]) / o["energy_cf"][0]
        assert np.all(np.abs(s_g - s_o) <= 1e-5 * s_o + 1e-12)
    assert res[0]["offset"] == 0 and res[1]["offset"] == len(res[0]["top"])
    np.testing.assert_array_equal(np.concatenate([r["top"] for r in res]), o["top_idx"])
    rho = np.concatenate([r["rho"] for r in res])
    assert np.max(np.abs(rho - o["rho"])) <= 1e-3
    # the replicated eigensolver sees the same exchanged Gram on both ranks
    np.testing.assert_array_equal(res[0]["sigma"], res[1]["sigma"])


def _c_worker(rank, world, port, spec, out):
    """avd_decompose_sharded: the C library drives every stage and exchange itself, calling back
    into a Python avd_exchange_fn that all-reduces the named workspace buffer (gloo)."""
    import ctypes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2603_10444_b200 import _lib as L
    from paper_2603_10444_b200.api import Decomposer
    from paper_2603_10444_b200.distributed import shard_rows
    r0, lr = shard_rows(spec.l, world, rank)
    X = generate(spec, r0, lr, device="cuda")
    dec = Decomposer(spec.l, spec.m, world=world, l_local=lr, row_offset=r0)
    dtypes = {L.AVD_DT_F64: torch.float64, L.AVD_DT_F32: torch.float32, L.AVD_DT_I64: torch.int64}
    ops = {L.AVD_OP_SUM: dist.ReduceOp.SUM, L.AVD_OP_MAX: dist.ReduceOp.MAX, L.AVD_OP_MIN: dist.ReduceOp.MIN}
    calls = []

    def cb(which, ptr, dtype, op, count, user):
        t = dec.buffer(L.BUF_NAME[which], dtypes[dtype])
        assert t.data_ptr() == ptr and t.numel() == count
        dist.all_reduce(t, op=ops[op])
        calls.append(L.BUF_NAME[which])
        return 0
    fn = L.EXCHANGE_FN(cb)
    o = dec._outputs()
    L.avd_decompose_sharded(dec.h, X.data_ptr(), rank, o, fn, None)
    torch.cuda.synchronize()
    r = dec._result(o, 0)
    out[rank] = dict(mu=r.mu.cpu().numpy(), sigma=r.sigma.cpu().numpy(), top=r.top_idx.cpu().numpy(),
                     rho=r.rho.cpu().numpy(), offset=int(r.top_offset), calls=list(calls))
    dec.close()
    dist.barrier()
    dist.destroy_process_group()


def test_c_driven_sharded_pass(cuda_device):
    """include/avd.h avd_decompose_sharded over two ranks on one GPU: the library's own exchange
    schedule (packed Gram, distributed eigensolve) matches the oracle."""
    from oracle import oracle as O
    spec = SynthSpec(4096, 256, seed=21, f_mean=0.8)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_c_worker, args=(2, _free_port(), spec, out), nprocs=2, join=True)
    res = [out[0], out[1]]
    o = O.decompose(generate(spec).numpy())
    for r in res:
        assert np.max(np.abs(r["mu"] - o["mu"])) <= 1e-6 * np.max(np.abs(o["mu"]))
        np.testing.assert_allclose(r["sigma"], o["sigma"], rtol=1e-4)
        assert "GRAMP" in r["calls"] and "EIGY" in r["calls"] and "EIGZ" in r["calls"]
    np.testing.assert_array_equal(np.concatenate([r["top"] for r in res]), o["top_idx"])
    assert np.max(np.abs(np.concatenate([r["rho"] for r in res]) - o["rho"])) <= 1e-3
    np.testing.assert_array_equal(res[0]["sigma"], res[1]["sigma"])
