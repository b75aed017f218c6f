"""Full-size parity at BASELINE.json's bench configurations in the launch configuration bench.py
times (one B200, default = automatic digits):

  * c4 (131072 x 4096, k = 40, |E_top| = 536870) against the fp64 ORACLE's own outputs at that
    size, cached by `python tools/oracle_cache.py c4` (oracle/ only; tests/golden/oracle_c4.npz):
    mu (1e-6, R14), sigma_k (1e-4), the V_k subspace, sigma_{k+1}, the energy shares (1e-5,
    R15), E_top exactly (SHA-256 of the ascending int64 index list), rho at 4096 seeded entries
    of E_top (1e-3), the rho aggregates, the cross terms and column means of spike / tail;
  * c4 properties that hold at any size, recomputed in fp64 numpy on the host (mu, ||X||^2,
    E_top by a host composite-key selection, sigma_r = ||Xc v_r||, rho at sampled entries);
  * c4 on the PLANTED EXACT generator (sigma_t = 0, dyadic mu and c_r, Walsh-Hadamard factors):
    every output has a closed form at this size (SURVEY §8(c) "closed form at any size");
  * c5 (1048576 x 8192, k = 81, one B200 — the north star's target matrix) against the cached
    oracle (eig step by LAPACK, `tools/oracle_cache.py c5 --eig lapack`), when that cache exists.
"""
import hashlib
import math
import os

import numpy as np
import pytest
import torch

from synth.gen import SynthSpec, config_spec, generate, planted, walsh

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _run(spec, **kw):
    from paper_2603_10444_b200 import Decomposer
    Xd = generate(spec, device="cuda")
    dec = Decomposer(spec.l, spec.m, seed=0, **kw)
    r = dec(Xd)
    torch.cuda.synchronize()
    out = dict(res=r, mu=r.mu.cpu().numpy(), V=r.V.cpu().numpy(), sigma=r.sigma.cpu().numpy(),
               top=r.top_idx.cpu().numpy(), rho=r.rho.cpu().numpy(), n_top=dec.n_top)
    dec.close()
    return Xd, out


def _subspace_sin(A, B):
    s = np.linalg.svd(A.T @ B, compute_uv=False)
    return float(np.sqrt(max(0.0, 1.0 - float(s.min()) ** 2)))


def _against_cache(name, g):
    path = os.path.join(GOLD, f"oracle_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (python tools/oracle_cache.py {name})")
    o = np.load(path)
    r = g["res"]
    mu_o = o["mu"]
    assert np.max(np.abs(g["mu"] - mu_o)) <= 1e-6 * np.max(np.abs(mu_o))
    np.testing.assert_allclose(g["sigma"], o["sigma"], rtol=1e-4)
    assert _subspace_sin(g["V"], o["V"].astype(np.float64)) <= 1e-3
    so = float(o["sigma_next"])  # Ritz lower bound of sigma_{k+1} (include/avd.h)
    assert 0.9 * so <= r.sigma_next <= so * (1 + 1e-4)
    e_o = o["energy_cf"]
    s_g = np.array(r.energy_cf[1:]) / r.energy_cf[0]
    s_o = e_o[1:] / e_o[0]
    assert np.all(np.abs(s_g - s_o) <= 1e-5 * s_o + 1e-12), (s_g, s_o)
    np.testing.assert_allclose(r.energy_el, o["energy_el"], rtol=0, atol=1e-5 * e_o[0])
    np.testing.assert_allclose(r.cross_el, o["cross_el"], rtol=0, atol=1e-6 * e_o[0])
    np.testing.assert_allclose(r.colmean_absmax, o["colmean_absmax"], rtol=0, atol=1e-6 * np.max(np.abs(mu_o)))
    # E_top bit-exact
    assert r.n_top_global == int(o["n_top"])
    sha = hashlib.sha256(np.ascontiguousarray(g["top"], "<i8").tobytes()).hexdigest()
    assert sha == str(o["top_sha256"])
    pos = o["sample_pos"]
    np.testing.assert_array_equal(g["top"][pos], o["sample_idx"])
    assert np.max(np.abs(g["rho"][pos] - o["sample_rho"])) <= 1e-3
    np.testing.assert_allclose(r.rho_mean_aggr, o["rho_mean_aggr"], atol=1e-3)
    np.testing.assert_allclose(r.rho_energy_aggr, o["rho_energy_aggr"], atol=1e-3)
    return r


def test_c4_against_cached_oracle(cuda_device):
    _, g = _run(config_spec("c4"))
    r = _against_cache("c4", g)
    assert r.precision_sigma <= 5e-5 and r.precision_share <= 5e-6


def test_c4_fullsize_properties(cuda_device):
    spec = config_spec("c4")
    l, m = spec.l, spec.m
    Xd, g = _run(spec)
    r, mu_g, V, sigma, top, rho = g["res"], g["mu"], g["V"], g["sigma"], g["top"], g["rho"]
    k, n_top = V.shape[1], g["n_top"]
    X = Xd.cpu().numpy()
    del Xd
    torch.cuda.empty_cache()

    mu = X.sum(axis=0, dtype=np.float64) / l
    assert np.max(np.abs(mu_g - mu)) <= 1e-6 * np.max(np.abs(mu))
    total = float(np.einsum("ij,ij->", X, X, dtype=np.float64))
    assert abs(r.energy_cf[0] - total) <= 1e-9 * total
    assert abs(r.energy_cf[1] - l * float(mu @ mu)) <= 1e-9 * total

    # E_top: composite key (|x| bits, then smaller linear index first), zeros excluded
    key = (X.view(np.uint32) & np.uint32(0x7FFFFFFF)).astype(np.int64).ravel()
    comp = (key << 32) | (np.int64(0xFFFFFFFF) - np.arange(l * m, dtype=np.int64))
    nz = int(np.count_nonzero(key))
    n_eff = min(n_top, nz)
    want = np.sort(np.argpartition(comp, comp.size - n_eff)[comp.size - n_eff:])
    assert r.n_top_global == n_eff
    np.testing.assert_array_equal(top, want)
    del comp, key

    # V orthonormal; sigma_r = ||Xc v_r|| (fp64 Rayleigh quotient at the returned vectors)
    assert np.max(np.abs(V.T @ V - np.eye(k))) <= 1e-6
    xv = np.zeros((l, k))
    for r0 in range(0, l, 8192):
        blk = X[r0:r0 + 8192].astype(np.float64) - mu
        xv[r0:r0 + 8192] = blk @ V
    sig_rq = np.sqrt(np.sum(xv * xv, axis=0))
    np.testing.assert_allclose(sigma, sig_rq, rtol=1e-4)
    assert r.sigma_next / sigma[-1] < 0.8

    # rho at sampled entries of E_top, recomputed in fp64
    rng = np.random.default_rng(0)
    pick = np.sort(rng.choice(len(top), size=2000, replace=False))
    li = top[pick]
    i, j = li // m, li % m
    x = X[i, j].astype(np.float64)
    S = np.sum(xv[i] * V[j], axis=1)
    Tt = (x - mu[j]) - S
    ref = np.stack([mu[j] ** 2, S ** 2, Tt ** 2], 1) / (x * x)[:, None]
    assert np.max(np.abs(rho[pick, :3] - ref)) <= 1e-3
    np.testing.assert_allclose(rho[pick, 3], 1.0 - rho[pick, :3].sum(1), atol=1e-12)

    e_el, e_cf = np.array(r.energy_el), np.array(r.energy_cf)
    assert np.all(np.abs(e_el - e_cf) <= 1e-5 * e_cf[0])
    assert abs(e_cf[1] + e_cf[2] + e_cf[3] - e_cf[0]) <= 1e-6 * e_cf[0]


def test_c4_planted_exact_closed_forms(cuda_device):
    """sigma_t = 0: X = 1 mu^T + sum_{r < 48} c_r h(a_r, i) h(b_r, j) exactly in fp32 at c4 size;
    k = 40 < 48 planted directions, so the tail is the 8 smallest planted terms.  Closed forms:
    mu exact, sigma_r = c_r sqrt(l m), E_mean = l ||mu||^2, E_spike = sum_{r<40} sigma_r^2,
    E_tail = sum_{r>=40} sigma_r^2, M / spike / tail and rho of every entry."""
    spec = SynthSpec(131072, 4096, seed=77, exact=True, k_s=48)
    l, m, k = spec.l, spec.m, 40
    Xd, g = _run(spec)
    r = g["res"]
    a, b, c, mu = planted(spec)
    mu = mu.numpy()
    order = np.argsort(-np.array(c), kind="stable")
    sig = np.array(c)[order] * math.sqrt(l * m)
    np.testing.assert_array_equal(g["mu"], mu)
    np.testing.assert_allclose(g["sigma"], sig[:k], rtol=1e-9)
    assert 0.9 * sig[k] <= r.sigma_next <= sig[k] * (1 + 1e-6)
    e_mean = l * float(mu @ mu)
    e_spike = float(np.sum(sig[:k] ** 2))
    e_tail = float(np.sum(sig[k:] ** 2))
    e_tot = e_mean + e_spike + e_tail  # the planted terms are orthogonal to 1 and to each other
    np.testing.assert_allclose(r.energy_cf, [e_tot, e_mean, e_spike, e_tail], rtol=1e-9)
    np.testing.assert_allclose(r.energy_el, [e_tot, e_mean, e_spike, e_tail], rtol=1e-6)
    # V_k spans the planted right factors of the 40 largest c_r
    jj = torch.arange(m, dtype=torch.int64)
    Vp = np.stack([walsh(b[q], jj).numpy() / math.sqrt(m) for q in order[:k]], 1)
    assert _subspace_sin(g["V"], Vp) <= 1e-5  # eig_tol 1e-6 on residuals / lambda_1
    # E_top by the composite key over the closed-form X (massive ties), then rho per entry
    X = Xd.cpu().numpy()
    del Xd
    torch.cuda.empty_cache()
    key = (X.view(np.uint32) & np.uint32(0x7FFFFFFF)).astype(np.int64).ravel()
    comp = (key << 32) | (np.int64(0xFFFFFFFF) - np.arange(l * m, dtype=np.int64))
    n_eff = min(g["n_top"], int(np.count_nonzero(key)))
    want = np.sort(np.argpartition(comp, comp.size - n_eff)[comp.size - n_eff:])
    del comp, key
    np.testing.assert_array_equal(g["top"], want)
    i, j = want // m, want % m
    ii, jt = torch.from_numpy(i), torch.from_numpy(j)
    S = np.zeros(len(want))
    T = np.zeros(len(want))
    for q, cr in enumerate(np.array(c)[order]):
        term = cr * walsh(a[order[q]], ii).numpy() * walsh(b[order[q]], jt).numpy()
        if q < k:
            S += term
        else:
            T += term
    x2 = X[i, j].astype(np.float64) ** 2
    ref = np.stack([mu[j] ** 2 / x2, S ** 2 / x2, T ** 2 / x2], 1)
    assert np.max(np.abs(g["rho"][:, :3] - ref)) <= 1e-6


def test_c5_against_cached_oracle(cuda_device):
    path = os.path.join(GOLD, "oracle_c5.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (python tools/oracle_cache.py c5 --eig lapack)")
    _, g = _run(config_spec("c5"))
    _against_cache("c5", g)
