"""Pins of the fp64 CPU oracle (oracle/) against what the paper and the mathematics fix —
never against the oracle itself and never against the CUDA path.

  * worked examples (tests/golden/*.json, each with its citation),
  * closed forms of the planted exact generator (synth/, sigma_t = 0): mu, sigma_r, energies,
    per-entry M/S/T and rho, at sizes up to a few hundred thousand entries,
  * a library routine (numpy SVD / eigh) for the truncated SVD on small inputs,
  * brute force (numpy lexsort) for the top set, including massive ties and zeros,
  * invariants the paper states (zero column means, exact energy split,
    orthogonality; rho + cross = 1).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from synth.gen import SynthSpec, generate, planted, walsh

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- worked examples
def test_worked_example_2x2():
    g = _gold("worked_2x2.json")
    X = np.array(g["X"], np.float32)
    r = O.decompose(X)
    assert r["k"] == g["k"] and r["n_top"] == g["n_top"]
    np.testing.assert_allclose(r["mu"], g["mu"], rtol=0, atol=0)
    np.testing.assert_allclose(r["sigma"], g["sigma"], rtol=1e-14)
    np.testing.assert_allclose(np.abs(r["V"][:, 0]), g["v1"], rtol=1e-14)
    np.testing.assert_allclose(r["energy_cf"], g["energy_cf"], rtol=1e-14, atol=1e-13)
    np.testing.assert_array_equal(r["top_idx"], g["top_idx"])
    np.testing.assert_allclose(r["rho"], g["rho"], atol=1e-14)
    np.testing.assert_allclose(r["rho_mean_aggr"], g["rho_mean_aggr"], atol=1e-14)
    np.testing.assert_allclose(r["rho_energy_aggr"], g["rho_energy_aggr"], atol=1e-14)
    np.testing.assert_allclose(r["cross_el"], g["cross_el"], atol=1e-13)
    np.testing.assert_allclose(r["colmean_absmax"], g["colmean_absmax"], atol=1e-14)
    np.testing.assert_allclose(r["energy_el"], g["energy_el"], rtol=1e-14, atol=1e-13)
    assert abs(r["sigma_next"] - g["sigma_next"]) <= 1e-7  # sqrt of a ~1e-16 rounding residue


def test_column_mean_and_center_examples():
    for case in _gold("column_mean_examples.json")["cases"]:
        X = np.array(case["X"], np.float32)
        mu = O.column_mean(X)
        np.testing.assert_array_equal(mu, case["mu"])
        np.testing.assert_array_equal(O.center(X, mu), case["Xc"])


def test_center_idempotent_and_zero_colmeans():
    rng = np.random.default_rng(0)
    X = (rng.standard_normal((37, 11)) * 3 + 5).astype(np.float32)
    mu = O.column_mean(X)
    Xc = O.center(X, mu)
    # column means of Xc vanish to fp64 rounding of the fp32 data
    assert np.abs(Xc.mean(axis=0)).max() <= 1e-12 * np.abs(X).max()
    # mean equals the exact rational mean of the fp32 values (math.fsum is exact)
    exact = np.array([math.fsum(map(float, X[:, j])) / X.shape[0] for j in range(X.shape[1])])
    np.testing.assert_allclose(mu, exact, rtol=1e-15, atol=0)


def test_mean_exact_on_planted_generator():
    spec = SynthSpec(256, 64, seed=3, exact=True, k_s=3)
    X = generate(spec).numpy()
    _, _, _, mu = planted(spec)
    # Walsh rows with a != 0 sum to zero over a power-of-two l: the mean is exactly mu
    np.testing.assert_array_equal(O.column_mean(X), mu.numpy())


# ---------------------------------------------------------------- Gram + Jacobi
def test_gram_matches_numpy_matmul():
    rng = np.random.default_rng(1)
    Xc = rng.standard_normal((50, 23))
    np.testing.assert_allclose(O.gram(Xc), Xc.T @ Xc, rtol=1e-13, atol=1e-12)


def test_jacobi_diag_example():
    g = _gold("svd_examples.json")["diag"]
    lam, V, _ = O.jacobi_eig(np.array(g["G"], float))
    np.testing.assert_allclose(lam, g["lam"], rtol=0, atol=0)
    np.testing.assert_allclose(np.abs(V), np.eye(3), atol=0)


def test_jacobi_matches_numpy_eigh():
    rng = np.random.default_rng(2)
    A = rng.standard_normal((60, 40))
    G = A.T @ A
    lam, V, sweeps = O.jacobi_eig(G)
    ref = np.linalg.eigh(G)[0][::-1]
    np.testing.assert_allclose(lam, ref, rtol=1e-11, atol=1e-11 * ref[0])
    np.testing.assert_allclose(V.T @ V, np.eye(40), atol=1e-12)
    np.testing.assert_allclose(G @ V, V * lam, atol=1e-10 * ref[0])
    # sign rule: the largest-|.| entry of every eigenvector is positive
    for r in range(40):
        assert V[np.argmax(np.abs(V[:, r])), r] > 0
    assert sweeps < 20


def test_jacobi_zero_and_rank_deficient():
    lam, V, _ = O.jacobi_eig(np.zeros((5, 5)))
    np.testing.assert_array_equal(lam, 0)
    g = _gold("svd_examples.json")["rank1"]
    a, b = np.array(g["a"]), np.array(g["b"])
    X = np.outer(a, b).astype(np.float32)  # exact in fp32
    r = O.decompose(X, k=1)
    Xc = X - X.astype(np.float64).mean(0)
    sv = np.linalg.svd(Xc, compute_uv=False)
    np.testing.assert_allclose(r["sigma"][0], sv[0], rtol=1e-12)
    # rank-1 reconstruction: tail energy is ~0
    assert r["energy_cf"][3] <= 1e-8 * r["energy_cf"][0]


# ---------------------------------------------------------------- top set (brute force)
def _brute_top(X, n):
    a = np.abs(X.astype(np.float64)).ravel()
    idx = np.arange(a.size)
    keep = a != 0
    a, idx = a[keep], idx[keep]
    order = np.lexsort((idx, -a))  # |x| desc, then linear index asc
    return np.sort(idx[order[:n]])


@pytest.mark.parametrize("heap", [False, True])
def test_top_set_brute_force_random(heap):
    rng = np.random.default_rng(4)
    X = rng.standard_normal((97, 31)).astype(np.float32)
    X[rng.random(X.shape) < 0.05] = 0.0
    X[3, :] = 2.5  # a tied row
    X[:, 7] = -2.5  # ties of equal magnitude, opposite sign
    for n in (1, 5, 40, 200, 3000):
        np.testing.assert_array_equal(O.top_set(X, n, heap=heap), _brute_top(X, n))


@pytest.mark.parametrize("heap", [False, True])
def test_top_set_massive_ties_pure_mean(heap):
    # X = 1 mu^T with a unique argmax |mu_j*| : E_top = {i*m + j* : i < n_top}
    mu = np.array([1.0, -3.0, 2.0, 0.5], np.float32)
    X = np.tile(mu, (50, 1))
    np.testing.assert_array_equal(O.top_set(X, 20, heap=heap), np.arange(20) * 4 + 1)
    # two equal-magnitude columns: row-major interleaving
    mu2 = np.array([3.0, -1.0, -3.0, 0.5], np.float32)
    X2 = np.tile(mu2, (50, 1))
    want = np.sort(np.concatenate([np.arange(10) * 4, np.arange(10) * 4 + 2]))
    np.testing.assert_array_equal(O.top_set(X2, 20, heap=heap), want)


def test_top_set_zeros_excluded_and_negzero():
    X = np.zeros((4, 4), np.float32)
    X[1, 2] = -0.0
    X[2, 3] = 1e-30
    np.testing.assert_array_equal(O.top_set(X, 5), [11])


# ---------------------------------------------------------------- planted closed forms
def _closed_form(spec, k):
    """Every output of the pass from the planted parameters alone (no decomposition)."""
    a, b, c, mu = planted(spec)
    l, m = spec.l, spec.m
    ii = torch.arange(l, dtype=torch.int64)
    jj = torch.arange(m, dtype=torch.int64)
    mu = mu.numpy()
    S = np.zeros((l, m))
    T = np.zeros((l, m))
    for r in range(len(c)):
        term = c[r] * np.outer(walsh(a[r], ii).numpy(), walsh(b[r], jj).numpy())
        if r < k:
            S += term
        else:
            T += term
    X = mu[None, :] + S + T
    sig = np.array(sorted(c, reverse=True)) * math.sqrt(l * m)
    return X, mu, S, T, sig


@pytest.mark.parametrize("l,m,ks,k", [(64, 32, 3, 3), (256, 128, 4, 2), (1024, 256, 2, 2),
                                      (512, 512, 6, 5)])
def test_decompose_planted_exact_closed_forms(l, m, ks, k):
    spec = SynthSpec(l, m, seed=l + m, exact=True, k_s=ks)
    X32 = generate(spec).numpy()
    Xcf, mu, S, T, sig = _closed_form(spec, k)
    np.testing.assert_array_equal(X32.astype(np.float64), Xcf)  # exact in fp32
    n_top = max(1, int(math.floor(0.001 * l * m)))
    r = O.decompose(X32, k=k, n_top=n_top)
    np.testing.assert_array_equal(r["mu"], mu)
    np.testing.assert_allclose(r["sigma"], sig[:k], rtol=1e-11)
    e_tot = float(np.sum(Xcf ** 2))
    want = [e_tot, l * float(np.sum(mu ** 2)), float(np.sum(sig[:k] ** 2)),
            float(np.sum(sig[k:] ** 2))]
    np.testing.assert_allclose(r["energy_cf"], want, rtol=1e-11, atol=1e-9 * e_tot)
    np.testing.assert_allclose(r["energy_el"], want, rtol=1e-11, atol=1e-9 * e_tot)
    top = _brute_top(Xcf, n_top)
    np.testing.assert_array_equal(r["top_idx"], top)
    i, j = top // m, top % m
    x2 = Xcf[i, j] ** 2
    rho = np.stack([mu[j] ** 2 / x2, S[i, j] ** 2 / x2, T[i, j] ** 2 / x2], 1)
    np.testing.assert_allclose(r["rho"][:, :3], rho, atol=1e-10)
    np.testing.assert_allclose(r["rho"].sum(1), 1.0, atol=1e-12)


def test_pure_mean_rho_mean_is_one():
    spec = SynthSpec(128, 64, seed=5, exact=True, k_s=1, spike_scale=0.0)
    X = generate(spec).numpy()
    r = O.decompose(X)
    np.testing.assert_allclose(r["rho"][:, 0], 1.0, atol=0)
    np.testing.assert_allclose(r["energy_cf"][2:], 0.0, atol=0)
    np.testing.assert_allclose(r["rho_mean_aggr"][0], 1.0, atol=0)


def test_centred_rank_k_rho_spike_is_one():
    spec = SynthSpec(256, 128, seed=6, exact=True, k_s=1, mean_scale=0.0)
    X = generate(spec).numpy()
    r = O.decompose(X)  # k = 1 = planted rank
    np.testing.assert_allclose(r["rho"][:, 1], 1.0, atol=1e-12)
    np.testing.assert_allclose(r["rho"][:, [0, 2]], 0.0, atol=1e-12)


# ---------------------------------------------------------------- numpy SVD (library routine)
@pytest.mark.parametrize("l,m,k", [(200, 128, 1), (300, 100, 4), (64, 96, 3)])
def test_decompose_vs_numpy_svd(l, m, k):
    spec = SynthSpec(l, m, seed=l * 7 + m, k_s=k, f_mean=0.7)
    X = generate(spec).numpy()
    r = O.decompose(X, k=k)
    Xd = X.astype(np.float64)
    mu = Xd.mean(axis=0)
    Xc = Xd - mu
    U, s, Vt = np.linalg.svd(Xc, full_matrices=False)
    np.testing.assert_allclose(r["sigma"], s[:k], rtol=1e-10)
    np.testing.assert_allclose(r["sigma_next"], s[k], rtol=1e-9)
    spike = (U[:, :k] * s[:k]) @ Vt[:k]
    tail = Xc - spike
    e = [np.sum(Xd ** 2), l * np.sum(mu ** 2), np.sum(spike ** 2), np.sum(tail ** 2)]
    np.testing.assert_allclose(r["energy_cf"], e, rtol=1e-9)
    np.testing.assert_allclose(r["energy_el"], e, rtol=1e-9)
    top = _brute_top(X, r["n_top_req"])
    np.testing.assert_array_equal(r["top_idx"], top)
    i, j = top // m, top % m
    x2 = Xd[i, j] ** 2
    rho = np.stack([mu[j] ** 2 / x2, spike[i, j] ** 2 / x2, tail[i, j] ** 2 / x2], 1)
    np.testing.assert_allclose(r["rho"][:, :3], rho, atol=1e-9)
    # aggregates over E_top (R10): mean of the per-entry shares, energy-weighted shares
    np.testing.assert_allclose(r["rho_mean_aggr"][:3], rho.mean(axis=0), atol=1e-10)
    np.testing.assert_allclose(r["rho_mean_aggr"][3], 1.0 - rho.sum(1).mean(), atol=1e-10)
    comp = np.stack([mu[j] ** 2, spike[i, j] ** 2, tail[i, j] ** 2], 1)
    np.testing.assert_allclose(r["rho_energy_aggr"], comp.sum(0) / x2.sum(), rtol=1e-9, atol=1e-12)
    # cross terms and column means of the spike / tail from the numpy SVD
    M = np.broadcast_to(mu, Xd.shape)
    cross = [np.sum(M * spike), np.sum(M * tail), np.sum(spike * tail)]
    np.testing.assert_allclose(r["cross_el"], cross, atol=1e-9 * e[0])
    np.testing.assert_allclose(r["colmean_absmax"], [np.abs(spike.mean(0)).max(), np.abs(tail.mean(0)).max()],
                               atol=1e-10 * np.abs(Xd).max())
    # subspace: V_k spans the top right singular vectors
    np.testing.assert_allclose(np.abs(Vt[:k] @ r["V"]), np.eye(k), atol=1e-8)


# ---------------------------------------------------------------- invariants
def test_invariants_on_generator_data():
    spec = SynthSpec(512, 256, seed=9)
    X = generate(spec).numpy()
    r = O.decompose(X)
    e_cf, e_el = r["energy_cf"], r["energy_el"]
    assert abs(e_cf[1] + e_cf[2] + e_cf[3] - e_cf[0]) <= 1e-8 * e_cf[0]  # exact split
    np.testing.assert_allclose(e_el, e_cf, rtol=1e-8)
    assert np.all(np.abs(r["cross_el"]) <= 1e-6 * e_cf[0])  # orthogonality
    assert np.all(r["colmean_absmax"] <= 1e-10 * np.abs(X).max())  # zero column means
    np.testing.assert_allclose(r["rho"].sum(1), 1.0, atol=1e-12)
    assert np.all(r["rho"][:, :3] >= 0)
    assert r["n_top"] == 131  # BASELINE.json configs[0]


def test_validation_errors():
    with pytest.raises(ValueError):
        O.decompose(np.ones((1, 5), np.float32))
    X = np.ones((4, 4), np.float32)
    X[2, 2] = np.nan
    with pytest.raises(ValueError):
        O.decompose(X)
    with pytest.raises(ValueError):
        O.decompose(np.ones((4, 3), np.float32), k=4)


def test_plan_rules():
    assert O.rank_k(256) == 2 and O.rank_k(2048) == 20 and O.rank_k(4096) == 40
    assert O.rank_k(8192) == 81 and O.rank_k(99) == 1 and O.rank_k(100) == 1
    assert O.n_top_of(512, 256) == 131 and O.n_top_of(131072, 4096) == 536870
    assert O.n_top_of(1048576, 8192) == 8589934 and O.n_top_of(2, 2) == 1


# ---------------------------------------------------------------- generator
def test_generator_shard_invariant_and_deterministic():
    spec = SynthSpec(300, 70, seed=11)
    X = generate(spec)
    Y = torch.cat([generate(spec, 0, 123), generate(spec, 123, 177)])
    assert torch.equal(X, Y)
    assert torch.equal(X, generate(spec))
    assert not torch.equal(X, generate(SynthSpec(300, 70, seed=12)))


# ---- mean-bias diagnostics -----------------------
def test_mean_diagnostics_worked_2x2():
    """X = [[1,2],[3,4]] by hand: mu = (2,3), ||X||^2 = 30, X^T X = [[10,14],[14,20]] with
    eigenvalues 15 +- sqrt(221); p = X mu_hat = (8, 18)/sqrt(13) > 0."""
    d = O.mean_diagnostics(np.array([[1, 2], [3, 4]], np.float32))
    lam1 = 15 + math.sqrt(221)
    v1 = np.array([14.0, lam1 - 10.0])
    v1 /= np.linalg.norm(v1)
    mu = np.array([2.0, 3.0])
    assert d["p_pos"] == 2 and d["p_neg"] == 0 and d["sign_fraction"] == 1.0
    assert abs(d["R"] - math.sqrt(13) / math.sqrt(15)) < 1e-14
    assert abs(d["sigma1_u"] - math.sqrt(lam1)) < 1e-12
    assert abs(d["alpha1"] - mu @ v1) < 1e-12
    assert abs(d["cos_mu_v1"] - (mu @ v1) / math.sqrt(13)) < 1e-12


@pytest.mark.parametrize("l,m,rank", [(256, 64, 2), (512, 128, 3)])
def test_mean_diagnostics_planted_constant_mean(l, m, rank):
    """X = 1 c 1^T + sum_r c_r h(a_r, .) h(b_r, .)^T with Walsh codes a_r, b_r != 0: every spike
    direction is orthogonal to 1 (the mean direction), so X^T X = l c^2 1 1^T + sum_r sigma_r^2
    v_r v_r^T exactly: v_1 = mu_hat when l m c^2 > sigma_r^2, cos = 1, sigma_1 = c sqrt(l m),
    alpha_1 = ||mu|| = c sqrt(m); p_i = ||mu|| for every row (sign fraction 1); closed-form R."""
    c = 0.75
    ii, jj = torch.arange(l), torch.arange(m)
    X = torch.full((l, m), c, dtype=torch.float64)
    sig2 = 0.0
    for r in range(rank):
        cr = 0.125 * (r + 1)
        X += cr * torch.outer(walsh(r + 1, ii), walsh(2 * r + 3, jj))
        sig2 += cr * cr * l * m
    d = O.mean_diagnostics(X.float().numpy())
    assert d["sign_fraction"] == 1.0 and d["p_pos"] == l
    assert abs(d["cos_mu_v1"] - 1.0) < 1e-12
    assert abs(d["sigma1_u"] - c * math.sqrt(l * m)) < 1e-9 * c * math.sqrt(l * m)
    assert abs(d["alpha1"] - c * math.sqrt(m)) < 1e-12 * m
    assert abs(d["R"] - c * math.sqrt(m) / math.sqrt((l * m * c * c + sig2) / l)) < 1e-12


def test_mean_diagnostics_vs_numpy_svd():
    """Library routine: numpy's SVD of the uncentred X gives sigma_1 and v_1."""
    rng = np.random.default_rng(7)
    X = (rng.standard_normal((300, 40)) + rng.standard_normal(40) * 3).astype(np.float32)
    d = O.mean_diagnostics(X)
    U, S, Vt = np.linalg.svd(X.astype(np.float64), full_matrices=False)
    mu = X.astype(np.float64).mean(0)
    assert abs(d["sigma1_u"] - S[0]) < 1e-10 * S[0]
    assert abs(d["cos_mu_v1"] - abs(mu @ Vt[0]) / np.linalg.norm(mu)) < 1e-10
    assert abs(d["alpha1"] - abs(S[0] / 300 * U[:, 0].sum())) < 1e-10 * d["alpha1"]
    p = X.astype(np.float64) @ (mu / np.linalg.norm(mu))  # brute force
    assert d["p_pos"] == int((p > 0).sum()) and d["p_neg"] == int((p < 0).sum())


@pytest.mark.parametrize("l,m,rank", [(256, 64, 2), (512, 128, 3)])
def test_mean_topk_planted_closed_forms(l, m, rank):
    """Top-k uncentred pairs on the planted constant-mean data: X^T X =
    l m c^2 (1/sqrt(m))(1/sqrt(m))^T + sum_r sigma_r^2 v_r v_r^T with v_r (Walsh) orthogonal to the
    mean direction, so the pairs are (c sqrt(l m), mu_hat) then (sigma_r, v_r): alpha = (||mu||,
    0, ..., 0) exactly and cos = (1, 0, ..., 0); sigma_i in descending order."""
    c = 0.75
    ii, jj = torch.arange(l), torch.arange(m)
    X = torch.full((l, m), c, dtype=torch.float64)
    sig = []
    for r in range(rank):
        cr = 0.125 * (r + 1)
        X += cr * torch.outer(walsh(r + 1, ii), walsh(2 * r + 3, jj))
        sig.append(cr * math.sqrt(l * m))
    d = O.mean_diagnostics(X.float().numpy(), k=rank + 1)
    want_sig = np.array([c * math.sqrt(l * m)] + sorted(sig, reverse=True))
    np.testing.assert_allclose(d["sigma_u"], want_sig, rtol=1e-12)
    np.testing.assert_allclose(d["alpha"], [c * math.sqrt(m)] + [0.0] * rank, atol=1e-10 * m)
    np.testing.assert_allclose(d["cos"], [1.0] + [0.0] * rank, atol=1e-10)


def test_mean_topk_vs_numpy_svd():
    """Library routine: numpy's SVD of the uncentred X gives every sigma_i and |mu . v_i|."""
    rng = np.random.default_rng(8)
    X = (rng.standard_normal((400, 50)) * np.linspace(3, 0.5, 50) + rng.standard_normal(50) * 2).astype(np.float32)
    d = O.mean_diagnostics(X, k=6)
    _, S, Vt = np.linalg.svd(X.astype(np.float64), full_matrices=False)
    mu = X.astype(np.float64).mean(0)
    np.testing.assert_allclose(d["sigma_u"], S[:6], rtol=1e-10)
    np.testing.assert_allclose(d["alpha"], np.abs(Vt[:6] @ mu), rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(d["cos"], np.abs(Vt[:6] @ mu) / np.linalg.norm(mu), rtol=1e-8, atol=1e-12)


def test_mean_diagnostics_zero_mean():
    """Exactly zero column means: no mean direction -> sign fraction 0, cos 0, R 0 (R19)."""
    ii, jj = torch.arange(64), torch.arange(16)
    X = torch.outer(walsh(3, ii), walsh(5, jj)).float().numpy()
    d = O.mean_diagnostics(X)
    assert d["mu_norm"] == 0.0 and d["sign_fraction"] == 0.0 and d["cos_mu_v1"] == 0.0 and d["R"] == 0.0


# ---------------------------------------------------------------- scaled oracle
def test_gram_x_equals_explicit_centring():
    """The row-chunked Gram from fp32 X (no l x m fp64 copy) is bit-identical to the Gram of
    the explicit Xc, and both equal numpy's fp64 product to rounding."""
    X = generate(SynthSpec(700, 96, seed=41)).numpy()
    mu = O.column_mean(X)
    G1 = O.gram_x(X, mu)
    G2 = O.gram(O.center(X, mu))
    np.testing.assert_array_equal(G1, G2)
    Xc = X.astype(np.float64) - mu
    np.testing.assert_allclose(G1, Xc.T @ Xc, rtol=1e-12, atol=1e-12 * np.abs(G1).max())


@pytest.mark.parametrize("m", [7, 8, 33])
def test_parallel_jacobi_odd_even_sizes(m):
    """Round-robin parallel Jacobi on even and odd m (padding index) against numpy eigh."""
    rng = np.random.default_rng(m)
    A = rng.standard_normal((3 * m, m))
    G = A.T @ A
    lam, V, sweeps = O.jacobi_eig(G)
    w = np.linalg.eigvalsh(G)[::-1]
    np.testing.assert_allclose(lam, w, rtol=1e-12, atol=1e-12 * w[0])
    np.testing.assert_allclose(V.T @ V, np.eye(m), atol=1e-12)
    np.testing.assert_allclose(G @ V, V * lam, atol=1e-11 * w[0])
    assert sweeps < 20


def test_lapack_eig_step_matches_jacobi():
    """decompose(eig="lapack") (numpy eigh as the eigen step) gives the Jacobi oracle's outputs."""
    X = generate(SynthSpec(2048, 256, seed=43)).numpy()
    a = O.decompose(X)
    b = O.decompose(X, eig="lapack")
    np.testing.assert_allclose(b["sigma"], a["sigma"], rtol=1e-11)
    np.testing.assert_allclose(b["V"], a["V"], atol=1e-9)
    np.testing.assert_array_equal(b["top_idx"], a["top_idx"])
    np.testing.assert_allclose(b["rho"], a["rho"], atol=1e-10)
    np.testing.assert_allclose(b["energy_cf"], a["energy_cf"], rtol=1e-11)


@pytest.mark.parametrize("spec", [SynthSpec(300, 77, seed=3), SynthSpec(256, 128, seed=5, exact=True, k_s=4),
                                  SynthSpec(1024, 96, seed=9, k_s=3, f_mean=0.5)])
def test_fast_generator_bit_identical(spec):
    """synth/gen_fast.c (host fill for bench-scale oracle runs) == synth.gen.generate, bit for bit,
    including a shard that starts mid-matrix."""
    from synth.fast import generate_np
    np.testing.assert_array_equal(generate_np(spec).view(np.uint32), generate(spec).numpy().view(np.uint32))
    np.testing.assert_array_equal(generate_np(spec, 37, 100).view(np.uint32),
                                  generate(spec, 37, 100).numpy().view(np.uint32))
