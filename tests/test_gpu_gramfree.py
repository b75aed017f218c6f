"""GPU parity of the Gram-free eigensolve (AVD_FLAG_GRAM_FREE; SPEC.md:91;
PAPER.md:311-313): every product G Q of the subspace iteration is X_hat^T (X_hat Q) by two
tensor-core passes over the digit planes, the m x m Gram is never formed.  The method still
reaches the truncated SVD of the centred matrix, so the oracle is the same plain definition
(oracle/oracle.py) with the same north-star tolerances as the Gram path (tests/test_gpu_parity.py):
shapes through both P widths (KQ = 64 / 128), ragged tails, 3 digits, the unsampled massive
activation, the device-graph loop against the host loop, and c4 against the cached fp64 oracle."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from synth.gen import SynthSpec, config_spec, generate

from test_gpu_parity import _gpu, assert_parity

pytestmark = pytest.mark.gpu


def _gf(X, flags=0, **kw):
    from paper_2603_10444_b200._lib import AVD_FLAG_GRAM_FREE
    return _gpu(X, flags=AVD_FLAG_GRAM_FREE | flags, **kw)


@pytest.mark.parametrize("l,m,seed", [(512, 256, 0), (3000, 300, 1), (777, 130, 3), (4096, 512, 4), (1024, 1024, 2)])
def test_gram_free_parity(cuda_device, l, m, seed):
    X = generate(SynthSpec(l, m, seed=seed, f_mean=0.8))
    o = O.decompose(X.numpy())
    g = _gf(X)
    r = g["res"]
    assert r.digits_used == _gpu(X)["res"].digits_used  # the same automatic digits as the Gram path
    assert_parity(g, o)
    assert np.isnan(r.sigma1_u) and np.isnan(r.cos_mu_v1)  # the uncentred pair needs G


@pytest.mark.parametrize("k", [7, 81])
def test_gram_free_large_k(cuda_device, k):
    """p = 16 -> KQ = 64 and p = 96 -> KQ = 128 (SWIZZLE_64B / 128B P operand)."""
    X = generate(SynthSpec(2048, 512, seed=30 + k, k_s=k, f_mean=0.7))
    o = O.decompose(X.numpy(), k=k)
    assert_parity(_gf(X, k=k), o)


def test_gram_free_three_digits_and_outlier(cuda_device):
    X = generate(SynthSpec(65536, 128, seed=13, f_mean=0.8))
    X[17, 3] = 5000.0  # unsampled massive activation: exact-range requant
    o = O.decompose(X.numpy())
    g = _gf(X)
    assert g["res"].requantised == 1
    assert_parity(g, o)
    g3 = _gf(X, digits=3)
    assert g3["res"].digits_used == 3
    assert_parity(g3, o)


def test_gram_free_deterministic(cuda_device):
    X = generate(SynthSpec(4096, 512, seed=9, f_mean=0.8))
    a = _gf(X)
    b = _gf(X)
    np.testing.assert_array_equal(a["sigma"], b["sigma"])
    np.testing.assert_array_equal(a["V"], b["V"])
    np.testing.assert_array_equal(a["rho"], b["rho"])
    # the host entry point (avd_decompose_host: H2D and D2H inside) gives the same bits
    from paper_2603_10444_b200 import Decomposer
    from paper_2603_10444_b200._lib import AVD_FLAG_GRAM_FREE
    dec = Decomposer(4096, 512, flags=AVD_FLAG_GRAM_FREE)
    r = dec.run_host(X.pin_memory())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(np.asarray(r.sigma.cpu()), a["sigma"])
    np.testing.assert_array_equal(np.asarray(r.top_idx.cpu()), a["top_idx"])
    dec.close()


def test_gram_free_c4_against_cached_oracle(cuda_device):
    from paper_2603_10444_b200._lib import AVD_FLAG_GRAM_FREE
    from test_gpu_fullsize import _against_cache, _run
    _, g = _run(config_spec("c4"), flags=AVD_FLAG_GRAM_FREE)
    _against_cache("c4", g)


@pytest.mark.parametrize("l,m,k,gram_free,outlier", [(3000, 300, None, True, False), (2048, 512, 81, True, False),
                                                     (3000, 300, None, False, False), (65536, 128, None, True, True),
                                                     (65536, 128, None, False, True)])
def test_gram_product_matches_fp64(cuda_device, l, m, k, gram_free, outlier):
    """avd_gram_product: Y = G In against fp64 numpy Xc^T (Xc In) (Xc = X - 1 mu^T from the same
    X), element-wise within the Gram operand's quantisation (2 digits: ~2^-13 of each column's
    range, dithered) — the product the Gram-free eigensolve iterates with, checked on its own."""
    from paper_2603_10444_b200 import Decomposer
    from paper_2603_10444_b200 import _lib as L
    X = generate(SynthSpec(l, m, seed=21, f_mean=0.8))
    if outlier:
        X[17, 3] = 5000.0  # a massive activation: its diagonal must be the exact energy (k_gramfree.cu F4)
    dec = Decomposer(l, m, k=k, flags=L.AVD_FLAG_GRAM_FREE if gram_free else 0)
    dec(X.cuda())
    torch.cuda.synchronize()
    p = dec.plan.p
    rng = np.random.default_rng(5)
    In = rng.standard_normal((m, p))
    In[:, 0] = 0.0
    In[3, 0] = 1.0  # e_3: the diagonal entry G_33 itself
    Y = torch.zeros(m, p, dtype=torch.float64, device="cuda")
    Ind = torch.from_numpy(In).cuda()
    L.avd_gram_product(dec.h, Ind.data_ptr(), Y.data_ptr())
    Xc = X.numpy().astype(np.float64)
    Xc -= Xc.mean(0)
    ref = Xc.T @ (Xc @ In)
    err = np.abs(Y.cpu().numpy() - ref)
    scale = np.abs(Xc).T @ np.abs(Xc @ In)          # |Xc|^T |Xc In|: the magnitudes summed
    # the formed Gram (gram2_kernel) keeps the digit-product classes c <= nd - 1; in a column whose
    # scale a massive activation sets, the other rows live in the low digits, so its off-diagonal
    # entries there carry ~1e-4 of |Xc|^T|Xc In| (they reach eigenvalues at second order only, and
    # its diagonal is exact); the Gram-free products keep every class
    tol = 1e-3 if (outlier and not gram_free) else 1e-4
    assert np.max(err / scale) < tol, float(np.max(err / scale))
    assert np.linalg.norm(Y.cpu().numpy() - ref) <= 1e-5 * np.linalg.norm(ref)
    assert abs(Y[3, 0].item() - ref[3, 0]) <= 1e-6 * ref[3, 0]
    dec.close()
