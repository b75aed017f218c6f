"""GPU parity of the Averis NVFP4 forward GeMM through the C ABI
(include/avd_averis.h) against the numpy oracle (oracle/averis.py) on the same seeded inputs:

  * bit-exact: every E2M1 code and UE4M3 scale of X_R, W and mu_bar, and the tensor scales
    (integer decisions taken in the same fp32 order on both sides, A1-A8);
  * mu_X to 1e-12 relative (fp64 sums in different orders);
  * Y_hat within the fp32-accumulation bound derived in DESIGN.md A9:
        |dY_ij| <= (m * 2^-23 + 2^-20) * (|X_R_bar| |W_bar|)_ij + 2^-20 |bias_j|
    and, as a sharper statistical check, the median relative error below 2^-18.
Shapes span several 128 x 128 tiles, ragged l, n and a K tail (m % 256 != 0)."""
import numpy as np
import pytest
import torch

from oracle import averis as A
from synth.gen import SynthSpec, generate, generate_weight

pytestmark = pytest.mark.gpu


def _unpack(codes: torch.Tensor, rows: int, m: int) -> np.ndarray:
    b = codes.cpu().numpy()[: rows * (m // 2)].reshape(rows, m // 2)
    out = np.empty((rows, m), np.uint8)
    out[:, 0::2] = b & 15
    out[:, 1::2] = b >> 4
    return out


def _unswizzle(sf: torch.Tensor, rows: int, m: int) -> np.ndarray:
    kb4 = 4 * (-(-m // 256))
    r = np.arange(rows)[:, None]
    b = np.arange(m // 16)[None, :]
    off = ((r >> 7) * kb4 + (b >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (b & 3)
    return sf.cpu().numpy()[off]


def _check(l, m, n, stochastic=False, vanilla=False, seed=0):
    from paper_2603_10444_b200.averis import AverisGemm
    X = generate(SynthSpec(l, m, seed=seed))
    W = generate_weight(m, n, seed=seed)
    o = A.averis_forward(X.numpy(), W.numpy(), stochastic=stochastic, seed=seed, split=not vanilla)
    g = AverisGemm(l, m, n, stochastic=stochastic, vanilla=vanilla, seed=seed)
    g.set_weight(W.cuda())
    Y = g(X.cuda())
    torch.cuda.synchronize()
    gs = g.buffer("GSCALE").cpu().numpy()
    # tensor scales and every code / block scale, bit for bit
    assert gs[0] == o["qx"]["g"] and gs[1] == o["qw"]["g"]
    np.testing.assert_array_equal(_unpack(g.buffer("WCODES"), n, m), o["qw"]["codes"])
    np.testing.assert_array_equal(_unswizzle(g.buffer("WSF"), n, m), o["qw"]["scale"])
    np.testing.assert_array_equal(_unswizzle(g.buffer("XSF"), l, m), o["qx"]["scale"])
    np.testing.assert_array_equal(_unpack(g.buffer("XCODES"), l, m), o["qx"]["codes"])
    if not vanilla:
        mu = g.buffer("MU").cpu().numpy()
        np.testing.assert_allclose(mu, o["mu"], rtol=1e-12, atol=1e-12 * np.abs(o["mu"]).max())
        assert gs[2] == o["qmu"]["g"]
        np.testing.assert_array_equal(_unpack(g.buffer("MUCODES"), 1, m), o["qmu"]["codes"])
        np.testing.assert_array_equal(g.buffer("MUSF").cpu().numpy(), o["qmu"]["scale"][0])
        bias = g.buffer("BIAS").cpu().numpy().astype(np.float64)
        np.testing.assert_allclose(bias, o["bias"], rtol=2.0 ** -22, atol=1e-30)
    Yg = Y.cpu().numpy().astype(np.float64)
    err = np.abs(Yg - o["Y"])
    bound = (m * 2.0 ** -23 + 2.0 ** -20) * o["absY"] + 2.0 ** -20 * np.abs(o["bias"])[None, :] + 1e-30
    assert np.all(err <= bound), float(np.max(err / bound))
    rel = err / np.maximum(o["absY"], 1e-30)
    assert np.median(rel) < 2.0 ** -18, float(np.median(rel))
    launches = g.launches()
    g.close()
    return launches


@pytest.mark.parametrize("l,m,n", [(128, 256, 128), (300, 320, 144), (1024, 1024, 512), (513, 2048, 384)])
def test_averis_matches_oracle(cuda_device, l, m, n):
    assert _check(l, m, n) > 0


@pytest.mark.parametrize("l,m,n", [(256, 512, 256), (300, 320, 144)])
def test_averis_stochastic_rounding(cuda_device, l, m, n):
    _check(l, m, n, stochastic=True, seed=3)


def test_vanilla_fp4(cuda_device):
    _check(384, 512, 256, vanilla=True, seed=1)


def test_repeat_calls_identical(cuda_device):
    from paper_2603_10444_b200.averis import AverisGemm
    X = generate(SynthSpec(512, 1024, seed=2)).cuda()
    W = generate_weight(1024, 256, seed=2).cuda()
    g = AverisGemm(512, 1024, 256)
    g.set_weight(W)
    Y1 = g(X).clone()
    Y2 = g(X)
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    # host entry point: same bits
    Yh = torch.empty(512, 256).pin_memory()
    g.forward_host(X.cpu().pin_memory(), Yh)
    assert torch.equal(Yh, Y1.cpu())
    g.close()


def test_full_size_sampled_rows(cuda_device):
    """The bench workload (l = 131072, m = n = 4096) in the bench's launch configuration: every
    code of W and of 48 sampled rows of X_R, and those rows of Y_hat, against the oracle."""
    from paper_2603_10444_b200.averis import AverisGemm
    l, m, n = 131072, 4096, 4096
    spec = SynthSpec(l, m, seed=0)
    Xd = generate(spec, device="cuda")
    W = generate_weight(m, n, seed=0, device="cuda")
    g = AverisGemm(l, m, n)
    g.set_weight(W)
    Y = g(Xd)
    torch.cuda.synchronize()
    X = Xd.cpu().numpy()
    del Xd
    mu = np.zeros(m)
    for r0 in range(0, l, 8192):
        mu += X[r0:r0 + 8192].astype(np.float64).sum(0)
    mu /= l
    corr = np.zeros(m)
    for r0 in range(0, l, 8192):
        corr += (X[r0:r0 + 8192].astype(np.float64) - mu).sum(0)
    mu += corr / l                                     # the oracle's two-pass mean (A.column_mean)
    mu_f = mu.astype(np.float32)
    amax = 0.0
    for r0 in range(0, l, 8192):
        amax = max(amax, float(np.max(np.abs(X[r0:r0 + 8192] - mu_f))))
    np.testing.assert_allclose(g.buffer("MU").cpu().numpy(), mu, rtol=1e-12, atol=1e-12 * np.abs(mu).max())
    qw = A.quantize(W.cpu().numpy().T, lin=np.arange(m)[None, :] * n + np.arange(n)[:, None])
    np.testing.assert_array_equal(_unpack(g.buffer("WCODES"), n, m), qw["codes"])
    rows = np.unique(np.concatenate([[0, 17, 127, 128, l - 1], np.random.default_rng(0).integers(0, l, 43)]))
    XR = (X[rows] - mu_f).astype(np.float32)
    qx = A.quantize(XR, lin=rows[:, None] * m + np.arange(m)[None, :], amax=amax)
    codes = _unpack(g.buffer("XCODES"), l, m)[rows]
    np.testing.assert_array_equal(codes, qx["codes"])
    qmu = A.quantize(mu_f[None, :], amax=float(np.max(np.abs(mu_f))))
    Wd = A.dequantize(qw).T
    bias = A.dequantize(qmu)[0] @ Wd
    Yo = bias[None, :] + A.dequantize(qx) @ Wd
    absY = np.abs(A.dequantize(qx)) @ np.abs(Wd)
    Yg = Y[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.float64)
    bound = (m * 2.0 ** -23 + 2.0 ** -20) * absY + 2.0 ** -20 * np.abs(bias)[None, :]
    assert np.all(np.abs(Yg - Yo) <= bound)
    g.close()


@pytest.mark.parametrize("l,m,n", [(300, 320, 144), (1024, 1024, 512)])
def test_averis_bf16_output(cuda_device, l, m, n):
    """AVD_AVERIS_BF16_OUT: the same fp32 epilogue value rounded to bf16 (RNE): within A9's bound
    plus half a bf16 ulp (2^-8 relative: 8 significant bits), and equal to torch's RNE cast of the fp32 path's Y."""
    from paper_2603_10444_b200.averis import AverisGemm
    X = generate(SynthSpec(l, m, seed=4))
    W = generate_weight(m, n, seed=4)
    o = A.averis_forward(X.numpy(), W.numpy())
    g32 = AverisGemm(l, m, n)
    g32.set_weight(W.cuda())
    Y32 = g32(X.cuda())
    g16 = AverisGemm(l, m, n, bf16_out=True)
    g16.set_weight(W.cuda())
    Y16 = g16(X.cuda())
    torch.cuda.synchronize()
    assert Y16.dtype == torch.bfloat16
    assert torch.equal(Y16, Y32.to(torch.bfloat16))
    Yg = Y16.float().cpu().numpy().astype(np.float64)
    bound = (m * 2.0 ** -23 + 2.0 ** -20) * o["absY"] + 2.0 ** -20 * np.abs(o["bias"])[None, :] + 2.0 ** -8 * np.abs(o["Y"]) + 1e-30
    assert np.all(np.abs(Yg - o["Y"]) <= bound)
    g32.close()
    g16.close()
