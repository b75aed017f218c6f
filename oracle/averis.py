"""Plain numpy oracle of the Averis mean-residual NVFP4 forward GeMM.

TEST INFRASTRUCTURE ONLY — may be imported only by tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs.  The product package never imports it
and shares no code, table or constant generator with it.

What it computes (section "Averis", paragraph "Forward pass: activation
mean--residual splitting"; format PAPER.md:488-491 "E2M1 NVFP4"):

    mu_X = (1/l) 1^T X
    X_R  = X - 1 mu_X
    mu_bar = Q_b(mu_X), X_R_bar = Q_b(X_R), W_bar = Q_b(W)
    Y_hat = 1 (mu_bar W_bar) + X_R_bar W_bar             (Eq. averis_forward)

and the paper's baseline "Vanilla FP4" Y = Q_b(X) Q_b(W) with split=False.

Q_b is NVFP4 as DESIGN.md §3 readings A1-A8 fix it (the paper names the format only):
  * E2M1 elements on the grid +-{0, 0.5, 1, 1.5, 2, 3, 4, 6} (1 sign, 2 exponent,
    1 mantissa bit with subnormal 0.5), code = sign << 3 | grid index;
  * blocks of 16 consecutive elements along the contraction dimension K (rows of X and of mu along
    m; columns of W along m) with a UE4M3 block scale, and one fp32 tensor scale
    g = amax / (6 * 448) (the two-level NVFP4 convention; "e4m3-emulated scale mode");
  * every decision in fp32, in this order (both sides take it in the same precision):
        x_r  = fl32(x - fl32(mu))                                  (A6)
        g    = fl32(amax_T / 2688), 1 when that is 0               (A2)
        d6   = fl32(6 * g)
        s    = e4m3_rne(fl32(amax_b / d6)), saturating at 448      (A2)
        S    = fl32(e4m3(s) * g),   R = fl32(1 / S)
        v    = fl32(x_r * R)
        code = nearest grid point of |v| (ties to the even grid index) clamped to 6,
               or stochastic rounding up with probability (|v| - g_lo) / (g_hi - g_lo)
               ("Stochastic rounding (SR) is applied by default")
               decided by u24 < frac * 2^24 with u24 from the counter hash below (A3);
        a block whose scale code is 0 has all codes 0 (A7);
  * dequantised value = grid(code) * e4m3(s) * g, in fp64.
"""
from __future__ import annotations

import numpy as np

BLOCK = 16
E2M1_GRID = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0], np.float64)
E2M1_MAX = 6.0
E4M3_MAX = 448.0
TID_X, TID_MU, TID_W = 1, 2, 3  # stream ids of the stochastic-rounding counter hash (A3)

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def e4m3_value(code) -> np.ndarray:
    """Value of a non-negative UE4M3 code 0..126 (bias 7; exponent 0 = subnormal m * 2^-9)."""
    c = np.asarray(code, np.int64)
    e = c >> 3
    f = c & 7
    return np.where(e == 0, f * 2.0 ** -9, (1.0 + f / 8.0) * np.exp2(e - 7.0))


_E4M3_VALUES = e4m3_value(np.arange(127))  # strictly increasing, 0 .. 448


def e4m3_rne(s) -> np.ndarray:
    """Nearest UE4M3 code of s >= 0 (ties to the even code), saturating at 448 (code 126)."""
    s = np.asarray(s, np.float64)
    hi = np.searchsorted(_E4M3_VALUES, s, side="left")  # first value >= s
    hi = np.clip(hi, 0, 126)
    lo = np.clip(hi - 1, 0, 126)
    dlo = np.abs(s - _E4M3_VALUES[lo])
    dhi = np.abs(_E4M3_VALUES[hi] - s)
    pick_hi = (dhi < dlo) | ((dhi == dlo) & (hi % 2 == 0))
    code = np.where(pick_hi, hi, lo)
    return np.where(s >= E4M3_MAX, 126, code).astype(np.uint8)


def counter_u24(seed: int, tid: int, idx) -> np.ndarray:
    """24-bit uniform integers from a counter hash of (seed, tensor id, linear index): the
    splitmix64 finaliser of idx + tid * 0x9E3779B97F4A7C15 + seed * 0xD1B54A32D192ED03 (mod 2^64),
    top 24 bits.  Both sides implement it independently (A3)."""
    with np.errstate(over="ignore"):
        z = np.asarray(idx, np.uint64) + np.uint64(tid) * np.uint64(0x9E3779B97F4A7C15) \
            + np.uint64(seed) * np.uint64(0xD1B54A32D192ED03)
        z = z ^ (z >> np.uint64(30))
        z = z * np.uint64(0xBF58476D1CE4E5B9)
        z = z ^ (z >> np.uint64(27))
        z = z * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(40)).astype(np.int64)


def tensor_scale(amax: float) -> np.float32:
    """g = fl32(amax / 2688) (2688 = 6 * 448), 1 when that is 0 (A2)."""
    g = np.float32(amax) / np.float32(6.0 * 448.0)
    return np.float32(1.0) if g == 0 else np.float32(g)


def e2m1_round(v: np.ndarray, stochastic: bool, u24=None) -> np.ndarray:
    """E2M1 code (sign << 3 | index) of fp32 values v (A3)."""
    v = np.asarray(v, np.float32)
    a = np.minimum(np.abs(v).astype(np.float64), E2M1_MAX)
    lo = np.searchsorted(E2M1_GRID, a, side="right") - 1           # grid[lo] <= a
    lo = np.clip(lo, 0, 7)
    hi = np.minimum(lo + 1, 7)
    glo, ghi = E2M1_GRID[lo], E2M1_GRID[hi]
    if stochastic:
        frac = np.where(hi > lo, (a - glo) / np.where(hi > lo, ghi - glo, 1.0), 0.0)
        up = np.asarray(u24, np.float64) < frac * 2.0 ** 24
        idx = np.where(up & (hi > lo), hi, lo)
    else:
        dlo, dhi = a - glo, ghi - a
        pick_hi = (hi > lo) & ((dhi < dlo) | ((dhi == dlo) & (hi % 2 == 0)))
        idx = np.where(pick_hi, hi, lo)
    sign = np.signbit(v).astype(np.int64)
    return ((sign << 3) | idx).astype(np.uint8)


def e2m1_value(code) -> np.ndarray:
    c = np.asarray(code, np.int64)
    return np.where(c & 8, -1.0, 1.0) * E2M1_GRID[c & 7]


def quantize(A, stochastic: bool = False, seed: int = 0, tid: int = TID_X, lin=None, amax=None) -> dict:
    """NVFP4 Q_b of a matrix A (rows x K, fp32), blocks of 16 along K (the last axis).

    lin: linear indices (same shape as A) fed to the counter hash (the element's position in the
    tensor as the caller stores it); default row-major.  amax: the tensor amax (default max|A|).
    Returns codes [rows, K] (one E2M1 code per element), scale codes [rows, ceil(K/16)], g."""
    A = np.asarray(A, np.float32)
    rows, K = A.shape
    nb = -(-K // BLOCK)
    Ap = np.zeros((rows, nb * BLOCK), np.float32)
    Ap[:, :K] = A
    if amax is None:
        amax = float(np.max(np.abs(A))) if A.size else 0.0
    g = tensor_scale(amax)
    d6 = np.float32(np.float32(6.0) * g)
    blocks = Ap.reshape(rows, nb, BLOCK)
    amax_b = np.max(np.abs(blocks), axis=2)                              # fp32, exact
    s_code = e4m3_rne((amax_b / d6).astype(np.float32))
    S = (e4m3_value(s_code).astype(np.float32) * g).astype(np.float32)
    with np.errstate(divide="ignore"):
        R = np.where(s_code > 0, np.float32(1.0) / np.where(S > 0, S, np.float32(1)), np.float32(0)).astype(np.float32)
    v = (blocks * R[:, :, None]).astype(np.float32)
    u = None
    if stochastic:
        if lin is None:
            lin = np.arange(rows * K, dtype=np.int64).reshape(rows, K)
        linp = np.zeros((rows, nb * BLOCK), np.int64)
        linp[:, :K] = lin
        u = counter_u24(seed, tid, linp.reshape(rows, nb, BLOCK))
    codes = e2m1_round(v, stochastic, u)
    codes = np.where((s_code > 0)[:, :, None], codes, 0).astype(np.uint8)
    return {"codes": codes.reshape(rows, nb * BLOCK)[:, :K], "scale": s_code, "g": g}


def dequantize(q: dict) -> np.ndarray:
    """fp64 values grid(code) * e4m3(scale) * g."""
    codes, s_code, g = q["codes"], q["scale"], float(q["g"])
    rows, K = codes.shape
    sc = np.repeat(e4m3_value(s_code), BLOCK, axis=1)[:, :K]
    return e2m1_value(codes) * sc * g


def column_mean(X) -> np.ndarray:
    """mu_X = (1/l) 1^T X, two-pass fp64."""
    X = np.asarray(X, np.float64)
    mu = X.sum(axis=0) / X.shape[0]
    mu += (X - mu).sum(axis=0) / X.shape[0]
    return mu


def averis_forward(X, W, stochastic: bool = False, seed: int = 0, split: bool = True) -> dict:
    """Eq. averis_forward: Y_hat = 1 (mu_bar W_bar) + X_R_bar W_bar, fp64.

    X: [l, m] fp32 activations, W: [m, n] fp32 weights.  split=False is the
    paper's "Vanilla FP4" baseline Q(X) Q(W).  Quantised operands are returned
    with their codes and scales (codes of W as [n, m]: the blocks of column j of W along m)."""
    X = np.asarray(X, np.float32)
    W = np.asarray(W, np.float32)
    l, m = X.shape
    m2, n = W.shape
    assert m == m2
    if split:
        mu = column_mean(X)
        mu_f = mu.astype(np.float32)
    else:
        mu = np.zeros(m)
        mu_f = np.zeros(m, np.float32)
    XR = (X - mu_f[None, :]).astype(np.float32)                          # A6
    lin_x = np.arange(l * m, dtype=np.int64).reshape(l, m)
    qx = quantize(XR, stochastic, seed, TID_X, lin_x)
    lin_w = (np.arange(m, dtype=np.int64)[None, :] * n + np.arange(n, dtype=np.int64)[:, None])  # W[k][j] at k*n + j
    qw = quantize(W.T, stochastic, seed, TID_W, lin_w)
    Wd = dequantize(qw).T                                                # [m, n]
    Xd = dequantize(qx)
    out = {"mu": mu, "mu_f": mu_f, "qx": qx, "qw": qw}
    if split:
        qmu = quantize(mu_f[None, :], stochastic, seed, TID_MU, np.arange(m, dtype=np.int64)[None, :])
        bias = dequantize(qmu)[0] @ Wd                                   # mu_bar W_bar  [n]
        out["qmu"] = qmu
    else:
        bias = np.zeros(n)
    out["bias"] = bias
    out["Y"] = bias[None, :] + Xd @ Wd
    out["absY"] = np.abs(Xd) @ np.abs(Wd)                                # for the accumulation bound
    return out


def forward_identity(X, W) -> np.ndarray:
    """The same split with a pass-through quantiser: 1 (mu W) + (X - 1 mu) W."""
    X = np.asarray(X, np.float64)
    W = np.asarray(W, np.float64)
    mu = column_mean(X)
    return (mu @ W)[None, :] + (X - mu[None, :]) @ W


def quantization_error(A, stochastic: bool = False, seed: int = 0) -> float:
    """||deq(Q(A)) - A||_F / ||A||_F (0 for the zero matrix)."""
    A = np.asarray(A, np.float32)
    nrm = np.linalg.norm(A.astype(np.float64))
    if nrm == 0:
        return 0.0
    return float(np.linalg.norm(dequantize(quantize(A, stochastic, seed)) - A) / nrm)
