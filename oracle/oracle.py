"""ctypes front end of the fp64 CPU oracle (oracle/avd_oracle.c).

TEST INFRASTRUCTURE ONLY — may be imported only by tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs.  The product package
(``paper_2603_10444_b200``) never imports this module and shares no code with it.

Every quantity follows PAPER.md:1-27 (section "Mean Bias as the Dominant Source of Activation
Outliers"); the readings used where the paper is silent are DESIGN.md R1..R13.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import sys
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "avd_oracle.c")
_LIB = os.path.join(_HERE, "_build", "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, fp64, IEEE order: -ffp-contract=off, no fast-math)."""
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O3", "-mavx2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class OracleReport(ctypes.Structure):
    _fields_ = [
        ("n_top", ctypes.c_int64),
        ("energy_cf", ctypes.c_double * 4),
        ("energy_el", ctypes.c_double * 4),
        ("cross_el", ctypes.c_double * 3),
        ("colmean_absmax", ctypes.c_double * 2),
        ("rho_mean_aggr", ctypes.c_double * 4),
        ("rho_energy_aggr", ctypes.c_double * 3),
        ("sigma_next", ctypes.c_double),
        ("trace_g", ctypes.c_double),
        ("sweeps", ctypes.c_int32),
        ("status", ctypes.c_int32),
    ]


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        lib.oracle_column_mean.argtypes = [P, I64, I64, P]
        lib.oracle_center.argtypes = [P, I64, I64, P, P]
        lib.oracle_gram.argtypes = [P, I64, I64, P]
        lib.oracle_jacobi_eig.argtypes = [P, I64, P, P, ctypes.c_int]
        lib.oracle_jacobi_eig.restype = ctypes.c_int
        lib.oracle_top_set_sort.argtypes = [P, I64, I64, I64, P]
        lib.oracle_top_set_sort.restype = I64
        lib.oracle_top_set_heap.argtypes = [P, I64, I64, I64, P]
        lib.oracle_top_set_heap.restype = I64
        lib.oracle_decompose.argtypes = [P, I64, I64, ctypes.c_int32, I64, ctypes.c_int32,
                                         P, P, P, P, P, P, ctypes.POINTER(OracleReport)]
        lib.oracle_decompose.restype = ctypes.c_int
        lib.oracle_gram_x.argtypes = [P, I64, I64, P, P]
        lib.oracle_gram_x.restype = ctypes.c_int
        lib.oracle_mean_gram.argtypes = [P, I64, I64, ctypes.c_int32, P, P]
        lib.oracle_mean_gram.restype = ctypes.c_int
        lib.oracle_finish.argtypes = [P, I64, I64, ctypes.c_int32, I64, ctypes.c_int32, P, P, P,
                                      ctypes.c_double, P, P, P, ctypes.POINTER(OracleReport)]
        lib.oracle_finish.restype = ctypes.c_int
        lib.oracle_sign_fix.argtypes = [P, I64, I64]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(X) -> np.ndarray:
    X = np.ascontiguousarray(np.asarray(X, dtype=np.float32))
    assert X.ndim == 2
    return X


# ---- plan rules (R1, R2) -------------------------------------------------------
def _floor_frac(frac: float, n: int) -> int:
    v = frac * n
    r = round(v)
    return int(r) if abs(v - r) < 1e-9 else int(math.floor(v))


def rank_k(m: int, k_frac: float = 0.01) -> int:
    """k = max(1, floor(0.01 m)) — PAPER.md:14 ("top k = floor(0.01 m)"), R1."""
    return max(1, _floor_frac(k_frac, m))


def n_top_of(l: int, m: int, top_frac: float = 0.001) -> int:
    """|E_top| = max(1, floor(0.001 l m)) — PAPER.md:22 ("top 0.1% of entries"), R2."""
    return max(1, _floor_frac(top_frac, l * m))


# ---- single steps ------------------------------------------------------------------------
def column_mean(X) -> np.ndarray:
    """mu = (1/l) X^T 1, two-pass in fp64."""
    X = _f32(X)
    mu = np.empty(X.shape[1], np.float64)
    _load().oracle_column_mean(_ptr(X), X.shape[0], X.shape[1], _ptr(mu))
    return mu


def center(X, mu) -> np.ndarray:
    """Xc = X - 1 mu^T."""
    X = _f32(X)
    mu = np.ascontiguousarray(mu, np.float64)
    Xc = np.empty(X.shape, np.float64)
    _load().oracle_center(_ptr(X), X.shape[0], X.shape[1], _ptr(mu), _ptr(Xc))
    return Xc


def gram(Xc) -> np.ndarray:
    """G = Xc^T Xc (fp64, row-order sums)."""
    Xc = np.ascontiguousarray(Xc, np.float64)
    G = np.empty((Xc.shape[1], Xc.shape[1]), np.float64)
    _load().oracle_gram(_ptr(Xc), Xc.shape[0], Xc.shape[1], _ptr(G))
    return G


def jacobi_eig(G, max_sweeps: int = 60):
    """Cyclic Jacobi eigendecomposition; returns (lam desc, V with V[:, r] = eigvec r, sweeps)."""
    G = np.ascontiguousarray(G, np.float64)
    m = G.shape[0]
    lam = np.empty(m, np.float64)
    V = np.empty((m, m), np.float64)
    sweeps = _load().oracle_jacobi_eig(_ptr(G), m, _ptr(lam), _ptr(V), max_sweeps)
    return lam, V, sweeps


def top_set(X, n_top: int, heap: bool = False) -> np.ndarray:
    """E_top: linear indices i*m+j of the n_top largest |X_ij| (ties: smaller index first,
    zeros excluded), ascending (R3, R4)."""
    X = _f32(X)
    idx = np.empty(max(n_top, 1), np.int64)
    f = _load().oracle_top_set_heap if heap else _load().oracle_top_set_sort
    n = f(_ptr(X), X.shape[0], X.shape[1], n_top, _ptr(idx))
    return idx[:n].copy()


# ---- the whole pass ----------------------------------------------------------------------
def decompose(X, k: int | None = None, n_top: int | None = None, k_frac: float = 0.01,
              top_frac: float = 0.001, heap: bool | None = None, eig: str = "jacobi") -> dict:
    """Full mean/spike/tail decomposition + top-0.1% attribution of X (fp32 l x m).

    eig = "jacobi": the oracle's own parallel cyclic Jacobi eigensolve of G (the default; every
    pin runs it).  eig = "lapack": the eigen step is numpy.linalg.eigh (LAPACK dsyevd) on the same
    G — a library primitive serving as that one step, for m in the thousands where
    the Jacobi sweeps take hours; the Gram, E_top, energies and rho stay the oracle's C code."""
    X = _f32(X)
    l, m = X.shape
    k = rank_k(m, k_frac) if k is None else int(k)
    n_top = n_top_of(l, m, top_frac) if n_top is None else int(n_top)
    if heap is None:
        heap = l * m > (1 << 26)
    mu = np.empty(m, np.float64)
    V = np.empty((m, max(k, 1)), np.float64)
    sigma = np.empty(max(k, 1), np.float64)
    lam = np.empty(m, np.float64)
    idx = np.empty(max(n_top, 1), np.int64)
    rho = np.empty((max(n_top, 1), 4), np.float64)
    rep = OracleReport()
    lib = _load()
    if eig == "jacobi":
        st = lib.oracle_decompose(_ptr(X), l, m, k, n_top, int(heap), _ptr(mu), _ptr(V),
                                  _ptr(sigma), _ptr(lam), _ptr(idx), _ptr(rho),
                                  ctypes.byref(rep))
    elif eig == "lapack":
        G = np.empty((m, m), np.float64)
        st = lib.oracle_mean_gram(_ptr(X), l, m, k, _ptr(mu), _ptr(G))
        if st == 0:
            trace = float(sum(float(G[j, j]) for j in range(m)))  # row order, as the C pass
            w, U = np.linalg.eigh(G)
            order = np.lexsort((np.arange(m), -w))  # descending, ties by index
            lam[:] = w[order]
            V[:] = U[:, order[:k]]
            lib.oracle_sign_fix(_ptr(V), m, k)
            del G, U
            st = lib.oracle_finish(_ptr(X), l, m, k, n_top, int(heap), _ptr(mu), _ptr(lam), _ptr(V),
                                   trace, _ptr(sigma), _ptr(idx), _ptr(rho), ctypes.byref(rep))
    else:
        raise ValueError(eig)
    if st != 0:
        raise ValueError(f"oracle_decompose status {st}")
    n = rep.n_top
    e_cf = np.array(rep.energy_cf[:])
    return dict(
        l=l, m=m, k=k, n_top_req=n_top, n_top=n, mu=mu, V=V, sigma=sigma, lam=lam,
        sigma_next=rep.sigma_next, top_idx=idx[:n].copy(), rho=rho[:n].copy(),
        energy_cf=e_cf, energy_el=np.array(rep.energy_el[:]),
        shares_cf=e_cf[1:] / e_cf[0] if e_cf[0] > 0 else np.zeros(3),
        cross_el=np.array(rep.cross_el[:]), colmean_absmax=np.array(rep.colmean_absmax[:]),
        rho_mean_aggr=np.array(rep.rho_mean_aggr[:]),
        rho_energy_aggr=np.array(rep.rho_energy_aggr[:]),
        trace_g=rep.trace_g, sweeps=rep.sweeps, eig=eig,
    )


def gram_x(X, mu) -> np.ndarray:
    """G = Xc^T Xc formed from fp32 X and mu in row chunks (no l x m fp64 copy)."""
    X = _f32(X)
    mu = np.ascontiguousarray(mu, np.float64)
    G = np.empty((X.shape[1], X.shape[1]), np.float64)
    _load().oracle_gram_x(_ptr(X), X.shape[0], X.shape[1], _ptr(mu), _ptr(G))
    return G


def mean_diagnostics(X, k=None) -> dict:
    """Mean-bias diagnostics of the paper's section "Mean bias phenomenon" and
    Eq. R, in the paper's order and notation, fp64:
      mu = (1/l) X^T 1; mu_hat = mu / ||mu||; p_i = x_i^T mu_hat;
      sign fraction = max(#p_i > 0, #p_i < 0) / l ("max fraction of tokens whose
      x_i^T mu_hat shares one sign"); R = ||mu|| / sqrt(||X||_F^2 / l) (N read as l);
      X = U S V^T (uncentred): v_1, sigma_1 from the Jacobi eigendecomposition of
      X^T X; u_1 = X v_1 / sigma_1; alpha_1 = (sigma_1 / l) u_1^T 1 (sign of v_1
      such that alpha_1 >= 0); cos_mu_v1 = |mu_hat^T v_1| (0 when mu = 0).
    Top k (default all m) uncentred pairs: sigma_u[i], alpha[i] = |mu . v_i|, cos[i] = alpha[i]/||mu||.
    Readings (R19): with mu = 0 the sign fraction and cos are 0."""
    X = _f32(X)
    l, m = X.shape
    Xd = X.astype(np.float64)
    mu = column_mean(X)
    nmu = math.sqrt(float(mu @ mu))
    if nmu > 0.0:
        p = Xd @ (mu / nmu)
        pos, neg = int(np.count_nonzero(p > 0)), int(np.count_nonzero(p < 0))
        frac = max(pos, neg) / l
    else:
        pos = neg = 0
        frac = 0.0
    R = nmu / math.sqrt(float(np.sum(Xd * Xd)) / l)
    lam, V, _ = jacobi_eig(gram(Xd))
    v1 = V[:, 0].copy()
    s1 = math.sqrt(max(lam[0], 0.0))
    u1 = (Xd @ v1) / s1 if s1 > 0 else np.zeros(l)
    alpha1 = s1 / l * float(np.sum(u1))
    if alpha1 < 0:
        v1, u1, alpha1 = -v1, -u1, -alpha1
    cos = abs(float(mu @ v1)) / nmu if nmu > 0 else 0.0
    # the top-k uncentred pairs ("the other right singular directions"):
    # sigma_i = sqrt(lambda_i(X^T X)), alpha_i = |mu . v_i| (the coefficients of mu = sum_i
    # alpha_i v_i, sign-free), cos_i = alpha_i / ||mu||
    kk = m if k is None else min(int(k), m)
    sig_u = np.sqrt(np.maximum(lam[:kk], 0.0))
    alpha = np.abs(mu @ V[:, :kk])
    cos_k = alpha / nmu if nmu > 0 else np.zeros(kk)
    return dict(mu_norm=nmu, p_pos=pos, p_neg=neg, sign_fraction=frac, R=R, sigma1_u=s1, v1=v1,
                alpha1=alpha1, cos_mu_v1=cos, sigma_u=sig_u, alpha=alpha, cos=cos_k)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


if __name__ == "__main__":  # tiny self-demo
    X = np.array([[1, 2], [3, 4]], np.float32)
    t = time.time()
    r = decompose(X)
    print({k: v for k, v in r.items() if k in ("mu", "sigma", "energy_cf", "top_idx", "rho")},
          f"{time.time() - t:.3f}s", file=sys.stderr)
