"""User-facing Python API over the C ABI (argument marshalling only; the work is in libavd.so).

    from paper_2603_10444_b200 import Decomposer
    dec = Decomposer(l, m)                 # plans + allocates the workspace once
    res = dec(X)                           # X: CUDA fp32 [l, m], contiguous
    res.mu, res.V, res.sigma, res.top_idx, res.rho, res.energy_cf, ...

PyTorch is used only for device memory and the current CUDA stream.
"""
from __future__ import annotations

import ctypes
import dataclasses

import torch

from . import _lib as L


@dataclasses.dataclass
class Result:
    mu: torch.Tensor            # [m] f64
    V: torch.Tensor             # [m, k] f64, columns = top-k right singular vectors of Xc
    sigma: torch.Tensor         # [k] f64, descending
    top_idx: torch.Tensor       # [n] int64 global linear indices (this rank's slice), ascending
    rho: torch.Tensor           # [n, 4] f64: rho_mean, rho_spike, rho_tail, cross
    n_top_global: int
    top_offset: int
    energy_cf: list             # total, mean, spike, tail (closed forms)
    energy_el: list             # elementwise sum x^2, M^2, spike^2, tail^2
    cross_el: list              # <M,S>, <M,T>, <S,T>
    colmean_absmax: list        # max_j |mean_i spike_ij|, |mean_i tail_ij|
    rho_mean_aggr: list
    rho_energy_aggr: list
    sigma_next: float
    trace_g: float
    iters: int
    max_resid: float
    status: int
    rr_checks: int = 0
    jacobi_sweeps: int = 0
    requantised: int = 0        # 1: Gram operand re-quantised with the exact column ranges
    digits_used: int = 2        # digit planes of the final Gram (3 after an automatic escalation)
    precision_sigma: float = 0.0  # 5-sigma bound of the quantisation error on sigma (relative)
    precision_share: float = 0.0  # 5-sigma bound of the quantisation error on the shares
    # mean-bias diagnostics (include/avd.h)
    mean_R: float = 0.0
    sign_fraction: float = 0.0
    cos_mu_v1: float = 0.0
    alpha1: float = 0.0
    sigma1_u: float = 0.0
    iters_u: int = 0
    # AVD_FLAG_MEAN_TOPK: top-k singular values of the uncentred X and alpha_i = |mu . v_i|
    mean_sigma: torch.Tensor | None = None
    mean_alpha: torch.Tensor | None = None
    iters_uk: int = 0
    resid_uk: float = 0.0

    @property
    def shares_cf(self):
        t = self.energy_cf[0]
        return [e / t for e in self.energy_cf[1:]] if t > 0 else [0.0, 0.0, 0.0]


def _to_list(a):
    return [float(x) for x in a]


class Decomposer:
    """One context (plan + device workspace) for a fixed shape; call it on many matrices."""

    def __init__(self, l: int, m: int, *, k: int | None = None, n_top: int | None = None,
                 k_frac: float = 0.01, top_frac: float = 0.001, seed: int = 0, digits: int = 0,
                 max_iters: int = 0, eig_tol: float = 0.0, device: int | None = None,
                 world: int = 1, l_local: int | None = None, row_offset: int = 0,
                 stream: torch.cuda.Stream | None = None, flags: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2603_10444_b200 needs a CUDA device (sm_100a); no CPU path")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.stream = stream or torch.cuda.current_stream(self.device)
        cfg = L.avd_config()
        cfg.l_global, cfg.m = int(l), int(m)
        cfg.l_local = int(l if l_local is None else l_local)
        cfg.row_offset = int(row_offset)
        cfg.k_frac, cfg.top_frac = float(k_frac), float(top_frac)
        cfg.k_override = int(k or 0)
        cfg.n_top_override = int(n_top or 0)
        cfg.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        cfg.max_iters, cfg.eig_tol, cfg.digits = int(max_iters), float(eig_tol), int(digits)
        cfg.world, cfg.device = int(world), self.device
        cfg.stream = ctypes.c_void_p(self.stream.cuda_stream)
        cfg.flags = int(flags)
        self.cfg = cfg
        with torch.cuda.device(self.device):
            self.h = L.avd_create(cfg)
        self.plan = L.avd_get_plan(self.h)
        self.l, self.m, self.k, self.n_top = int(l), int(m), self.plan.k, self.plan.n_top
        dev = torch.device("cuda", self.device)
        self.mu = torch.empty(self.m, dtype=torch.float64, device=dev)
        self.V = torch.empty((self.m, self.k), dtype=torch.float64, device=dev)
        self.sigma = torch.empty(self.k, dtype=torch.float64, device=dev)
        self.top_idx = torch.empty(max(self.n_top, 1), dtype=torch.int64, device=dev)
        self.rho = torch.empty((max(self.n_top, 1), 4), dtype=torch.float64, device=dev)
        self.topk_u = bool(int(flags) & L.AVD_FLAG_MEAN_TOPK)  # uncentred top-k pairs requested
        self.mean_sigma = torch.empty(self.k, dtype=torch.float64, device=dev) if self.topk_u else None
        self.mean_alpha = torch.empty(self.k, dtype=torch.float64, device=dev) if self.topk_u else None

    def close(self):
        if getattr(self, "h", None):
            L.avd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _outputs(self) -> L.avd_outputs:
        o = L.avd_outputs()
        o.mu_dev, o.V_dev, o.sigma_dev = self.mu.data_ptr(), self.V.data_ptr(), self.sigma.data_ptr()
        o.top_idx_dev, o.rho_dev = self.top_idx.data_ptr(), self.rho.data_ptr()
        if self.topk_u:
            o.mean_sigma_dev, o.mean_alpha_dev = self.mean_sigma.data_ptr(), self.mean_alpha.data_ptr()
        return o

    def _result(self, o: L.avd_outputs, st: int, host=None) -> Result:
        n = int(o.n_top_local)
        mu, V, sigma, idx, rho = host if host is not None else (self.mu, self.V, self.sigma,
                                                                self.top_idx, self.rho)
        return Result(mu=mu, V=V, sigma=sigma, top_idx=idx[:n], rho=rho[:n],
                      n_top_global=int(o.n_top_global), top_offset=int(o.top_offset),
                      energy_cf=_to_list(o.energy_cf), energy_el=_to_list(o.energy_el),
                      cross_el=_to_list(o.cross_el), colmean_absmax=_to_list(o.colmean_absmax),
                      rho_mean_aggr=_to_list(o.rho_mean_aggr),
                      rho_energy_aggr=_to_list(o.rho_energy_aggr), sigma_next=float(o.sigma_next),
                      trace_g=float(o.trace_g), iters=int(o.iters), max_resid=float(o.max_resid),
                      status=st, rr_checks=int(o.rr_checks), jacobi_sweeps=int(o.jacobi_sweeps),
                      requantised=int(o.requantised), digits_used=int(o.digits_used),
                      precision_sigma=float(o.precision_sigma),
                      precision_share=float(o.precision_share), mean_R=float(o.mean_R),
                      sign_fraction=float(o.sign_fraction), cos_mu_v1=float(o.cos_mu_v1),
                      alpha1=float(o.alpha1), sigma1_u=float(o.sigma1_u), iters_u=int(o.iters_u),
                      mean_sigma=self.mean_sigma if host is None else None,
                      mean_alpha=self.mean_alpha if host is None else None,
                      iters_uk=int(o.iters_uk), resid_uk=float(o.resid_uk))

    def _check_X(self, X: torch.Tensor):
        if not (X.is_cuda and X.dtype == torch.float32 and X.is_contiguous()):
            raise ValueError("X must be a contiguous CUDA float32 tensor")
        if tuple(X.shape) != (self.cfg.l_local, self.m):
            raise ValueError(f"X shape {tuple(X.shape)} != ({self.cfg.l_local}, {self.m})")

    def __call__(self, X: torch.Tensor) -> Result:
        """Whole pass on one GPU (world == 1); outputs stay on the device."""
        self._check_X(X)
        o = self._outputs()
        st = L.avd_decompose(self.h, X.data_ptr(), o)
        return self._result(o, st)

    def run_host(self, X_host: torch.Tensor) -> Result:
        """Same pass from host memory through avd_decompose_host (H2D + D2H inside)."""
        if X_host.is_cuda or X_host.dtype != torch.float32 or not X_host.is_contiguous():
            raise ValueError("X_host must be a contiguous CPU float32 tensor")
        if not hasattr(self, "_host_out"):
            pin = torch.cuda.is_available()
            self._host_out = (torch.empty(self.m, dtype=torch.float64, pin_memory=pin),
                              torch.empty((self.m, self.k), dtype=torch.float64, pin_memory=pin),
                              torch.empty(self.k, dtype=torch.float64, pin_memory=pin),
                              torch.empty(max(self.n_top, 1), dtype=torch.int64, pin_memory=pin),
                              torch.empty((max(self.n_top, 1), 4), dtype=torch.float64, pin_memory=pin))
        mu, V, sigma, idx, rho = self._host_out
        o = L.avd_outputs()
        o.mu_dev, o.V_dev, o.sigma_dev = mu.data_ptr(), V.data_ptr(), sigma.data_ptr()
        o.top_idx_dev, o.rho_dev = idx.data_ptr(), rho.data_ptr()
        st = L.avd_decompose_host(self.h, X_host.data_ptr(), o)
        return self._result(o, st, host=self._host_out)

    def launches(self) -> int:
        return L.avd_launch_count(self.h)

    def buffer(self, which: str, dtype: torch.dtype, shape=None) -> torch.Tensor:
        """Zero-copy torch view of a workspace buffer (exchange buffers / diagnostics)."""
        ptr, nbytes = L.avd_buffer(self.h, L.BUF[which])
        return _view(ptr, nbytes, dtype, self.device, shape)


class _CudaArray:
    def __init__(self, ptr, n, typestr, shape):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": shape, "typestr": typestr,
                                         "version": 3, "strides": None}


_TYPESTR = {torch.float64: "<f8", torch.float32: "<f4", torch.int64: "<i8", torch.int32: "<i4",
            torch.int8: "|i1", torch.uint8: "|u1"}


def _view(ptr: int, nbytes: int, dtype: torch.dtype, device: int, shape=None) -> torch.Tensor:
    item = torch.empty((), dtype=dtype).element_size()
    n = nbytes // item
    shape = (n,) if shape is None else tuple(shape)
    with torch.cuda.device(device):
        return torch.as_tensor(_CudaArray(ptr, n, _TYPESTR[dtype], shape), device=f"cuda:{device}")


def decompose(X: torch.Tensor, **kw) -> Result:
    """One-shot convenience: plan, run, free the workspace (outputs are torch-owned)."""
    dec = Decomposer(X.shape[0], X.shape[1], device=X.device.index, **kw)
    r = dec(X)
    torch.cuda.current_stream(X.device).synchronize()
    dec.close()
    return r
