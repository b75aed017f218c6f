"""Averis mean-residual NVFP4 forward GeMM (Eq. averis_forward)
over the C ABI of include/avd_averis.h — argument marshalling only: every step (column mean,
residual, NVFP4 quantisation of mu, X_R and W, mu_bar W_bar, the block-scaled tcgen05 GeMM) runs in
libavd.so's kernels.  torch is used for device memory and streams."""
from __future__ import annotations

import torch

from . import _lib as L
from .api import _view


class AverisGemm:
    """Y_hat = 1 (mu_bar W_bar) + X_R_bar W_bar for X [l, m] fp32 and W [m, n] fp32 on a B200.

    stochastic: stochastic rounding of the E2M1 codes; vanilla: the paper's
    baseline Q(X) Q(W) without the split."""

    def __init__(self, l: int, m: int, n: int, stochastic: bool = False, vanilla: bool = False,
                 seed: int = 0, device: int = 0, stream: torch.cuda.Stream | None = None,
                 timing: bool = False, bf16_out: bool = False):
        self.l, self.m, self.n = l, m, n
        self.stream = stream or torch.cuda.current_stream(device)
        cfg = L.avd_averis_config()
        cfg.l, cfg.m, cfg.n = l, m, n
        cfg.flags = (L.AVD_AVERIS_STOCHASTIC if stochastic else 0) | (L.AVD_AVERIS_VANILLA if vanilla else 0) | \
            (L.AVD_AVERIS_TIMING if timing else 0) | (L.AVD_AVERIS_BF16_OUT if bf16_out else 0)
        cfg.seed, cfg.device, cfg.stream = seed, device, self.stream.cuda_stream
        self.device = torch.device("cuda", device)
        self.out_dtype = torch.bfloat16 if bf16_out else torch.float32
        self.h = L.avd_averis_create(cfg)

    def set_weight(self, W: torch.Tensor) -> None:
        assert W.dtype == torch.float32 and W.is_contiguous() and tuple(W.shape) == (self.m, self.n)
        self._W = W  # kept alive until the stream-ordered quantisation has read it
        L.avd_averis_set_weight(self.h, W.data_ptr())

    def forward(self, X: torch.Tensor, Y: torch.Tensor | None = None) -> torch.Tensor:
        assert X.dtype == torch.float32 and X.is_contiguous() and tuple(X.shape) == (self.l, self.m)
        if Y is None:
            Y = torch.empty(self.l, self.n, dtype=self.out_dtype, device=self.device)
        L.avd_averis_forward(self.h, X.data_ptr(), Y.data_ptr())
        return Y

    __call__ = forward

    def forward_host(self, X: torch.Tensor, Y: torch.Tensor) -> torch.Tensor:
        """X, Y host tensors (pinned for asynchronous copies); synchronises."""
        L.avd_averis_forward_host(self.h, X.data_ptr(), Y.data_ptr())
        return Y

    def buffer(self, name: str) -> torch.Tensor:
        """A workspace buffer as a torch view (include/avd_averis.h, AVD_AV_*)."""
        ptr, nbytes = L.avd_averis_buffer(self.h, L.AV_BUF[name])
        dt = {"MU": torch.float64, "GSCALE": torch.float32, "BIAS": torch.float32}.get(name, torch.uint8)
        return _view(ptr, nbytes, dt, self.device.index)

    def stage_ms(self) -> list[float]:
        """[stats + mu_bar + bias, quantise X_R, GeMM] of the last forward (timing=True)."""
        return L.avd_averis_stage_ms(self.h)

    def launches(self) -> int:
        return L.avd_averis_launch_count(self.h)

    def close(self) -> None:
        if self.h:
            L.avd_averis_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
