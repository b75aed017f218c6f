"""Candidate-list density at c4: the library's candidate count (BUF CAND) vs n_top, and the
fraction of fused-pass warp row-groups (4 rows x 128 columns) that hold a candidate, for the
library's threshold and for tighter ones (k-th largest |x| at 1.0, 1.25, 1.5 x n_top)."""
import torch

from paper_2603_10444_b200 import Decomposer
from synth.gen import config_spec, generate

spec = config_spec("c4")
X = generate(spec, device="cuda")
dec = Decomposer(spec.l, spec.m, seed=0)
r = dec(X)
torch.cuda.synchronize()
cx = dec.buffer("CAND", torch.int64)[:2].cpu().tolist()
n_top = dec.n_top
print(f"n_top {n_top}  candidates {cx[0]} ({cx[0] / n_top:.2f} x n_top)  overflow {cx[1]}")
A = X.abs().flatten()
for f in (cx[0] / n_top, 1.5, 1.25, 1.0):
    k = int(f * n_top)
    thr = torch.topk(A, k, sorted=False).values.min()
    g = (X.abs() >= thr).view(spec.l // 4, 4, spec.m // 128, 128).any(dim=3).any(dim=1)
    print(f"  {f:.2f} x n_top: thr {thr.item():.4g}  density {k / A.numel():.4%}  groups with a candidate {g.float().mean().item():.1%}")
