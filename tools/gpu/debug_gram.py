"""Debug helper (not product code): compare the library's fp64 G (AVD_BUF_G) with the exact
centred Gram of X computed in numpy fp64, on an outlier case."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from synth.gen import SynthSpec, generate
from paper_2603_10444_b200 import Decomposer

X = generate(SynthSpec(65536, 128, seed=13, f_mean=0.8))
if len(sys.argv) < 2 or sys.argv[1] != "clean":
    X[17, 3] = 5000.0
Xn = X.numpy().astype(np.float64)
Xc = Xn - Xn.mean(0)
Gt = Xc.T @ Xc
for nd in (2, 3):
    dec = Decomposer(65536, 128, digits=nd)
    r = dec(X.cuda())
    torch.cuda.synchronize()
    mp = (128 + 127) // 128 * 128
    G = dec.buffer("G", torch.float64).view(-1)[: mp * mp].view(mp, mp)[:128, :128].cpu().numpy()
    d = G - Gt
    print(f"nd={nd} requant={r.requantised} sigma={r.sigma.cpu().numpy()} "
          f"max|dG|/max|G|={np.abs(d).max() / np.abs(Gt).max():.3e} "
          f"diag rel err max={np.max(np.abs(np.diag(d)) / np.diag(Gt)):.3e} at {np.argmax(np.abs(np.diag(d)) / np.diag(Gt))} "
          f"offdiag max={np.abs(d - np.diag(np.diag(d))).max():.3e}  G33 {G[3,3]:.6e} vs {Gt[3,3]:.6e}  row3 max err {np.abs(d[3]).max():.3e}")
    lam = np.linalg.eigvalsh(Gt)[::-1][:2]
    print("   true sigma", np.sqrt(lam), " eig(G gpu)", np.sqrt(np.linalg.eigvalsh(G)[::-1][:2]))
    dec.close()

# ---- digit-level check of column 3 (outlier case)
X = generate(SynthSpec(65536, 128, seed=13, f_mean=0.8))
X[17, 3] = 5000.0
for nd in (2, 3):
    dec = Decomposer(65536, 128, digits=nd)
    r = dec(X.cuda())
    torch.cuda.synchronize()
    Dg = dec.buffer("DIGITS", torch.int8).cpu().numpy()
    lp, mp = 65536, 128
    D = Dg[: nd * lp * mp].reshape(nd, lp, mp).astype(np.int64)
    q = D[0] * 128 + D[1] if nd == 2 else (D[0] * 128 + D[1]) * 128 + D[2]
    sh = dec.buffer("SCALE", torch.int32).cpu().numpy()[:128]
    qs = dec.buffer("QSUM", torch.int64).cpu().numpy()
    qe = dec.buffer("QERR", torch.float64).cpu().numpy()
    j = 3
    print("nd", nd, "shift", sh[j], "S lib", qs[j], "S digits", q[:, j].sum(), "Sq2 lib", qs[128 + j], "Sq2 digits", (q[:, j] ** 2).sum(), "qerr", qe[j])
    y = (Xn[:, j] + 2.39048615) * 2.0 ** sh[j]
    print("  q[17,3]", q[17, j], "y", y[17])
    c = ((q[:, j] - q[:, j].mean()) ** 2).sum()
    print("  centred sum q^2 (x units)", c * 2.0 ** (-2 * sh[j]), "- qerr", (c - qe[j]) * 2.0 ** (-2 * sh[j]), "true", ((Xn[:, j] - Xn[:, j].mean()) ** 2).sum())
    dec.close()
