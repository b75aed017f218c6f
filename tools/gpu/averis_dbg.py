"""Diagnostics of the Averis path on one small case: which stage departs from the oracle."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import averis as A
from synth.gen import SynthSpec, generate, generate_weight
from paper_2603_10444_b200.averis import AverisGemm
sys.path.insert(0, "tests")
from test_gpu_averis import _unpack, _unswizzle

for (l, m, n, sr) in [(128, 256, 128, False), (300, 320, 144, False), (256, 512, 256, True)]:
    X = generate(SynthSpec(l, m, seed=0)); W = generate_weight(m, n, seed=0)
    o = A.averis_forward(X.numpy(), W.numpy(), stochastic=sr, seed=0)
    g = AverisGemm(l, m, n, stochastic=sr); g.set_weight(W.cuda()); Y = g(X.cuda()); torch.cuda.synchronize()
    gs = g.buffer("GSCALE").cpu().numpy()
    print(f"== l={l} m={m} n={n} sr={sr}: g gpu {gs} oracle {o['qx']['g']}, {o['qw']['g']}, {o['qmu']['g']}")
    for nm, gc, oc in [("W codes", _unpack(g.buffer("WCODES"), n, m), o["qw"]["codes"]),
                       ("W sf", _unswizzle(g.buffer("WSF"), n, m), o["qw"]["scale"]),
                       ("X codes", _unpack(g.buffer("XCODES"), l, m), o["qx"]["codes"]),
                       ("X sf", _unswizzle(g.buffer("XSF"), l, m), o["qx"]["scale"]),
                       ("mu codes", _unpack(g.buffer("MUCODES"), 1, m), o["qmu"]["codes"]),
                       ("mu sf", g.buffer("MUSF").cpu().numpy()[None, :], o["qmu"]["scale"])]:
        bad = np.argwhere(gc != oc)
        print(f"  {nm}: {len(bad)} mismatches of {gc.size}", "" if not len(bad) else
              f"first {bad[:4].tolist()} gpu {gc[tuple(bad[:4].T)]} ora {oc[tuple(bad[:4].T)]}")
    mu = g.buffer("MU").cpu().numpy(); print("  mu max rel", np.max(np.abs(mu - o["mu"])) / np.abs(o["mu"]).max())
    b = g.buffer("BIAS").cpu().numpy(); print("  bias max rel", np.max(np.abs(b - o["bias"]) / (np.abs(o["bias"]) + 1e-30)))
    Yg = Y.cpu().numpy().astype(np.float64); err = np.abs(Yg - o["Y"])
    rel = err / np.maximum(o["absY"], 1e-30)
    print("  Y rel err max", rel.max(), "median", np.median(rel), "Y[0,:4]", Yg[0, :4], o["Y"][0, :4])
    if rel.max() > 1e-3:
        # diagnose: ratio pattern
        Xd = A.dequantize(o["qx"]); Wd = A.dequantize(o["qw"]).T
        Yr = (Yg - o["bias"][None, :])
        print("  resid-only ratio sample", (Yr / (Xd @ Wd))[:2, :6])
        print("  per-row-block max rel", [float(rel[i:i+32].max()) for i in range(0, min(l, 128), 32)])
        print("  per-col-block max rel", [float(rel[:, j:j+32].max()) for j in range(0, min(n, 128), 32)])
    g.close()
