"""Gram-free vs Gram path at fixed 2 digits: precision bounds and errors against the oracle."""
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np, torch
from oracle import oracle as O
from synth.gen import SynthSpec, generate
from paper_2603_10444_b200 import _lib as L
from test_gpu_parity import _gpu
for (l, m, k) in [(512, 256, None), (3000, 300, None), (2048, 512, 81)]:
    X = generate(SynthSpec(l, m, seed=1, f_mean=0.8, **({"k_s": k} if k else {})))
    o = O.decompose(X.numpy(), k=k)
    for fl in (0, L.AVD_FLAG_GRAM_FREE):
        for d in (2, 0):
            g = _gpu(X, flags=fl, digits=d, **({"k": k} if k else {}))
            r = g["res"]
            s_g = np.array(r.energy_cf[1:]) / r.energy_cf[0]; s_o = np.array(o["energy_cf"][1:]) / o["energy_cf"][0]
            print(f"l={l} m={m} k={k} gf={fl!=0} digits={d}->{r.digits_used}: iters {r.iters} resid {r.max_resid:.2e} "
                  f"prec_sigma {r.precision_sigma:.2e} prec_share {r.precision_share:.2e} "
                  f"sigma_err {np.max(np.abs(g['sigma']-o['sigma'])/o['sigma']):.2e} share_err {np.max(np.abs(s_g-s_o)):.2e} "
                  f"trace {r.trace_g:.6e} E_tot {r.energy_cf[0]:.6e}", flush=True)
