import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
from oracle import oracle as O
from synth.gen import SynthSpec, generate
from paper_2603_10444_b200 import _lib as L
from test_gpu_parity import _gpu
X = generate(SynthSpec(65536, 128, seed=13, f_mean=0.8))
X[17, 3] = 5000.0
o = O.decompose(X.numpy())
print("oracle sigma", o["sigma"], "shares", np.array(o["energy_cf"][1:]) / o["energy_cf"][0], flush=True)
for fl in (0, L.AVD_FLAG_GRAM_FREE):
    for d in (0, 3):
        g = _gpu(X, flags=fl, digits=d)
        r = g["res"]
        s_g = np.array(r.energy_cf[1:]) / r.energy_cf[0]; s_o = np.array(o["energy_cf"][1:]) / o["energy_cf"][0]
        print(f"gf={fl!=0} digits={d}->{r.digits_used} req={r.requantised}: sigma {g['sigma']} prec {r.precision_sigma:.2e} {r.precision_share:.2e} "
              f"sigma_err {np.max(np.abs(g['sigma']-o['sigma'])/o['sigma']):.2e} share_err {np.max(np.abs(s_g-s_o)):.2e} "
              f"trace {r.trace_g:.9e} oracle trace {o.get('trace_g', float('nan'))}", flush=True)
