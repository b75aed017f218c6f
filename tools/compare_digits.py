"""Compare the Gram operand precision (digits=2: 14-bit, digits=3: 21-bit dithered fixed point)
on the c4 workload: sigma, energy shares, rho and the top set (GPU vs GPU; nd=3 is ~2^-21 exact)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_10444_b200 import Decomposer  # noqa: E402
from synth.gen import config_spec, generate  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
spec = config_spec(name)
X = generate(spec, device="cuda")
res = {}
for nd in (3, 2):
    dec = Decomposer(spec.l, spec.m, digits=nd)
    r = dec(X)
    torch.cuda.synchronize()
    res[nd] = dict(sigma=r.sigma.cpu().numpy().copy(), shares=np.array(r.shares_cf), rho=r.rho.cpu().numpy().copy(),
                   idx=r.top_idx.cpu().numpy().copy(), el=np.array(r.energy_el), cf=np.array(r.energy_cf),
                   V=r.V.cpu().numpy().copy())
    dec.close()
a, b = res[3], res[2]
out = {
    "config": name,
    "sigma_max_rel_diff": float(np.max(np.abs(a["sigma"] - b["sigma"]) / a["sigma"])),
    "shares_max_rel_diff": float(np.max(np.abs(a["shares"] - b["shares"]) / a["shares"])),
    "rho_max_abs_diff": float(np.max(np.abs(a["rho"] - b["rho"]))),
    "top_set_equal": bool(np.array_equal(a["idx"], b["idx"])),
    "V_min_abs_cos": float(np.min(np.abs(np.sum(a["V"] * b["V"], axis=0)))),
    "nd3_el_vs_cf_rel": (np.abs(a["el"] - a["cf"]) / a["cf"][0]).tolist(),
    "nd2_el_vs_cf_rel": (np.abs(b["el"] - b["cf"]) / b["cf"][0]).tolist(),
    "shares_nd3": a["shares"].tolist(),
}
print(json.dumps(out))
