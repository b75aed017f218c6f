import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2603_10444_b200 import Decomposer, _lib as L
from paper_2603_10444_b200.api import _view
from synth.gen import SynthSpec, generate
l, m = 512, 256
X = generate(SynthSpec(l, m, seed=0)).cuda()
d = Decomposer(l, m)
r = d(X); torch.cuda.synchronize()
def buf(i, dt):
    ptr, nb = L.avd_buffer(d.h, i)
    return _view(ptr, nb, dt, d.device).cpu().numpy()
Pd = buf(30, torch.int8).reshape(3, -1, 128); ps = buf(31, torch.float32)
Vd = buf(32, torch.int8).reshape(3, -1, 128); vs = buf(33, torch.float32)
P = buf(18, torch.float32).reshape(l, -1)
V = r.V.cpu().numpy()
k = d.k
zp = Pd[0].astype(np.int64) * 16384 + Pd[1].astype(np.int64) * 128 + Pd[2]
zv = Vd[0].astype(np.int64) * 16384 + Vd[1].astype(np.int64) * 128 + Vd[2]
print("k", k, "P[:2,:k]", P[:2, :k], "ps", ps[:2], "zp", zp[:2, :4])
print("recon P", (zp[:2, :k] * ps[:2, None]))
print("V", V[:2], "vs", vs[:2], "zv", zv[:2, :4], "recon", zv[:2, :k] * vs[:2, None])
print("energy_el", r.energy_el, "cf", r.energy_cf)
