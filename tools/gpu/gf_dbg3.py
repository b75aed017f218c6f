import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np, torch
from synth.gen import SynthSpec, generate
from paper_2603_10444_b200 import Decomposer
from paper_2603_10444_b200 import _lib as L
X = generate(SynthSpec(65536, 128, seed=13, f_mean=0.8))
X[17, 3] = 5000.0
Xc = X.numpy().astype(np.float64); Xc -= Xc.mean(0)
G = Xc.T @ Xc
for fl in (0, L.AVD_FLAG_GRAM_FREE):
    dec = Decomposer(65536, 128, flags=fl)
    r = dec(X.cuda()); torch.cuda.synchronize()
    p = dec.plan.p
    In = np.random.default_rng(1).standard_normal((128, p)); In[:, 0] = 0; In[3, 0] = 1.0
    In[:, 1] = 0; In[5, 1] = 1.0
    Y = torch.zeros(128, p, dtype=torch.float64, device="cuda")
    Ind = torch.from_numpy(In).cuda()
    L.avd_gram_product(dec.h, Ind.data_ptr(), Y.data_ptr())
    Yg = Y.cpu().numpy(); ref = G @ In
    print("gf" if fl else "gram", "digits", r.digits_used, "sigma", r.sigma.cpu().numpy())
    print("  col0 (e_3): G33 ref", ref[3, 0], "gpu", Yg[3, 0], "diff", Yg[3, 0] - ref[3, 0], " max|diff| col0", np.max(np.abs(Yg[:, 0] - ref[:, 0])))
    print("  col1 (e_5): max|diff|", np.max(np.abs(Yg[:, 1] - ref[:, 1])), "G55", ref[5, 1], Yg[5, 1])
    print("  rest: max rel", np.max(np.abs(Yg[:, 2:] - ref[:, 2:])) / np.max(np.abs(ref[:, 2:])))
    dec.close()
