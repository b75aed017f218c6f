import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from synth.gen import SynthSpec, generate
from paper_2603_10444_b200 import Decomposer
from paper_2603_10444_b200 import _lib as L
X = generate(SynthSpec(65536, 128, seed=13, f_mean=0.8))
X[17, 3] = 5000.0
Xc = X.numpy().astype(np.float64); mu = Xc.mean(0); Xc -= mu
print("x[14:20,3] - mu", Xc[14:20, 3], "sum xc3^2", (Xc[:, 3]**2).sum(), flush=True)
dec = Decomposer(65536, 128, flags=L.AVD_FLAG_GRAM_FREE)
r = dec(X.cuda()); torch.cuda.synchronize()
p = dec.plan.p
In = np.zeros((128, p)); In[3, 0] = 1.0
Y = torch.zeros(128, p, dtype=torch.float64, device="cuda")
Ind = torch.from_numpy(In).cuda()
os.environ["AVD_GF_DUMP"] = "gpurun_out/gfdump.bin"
L.avd_gram_product(dec.h, Ind.data_ptr(), Y.data_ptr())
print("Y33", Y[3, 0].item(), "exact", (Xc[:, 3]**2).sum(), flush=True)
