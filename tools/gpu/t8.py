import sys, os; sys.path.insert(0, ".")
import torch
from paper_2603_10444_b200 import Decomposer
from paper_2603_10444_b200._lib import AVD_FLAG_EIG_HOST_LOOP
from synth.gen import SynthSpec, generate
for flags in [AVD_FLAG_EIG_HOST_LOOP, 0]:
    for (l, m) in [(4096, 512), (512, 256), (4096, 2048)]:
        X = generate(SynthSpec(l, m, seed=1)).cuda()
        d = Decomposer(l, m, flags=flags)
        try:
            r = d(X); torch.cuda.synchronize()
            print(flags, l, m, "ok", r.sigma[:2].tolist(), r.iters, r.max_resid, flush=True)
        except Exception as e:
            print(flags, l, m, "ERR", e, flush=True); sys.exit(1)
        d.close()
