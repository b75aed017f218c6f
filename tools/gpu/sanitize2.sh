#!/bin/bash
mkdir -p gpurun_out
cat > /tmp/san_case.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_2603_10444_b200 import Decomposer
from synth.gen import SynthSpec, generate
for (l, m) in [(512, 256), (777, 130), (3000, 300)]:
    X = generate(SynthSpec(l, m, seed=1)).cuda()
    d = Decomposer(l, m)
    r = d(X)
    torch.cuda.synchronize()
    print(l, m, "sigma", r.sigma[:2].tolist(), "top", r.n_top_global)
    d.close()
PY
AVD_EIG_NOGRAPH=1 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python /tmp/san_case.py > gpurun_out/san_memcheck_nograph.txt 2>&1; echo "exit=$?" >> gpurun_out/san_memcheck_nograph.txt
AVD_EIG_NOGRAPH=1 timeout 900 compute-sanitizer --tool synccheck --error-exitcode 99 --print-limit 20 python /tmp/san_case.py > gpurun_out/san_synccheck_nograph.txt 2>&1; echo "exit=$?" >> gpurun_out/san_synccheck_nograph.txt
compute-sanitizer --version > gpurun_out/san_version.txt 2>&1
