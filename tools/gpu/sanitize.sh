#!/bin/bash
# compute-sanitizer memcheck / synccheck / racecheck of the c1 smoke pass and a ragged shape
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
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 python /tmp/san_case.py > gpurun_out/san_$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/san_$tool.txt
done
