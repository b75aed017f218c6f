#!/usr/bin/env python
"""Cache the fp64 CPU oracle's outputs at the bench-scale configurations (c4, c5) so the GPU
parity tests can assert them at full size (tests/test_gpu_fullsize.py).  Calls ONLY oracle/
(and synth/ for the seeded input); nothing here touches the CUDA path.

    python tools/oracle_cache.py c4 [--eig jacobi|lapack]     (c4: ~6 min on 8 cores, jacobi)
    python tools/oracle_cache.py c5 --eig lapack              (c5: ~25 min, 36 GB of host RAM)

Writes tests/golden/oracle_<cfg>.npz: mu, sigma, sigma_next, lam (first k+8), V_k (fp32), the
energy / cross / column-mean / aggregate scalars, |E_top|, the SHA-256 of E_top (int64 little
endian, ascending), and rho at 4096 seeded positions of E_top (their linear indices included).
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from synth.fast import generate_np  # noqa: E402
from synth.gen import config_spec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c2", "c4", "c5"])
    ap.add_argument("--eig", default="jacobi", choices=["jacobi", "lapack"])
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    spec = config_spec(args.config, args.seed)
    t0 = time.time()
    X = generate_np(spec)  # bit-identical to synth.gen.generate (pinned)
    t_gen = time.time() - t0
    t0 = time.time()
    r = O.decompose(X, eig=args.eig)
    t_run = time.time() - t0
    top = r["top_idx"]
    rng = np.random.default_rng(1234)
    pick = np.sort(rng.choice(len(top), size=min(4096, len(top)), replace=False))
    out = dict(
        mu=r["mu"], sigma=r["sigma"], sigma_next=r["sigma_next"], lam=r["lam"][:r["k"] + 8],
        V=r["V"].astype(np.float32), energy_cf=r["energy_cf"], energy_el=r["energy_el"],
        cross_el=r["cross_el"], colmean_absmax=r["colmean_absmax"],
        rho_mean_aggr=r["rho_mean_aggr"], rho_energy_aggr=r["rho_energy_aggr"],
        trace_g=r["trace_g"], n_top=r["n_top"], k=r["k"],
        top_sha256=hashlib.sha256(np.ascontiguousarray(top, "<i8").tobytes()).hexdigest(),
        sample_pos=pick, sample_idx=top[pick], sample_rho=r["rho"][pick],
        meta=json.dumps({"config": args.config, "seed": args.seed, "l": spec.l, "m": spec.m,
                         "eig": args.eig, "sweeps": r["sweeps"], "cores": O.host_cores(),
                         "seconds_generate": t_gen, "seconds_oracle": t_run,
                         "cmd": "python tools/oracle_cache.py " + " ".join(sys.argv[1:])}),
    )
    path = os.path.join(ROOT, "tests", "golden", f"oracle_{args.config}.npz")
    np.savez_compressed(path, **out)
    print(json.loads(str(out["meta"])), "->", path, flush=True)


if __name__ == "__main__":
    main()
