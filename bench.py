#!/usr/bin/env python
"""Benchmark of the activation outlier-attribution pass (arXiv 2603.10444).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One step = the whole hot path (stats+histogram, centre+digits,
Gram, eigensolve, projections+energies, exact top set, rho gather) over one synthetic matrix
(synth/gen.py; default c4 = 131072 x 4096, k = 40, |E_top| = 536870; BASELINE.json configs[3],
the configuration the metric is quoted on at 1/2/4/8 B200).  X (2.1 GB) is larger than L2, so no
flush is needed between steps.  N > 1: torchrun, one process per GPU, rows sharded in rank
order, NCCL all-reduces of the exchange buffers (strong scaling of one matrix); time is the max
over ranks.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth.gen import config_spec, generate, sweep_specs  # noqa: E402

METRIC = "activation entries decomposed/sec (l*m/s)"
UNIT = "entries/s"
WORKLOADS = {
    "c1": "c1: single matrix l=512, m=256 (k=2, |E_top|=131)",
    "c2": "c2: single layer l=8192, m=2048 (k=20)",
    "c3": "c3: 29-module sweep (embedding + 28 layers) x early/late mean-bias strength = 58 matrices "
          "of l=32768, m=2048 (k=20)",
    "c4": "c4: single matrix l=131072, m=4096 (k=40), row-sharded over the GPUs",
    "c5": "c5: single matrix l=1048576, m=8192 (k=81), row-sharded over the GPUs",
    "averis": "f3: Averis mean-residual NVFP4 forward GeMM, X l=131072 x m=4096 (the c4 activations) "
              "times W m=4096 x n=4096 (PAPER.md:391-429)",
}
AVERIS_SHAPE = (131072, 4096, 4096)
AVERIS_METRIC = "Averis NVFP4 forward GeMM throughput (2*l*m*n flop/s, mean split + quantisation inside)"


def _traffic(key):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(key)
    except OSError:
        return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thr = threading.Thread(target=self._read, daemon=True)
            self.thr.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ timed stage wrapper
class TimedBackend:
    """Wraps the library stage backend and records CUDA events around every stage (on the
    stream the library launches on, which is torch's current stream)."""

    STAGES = ["stage_stats", "stage_split", "stage_gram", "stage_eig", "stage_project",
              "stage_select", "stage_gather", "stage_report"]

    def __init__(self, inner):
        self.inner = inner
        self.events = []  # (name, start, end)
        self.record = False

    def exchange_buffer(self, name, dtype):
        return self.inner.exchange_buffer(name, dtype)

    def __getattr__(self, name):
        fn = getattr(self.inner, name)
        if name not in self.STAGES:
            return fn

        def wrapped(*a, **k):
            if not self.record:
                return fn(*a, **k)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            r = fn(*a, **k)
            e.record()
            self.events.append((name, s, e))
            return r
        return wrapped

    def stage_ms(self, steps):
        torch.cuda.synchronize()
        acc = {}
        for name, s, e in self.events:
            acc[name] = acc.get(name, 0.0) + s.elapsed_time(e)
        return {k.replace("stage_", ""): v / steps for k, v in acc.items()}


class LocalComm:
    rank, world = 0, 1

    def all_reduce(self, t, op):  # pragma: no cover - world 1 never exchanges
        pass


# ------------------------------------------------------------------ CPU baseline (the oracle)
def cpu_baseline(spec, rows: int, eig: str):
    """The fp64 oracle as it stands on rows [0, rows) x ALL m columns of the bench matrix (the
    Gram, the eigen step and the column work keep the workload's width; only l is sampled).
    eig='lapack': the oracle's LAPACK eigen step (numpy eigh, a library primitive); 'jacobi':
    its parallel round-robin Jacobi (O(m^3) per sweep, minutes at m = 4096).  rows = l: the whole
    matrix (c4: ~11 min on 8 cores)."""
    from oracle import oracle as O
    O.build()
    Xs = generate(spec, 0, rows).numpy()
    t0 = time.perf_counter()
    O.decompose(Xs, eig=eig)
    dt = time.perf_counter() - t0
    what = "the whole matrix" if rows == spec.l else f"rows [0,{rows}) x all {spec.m} columns"
    return {"value": rows * spec.m / dt, "unit": UNIT, "cores": O.host_cores(), "kind": "oracle",
            "sample": f"{what} of the {spec.l}x{spec.m} matrix (full oracle pass: two-pass mean, "
                      f"row-blocked fp64 Gram of Xc, {eig} eigen step, top set, spike/tail, rho); "
                      f"{dt:.2f} s", "seconds": dt}


def averis_cpu_baseline(rows: int):
    """oracle/averis.py as it stands (numpy: fp32 quantiser decisions, fp64 GeMM) on rows
    [0, rows) of the bench X with the full W."""
    from oracle import averis as A
    from oracle import oracle as O
    from synth.gen import generate_weight
    l, m, n = AVERIS_SHAPE
    Xs = generate(config_spec("c4"), 0, rows).numpy()
    W = generate_weight(m, n, seed=0).numpy()
    t0 = time.perf_counter()
    A.averis_forward(Xs, W)
    dt = time.perf_counter() - t0
    return {"value": 2.0 * rows * m * n / dt / 1e12, "unit": "TFLOP/s", "cores": O.host_cores(), "kind": "oracle",
            "sample": f"rows [0,{rows}) of X x the full {m}x{n} W (quantise W, mu of the sample, X_R, fp64 "
                      f"GeMM); {dt:.2f} s", "seconds": dt}


def run_reference(args):
    """--impl reference: the fp64 CPU oracle as it stands, on a bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.config == "averis":
        for _ in range(args.warmup):
            averis_cpu_baseline(256)
        cb = [averis_cpu_baseline(512) for _ in range(args.steps)]
        v = statistics.median(c["value"] for c in cb)
        line = {"impl": "reference", "metric": AVERIS_METRIC, "value": v, "unit": "TFLOP/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": statistics.median(c["seconds"] for c in cb) * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOADS["averis"], "sample_rows": 512},
                "cpu_baseline": {k: cb[0][k] for k in ("unit", "cores", "kind", "sample")} | {"value": v},
                "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "gpu_launches": 0}
        print(json.dumps(line), flush=True)
        return
    from oracle import oracle as O
    O.build()
    spec = config_spec(args.config)
    rows, cols = 2048, 256
    Xs = generate(spec, 0, rows)[:, :cols].contiguous().numpy()
    for _ in range(args.warmup):
        O.decompose(Xs)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.decompose(Xs)
    dt = (time.perf_counter() - t0) / args.steps
    v = rows * cols / dt
    sample = (f"rows [0,{rows}) x cols [0,{cols}) of the {args.config} matrix per step "
              f"(oracle: fp64 two-pass mean, Gram, cyclic Jacobi, full sort, rho)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOADS.get(args.config, args.config),
                                            "sample_rows": rows, "sample_cols": cols},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": O.host_cores(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# massive activations of ONE token in two hidden dimensions (the attention-sink pattern of
# PAPER.md:245-246): row 17 is not in the 1/16 row sample, so the sampled quantiser range misses it
MASSIVE = ((17, 3, 5000.0), (17, 1027, -3000.0))


def plant_massive(X, row0, m):
    for i, j, v in MASSIVE:
        if row0 <= i < row0 + X.shape[0] and j < m:
            X[i - row0, j] = v


# ------------------------------------------------------------------ c3: the 58-matrix sweep
def run_c3(args, rank, world, local):
    """BASELINE.json configs[2]: one step = the whole pass over each of the 58 matrices of the
    sweep (synth.gen.sweep_specs).  Four contexts on four CUDA streams, each
    driven by its own host thread (the C calls release the GIL), so other matrices' fused passes /
    Grams run while one is in its latency-bound eigensolve (2 streams: 60.3 ms per sweep, 3: 50.0,
    4: 44.6, 6: 44.2).  N > 1: the matrices are dealt round-robin to
    the ranks (independent problems, no collective)."""
    import torch.distributed as dist
    from concurrent.futures import ThreadPoolExecutor
    from paper_2603_10444_b200.api import Decomposer
    specs = sweep_specs(0)
    mine = [i for i in range(len(specs)) if i % world == rank]
    l, m = specs[0].l, specs[0].m
    Xs = [generate(specs[i], device="cuda") for i in mine]
    torch.cuda.synchronize()
    NW = args.c3_streams
    streams = [torch.cuda.Stream() for _ in range(NW)]
    decs = [Decomposer(l, m, seed=0, stream=st) for st in streams]

    def worker(w, mats, host=None):
        out = []
        with torch.cuda.stream(streams[w]):
            for j in range(w, len(mats), NW):
                out.append(decs[w](mats[j]) if host is None else decs[w].run_host(host[j]))
        return out

    pool = ThreadPoolExecutor(NW)

    def step(mats, host=None):
        fut = [pool.submit(worker, w, mats, host) for w in range(NW)]
        return [r for f in fut for r in f.result()]

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        res = step(Xs)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.15)
    l0 = sum(d.launches() for d in decs)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(streams[0])
    for st in streams[1:]:
        st.wait_event(ev0)
    for _ in range(args.steps):
        res = step(Xs)
    for st in streams[1:]:
        ev_b = torch.cuda.Event()
        ev_b.record(st)
        streams[0].wait_event(ev_b)
    ev1.record(streams[0])
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = sum(d.launches() for d in decs) - l0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    n_all = len(specs)
    entries = n_all * l * m
    bad = [f"matrix {mine[i]}: status {r.status}, residual {r.max_resid}" for i, r in enumerate(res)
           if r.status != 0 or not (r.max_resid <= 1e-6)]
    # e2e: host buffers through avd_decompose_host (H2D of X and D2H of the results inside), on
    # the first 8 of this rank's matrices, both threads
    ne = min(8, len(Xs))
    Xh = [x.cpu().pin_memory() for x in Xs[:ne]]
    step(Xs[:ne], Xh)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(max(1, args.e2e_steps)):
        step(Xs[:ne], Xh)
    torch.cuda.synchronize()
    e_ms = (time.perf_counter() - t0) * 1e3 / max(1, args.e2e_steps)
    k = decs[0].k
    d2h = ne * (8 * (m + m * k + k) + 40 * decs[0].n_top)
    line = {
        "metric": METRIC, "value": entries / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "i8/i32 Gram + f64 eig + i8/f32 projection", "data":
            "synthetic (synth/gen.py sweep_specs: 29 modules x early/late, invented monotone schedule)",
        "matrices_per_s": n_all / (ms_step * 1e-3),
        "config": {"workload": WORKLOADS["c3"], "matrices": n_all, "l": l, "m": m, "k": k,
                   "streams": NW, "l2": "each matrix (268 MB) is larger than L2; no flush",
                   "parallelism": f"matrices dealt round-robin to {world} rank(s)"},
        "clocks": clocks, "gpu_launches": int(launches),
        "e2e": {"value": ne * l * m / (e_ms * 1e-3), "unit": UNIT, "matrices_per_s": ne / (e_ms * 1e-3),
                "h2d_bytes_per_step": ne * l * m * 4, "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms,
                "sample": f"the first {ne} matrices of this rank, pinned host buffers"},
        "eig_iters": [r.iters for r in res[:4]], "digits_used": sorted({r.digits_used for r in res}),
    }
    if bad:
        line["invalid"] = "; ".join(bad[:4])
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(specs[0], min(l, 8192), args.cpu_baseline_eig)
    if rank == 0:
        print(json.dumps(line), flush=True)
    for d in decs:
        d.close()
    pool.shutdown()
    if world > 1:
        dist.destroy_process_group()
    if bad:
        print("bench: INVALID run: " + "; ".join(bad[:4]), file=sys.stderr)
        sys.exit(3)


# ------------------------------------------------------------------ f3: Averis NVFP4 GeMM
def run_averis(args, rank, world, local):
    """one step = avd_averis_forward on the c4 activations X (131072 x 4096) with a
    4096 x 4096 weight: column statistics, mu_bar and mu_bar W_bar, NVFP4 quantisation of X_R, the
    block-scaled tcgen05 GeMM and its epilogue (W quantised once, outside the step, as a weight
    is between optimizer updates).  N > 1: replicas only — every rank runs its own micro-batch
    (the split's mean is per micro-batch, the GeMM is local to the data-parallel rank)."""
    import torch.distributed as dist
    from paper_2603_10444_b200.averis import AverisGemm
    from synth.gen import generate_weight
    l, m, n = AVERIS_SHAPE
    X = generate(config_spec("c4"), device="cuda")
    W = generate_weight(m, n, seed=0, device="cuda")
    bf = args.variant == "bf16"
    Y = torch.empty(l, n, dtype=torch.bfloat16 if bf else torch.float32, device="cuda")
    g = AverisGemm(l, m, n, timing=True, bf16_out=bf)
    g.set_weight(W)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        g(X, Y)
    torch.cuda.synchronize()
    # per-stage times (events inside the library, on its stream), one synchronised step at a time
    st = []
    for _ in range(max(3, args.steps // 2)):
        g(X, Y)
        st.append(g.stage_ms())
    stage = [statistics.median(s[i] for s in st) for i in range(3)]
    barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.15)
    l0 = g.launches()
    t_s, t_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_s.record()
    for _ in range(args.steps):
        g(X, Y)
    t_e.record()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = g.launches() - l0
    ms = t_s.elapsed_time(t_e)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    flops = 2.0 * l * m * n
    value = world * flops / (ms_step * 1e-3) / 1e12
    e2e = None
    if not args.no_e2e:
        Xh = X.cpu().pin_memory()
        Yh = torch.empty(l, n, dtype=Y.dtype).pin_memory()
        g.forward_host(Xh, Yh)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            g.forward_host(Xh, Yh)
        e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        e2e = {"value": world * flops / (e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": l * m * 4,
               "d2h_bytes_per_step": l * n * Y.element_size(), "ms_per_step": e_ms}
    peaks, which = _peaks()
    fp4_peak = 4.0 * peaks.get("bf16_tflops")
    t_gemm = stage[2] * 1e-3
    hbm = peaks.get("hbm_gbs", 6650.0)
    line = {
        "metric": AVERIS_METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "nvfp4 (e2m1 + ue4m3/16) x nvfp4 -> " + ("bf16" if bf else "f32"),
        "data": "synthetic (X: synth/gen.py c4 seed 0, mean-biased with massive columns; W: generate_weight seed 0)",
        "config": {"workload": WORKLOADS["averis"], "l": l, "m": m, "n": n, "rounding": "nearest",
                   "l2": "X (2.1 GB) and Y (2.1 GB) larger than L2; no flush", "parallelism": f"replicas x{world}"},
        "clocks": clocks, "e2e": e2e, "gpu_launches": int(launches),
        "stage_ms": {"stats+mu_bar+bias": stage[0], "quantise X_R": stage[1], "gemm": stage[2]},
        "roofline": {"bound": "tensor", "kernel": "av_gemm_kernel (tcgen05.mma.cta_group::2 kind::mxf4nvf4 block16)",
                     "achieved": flops / t_gemm / 1e12, "peak": fp4_peak, "unit": "TFLOP/s",
                     "frac": flops / t_gemm / 1e12 / fp4_peak, "traffic": _traffic("averis_gemm"),
                     "traffic_note": "ncu dram bytes of one launch (fp32 Y): X_R codes + W codes read, Y (2.15 GB) written",
                     "peak_source": f"{which}: 4 x bf16_tflops (burst; fp4 dense = 4x bf16 nominal)",
                     "algorithmic_flops_per_launch": flops, "launch_ms": stage[2]},
        "streaming_roofline": {
            "column stats (read X 4 B/entry)": {"alg_GB/s": l * m * 4 / (stage[0] * 1e-3) / 1e9,
                                                "frac_hbm": l * m * 4 / (stage[0] * 1e-3) / 1e9 / hbm},
            "quantise X_R (read 4 B, write 0.5625 B/entry)": {
                "alg_GB/s": l * m * 4.5625 / (stage[1] * 1e-3) / 1e9,
                "frac_hbm": l * m * 4.5625 / (stage[1] * 1e-3) / 1e9 / hbm}},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = averis_cpu_baseline(1024)
    if rank == 0:
        print(json.dumps(line), flush=True)
    g.close()
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--digits", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-baseline-rows", type=int, default=0,
                    help="rows of the oracle sample (0: 8192 for c4/c5, all rows below; -1: all rows)")
    ap.add_argument("--cpu-baseline-eig", default="lapack", choices=["lapack", "jacobi"])
    ap.add_argument("--variant", default="base", choices=["base", "massive", "gramfree", "bf16"],
                    help="massive: plant single-token massive activations (PAPER.md:245-246) in an "
                         "unsampled row, which forces the exact-range requantisation and exercises "
                         "the automatic digit escalation inside the timed region; gramfree: the "
                         "Gram-free eigensolve (AVD_FLAG_GRAM_FREE, SURVEY 8(f4)); bf16 (--config averis): "
                         "Y in bf16")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (huge configs)")
    ap.add_argument("--c3-streams", type=int, default=4, help="c3: contexts / streams / host threads in flight")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.config == "c3":
        run_c3(args, rank, world, local)
        return
    if args.config == "averis":
        run_averis(args, rank, world, local)
        return
    from paper_2603_10444_b200.distributed import ShardedDecomposer, TorchComm, _LibBackend, run_stages, shard_rows
    from paper_2603_10444_b200.api import Decomposer

    spec = config_spec(args.config)
    l, m = spec.l, spec.m
    r0, lloc = shard_rows(l, world, rank)
    X = generate(spec, r0, lloc, device="cuda")
    if args.variant == "massive":
        plant_massive(X, r0, m)
    torch.cuda.synchronize()

    flags = 0
    if args.variant == "gramfree":
        from paper_2603_10444_b200._lib import AVD_FLAG_GRAM_FREE
        flags = AVD_FLAG_GRAM_FREE
    if world == 1:
        dec = Decomposer(l, m, digits=args.digits, seed=0, flags=flags)
        comm = LocalComm()
    else:
        sd = ShardedDecomposer(l, m, digits=args.digits, seed=0)
        dec, comm = sd.dec, sd.comm
    backend = TimedBackend(_LibBackend(dec))

    def step():
        return run_stages(backend, comm, X)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.15)
    launches0 = dec.launches()
    backend.record = True
    t_s, t_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_s.record()
    for _ in range(args.steps):
        res = step()
    t_e.record()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    backend.record = False
    launches = dec.launches() - launches0
    clocks = sampler.stop()
    ms = t_s.elapsed_time(t_e)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    stage_ms = backend.stage_ms(args.steps)
    ms_step = ms / args.steps
    value = l * m / (ms_step * 1e-3)

    # ---------------- e2e: host buffers through the public API, copies inside the timed region
    e2e = None
    n_loc = int(res.top_idx.numel())
    d2h = 8 * (m + m * dec.k + dec.k) + 8 * n_loc + 32 * n_loc
    Xh = None if args.no_e2e else X.cpu().pin_memory()
    if args.no_e2e:
        e_ms = float("nan")
    elif world == 1:
        for _ in range(1):
            dec.run_host(Xh)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            dec.run_host(Xh)
        torch.cuda.synchronize()
        e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
    else:
        Xd = torch.empty_like(X)
        outs = None

        def e2e_step():
            Xd.copy_(Xh, non_blocking=True)
            r = run_stages(_LibBackend(dec), comm, Xd)
            return [t.cpu() for t in (r.mu, r.V, r.sigma, r.top_idx, r.rho)]
        outs = e2e_step()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            outs = e2e_step()
        torch.cuda.synchronize()
        barrier()
        e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        t = torch.tensor([e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
        del outs
    e2e = None if args.no_e2e else {"value": l * m / (e_ms * 1e-3), "unit": UNIT,
                                    "h2d_bytes_per_step": int(lloc * m * 4),
                                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms}

    # ---------------- roofline of the dominant kernel (the tcgen05 Gram, stage "gram")
    peaks, which = _peaks()
    nd = dec.plan.digits
    t_gram = stage_ms.get("gram", float("nan")) * 1e-3
    alg_ops = lloc * m * (m + 1)                       # symmetric Gram, SURVEY §8(d) K3
    T = (m + 127) // 128
    lpad = (lloc + 127) // 128 * 128
    exec_ops = (4 if nd == 2 else 6) * 2 * lpad * 128 * 128 * (T * (T + 1) // 2)
    # the Gram runs ~3 ms inside a ~8 ms step: the BURST peak is the denominator (the guide's
    # nominal int8 = 2 x bf16 ratio applied to the measured bf16 burst figure)
    int8_peak = 2.0 * peaks.get("bf16_tflops")
    int8_sus = 2.0 * peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    achieved = alg_ops / t_gram / 1e12
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get(f"{args.config}_gram_nd{nd}")
        traffic_src = tj.get("_source")
    except OSError:
        pass
    roofline = {"bound": "tensor", "kernel": "gram2_kernel (K3, tcgen05.mma.cta_group::2 kind::i8)",
                "achieved": achieved, "peak": int8_peak, "unit": "TFLOP/s",
                "frac": achieved / int8_peak, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": f"{which}: 2 x bf16_tflops (burst; int8 dense = 2x bf16 nominal)",
                "frac_vs_sustained": achieved / int8_sus,
                "algorithmic_ops_per_launch": alg_ops, "executed_int8_ops_per_launch": exec_ops,
                "executed_frac": exec_ops / t_gram / 1e12 / int8_peak,
                "launch_ms": t_gram * 1e3}
    hbm = peaks.get("hbm_gbs", 6650.0)
    samp = max(1, min(16, l // 4096))
    samp = 1 << (samp.bit_length() - 1)
    # (algorithmic bytes per SURVEY §8(d), executed bytes, stage ms); stage times include the
    # stage's small helper kernels
    streams = {
        "row sample (K1s, 1/%d of the rows)" % samp: (lloc * m * 4 // samp, lloc * m * 4 // samp, stage_ms.get("stats")),
        "fused pass (K1+K2: read X 4 B; writes nd digit bytes)": (lloc * m * 4, lloc * m * (4 + nd), stage_ms.get("split")),
        # K5 reads the nd digit planes of the Gram operand, K8 reads X
        "project+energy (K5/K8: two passes over X; K5 reads the digit planes)": (2 * lloc * m * 4, lloc * m * (nd + 4),
                                                                               stage_ms.get("project")),
    }
    stream_roof = {k: {"alg_GB/s": a / (t * 1e-3) / 1e9, "frac_hbm": a / (t * 1e-3) / 1e9 / hbm,
                       "exec_GB/s": b / (t * 1e-3) / 1e9, "exec_frac_hbm": b / (t * 1e-3) / 1e9 / hbm}
                   for k, (a, b, t) in streams.items() if t}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "i8/i32 Gram + f64 eig + f32 projection",
        "data": "synthetic (planted mean bias + rank-k Walsh spike + Irwin-Hall tail, synth/gen.py seed 0)",
        "config": {"workload": WORKLOADS[args.config], "l": l, "m": m, "k": dec.k,
                   "n_top": dec.n_top, "digits": nd, "l2": "inputs larger than L2 (X is "
                   f"{l * m * 4 / 1e9:.2f} GB > 126 MB); no flush",
                   "parallelism": f"row-shard x{world}"},
        "clocks": clocks, "e2e": e2e, "gpu_launches": int(launches),
        "roofline": roofline if args.variant != "gramfree" else None, "stage_ms": stage_ms, "streaming_roofline": stream_roof,
        "eig_iters": res.iters, "eig_max_resid": res.max_resid, "eig_rr_checks": res.rr_checks,
        "eig_jacobi_sweeps": res.jacobi_sweeps, "eig_status": res.status,
        "requantised": res.requantised, "digits_used": res.digits_used,
        "precision_bound": {"sigma": res.precision_sigma, "share": res.precision_share},
        "mean_diagnostics": {"R": res.mean_R, "sign_fraction": res.sign_fraction, "cos_mu_v1": res.cos_mu_v1,
                             "alpha1": res.alpha1, "sigma1_uncentred": res.sigma1_u, "power_iters": res.iters_u},
    }
    if args.variant != "base":
        line["config"]["variant"] = {"massive": f"single-token massive activations {list(MASSIVE)} "
                                                f"(row, col, value) in an unsampled row",
                                     "gramfree": "AVD_FLAG_GRAM_FREE: no Gram; every G Q of the eigensolve as "
                                                 "Xhat^T (Xhat Q) by two tensor-core passes (SURVEY 8(f4))"}[args.variant]
    bad = []
    if res.status != 0:
        bad.append(f"eigensolver status {res.status} (AVD_ENOCONV = 3): not converged")
    if not (res.max_resid <= 1e-6):
        bad.append(f"eigensolver residual {res.max_resid} above tol 1e-6")
    if bad:
        line["invalid"] = "; ".join(bad)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rows = args.cpu_baseline_rows
        rows = spec.l if rows < 0 else (rows or min(spec.l, 8192))
        line["cpu_baseline"] = cpu_baseline(spec, rows, args.cpu_baseline_eig)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if bad:
        print("bench: INVALID run: " + "; ".join(bad), file=sys.stderr)
        sys.exit(3)


if __name__ == "__main__":
    main()
