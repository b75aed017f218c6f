"""Seeded synthetic activation matrices X (l tokens x m hidden, fp32) — the ONLY module shared
by the oracle side (tests, bench cpu_baseline) and the CUDA side (tests, bench, smoke).

It holds none of the decomposition's arithmetic: it only draws inputs.  The draw is a pure
function of (spec, i, j) built from integer hashing and IEEE-exact fp64 ops issued as separate
torch ops (no fused multiply-add), so the same spec gives bit-identical X on CPU and on CUDA and
for any row shard (shard-invariant).

Recipe:
    x_ij = fl32( mu_j + sum_{r<k_s} c_r h(a_r,i) h(b_r,j) + sigma_t z_ij )
  * mean bias mu_j = beta sigma_t w_j, w_j = s_j (1 + 0.25 g_j), s_j = +1 w.p. 0.8 (coherent
    sign), ~0.5% "massive" columns x8; beta is set from the
    expected energies so that the mean-energy share is f_mean.
  * spike: Walsh–Hadamard rows h(a,i) = (-1)^popcount(a & i) with distinct a_r in [1,l),
    b_r in [1,m): u_r = h(a_r,.)/sqrt(l) is orthogonal to 1 (centred) and orthonormal when l, m
    are powers of two.  sigma_r = theta_r sigma_t (sqrt(l)+sqrt(m)), theta linear 8 -> 2,
    c_r = sigma_r / sqrt(l m); the planted gap sigma_{k+1}/sigma_k ~ 0.5 (tail edge ~ sqrt l + sqrt m).
  * tail z_ij: Irwin–Hall-12 (sum of 12 24-bit uniforms - 6): mean 0, variance 1, |z| <= 6.
  * exact=True: sigma_t = 0 and dyadic mu_j, c_r — X is exact in fp32 and every output of the
    pass has a closed form (the pins of tests/test_oracle_pins.py).
"""
from __future__ import annotations

import dataclasses
import math

import torch

M32 = 0xFFFFFFFF


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for x in [0, 2^32) held in int64, without int64 overflow."""
    lo = x & 0xFFFF
    hi = x >> 16
    return (lo * c + (((hi * c) & 0xFFFF) << 16)) & M32


def hash32(x: torch.Tensor) -> torch.Tensor:
    """'lowbias32' integer mixer on 32-bit values stored in int64."""
    x = x & M32
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _u24(h: torch.Tensor) -> torch.Tensor:
    return h >> 8  # top 24 bits


def _scalar_hash(*vals: int) -> int:
    h = 0x9E3779B9
    for v in vals:
        h = int(hash32(torch.tensor([(h ^ (v & M32)) & M32], dtype=torch.int64))[0])
        h = int(hash32(torch.tensor([(h ^ ((v >> 32) & M32)) & M32], dtype=torch.int64))[0])
    return h


def _parity(v: torch.Tensor) -> torch.Tensor:
    v = v ^ (v >> 32)
    v = v ^ (v >> 16)
    v = v ^ (v >> 8)
    v = v ^ (v >> 4)
    v = v ^ (v >> 2)
    v = v ^ (v >> 1)
    return v & 1


def walsh(a: int, idx: torch.Tensor) -> torch.Tensor:
    """h(a, i) = (-1)^popcount(a & i) as fp64 (+1/-1)."""
    return 1.0 - 2.0 * _parity(idx & a).to(torch.float64)


@dataclasses.dataclass(frozen=True)
class SynthSpec:
    l: int
    m: int
    seed: int = 0
    k_s: int | None = None        # planted spike rank (default k = max(1, floor(0.01 m)))
    theta_1: float = 8.0
    theta_k: float = 2.0
    sigma_t: float = 1.0
    f_mean: float = 0.9           # target mean-energy share l||mu||^2 / E_total
    coherent: float = 0.8         # P(s_j = +1)
    massive_frac: float = 0.005
    massive_mult: float = 8.0
    exact: bool = False           # sigma_t = 0, dyadic mu and c_r (closed-form pins)
    mean_scale: float = 1.0       # multiplies mu (0 => pure centred spike + tail)
    spike_scale: float = 1.0      # multiplies c_r (0 => no spike)

    @property
    def ks(self) -> int:
        return self.k_s if self.k_s is not None else max(1, int(math.floor(0.01 * self.m + 1e-9)))


def _distinct_codes(n: int, upper: int, seed: int, salt: int) -> list[int]:
    """n distinct integers in [1, upper) drawn by hashing (deterministic)."""
    out: list[int] = []
    seen = set()
    t = 0
    if upper - 1 < n:
        raise ValueError(f"cannot draw {n} distinct Walsh codes below {upper}")
    while len(out) < n:
        v = 1 + _scalar_hash(seed, salt, t) % (upper - 1)
        t += 1
        if v not in seen:
            seen.add(v)
            out.append(v)
    return out


def planted(spec: SynthSpec):
    """The planted parameters: (a_r, b_r, c_r, mu) with mu as fp64 tensor [m] (CPU)."""
    l, m, ks = spec.l, spec.m, spec.ks
    a = _distinct_codes(ks, l, spec.seed, 101)
    b = _distinct_codes(ks, m, spec.seed, 202)
    j = torch.arange(m, dtype=torch.int64)
    base = hash32(j ^ hash32(torch.full_like(j, (spec.seed * 7919 + 17) & M32)))
    if spec.exact:
        # dyadic, distinct: c_r = (ks + 1 - r)/16 ; mu_j = +-(1 + (h mod 64))/8
        c = [(ks + 1 - r) / 16.0 for r in range(ks)]
        mag = (1 + (hash32(base ^ 0x1234) % 64)).to(torch.float64) / 8.0
        sgn = torch.where((hash32(base ^ 0x5678) & 7) < 6, 1.0, -1.0).to(torch.float64)
        mu = sgn * mag * spec.mean_scale
        c = [ci * spec.spike_scale for ci in c]
        return a, b, c, mu
    scale = spec.sigma_t * (math.sqrt(l) + math.sqrt(m))
    if ks == 1:
        theta = [spec.theta_1]
    else:
        theta = [spec.theta_1 + (spec.theta_k - spec.theta_1) * r / (ks - 1) for r in range(ks)]
    sig = [t * scale for t in theta]
    c = [s / math.sqrt(l * m) * spec.spike_scale for s in sig]
    # mean-bias direction w_j
    u_sign = _u24(hash32(base ^ 0x0A0A)).to(torch.float64) / float(1 << 24)
    s = torch.where(u_sign < spec.coherent, 1.0, -1.0).to(torch.float64)
    g = torch.zeros(m, dtype=torch.float64)
    for t in range(12):
        g = g + _u24(hash32(base ^ (0x100 + t) * 0x9E3779B1)).to(torch.float64) / float(1 << 24)
    g = g - 6.0
    w = s * (1.0 + 0.25 * g)
    u_mass = _u24(hash32(base ^ 0xB0B0)).to(torch.float64) / float(1 << 24)
    w = torch.where(u_mass < spec.massive_frac, w * spec.massive_mult, w)
    e_rest = sum(ci * ci for ci in c) * l * m + l * m * spec.sigma_t ** 2
    f = spec.f_mean
    wn2 = float((w * w).sum())
    beta = math.sqrt(f / (1.0 - f) * e_rest / (l * spec.sigma_t ** 2 * wn2)) if f > 0 else 0.0
    mu = beta * spec.sigma_t * w * spec.mean_scale
    return a, b, c, mu


def generate(spec: SynthSpec, row0: int = 0, rows: int | None = None,
             device: str | torch.device = "cpu", chunk_rows: int | None = None) -> torch.Tensor:
    """Rows [row0, row0+rows) of X as a contiguous fp32 tensor on `device`."""
    rows = spec.l - row0 if rows is None else rows
    dev = torch.device(device)
    a, b, c, mu = planted(spec)
    mu = mu.to(dev)
    jj = torch.arange(spec.m, dtype=torch.int64, device=dev)
    Hb = [walsh(br, jj) for br in b]
    out = torch.empty((rows, spec.m), dtype=torch.float32, device=dev)
    if chunk_rows is None:
        chunk_rows = max(1, (1 << 22) // max(spec.m, 1)) if dev.type == "cpu" else max(1, (1 << 27) // max(spec.m, 1))
    seed_mix = (spec.seed * 0x85EBCA6B + 0x27D4EB2F) & M32
    hj = hash32(jj ^ seed_mix)
    for r0 in range(0, rows, chunk_rows):
        r1 = min(rows, r0 + chunk_rows)
        ii = torch.arange(row0 + r0, row0 + r1, dtype=torch.int64, device=dev)
        acc = mu.unsqueeze(0).expand(r1 - r0, spec.m).clone()
        for r in range(len(c)):
            if c[r] == 0.0:
                continue
            ha = walsh(a[r], ii) * c[r]
            acc = acc + ha.unsqueeze(1) * Hb[r].unsqueeze(0)
        if not spec.exact and spec.sigma_t != 0.0:
            base = hash32(hash32(ii ^ 0x3C6EF372).unsqueeze(1) ^ hj.unsqueeze(0))
            z = torch.zeros((r1 - r0, spec.m), dtype=torch.float64, device=dev)
            for t in range(12):
                z = z + _u24(hash32(base ^ ((0x632BE5AB * (t + 1)) & M32))).to(torch.float64)
            z = z / float(1 << 24) - 6.0
            acc = acc + spec.sigma_t * z
        out[r0:r1] = acc.to(torch.float32)
    return out


# ---- configs of BASELINE.json (SURVEY.md §8 config sheet) ---------------------------------
def config_spec(name: str, seed: int = 0) -> SynthSpec:
    if name == "c1":
        return SynthSpec(512, 256, seed=seed, f_mean=0.9)
    if name == "c2":
        return SynthSpec(8192, 2048, seed=seed, f_mean=0.9)
    if name == "c3":  # the first matrix of the 58-matrix sweep (embedding, early); see sweep_specs
        return sweep_specs(seed)[0]
    if name == "c4":
        return SynthSpec(131072, 4096, seed=seed, f_mean=0.9)
    if name == "c5":
        return SynthSpec(1048576, 8192, seed=seed, f_mean=0.9)
    raise KeyError(name)


def sweep_specs(seed: int = 0) -> list[SynthSpec]:
    """c3: embedding + 28 layers at early (10k) and late (170k) mean-bias strengths, l=32768,
    m=2048.  The paper's figures carry no numbers (PAPER.md:765-779 are placeholders), so the
    monotone schedule is invented: early f = 0.85 - 0.55 d/28, theta_1 = 8 + 8 d/28;
    late f = 0.97 - 0.17 d/28, theta_1 = 8."""
    out = []
    for stage in (0, 1):
        for d in range(29):
            if stage == 0:
                f, th = 0.85 - 0.55 * d / 28, 8.0 + 8.0 * d / 28
            else:
                f, th = 0.97 - 0.17 * d / 28, 8.0
            out.append(SynthSpec(32768, 2048, seed=seed * 1000 + 2 * d + stage, f_mean=f,
                                 theta_1=th))
    return out


def generate_weight(m: int, n: int, seed: int = 0, device: str | torch.device = "cpu") -> torch.Tensor:
    """W [m, n] fp32 for the Averis GeMM: Irwin-Hall-12 entries / sqrt(m) (mean 0,
    variance 1/m: a random-init linear layer), a pure function of (seed, k, j) like generate()."""
    dev = torch.device(device)
    kk = torch.arange(m, dtype=torch.int64, device=dev)
    jj = torch.arange(n, dtype=torch.int64, device=dev)
    base = hash32(hash32(kk ^ ((seed * 0x2545F491 + 0x68E31DA4) & M32)).unsqueeze(1) ^ hash32(jj ^ 0x5BD1E995).unsqueeze(0))
    z = torch.zeros((m, n), dtype=torch.float64, device=dev)
    for t in range(12):
        z = z + _u24(hash32(base ^ ((0x1B873593 * (t + 1)) & M32))).to(torch.float64)
    z = z / float(1 << 24) - 6.0
    return (z / math.sqrt(m)).to(torch.float32)
