"""Fast host-side fill of synth.gen matrices (C, OpenMP) — bit-identical to synth.gen.generate
(pinned by tests/test_oracle_pins.py::test_fast_generator_bit_identical).  Used by the oracle side
(tools/oracle_cache.py) for bench-scale matrices; holds none of the method's arithmetic."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .gen import M32, SynthSpec, planted

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen_fast.c")
_LIB = os.path.join(_HERE, "_build", "libgenfast.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        os.makedirs(os.path.dirname(_LIB), exist_ok=True)
        if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                                   "-fPIC", "-shared", _SRC, "-o", _LIB + ".tmp"])
            os.replace(_LIB + ".tmp", _LIB)
        L = ctypes.CDLL(_LIB)
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.synth_fill.argtypes = [P, I64, I64, I64, P, I32, P, P, P, I32, ctypes.c_double, ctypes.c_uint32]
        L.synth_fill.restype = ctypes.c_int
        _lib = L
    return _lib


def generate_np(spec: SynthSpec, row0: int = 0, rows: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    rows = spec.l - row0 if rows is None else rows
    a, b, c, mu = planted(spec)
    if len(c) > 128:
        raise ValueError("at most 128 planted directions")
    mu = np.ascontiguousarray(mu.numpy(), np.float64)
    a = np.asarray(a, np.int64)
    b = np.asarray(b, np.int64)
    c = np.asarray(c, np.float64)
    if out is None:
        out = np.empty((rows, spec.m), np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.shape == (rows, spec.m)
    tail = int((not spec.exact) and spec.sigma_t != 0.0)
    seed_mix = (spec.seed * 0x85EBCA6B + 0x27D4EB2F) & M32
    p = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    st = _load().synth_fill(p(out), row0, rows, spec.m, p(mu), len(c), p(a), p(b), p(c), tail,
                            float(spec.sigma_t), seed_mix)
    if st != 0:
        raise MemoryError("synth_fill")
    return out
