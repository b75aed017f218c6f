"""CPU-only checks of the C ABI (no device work): the library loads, exports every symbol
include/avd.h declares, plans sizes by the DESIGN.md R1/R2 rules, validates arguments, and the
host-only tie-quota logic is right.  Also guards the product/oracle separation."""
import ctypes
import os
import re

import pytest

from paper_2603_10444_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions(name="avd.h"):
    src = open(os.path.join(ROOT, "include", name)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(avd_[a-z_0-9]+)\s*\(", src)))


@pytest.mark.parametrize("header,exports", [("avd.h", L.EXPORTS), ("avd_averis.h", L.EXPORTS_AVERIS)])
def test_exports_match_header(header, exports):
    lib = L.lib()
    declared = _header_functions(header)
    assert set(declared) == set(exports), (declared, exports)
    for name in declared:
        assert hasattr(lib, name), name


def _cfg(l, m, **kw):
    c = L.avd_config()
    c.l_global = c.l_local = l
    c.m = m
    c.k_frac, c.top_frac, c.world = 0.01, 0.001, 1
    for k, v in kw.items():
        setattr(c, k, v)
    return c


@pytest.mark.parametrize("l,m,k,p,n_top", [(512, 256, 2, 16, 131), (8192, 2048, 20, 32, 16777),
                                           (131072, 4096, 40, 48, 536870),
                                           (1048576, 8192, 81, 96, 8589934), (2, 2, 1, 16, 1)])
def test_plan_sizes(l, m, k, p, n_top):
    pl = L.avd_plan(_cfg(l, m))
    assert (pl.k, pl.p, pl.n_top, pl.digits) == (k, p, n_top, 2)
    assert pl.workspace_bytes > l * m * 2  # digit planes dominate


def test_plan_rejects_bad_arguments():
    for cfg in (_cfg(1, 8), _cfg(8, 1), _cfg(64, 64, k_override=65), _cfg(64, 64, k_frac=0.0),
                _cfg(64, 64, top_frac=1.5), _cfg(64, 64, digits=5), _cfg(64, 64, l_local=63),
                _cfg(64, 4096, k_override=100)):
        with pytest.raises(L.AvdError) as e:
            L.avd_plan(cfg)
        assert e.value.status == L.AVD_EINVAL
    msg = L.lib().avd_last_error().decode()
    assert msg


def test_gram_free_plan_rules():
    """AVD_FLAG_GRAM_FREE is single-GPU and excludes AVD_FLAG_MEAN_TOPK (include/avd.h)."""
    pl = L.avd_plan(_cfg(4096, 512, flags=L.AVD_FLAG_GRAM_FREE))
    assert (pl.k, pl.p) == (5, 16)
    for cfg in (_cfg(4096, 512, flags=L.AVD_FLAG_GRAM_FREE, world=2, l_local=2048),
                _cfg(4096, 512, flags=L.AVD_FLAG_GRAM_FREE | L.AVD_FLAG_MEAN_TOPK)):
        with pytest.raises(L.AvdError) as e:
            L.avd_plan(cfg)
        assert e.value.status == L.AVD_EINVAL


def test_averis_create_validates():
    """avd_averis_create: m a multiple of 32, n of 16, l >= 1 (EINVAL), and no device -> ECUDA."""
    import torch
    for l, m, n in ((0, 64, 16), (16, 48, 16), (16, 64, 24)):
        c = L.avd_averis_config()
        c.l, c.m, c.n = l, m, n
        h = ctypes.c_void_p()
        assert L.lib().avd_averis_create(ctypes.byref(c), ctypes.byref(h)) == L.AVD_EINVAL and not h.value
    if not torch.cuda.is_available():
        c = L.avd_averis_config()
        c.l, c.m, c.n = 16, 64, 16
        h = ctypes.c_void_p()
        assert L.lib().avd_averis_create(ctypes.byref(c), ctypes.byref(h)) == L.AVD_ECUDA and not h.value


def test_tie_quota():
    # q = 4 ties to take; ranks hold 2, 3, 10 ties and 5, 3, 4 strictly-greater entries
    assert L.avd_tie_quota([5, 3, 4], [2, 3, 10], 0, 4) == (2, 0)
    assert L.avd_tie_quota([5, 3, 4], [2, 3, 10], 1, 4) == (2, 7)
    assert L.avd_tie_quota([5, 3, 4], [2, 3, 10], 2, 4) == (0, 12)
    assert L.avd_tie_quota([0, 0], [0, 0], 1, 0) == (0, 0)
    with pytest.raises(L.AvdError):
        L.avd_tie_quota([1], [1], 3, 0)


def test_strerror():
    lib = L.lib()
    assert lib.avd_strerror(L.AVD_ENONFINITE).decode().startswith("input contains")


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2603_10444_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("oracle/", ""), f


def test_create_needs_sm100():
    """avd_create refuses to run without an sm_100 device (no fallback path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    st = L.lib().avd_create(ctypes.byref(_cfg(64, 64)), ctypes.byref(h))
    assert st != L.AVD_OK and not h.value
