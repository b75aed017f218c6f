"""Thin ctypes binding of libavd.so (include/avd.h) — argument marshalling only.

Same names as the C ABI.  Every numerical step runs in the library's CUDA kernels; this module
never falls back to anything else: if libavd.so is missing or cannot load, it raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libavd.so")

AVD_FLAG_STREAM_SELECT, AVD_FLAG_EXACT_SCALE, AVD_FLAG_FORCE_ESCALATE, AVD_FLAG_EIG_HOST_LOOP = 1, 2, 4, 8
AVD_FLAG_MEAN_TOPK, AVD_FLAG_GRAM_FREE = 16, 32
AVD_OK, AVD_EINVAL, AVD_ENONFINITE, AVD_ENOCONV, AVD_ECUDA, AVD_ENOMEM, AVD_ESTATE = 0, 1, 2, 3, 4, 6, 8
AVD_EREPEAT, AVD_EEXCHANGE = 9, 10
BUF = dict(STATS=0, COLMAX=1, COLMIN=2, HIST1=3, GRAM=4, ENERGY=5, HIST2=6, HIST3=7, TIES=8, AGG=9,
           HIST0=10, CAND=11, SAMPLE=12, SMAX=13, SMIN=14, QSUM=15, QERR=21, DIAG=22,
           GRAMP=25, EIGZ=23, EIGY=24,
           MU=16, G=17, P=18, DIGITS=19, SCALE=20)
BUF_NAME = {v: k for k, v in BUF.items()}
AVD_DT_F64, AVD_DT_F32, AVD_DT_I64 = 0, 1, 2
AVD_OP_SUM, AVD_OP_MAX, AVD_OP_MIN = 0, 1, 2
# int (*avd_exchange_fn)(int32_t which, void* buf_dev, int32_t dtype, int32_t op, size_t count, void* user)
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                               ctypes.c_size_t, ctypes.c_void_p)

# every symbol include/avd.h declares
EXPORTS = ["avd_plan", "avd_create", "avd_destroy", "avd_get_plan", "avd_decompose",
           "avd_decompose_host", "avd_buffer", "avd_stage_stats", "avd_stage_split",
           "avd_stage_gram", "avd_stage_eig", "avd_stage_project", "avd_stage_select",
           "avd_stage_gather", "avd_stage_report", "avd_tie_quota", "avd_launch_count", "avd_strerror",
           "avd_last_error", "avd_stage_eig_dist", "avd_decompose_sharded", "avd_exchange_nccl", "avd_gram_product"]
# every symbol include/avd_averis.h declares
EXPORTS_AVERIS = ["avd_averis_create", "avd_averis_destroy", "avd_averis_set_weight", "avd_averis_forward",
                  "avd_averis_forward_host", "avd_averis_buffer", "avd_averis_launch_count",
                  "avd_averis_stage_ms"]
AVD_AVERIS_STOCHASTIC, AVD_AVERIS_VANILLA, AVD_AVERIS_TIMING, AVD_AVERIS_BF16_OUT = 1, 2, 4, 8
AV_BUF = dict(MU=0, XCODES=1, XSF=2, WCODES=3, WSF=4, MUCODES=5, MUSF=6, GSCALE=7, BIAS=8)


class avd_averis_config(ctypes.Structure):
    _fields_ = [("l", ctypes.c_int64), ("m", ctypes.c_int64), ("n", ctypes.c_int64),
                ("flags", ctypes.c_int32), ("seed", ctypes.c_uint64), ("device", ctypes.c_int32),
                ("stream", ctypes.c_void_p)]


class avd_plan_t(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("p", ctypes.c_int32), ("n_top", ctypes.c_int64),
                ("digits", ctypes.c_int32), ("workspace_bytes", ctypes.c_size_t)]


class avd_config(ctypes.Structure):
    _fields_ = [("l_global", ctypes.c_int64), ("l_local", ctypes.c_int64),
                ("row_offset", ctypes.c_int64), ("m", ctypes.c_int64),
                ("k_frac", ctypes.c_double), ("top_frac", ctypes.c_double),
                ("k_override", ctypes.c_int32), ("n_top_override", ctypes.c_int64),
                ("seed", ctypes.c_uint64), ("max_iters", ctypes.c_int32),
                ("eig_tol", ctypes.c_double), ("digits", ctypes.c_int32),
                ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("flags", ctypes.c_int32)]


class avd_outputs(ctypes.Structure):
    _fields_ = [("mu_dev", ctypes.c_void_p), ("V_dev", ctypes.c_void_p),
                ("sigma_dev", ctypes.c_void_p), ("top_idx_dev", ctypes.c_void_p),
                ("rho_dev", ctypes.c_void_p),
                ("n_top_local", ctypes.c_int64), ("top_offset", ctypes.c_int64),
                ("n_top_global", ctypes.c_int64),
                ("energy_cf", ctypes.c_double * 4), ("energy_el", ctypes.c_double * 4),
                ("cross_el", ctypes.c_double * 3), ("colmean_absmax", ctypes.c_double * 2),
                ("rho_mean_aggr", ctypes.c_double * 4), ("rho_energy_aggr", ctypes.c_double * 3),
                ("sigma_next", ctypes.c_double), ("trace_g", ctypes.c_double),
                ("iters", ctypes.c_int32), ("max_resid", ctypes.c_double),
                ("rr_checks", ctypes.c_int32), ("jacobi_sweeps", ctypes.c_int32),
                ("requantised", ctypes.c_int32), ("digits_used", ctypes.c_int32),
                ("precision_sigma", ctypes.c_double), ("precision_share", ctypes.c_double),
                ("mean_R", ctypes.c_double), ("sign_fraction", ctypes.c_double),
                ("p_pos", ctypes.c_int64), ("p_neg", ctypes.c_int64),
                ("cos_mu_v1", ctypes.c_double), ("alpha1", ctypes.c_double),
                ("sigma1_u", ctypes.c_double), ("resid_u", ctypes.c_double),
                ("iters_u", ctypes.c_int32),
                ("mean_sigma_dev", ctypes.c_void_p), ("mean_alpha_dev", ctypes.c_void_p),
                ("iters_uk", ctypes.c_int32), ("resid_uk", ctypes.c_double)]


_lib = None


class AvdError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: status {status} ({msg})")
        self.status = status


def lib() -> ctypes.CDLL:
    """Load libavd.so (raises if it is missing — there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run paper_2603_10444_b200/build.py "
                              "(or __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.avd_plan.argtypes = [ctypes.POINTER(avd_config), ctypes.POINTER(avd_plan_t)]
        L.avd_create.argtypes = [ctypes.POINTER(avd_config), ctypes.POINTER(P)]
        L.avd_destroy.argtypes = [P]
        L.avd_destroy.restype = None
        L.avd_get_plan.argtypes = [P, ctypes.POINTER(avd_plan_t)]
        L.avd_decompose.argtypes = [P, P, ctypes.POINTER(avd_outputs)]
        L.avd_decompose_host.argtypes = [P, P, ctypes.POINTER(avd_outputs)]
        L.avd_buffer.argtypes = [P, I32, ctypes.POINTER(P), ctypes.POINTER(ctypes.c_size_t)]
        L.avd_stage_stats.argtypes = [P, P]
        L.avd_stage_split.argtypes = [P, P]
        L.avd_stage_gram.argtypes = [P, P]
        L.avd_stage_eig.argtypes = [P]
        L.avd_stage_eig_dist.argtypes = [P, I32, EXCHANGE_FN, P]
        L.avd_decompose_sharded.argtypes = [P, P, I32, ctypes.POINTER(avd_outputs), EXCHANGE_FN, P]
        L.avd_exchange_nccl.argtypes = [I32, P, I32, I32, ctypes.c_size_t, P]
        L.avd_gram_product.argtypes = [P, P, P]
        L.avd_stage_project.argtypes = [P, P]
        L.avd_stage_select.argtypes = [P, P, I32, I32]
        L.avd_stage_gather.argtypes = [P, P, I32, ctypes.POINTER(avd_outputs)]
        L.avd_stage_report.argtypes = [P, ctypes.POINTER(avd_outputs)]
        L.avd_tie_quota.argtypes = [P, P, I32, I32, I64, P, P]
        L.avd_launch_count.argtypes = [P]
        L.avd_launch_count.restype = I64
        L.avd_strerror.argtypes = [ctypes.c_int]
        L.avd_strerror.restype = ctypes.c_char_p
        L.avd_last_error.argtypes = []
        L.avd_last_error.restype = ctypes.c_char_p
        L.avd_averis_create.argtypes = [ctypes.POINTER(avd_averis_config), ctypes.POINTER(P)]
        L.avd_averis_destroy.argtypes = [P]
        L.avd_averis_set_weight.argtypes = [P, P]
        L.avd_averis_forward.argtypes = [P, P, P]
        L.avd_averis_forward_host.argtypes = [P, P, P]
        L.avd_averis_buffer.argtypes = [P, I32, ctypes.POINTER(P), ctypes.POINTER(ctypes.c_size_t)]
        L.avd_averis_launch_count.argtypes = [P]
        L.avd_averis_launch_count.restype = I64
        L.avd_averis_stage_ms.argtypes = [P, P]
        for name in EXPORTS_AVERIS:
            if name != "avd_averis_launch_count":
                getattr(L, name).restype = ctypes.c_int
        for name in EXPORTS:
            if name not in ("avd_destroy", "avd_launch_count", "avd_strerror", "avd_last_error"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def check(status: int, where: str, ok=(AVD_OK,)) -> int:
    if status not in ok:
        L = lib()
        raise AvdError(status, where, f"{L.avd_strerror(status).decode()}: {L.avd_last_error().decode()}")
    return status


# ---- same-name wrappers -------------------------------------------------------------------
def avd_plan(cfg: avd_config) -> avd_plan_t:
    p = avd_plan_t()
    check(lib().avd_plan(ctypes.byref(cfg), ctypes.byref(p)), "avd_plan")
    return p


def avd_create(cfg: avd_config) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    check(lib().avd_create(ctypes.byref(cfg), ctypes.byref(h)), "avd_create")
    return h


def avd_destroy(h) -> None:
    lib().avd_destroy(h)


def avd_get_plan(h) -> avd_plan_t:
    p = avd_plan_t()
    check(lib().avd_get_plan(h, ctypes.byref(p)), "avd_get_plan")
    return p


def avd_decompose(h, X_ptr: int, out: avd_outputs) -> int:
    return check(lib().avd_decompose(h, ctypes.c_void_p(X_ptr), ctypes.byref(out)), "avd_decompose",
                 ok=(AVD_OK, AVD_ENOCONV))


def avd_decompose_host(h, X_ptr: int, out: avd_outputs) -> int:
    return check(lib().avd_decompose_host(h, ctypes.c_void_p(X_ptr), ctypes.byref(out)),
                 "avd_decompose_host", ok=(AVD_OK, AVD_ENOCONV))


def avd_buffer(h, which: int):
    p = ctypes.c_void_p()
    n = ctypes.c_size_t()
    check(lib().avd_buffer(h, which, ctypes.byref(p), ctypes.byref(n)), "avd_buffer")
    return p.value, n.value


def avd_stage_stats(h, X_ptr: int):
    return check(lib().avd_stage_stats(h, ctypes.c_void_p(X_ptr)), "avd_stage_stats")


def avd_stage_split(h, X_ptr: int):
    return check(lib().avd_stage_split(h, ctypes.c_void_p(X_ptr)), "avd_stage_split")


def avd_stage_gram(h, X_dev: int):
    return check(lib().avd_stage_gram(h, X_dev), "avd_stage_gram")


def avd_stage_eig(h):
    return check(lib().avd_stage_eig(h), "avd_stage_eig", ok=(AVD_OK, AVD_ENOCONV, AVD_EREPEAT))


def avd_stage_eig_dist(h, rank: int, fn, user=None):
    """fn: an EXCHANGE_FN (keep a reference alive for the call)."""
    return check(lib().avd_stage_eig_dist(h, rank, fn, user), "avd_stage_eig_dist",
                 ok=(AVD_OK, AVD_ENOCONV, AVD_EREPEAT))


def avd_decompose_sharded(h, X_ptr: int, rank: int, out: avd_outputs, fn, user=None):
    return check(lib().avd_decompose_sharded(h, ctypes.c_void_p(X_ptr), rank, ctypes.byref(out), fn, user),
                 "avd_decompose_sharded", ok=(AVD_OK, AVD_ENOCONV))


def avd_stage_project(h, X_ptr: int):
    return check(lib().avd_stage_project(h, ctypes.c_void_p(X_ptr)), "avd_stage_project")


def avd_stage_select(h, X_ptr: int, level: int, rank: int):
    return check(lib().avd_stage_select(h, ctypes.c_void_p(X_ptr), level, rank), "avd_stage_select")


def avd_stage_gather(h, X_ptr: int, rank: int, out: avd_outputs):
    return check(lib().avd_stage_gather(h, ctypes.c_void_p(X_ptr), rank, ctypes.byref(out)),
                 "avd_stage_gather")


def avd_stage_report(h, out: avd_outputs):
    return check(lib().avd_stage_report(h, ctypes.byref(out)), "avd_stage_report")


def avd_launch_count(h) -> int:
    return int(lib().avd_launch_count(h))


def avd_tie_quota(sel_counts, tie_counts, rank: int, q: int):
    """(quota, offset) of `rank` — host-only integer logic of the library (no GPU needed)."""
    world = len(sel_counts)
    S = (ctypes.c_int64 * world)(*[int(x) for x in sel_counts])
    T = (ctypes.c_int64 * world)(*[int(x) for x in tie_counts])
    quota, off = ctypes.c_int64(), ctypes.c_int64()
    check(lib().avd_tie_quota(S, T, world, rank, int(q), ctypes.byref(quota), ctypes.byref(off)),
          "avd_tie_quota")
    return quota.value, off.value


# ---- Averis NVFP4 forward GeMM (include/avd_averis.h) ---------------------------------------
def avd_averis_create(cfg: avd_averis_config) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    check(lib().avd_averis_create(ctypes.byref(cfg), ctypes.byref(h)), "avd_averis_create")
    return h


def avd_averis_destroy(h) -> None:
    check(lib().avd_averis_destroy(h), "avd_averis_destroy")


def avd_averis_set_weight(h, W_ptr: int):
    return check(lib().avd_averis_set_weight(h, ctypes.c_void_p(W_ptr)), "avd_averis_set_weight")


def avd_averis_forward(h, X_ptr: int, Y_ptr: int):
    return check(lib().avd_averis_forward(h, ctypes.c_void_p(X_ptr), ctypes.c_void_p(Y_ptr)), "avd_averis_forward")


def avd_averis_forward_host(h, X_ptr: int, Y_ptr: int):
    return check(lib().avd_averis_forward_host(h, ctypes.c_void_p(X_ptr), ctypes.c_void_p(Y_ptr)),
                 "avd_averis_forward_host")


def avd_averis_buffer(h, which: int):
    p = ctypes.c_void_p()
    n = ctypes.c_size_t()
    check(lib().avd_averis_buffer(h, which, ctypes.byref(p), ctypes.byref(n)), "avd_averis_buffer")
    return p.value, n.value


def avd_averis_launch_count(h) -> int:
    return int(lib().avd_averis_launch_count(h))


def avd_averis_stage_ms(h):
    ms = (ctypes.c_float * 3)()
    check(lib().avd_averis_stage_ms(h, ctypes.cast(ms, ctypes.c_void_p)), "avd_averis_stage_ms")
    return list(ms)


def avd_gram_product(h, In_ptr: int, Y_ptr: int):
    return check(lib().avd_gram_product(h, ctypes.c_void_p(In_ptr), ctypes.c_void_p(Y_ptr)), "avd_gram_product")
