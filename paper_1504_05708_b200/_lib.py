"""ctypes view of include/duquad.h (argument marshalling only).

Loads the in-tree `libduquad.so` built by `__graft_entry__.build()` /
`python -m paper_1504_05708_b200.build`.  There is no fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libduquad.so")

DUQUAD_OK = 0
DUQUAD_EINVAL = 1
DUQUAD_ENOMEM = 2
DUQUAD_ECUDA = 3
DUQUAD_ENCCL = 4
DUQUAD_ENONFINITE = 5
DUQUAD_ENODEV = 6
DUQUAD_ESTATE = 7
DUQUAD_EMAXITER = 8

DGM = 0
DFGM = 1
INNER_FGM = 0
INNER_GM = 1
INNER_FGM_SIGMA = 2
DENSE = 0
CSR = 1
CONE_ZERO = 0
CONE_NONPOS = 1


class Problem(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("p", C.c_int64), ("batch", C.c_int64),
        ("format", C.c_int32), ("on_device", C.c_int32),
        ("Q", C.c_void_p), ("ldQ", C.c_int64),
        ("G", C.c_void_p), ("ldG", C.c_int64),
        ("Q_rowptr", C.c_void_p), ("Q_col", C.c_void_p), ("Q_val", C.c_void_p), ("Q_nnz", C.c_int64),
        ("G_rowptr", C.c_void_p), ("G_col", C.c_void_p), ("G_val", C.c_void_p), ("G_nnz", C.c_int64),
        ("q", C.c_void_p), ("g", C.c_void_p), ("lb", C.c_void_p), ("ub", C.c_void_p),
        ("cone", C.c_void_p), ("cone_all", C.c_int32),
    ]


class Options(C.Structure):
    _fields_ = [
        ("dual_step_scale", C.c_double), ("project_dual", C.c_int32), ("inner_rule", C.c_int32),
        ("sigma", C.c_double), ("lambda_min_lb", C.c_double), ("l_mode", C.c_int32),
        ("use_graphs", C.c_int32), ("world_size", C.c_int32), ("rank", C.c_int32),
        ("nccl_id", C.c_void_p), ("stream", C.c_void_p), ("device", C.c_int32),
        ("time_passes", C.c_int32), ("small_path", C.c_int32), ("rho0_path", C.c_int32),
        ("emulate_ranks", C.c_int32), ("fused_path", C.c_int32), ("persist_path", C.c_int32),
        ("eq_precompute", C.c_int32), ("checkpoint", C.c_int32), ("dual_average", C.c_int32),
        ("nccl_self", C.c_int32), ("sell_path", C.c_int32), ("pair_rows", C.c_int32), ("pdl", C.c_int32),
    ]


class Monitor(C.Structure):
    _fields_ = [("outer_done", C.c_int64), ("inner_total", C.c_int64), ("passes_total", C.c_int64),
                ("checks", C.c_int32), ("converged", C.c_int32), ("F", C.c_double), ("dist", C.c_double),
                ("dual", C.c_double)]


class Result(C.Structure):
    _fields_ = [
        ("outer_iters", C.c_int64), ("inner_iters_total", C.c_int64),
        ("kernel_launches", C.c_int64), ("matrix_passes", C.c_int64),
        ("ms_device", C.c_double), ("ms_pass_a", C.c_double), ("ms_pass_b", C.c_double),
        ("n_timed_a", C.c_int64), ("n_timed_b", C.c_int64),
        ("bytes_pass_a", C.c_double), ("bytes_pass_b", C.c_double),
        ("flops_pass_a", C.c_double), ("flops_pass_b", C.c_double),
        ("path", C.c_int32), ("sparse_kernels", C.c_int32),
    ]


class Schedule(C.Structure):
    _fields_ = [
        ("eps_in", C.c_double), ("k_out", C.c_int64), ("k_in", C.c_int64), ("rho_star", C.c_double),
        ("k_total", C.c_int64), ("case_id", C.c_int32), ("reserved", C.c_int32),
    ]


class Bounds(C.Structure):
    _fields_ = [("dual_gap", C.c_double), ("drift", C.c_double), ("feas_last", C.c_double),
                ("feas_avg", C.c_double)]


PATHS = {0: "two_pass", 1: "byte_floor", 2: "rho0", 3: "rho0_floor", 4: "batched", 5: "csr", 6: "small",
         7: "persist", 8: "eq_h", 9: "eq_h_floor"}


_SIGS = {
    "duquad_abi_version": (C.c_int32, []),
    "duquad_struct_size": (C.c_int64, [C.c_int32]),
    "duquad_status_string": (C.c_char_p, [C.c_int32]),
    "duquad_default_options": (None, [C.POINTER(Options)]),
    "duquad_shard_range": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "duquad_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "duquad_setup": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(Problem), C.c_double, C.POINTER(Options)]),
    "duquad_lipschitz": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "duquad_set_constants": (C.c_int, [C.c_void_p, C.c_double, C.c_double]),
    "duquad_solve": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(Result)]),
    "duquad_get_result": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]),
    "duquad_set_trace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]),
    "duquad_solve_monitored": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                         C.c_double, C.c_double, C.POINTER(Monitor), C.POINTER(C.c_double),
                                         C.POINTER(Result)]),
    "duquad_residuals": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double)]),
    "duquad_solve_emulated": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "duquad_solve_eps_emulated": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                            C.c_double, C.c_double]),
    "duquad_solve_eps": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                   C.POINTER(Result)]),
    "duquad_get_inner_counts": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]),
    "duquad_set_initial": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]),
    "duquad_theory_schedule": (C.c_int, [C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(Schedule)]),
    "duquad_theory_bounds": (C.c_int, [C.c_int32, C.c_int64, C.c_double, C.c_double, C.c_double,
                                       C.POINTER(Bounds)]),
    "duquad_get_state": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_int32]),
    "duquad_set_state": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                   C.c_double, C.c_int32]),
    "duquad_local_ranges": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "duquad_destroy": (None, [C.c_void_p]),
    "duquad_last_error": (C.c_char_p, [C.c_void_p]),
}

EXPORTED = tuple(_SIGS)


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise RuntimeError(f"DuQuad CUDA library not built: {path} is missing "
                           "(run __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = load()
    return _lib


class DuquadError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


def check(status: int, ctx=None):
    if status != DUQUAD_OK:
        L = lib()
        msg = L.duquad_last_error(ctx).decode(errors="replace")
        raise DuquadError(status, f"{L.duquad_status_string(status).decode()}: {msg}")
