"""ctypes binding of libjtfs.so (include/jtfs.h). Argument marshalling only: every step of the path
runs in the CUDA kernels of the library; there is no Python or CPU fallback. Importing works
without a GPU (planning is host-only); compute calls need the CUDA device."""
from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libjtfs.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "jtfs.h")

STATUS = {0: "JTFS_OK", 1: "JTFS_ERR_CONFIG", 2: "JTFS_ERR_SIZE", 3: "JTFS_ERR_NUMERIC",
          4: "JTFS_ERR_CUDA", 5: "JTFS_ERR_OOM", 6: "JTFS_ERR_STATE"}


class JtfsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class PlanInfo(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("N_pad", ctypes.c_int64), ("pad_left", ctypes.c_int64),
                ("P", ctypes.c_int64), ("frames", ctypes.c_int64), ("n_coef", ctypes.c_int64),
                ("n_paths", ctypes.c_int64), ("N1", ctypes.c_int32), ("N2", ctypes.c_int32),
                ("N_fr", ctypes.c_int32), ("n_blocks", ctypes.c_int32), ("log2T", ctypes.c_int32),
                ("log2F", ctypes.c_int32)]


class PathT(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int32), ("n2", ctypes.c_int32), ("n_fr", ctypes.c_int32),
                ("spin", ctypes.c_int32), ("j2", ctypes.c_int32), ("j_fr", ctypes.c_int32),
                ("rows", ctypes.c_int32), ("frames", ctypes.c_int32), ("offset", ctypes.c_int64)]


class MetamerState(ctypes.Structure):
    _fields_ = [("y", ctypes.c_void_p), ("u", ctypes.c_void_p), ("y_prev", ctypes.c_void_p),
                ("g_prev", ctypes.c_void_p), ("mu", ctypes.c_void_p), ("loss_prev", ctypes.c_void_p),
                ("loss", ctypes.c_void_p), ("accepted", ctypes.c_void_p), ("iter", ctypes.c_int64),
                ("active", ctypes.c_void_p)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_SZ = ctypes.c_size_t
_SIGS = {
    "jtfs_plan": (_I, [_I64, _I, _I, _I, _I, _I64, _I64, ctypes.POINTER(_P)]),
    "jtfs_plan_q2": (_I, [_I64, _I, _I, _I, _I, _I, _I64, _I64, ctypes.POINTER(_P)]),
    "jtfs_plan_destroy": (_I, [_P]),
    "jtfs_plan_info": (_I, [_P, ctypes.POINTER(PlanInfo)]),
    "jtfs_plan_paths": (_I, [_P, ctypes.POINTER(PathT), _I64]),
    "jtfs_plan_filters": (_I, [_P, _I, _P, _P, _P, _I64, ctypes.POINTER(_I64)]),
    "jtfs_plan_response": (_I, [_P, _I, _I, _I, _P, _I64]),
    "jtfs_plan_prepare": (_I, [_P, _P]),
    "jtfs_workspace_size": (_SZ, [_P, _I64, _I]),
    "jtfs_forward": (_I, [_P, _P, _I64, _P, _P, _SZ, _P]),
    "jtfs_loss_grad": (_I, [_P, _P, _P, _I64, _P, _P, _I, _I, _P, _SZ, _P]),
    "metamer_step": (_I, [_P, ctypes.POINTER(MetamerState), _P, _I64, ctypes.c_float, ctypes.c_float,
                          ctypes.c_float, _P, _SZ, _P]),
    "jtfs_check_finite": (_I, [_P, _I64, _P]),
    "jtfs_debug_fft": (_I, [_P, _P, _P, _I64, _I64, _I64, _I, _I, _P]),
    "jtfs_plan_shards": (_I, [_P, _I, _P, _I64]),
    "jtfs_loss_report": (_I, [_P, _P, _P, _I64, _P, _P]),
    "jtfs_colored_noise": (_I, [_P, _P, _P, _I64, _P, _P, _SZ, _P]),
    "jtfs_host_staging_size": (_SZ, [_P, _I64, _I]),
    "jtfs_loss_grad_host": (_I, [_P, _P, _P, _I64, _P, _P, _P, _SZ, _P]),
    "jtfs_last_error": (ctypes.c_char_p, []),
    "jtfs_debug_stage": (_I, [_P, _I, _P, _I64, _P, _SZ, _P, _SZ, _P]),
    "jtfs_launch_count": (_I64, []),
    "jtfs_debug_tc_gemm": (_I, [_P, _P, _P, _I, _I, _I, _P]),
    "jtfs_debug_tc_gemm_ts": (_I, [_P, _P, _P, _I, _I, _I, _P]),
    "jtfs_plan_cost": (_I, [_P, _P, _I64]),
    "jtfs_prof_enable": (None, [_I]),
    "jtfs_prof_read": (_I, [_I, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64)]),
}

_lib = None


def header_symbols() -> list[str]:
    """Function names declared in include/jtfs.h."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(jtfs_[a-z_]+|metamer_step)\s*\(", txt)))


def load() -> ctypes.CDLL:
    """Load libjtfs.so (built in-tree by build.py). Raises if it is missing: no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(code: int) -> None:
    if code != 0:
        raise JtfsError(code, load().jtfs_last_error().decode())
