"""ctypes binding of the C ABI in include/dwt2d_b200.h.

The shared library is built in-tree (paper_1704_08657_b200/lib/
libdwt2d_b200.so, see build.py). There is no fallback: importing this module
raises if the library is missing, and every call raises on a non-zero status.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libdwt2d_b200.so"

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -m paper_1704_08657_b200.build` "
        "(there is no CPU fallback for the DWT path)")

lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL)

OK, EINVAL, ECUDA, ENOMEM, EUNSUPPORTED = range(5)
SHARD_HANDLE_BYTES = 64

SCHEMES = {
    "separable-convolution": 0,
    "separable-lifting": 1,
    "nonseparable-convolution": 2,
    "nonseparable-polyconvolution": 3,
    "nonseparable-lifting": 4,
    "inverse-lifting": 5,
}
FORWARD_SCHEMES = list(SCHEMES)[:5]
EXTENSIONS = {"periodic": 0, "symmetric": 1}
LOWERINGS = {"default": 0, "composed": 1, "factored": 2}


class PlanDesc(ctypes.Structure):
    _fields_ = [("wavelet", ctypes.c_char_p), ("scheme", ctypes.c_int), ("optimized", ctypes.c_int),
                ("extension", ctypes.c_int), ("lowering", ctypes.c_int), ("workers", ctypes.c_int)]


class Row(ctypes.Structure):
    _fields_ = [("identity", ctypes.c_int32), ("tap_begin", ctypes.c_int32),
                ("tap_end", ctypes.c_int32), ("scale", ctypes.c_float)]


class Tap(ctypes.Structure):
    _fields_ = [("comp", ctypes.c_int32), ("dm", ctypes.c_int32), ("dn", ctypes.c_int32),
                ("w", ctypes.c_float)]


class Program(ctypes.Structure):
    _fields_ = [("nsteps", ctypes.c_int32), ("rows", ctypes.POINTER(Row)), ("ntaps", ctypes.c_int32),
                ("taps", ctypes.POINTER(Tap)), ("logical_steps", ctypes.c_int32),
                ("extension", ctypes.c_int32), ("forward", ctypes.c_int32),
                ("fused_multiply_add", ctypes.c_int32),
                ("weights64", ctypes.POINTER(ctypes.c_double)), ("scales64", ctypes.POINTER(ctypes.c_double))]


class PlanInfo(ctypes.Structure):
    _fields_ = [("key", ctypes.c_char * 96), ("fingerprint", ctypes.c_uint64),
                ("logical_steps", ctypes.c_int32), ("substeps", ctypes.c_int32),
                ("operations", ctypes.c_int64), ("taps_per_quad", ctypes.c_int64),
                ("reach_left", ctypes.c_int32), ("reach_right", ctypes.c_int32),
                ("reach_up", ctypes.c_int32), ("reach_down", ctypes.c_int32),
                ("columns_per_lane", ctypes.c_int32), ("forward", ctypes.c_int32),
                ("extension", ctypes.c_int32), ("fused_multiply_add", ctypes.c_int32),
                ("generic", ctypes.c_int32)]


_p = ctypes.c_void_p
_sz = ctypes.c_size_t
_fp = ctypes.POINTER(ctypes.c_float)
_P4 = ctypes.c_void_p * 4
_S4 = ctypes.c_size_t * 4
# dwt2d_halo_fn (include/dwt2d_b200.h)
HaloFn = ctypes.CFUNCTYPE(ctypes.c_int, _p, _p, _sz, ctypes.c_int, ctypes.c_int, _p, _p, _sz, ctypes.c_int,
                          ctypes.c_int, _p)
_P3 = ctypes.c_void_p * 3
_S3 = ctypes.c_size_t * 3

_SIGS = {
    "dwt2d_plan_create": (ctypes.c_int, [ctypes.POINTER(PlanDesc), ctypes.POINTER(_p)]),
    "dwt2d_plan_create_from_program": (ctypes.c_int, [ctypes.POINTER(Program), ctypes.POINTER(_p)]),
    "dwt2d_plan_destroy": (None, [_p]),
    "dwt2d_plan_set_tuning": (ctypes.c_int, [_p, ctypes.c_char_p, ctypes.c_int]),
    "dwt2d_plan_get_info": (ctypes.c_int, [_p, ctypes.POINTER(PlanInfo)]),
    "dwt2d_plan_describe": (ctypes.c_int, [_p, ctypes.c_char_p, _sz]),
    "dwt2d_plan_get_tables": (ctypes.c_int, [_p, ctypes.POINTER(Row), ctypes.c_int32, ctypes.POINTER(Tap),
                                             ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                             ctypes.POINTER(ctypes.c_int32)]),
    "dwt2d_run_planar": (ctypes.c_int, [_p, _P4, _S4, _P4, _S4, ctypes.c_int, ctypes.c_int, _p]),
    "dwt2d_forward_level": (ctypes.c_int, [_p, _p, _sz, ctypes.c_int, ctypes.c_int, _P4, _S4, _p]),
    "dwt2d_inverse_level": (ctypes.c_int, [_p, _P4, _S4, _p, _sz, ctypes.c_int, ctypes.c_int, _p]),
    "dwt2d_forward_level_strip": (ctypes.c_int, [_p, _p, _sz, ctypes.c_int, ctypes.c_int, _p, _p, _sz, _P4,
                                                 _S4, _p]),
    "dwt2d_plan_has_pair": (ctypes.c_int, [_p]),
    "dwt2d_strip_workspace_bytes": (_sz, [_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "dwt2d_forward_mallat_strip": (ctypes.c_int, [_p, _p, _sz, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _sz,
                                                  _p, _p, _p, _p]),
    "dwt2d_forward_pair_strip": (ctypes.c_int, [_p, _p, _sz, ctypes.c_int, ctypes.c_int, _p, _p, _sz, _P3, _S3,
                                                _P4, _S4, _p]),
    "dwt2d_inverse_level_strip": (ctypes.c_int, [_p, _P4, _S4, _P4, _P4, _S4, _p, _sz, ctypes.c_int,
                                                 ctypes.c_int, _p]),
    "dwt2d_shard_create": (ctypes.c_int, [_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.POINTER(_p)]),
    "dwt2d_shard_destroy": (None, [_p]),
    "dwt2d_shard_export": (ctypes.c_int, [_p, ctypes.c_char_p, _sz]),
    "dwt2d_shard_connect": (ctypes.c_int, [_p, _p, _p]),
    "dwt2d_shard_connect_ipc": (ctypes.c_int, [_p, ctypes.c_char_p, ctypes.c_char_p]),
    "dwt2d_shard_forward_mallat": (ctypes.c_int, [_p, _p, _sz, _p, _sz, _p]),
    "dwt2d_shard_status": (ctypes.c_int, [_p, ctypes.POINTER(ctypes.c_int)]),
    "dwt2d_shard_forward_mallat_ex": (ctypes.c_int, [_p, _p, _sz, _p, _sz, ctypes.POINTER(ctypes.c_void_p), _p]),
    "dwt2d_shard_info": (ctypes.c_int, [_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(_sz)]),
    "dwt2d_forward_mallat_sharded": (ctypes.c_int, [_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                                    ctypes.POINTER(_p), ctypes.POINTER(_sz), ctypes.c_int,
                                                    ctypes.c_int, ctypes.c_int, ctypes.POINTER(_p),
                                                    ctypes.POINTER(_sz), ctypes.POINTER(_p)]),
    "dwt2d_workspace_bytes": (_sz, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "dwt2d_forward_mallat": (ctypes.c_int, [_p, _p, _sz, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _sz,
                                            _p, _p]),
    "dwt2d_forward_mallat_batch": (ctypes.c_int, [_p, ctypes.c_int, _p, _sz, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                  _p, _sz, ctypes.c_int, _p, _p]),
    "dwt2d_forward_mallat_ex": (ctypes.c_int, [_p, _p, _sz, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _sz,
                                               _p, ctypes.POINTER(ctypes.c_void_p), _p]),
    "dwt2d_event_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p)]),
    "dwt2d_event_destroy": (ctypes.c_int, [_p]),
    "dwt2d_event_elapsed_ms": (ctypes.c_int, [_p, _p, ctypes.POINTER(ctypes.c_float)]),
    "dwt2d_inverse_mallat": (ctypes.c_int, [_p, _p, _sz, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _sz,
                                            _p, _p]),
    "dwt2d_run_planar_host": (ctypes.c_int, [_p, _P4, _P4, ctypes.c_int, ctypes.c_int]),
    "dwt2d_run_planar_f64": (ctypes.c_int, [_p, _P4, _S4, _P4, _S4, ctypes.c_int, ctypes.c_int, _p]),
    "dwt2d_forward_level_f64": (ctypes.c_int, [_p, _p, _sz, ctypes.c_int, ctypes.c_int, _P4, _S4, _p]),
    "dwt2d_inverse_level_f64": (ctypes.c_int, [_p, _P4, _S4, _p, _sz, ctypes.c_int, ctypes.c_int, _p]),
    "dwt2d_run_planar_host_f64": (ctypes.c_int, [_p, _P4, _P4, ctypes.c_int, ctypes.c_int]),
    "dwt2d_forward_mallat_host": (ctypes.c_int, [_p, _p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p]),
    "dwt2d_inverse_mallat_host": (ctypes.c_int, [_p, _p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p]),
    "dwt2d_time_forward": (ctypes.c_int, [_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]),
    "dwt2d_last_error": (ctypes.c_char_p, []),
    "dwt2d_version": (ctypes.c_char_p, []),
    "dwt2d_registry_size": (ctypes.c_int, []),
    "dwt2d_registry_key": (ctypes.c_char_p, [ctypes.c_int]),
    "dwt2d_launch_count": (ctypes.c_uint64, []),
}
EXPORTED = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class DwtError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def check(rc: int) -> None:
    if rc != OK:
        msg = lib.dwt2d_last_error().decode()
        if rc == EINVAL:
            raise ValueError(msg)
        raise DwtError(rc, msg)


class Event:
    """A CUDA timing event owned by the library (for dwt2d_forward_mallat_ex)."""

    def __init__(self):
        h = ctypes.c_void_p()
        check(lib.dwt2d_event_create(ctypes.byref(h)))
        self.handle = h

    def elapsed_ms(self, end: "Event") -> float:
        ms = ctypes.c_float()
        check(lib.dwt2d_event_elapsed_ms(self.handle, end.handle, ctypes.byref(ms)))
        return float(ms.value)

    def __del__(self):
        if getattr(self, "handle", None) and lib is not None:
            lib.dwt2d_event_destroy(self.handle)
            self.handle = None


def registry_keys() -> list[str]:
    return [lib.dwt2d_registry_key(i).decode() for i in range(lib.dwt2d_registry_size())]


def launch_count() -> int:
    return int(lib.dwt2d_launch_count())
