"""TEST INFRASTRUCTURE ONLY — ctypes loader for the compiled reference.

Loads ``oracle/_ref/libdwt2d_ref.so`` (built by ``oracle/Makefile`` from the
unmodified reference sources under /root/reference/proj/src plus the shim
``oracle/ref_driver.cpp``). Only tests/, ``__graft_entry__.smoke()`` and the
cpu-baseline / ``--impl reference`` legs of ``bench.py`` may import this
module; the product path never does.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
REF_DIR = _HERE / "_ref"

_libs: dict[str, ctypes.CDLL] = {}

_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)


def available(fma: bool = False) -> bool:
    return (REF_DIR / ("libdwt2d_ref_fma.so" if fma else "libdwt2d_ref.so")).exists()


def lib(fma: bool = False) -> ctypes.CDLL:
    name = "libdwt2d_ref_fma.so" if fma else "libdwt2d_ref.so"
    if name not in _libs:
        path = REF_DIR / name
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run make -C oracle)")
        L = ctypes.CDLL(str(path), mode=os.RTLD_LOCAL)
        L.ref_last_error.restype = ctypes.c_char_p
        _libs[name] = L
    return _libs[name]


def _check(L, rc):
    if rc != 0:
        raise ValueError(L.ref_last_error().decode())


def random_image(w: int, h: int, seed: int, dtype=np.float32) -> np.ndarray:
    """random.hpp:31-37 — row-major LCG image in [0, 1)."""
    L = lib()
    out = np.empty((h, w), dtype=dtype)
    if dtype == np.float32:
        _check(L, L.ref_random_image_f32(w, h, ctypes.c_uint64(seed), out.ctypes.data_as(_f32p)))
    else:
        _check(L, L.ref_random_image_f64(w, h, ctypes.c_uint64(seed), out.ctypes.data_as(_f64p)))
    return out


def split(img: np.ndarray) -> list[np.ndarray]:
    """polyphase_split (image.hpp:73-94): ee, oe, eo, oo."""
    return [np.ascontiguousarray(img[(j >> 1)::2, (j & 1)::2]) for j in range(4)]


def merge(planes) -> np.ndarray:
    """polyphase_merge (image.hpp:96-113)."""
    h2, w2 = planes[0].shape
    img = np.empty((2 * h2, 2 * w2), dtype=planes[0].dtype)
    for j in range(4):
        img[(j >> 1)::2, (j & 1)::2] = planes[j]
    return img


def run(wavelet: str, scheme: str, planes, *, optimized=False, symmetric=False,
        workers=1, fma=False):
    """compile<T> + run<T> of the reference (executor.hpp:52-238).

    Returns (output planes, barrier_count). dtype follows the input planes.
    """
    L = lib(fma)
    planes = [np.ascontiguousarray(p) for p in planes]
    h2, w2 = planes[0].shape
    dt = planes[0].dtype
    outs = [np.empty_like(planes[0]) for _ in range(4)]
    bc = ctypes.c_long(0)
    if dt == np.float32:
        arr_t = _f32p * 4
        fn = L.ref_run_f32
        ins = arr_t(*[p.ctypes.data_as(_f32p) for p in planes])
        ous = arr_t(*[o.ctypes.data_as(_f32p) for o in outs])
    elif dt == np.float64:
        arr_t = _f64p * 4
        fn = L.ref_run_f64
        ins = arr_t(*[p.ctypes.data_as(_f64p) for p in planes])
        ous = arr_t(*[o.ctypes.data_as(_f64p) for o in outs])
    else:
        raise TypeError(dt)
    _check(L, fn(wavelet.encode(), scheme.encode(), int(optimized), int(symmetric),
                 int(workers), ins, w2, h2, ous, ctypes.byref(bc)))
    return outs, bc.value


def pyramid(wavelet: str, scheme: str, img: np.ndarray, levels: int, *,
            optimized=False, symmetric=False, workers=1, fma=False) -> np.ndarray:
    """Mallat loop over the reference API."""
    L = lib(fma)
    img = np.ascontiguousarray(img)
    H, W = img.shape
    out = np.empty_like(img)
    if img.dtype == np.float32:
        _check(L, L.ref_pyramid_f32(wavelet.encode(), scheme.encode(), int(optimized),
                                    int(symmetric), int(workers), img.ctypes.data_as(_f32p),
                                    W, H, levels, out.ctypes.data_as(_f32p)))
    else:
        _check(L, L.ref_pyramid_f64(wavelet.encode(), scheme.encode(), int(optimized),
                                    int(symmetric), int(workers), img.ctypes.data_as(_f64p),
                                    W, H, levels, out.ctypes.data_as(_f64p)))
    return out


def time_pyramid(wavelet: str, scheme: str, img: np.ndarray, levels: int, *,
                 optimized=False, workers=1, repeats=3) -> float:
    """Median seconds of `repeats` reference pyramid runs after one warm-up."""
    L = lib()
    img = np.ascontiguousarray(img, dtype=np.float32)
    H, W = img.shape
    out = np.empty_like(img)
    secs = ctypes.c_double(0.0)
    _check(L, L.ref_time_pyramid_f32(wavelet.encode(), scheme.encode(), int(optimized),
                                     int(workers), img.ctypes.data_as(_f32p), W, H, levels,
                                     int(repeats), out.ctypes.data_as(_f32p), ctypes.byref(secs)))
    return secs.value


def describe(wavelet: str, scheme: str, optimized=False) -> str:
    L = lib()
    buf = ctypes.create_string_buffer(1 << 20)
    _check(L, L.ref_describe(wavelet.encode(), scheme.encode(), int(optimized), buf, len(buf)))
    return buf.value.decode()


def count(wavelet: str, scheme: str, optimized=False) -> tuple[int, int]:
    L = lib()
    st, ops = ctypes.c_long(), ctypes.c_long()
    _check(L, L.ref_count(wavelet.encode(), scheme.encode(), int(optimized),
                          ctypes.byref(st), ctypes.byref(ops)))
    return st.value, ops.value


def taps(wavelet: str, scheme: str, optimized=False, symmetric=False):
    """compile<float> tap tables: list of kernels, each 4 rows of
    (identity, scale, [(comp, dm, dn, w), ...])."""
    L = lib()
    buf = (ctypes.c_double * (1 << 20))()
    n = ctypes.c_int(0)
    _check(L, L.ref_taps_f32(wavelet.encode(), scheme.encode(), int(optimized),
                             int(symmetric), buf, len(buf), ctypes.byref(n)))
    v = list(buf[: n.value])
    pos = 0
    nk = int(v[pos]); pos += 1
    kernels = []
    for _ in range(nk):
        rows = []
        for _r in range(4):
            ident, scale, nt = bool(v[pos]), float(v[pos + 1]), int(v[pos + 2])
            pos += 3
            tl = []
            for _t in range(nt):
                tl.append((int(v[pos]), int(v[pos + 1]), int(v[pos + 2]), float(v[pos + 3])))
                pos += 4
            rows.append((ident, scale, tl))
        kernels.append(rows)
    return kernels
