"""Python face of the C ABI: plans and transforms on torch CUDA tensors or
host numpy arrays. Mirrors the reference's call sequence
build_scheme -> optimize_constant_split -> compile -> run
(proj/src/bench.cpp:33-39, executor.hpp:52-238) with a GPU plan.

Device tensors are float32 CUDA tensors with unit stride along rows; their
row stride is passed as the pitch. Work is enqueued on the current torch
stream unless a stream is given.
"""
from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from . import native as N


def _stream_handle(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dev(t, name="tensor", dtype=None):
    import torch
    dtype = dtype or torch.float32
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dtype:
        raise TypeError(f"{name} must be a {str(dtype).replace('torch.', '')} CUDA tensor")
    if t.dim() != 2 or (t.size(1) > 1 and t.stride(1) != 1):
        raise ValueError(f"{name} must be 2-D with unit column stride")
    return t.data_ptr(), (t.stride(0) if t.size(0) > 1 else t.size(1))


class _CudaView:
    """A device pointer as a __cuda_array_interface__ object (zero-copy)."""

    def __init__(self, ptr, rows, cols, pitch):
        self.__cuda_array_interface__ = {"shape": (rows, cols), "strides": (pitch * 4, 4), "typestr": "<f4",
                                         "data": (ptr, False), "version": 3, "stream": None}


def _check_scratch(scratch, nbytes: int, device) -> None:
    """A caller's workspace must live on the transform's device and hold at
    least the library's workspace size (it is written without bounds)."""
    import torch
    if not isinstance(scratch, torch.Tensor) or not scratch.is_cuda or scratch.device != device:
        raise ValueError(f"scratch must be a CUDA tensor on {device}")
    if not scratch.is_contiguous() or scratch.numel() * scratch.element_size() < nbytes:
        raise ValueError(f"scratch must be contiguous with at least {nbytes} bytes")


def _wrap(ptr, rows, cols, pitch, device):
    import torch
    return torch.as_tensor(_CudaView(ptr, rows, cols, pitch), device=device)


class Plan:
    """A compiled transform plan (forward scheme or inverse lifting)."""

    def __init__(self, wavelet: str = "cdf97", scheme: str = "nonseparable-lifting",
                 optimized: bool = False, extension: str = "periodic",
                 lowering: str = "default", workers: int = 1):
        if scheme not in N.SCHEMES:
            raise ValueError(f"unknown scheme: {scheme} (valid: {' '.join(N.SCHEMES)})")
        desc = N.PlanDesc(wavelet.encode(), N.SCHEMES[scheme], int(optimized),
                          N.EXTENSIONS[extension], N.LOWERINGS[lowering], int(workers))
        h = ctypes.c_void_p()
        N.check(N.lib.dwt2d_plan_create(ctypes.byref(desc), ctypes.byref(h)))
        self._h = h
        self.wavelet, self.scheme, self.optimized = wavelet, scheme, bool(optimized)
        self.extension = extension

    @classmethod
    def from_program(cls, rows, taps, *, logical_steps: int, forward: bool = True,
                     extension: str = "periodic", fma: bool = False) -> "Plan":
        """compile<float> of explicit tables: rows = [(identity, tb, te, scale)]*4*nsteps,
        taps = [(comp, dm, dn, w)]."""
        R = (N.Row * max(1, len(rows)))(*[N.Row(*r) for r in rows])
        T = (N.Tap * max(1, len(taps)))(*[N.Tap(*t) for t in taps])
        prog = N.Program(len(rows) // 4, R, len(taps), T, logical_steps, N.EXTENSIONS[extension],
                         int(forward), int(fma))
        self = cls.__new__(cls)
        h = ctypes.c_void_p()
        N.check(N.lib.dwt2d_plan_create_from_program(ctypes.byref(prog), ctypes.byref(h)))
        self._h = h
        self.wavelet, self.scheme, self.optimized, self.extension = "program", "program", False, extension
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and N is not None and getattr(N, "lib", None) is not None:
            N.lib.dwt2d_plan_destroy(h)
        self._h = None

    def tune(self, **switches) -> "Plan":
        """Set run-time switches of this plan (dwt2d_plan_set_tuning), e.g.
        plan.tune(tma=2, chunk_rows=5). Returns the plan."""
        for k, v in switches.items():
            N.check(N.lib.dwt2d_plan_set_tuning(self._h, k.encode(), int(v)))
        return self

    # -- introspection -------------------------------------------------
    @property
    def info(self) -> dict:
        i = N.PlanInfo()
        N.check(N.lib.dwt2d_plan_get_info(self._h, ctypes.byref(i)))
        return {f: (getattr(i, f).decode() if f == "key" else getattr(i, f)) for f, _ in N.PlanInfo._fields_}

    def tables(self):
        """(rows, taps) the level kernel executes: rows = [(identity, tb, te, scale)],
        taps = [(comp, dm, dn, w)] (weights as float32 values)."""
        nr, nt = ctypes.c_int32(), ctypes.c_int32()
        N.check(N.lib.dwt2d_plan_get_tables(self._h, None, 0, None, 0, ctypes.byref(nr), ctypes.byref(nt)))
        R = (N.Row * max(1, nr.value))()
        T = (N.Tap * max(1, nt.value))()
        N.check(N.lib.dwt2d_plan_get_tables(self._h, R, nr.value, T, nt.value, ctypes.byref(nr),
                                            ctypes.byref(nt)))
        rows = [(bool(r.identity), r.tap_begin, r.tap_end, r.scale) for r in R[: nr.value]]
        taps = [(t.comp, t.dm, t.dn, t.w) for t in T[: nt.value]]
        return rows, taps

    def describe(self) -> str:
        buf = ctypes.create_string_buffer(1 << 18)
        N.check(N.lib.dwt2d_plan_describe(self._h, buf, len(buf)))
        return buf.value.decode()

    # -- device tensors ------------------------------------------------
    def run(self, planes: Sequence, out: Sequence | None = None, stream=None):
        """run<T> on four [h2, w2] CUDA tensors (ee, oe, eo, oo): float32
        planes run the fused kernels, float64 planes the float64 executor
        (compile<double>, dwt2d_run_planar_f64)."""
        import torch
        h2, w2 = planes[0].shape
        dt = planes[0].dtype if planes[0].dtype == torch.float64 else torch.float32
        if out is None:
            out = [torch.empty((h2, w2), dtype=dt, device=planes[0].device) for _ in range(4)]
        ip, op = zip(*[_dev(p, "plane", dt) for p in planes]), zip(*[_dev(o, "out", dt) for o in out])
        iptr, ipit = list(ip)
        optr, opit = list(op)
        fn = N.lib.dwt2d_run_planar_f64 if dt == torch.float64 else N.lib.dwt2d_run_planar
        N.check(fn(self._h, N._P4(*iptr), N._S4(*ipit), N._P4(*optr), N._S4(*opit), w2, h2, _stream_handle(stream)))
        return list(out)

    def forward_level(self, image, out: Sequence | None = None, stream=None):
        """One forward level of a float32 (fused kernels) or float64 image."""
        import torch
        H, W = image.shape
        dt = image.dtype if image.dtype == torch.float64 else torch.float32
        if out is None:
            out = [torch.empty((H // 2, W // 2), dtype=dt, device=image.device) for _ in range(4)]
        ptr, pitch = _dev(image, "image", dt)
        optr, opit = zip(*[_dev(o, "out", dt) for o in out])
        fn = N.lib.dwt2d_forward_level_f64 if dt == torch.float64 else N.lib.dwt2d_forward_level
        N.check(fn(self._h, ptr, pitch, W, H, N._P4(*optr), N._S4(*opit), _stream_handle(stream)))
        return list(out)

    def inverse_level(self, planes: Sequence, image=None, stream=None):
        import torch
        h2, w2 = planes[0].shape
        dt = planes[0].dtype if planes[0].dtype == torch.float64 else torch.float32
        if image is None:
            image = torch.empty((2 * h2, 2 * w2), dtype=dt, device=planes[0].device)
        iptr, ipit = zip(*[_dev(p, "plane", dt) for p in planes])
        ptr, pitch = _dev(image, "image", dt)
        fn = N.lib.dwt2d_inverse_level_f64 if dt == torch.float64 else N.lib.dwt2d_inverse_level
        N.check(fn(self._h, N._P4(*iptr), N._S4(*ipit), ptr, pitch, 2 * w2, 2 * h2, _stream_handle(stream)))
        return image

    def forward_level_strip(self, strip, top, bottom, out: Sequence | None = None, stream=None):
        """One forward level of a row strip; `top`/`bottom` are the 2*reach_up /
        2*reach_down image rows above/below it (same width, common pitch)."""
        import torch
        H, W = strip.shape
        if out is None:
            out = [torch.empty((H // 2, W // 2), dtype=torch.float32, device=strip.device) for _ in range(4)]
        ptr, pitch = _dev(strip, "strip")
        tptr, tpitch = _dev(top, "top")
        bptr, bpitch = _dev(bottom, "bottom")
        if tpitch != bpitch:
            raise ValueError("top and bottom halos must share a pitch")
        optr, opit = zip(*[_dev(o, "out") for o in out])
        N.check(N.lib.dwt2d_forward_level_strip(self._h, ptr, pitch, W, H, tptr, bptr, tpitch,
                                                N._P4(*optr), N._S4(*opit), _stream_handle(stream)))
        return list(out)

    def forward_mallat_strip(self, strip, levels: int, exchange=None, out=None, scratch=None, stream=None):
        """Whole forward pyramid of a row strip in the library (C++ driver,
        dwt2d_forward_mallat_strip): `exchange(cur, top_rows, bottom_rows,
        top, bottom)` fills the device tensors `top`/`bottom` with the rows
        above/below the level input `cur` in the global image (e.g.
        strips.HaloExchange); None = the strip is the whole periodic image.
        Returns the strip-Mallat buffer."""
        import torch
        H, W = strip.shape
        if out is None:
            out = torch.empty((H, W), dtype=torch.float32, device=strip.device)
        ptr, pitch = _dev(strip, "strip")
        optr, opitch = _dev(out, "out")
        nbytes = N.lib.dwt2d_strip_workspace_bytes(self._h, W, H, levels)
        if scratch is None:
            scratch = torch.empty(nbytes // 4 + 64, dtype=torch.float32, device=strip.device)
        _check_scratch(scratch, nbytes, strip.device)
        cb = None
        if exchange is not None:
            def _cb(user, cur, cpitch, w, h, top, bottom, hpitch, trows, brows, st):
                try:
                    dev = strip.device
                    args = (_wrap(cur, h, w, cpitch, dev), trows, brows, _wrap(top, trows, w, hpitch, dev),
                            _wrap(bottom, brows, w, hpitch, dev))
                    cur_stream = torch.cuda.current_stream(dev)
                    if (st or 0) == cur_stream.cuda_stream:
                        exchange(*args)
                    else:
                        # the exchange's copies and P2P ops run on torch's
                        # current stream: after the level the library
                        # enqueued on `st` that wrote `cur`, and before the
                        # kernel on `st` that reads the halo rows
                        lib_stream = torch.cuda.ExternalStream(st, device=dev)
                        cur_stream.wait_stream(lib_stream)
                        exchange(*args)
                        lib_stream.wait_stream(cur_stream)
                    return 0
                except Exception:  # surfaced as DWT2D_EINVAL by the library
                    import traceback
                    traceback.print_exc()
                    return 1
            cb = N.HaloFn(_cb)
        N.check(N.lib.dwt2d_forward_mallat_strip(self._h, ptr, pitch, W, H, levels, optr, opitch,
                                                 scratch.data_ptr(), cb, None, _stream_handle(stream)))
        return out

    @property
    def has_pair(self) -> bool:
        """Whether levels 1 and 2 can run fused (forward_pair_strip)."""
        return bool(N.lib.dwt2d_plan_has_pair(self._h))

    def forward_pair_strip(self, strip, top, bottom, out=None, stream=None):
        """Levels 1 and 2 of a row strip in one pass; `top`/`bottom` are the
        6*reach_up / 6*reach_down image rows above/below it. Returns (and
        writes into `out`, if given: pitched views are fine) (level-1 [HL,
        LH, HH], level-2 [LL, HL, LH, HH])."""
        import torch
        H, W = strip.shape
        d = strip.device
        if out is None:
            out1 = [torch.empty((H // 2, W // 2), dtype=torch.float32, device=d) for _ in range(3)]
            out2 = [torch.empty((H // 4, W // 4), dtype=torch.float32, device=d) for _ in range(4)]
        else:
            out1, out2 = out
        ptr, pitch = _dev(strip, "strip")
        tptr, tpitch = _dev(top, "top")
        bptr, bpitch = _dev(bottom, "bottom")
        if tpitch != bpitch:
            raise ValueError("top and bottom halos must share a pitch")
        p1, s1 = zip(*[_dev(o, "out") for o in out1])
        p2, s2 = zip(*[_dev(o, "out") for o in out2])
        N.check(N.lib.dwt2d_forward_pair_strip(self._h, ptr, pitch, W, H, tptr, bptr, tpitch, N._P3(*p1),
                                               N._S3(*s1), N._P4(*p2), N._S4(*s2), _stream_handle(stream)))
        return out1, out2

    def inverse_level_strip(self, planes: Sequence, tops: Sequence, bottoms: Sequence, image=None,
                            stream=None):
        import torch
        h2, w2 = planes[0].shape
        if image is None:
            image = torch.empty((2 * h2, 2 * w2), dtype=torch.float32, device=planes[0].device)
        iptr, ipit = zip(*[_dev(p, "plane") for p in planes])
        tptr, tpit = zip(*[_dev(t, "top") for t in tops])
        bptr, bpit = zip(*[_dev(b, "bottom") for b in bottoms])
        if tuple(tpit) != tuple(bpit):
            raise ValueError("top and bottom halos must share pitches")
        ptr, pitch = _dev(image, "image")
        N.check(N.lib.dwt2d_inverse_level_strip(self._h, N._P4(*iptr), N._S4(*ipit), N._P4(*tptr),
                                                N._P4(*bptr), N._S4(*tpit), ptr, pitch, 2 * w2, 2 * h2,
                                                _stream_handle(stream)))
        return image

    def forward_mallat(self, image, levels: int, out=None, scratch=None, stream=None, events=None):
        """Mallat pyramid. events: optional list of levels + 1 native.Event (or
        None entries) recorded before level 1 and after each level."""
        import torch
        H, W = image.shape
        if out is None:
            out = torch.empty((H, W), dtype=torch.float32, device=image.device)
        ptr, pitch = _dev(image, "image")
        optr, opitch = _dev(out, "out")
        scr = None
        if scratch is not None:
            _check_scratch(scratch, N.lib.dwt2d_workspace_bytes(W, H, levels), image.device)
            scr = scratch.data_ptr()
        if events is None:
            N.check(N.lib.dwt2d_forward_mallat(self._h, ptr, pitch, W, H, levels, optr, opitch, scr,
                                               _stream_handle(stream)))
        else:
            if len(events) != levels + 1:
                raise ValueError("events needs levels + 1 entries")
            arr = (ctypes.c_void_p * (levels + 1))(*[None if e is None else e.handle for e in events])
            N.check(N.lib.dwt2d_forward_mallat_ex(self._h, ptr, pitch, W, H, levels, optr, opitch, scr, arr,
                                                  _stream_handle(stream)))
        return out

    def forward_mallat_batch(self, images, levels: int, outs=None, devices=None, streams=None):
        """Forward pyramids of a batch of equally sized CUDA images
        (dwt2d_forward_mallat_batch): image i runs on devices[i % len(devices)]
        (its tensor must live there), overlapping with the batch's other images
        on library streams; ordered on streams[i % len(devices)] (torch
        streams or raw handles; default: each device's current torch stream)."""
        import torch
        if not images:
            return []
        H, W = images[0].shape
        pitch = _dev(images[0], "image")[1]
        if outs is None:
            outs = [torch.empty((H, W), dtype=torch.float32, device=im.device) for im in images]
        opitch = _dev(outs[0], "out")[1]
        for im, o in zip(images, outs):
            if tuple(im.shape) != (H, W) or tuple(o.shape) != (H, W):
                raise ValueError("batch: images and outputs must share one shape")
            if _dev(im, "image")[1] != pitch or _dev(o, "out")[1] != opitch:
                raise ValueError("batch: images (and outputs) must share one row pitch")
        devs = [images[0].device.index or 0] if devices is None else [int(d) for d in devices]
        for i, (im, o) in enumerate(zip(images, outs)):
            want = devs[i % len(devs)]
            if im.device.index != want or o.device.index != want:
                raise ValueError(f"batch: image {i} and its output must be on cuda:{want}")
        if streams is None:
            streams = [torch.cuda.current_stream(torch.device("cuda", d)) for d in devs]
        if len(streams) != len(devs):
            raise ValueError("batch: one stream per device")
        n = len(images)
        ims = (ctypes.c_void_p * n)(*[im.data_ptr() for im in images])
        ous = (ctypes.c_void_p * n)(*[o.data_ptr() for o in outs])
        dv = (ctypes.c_int * len(devs))(*devs)
        sts = (ctypes.c_void_p * len(devs))(*[_stream_handle(s) for s in streams])
        N.check(N.lib.dwt2d_forward_mallat_batch(self._h, n, ims, pitch, W, H, levels, ous, opitch, len(devs), dv, sts))
        return outs

    def inverse_mallat(self, coeffs, levels: int, image=None, scratch=None, stream=None):
        import torch
        H, W = coeffs.shape
        if image is None:
            image = torch.empty((H, W), dtype=torch.float32, device=coeffs.device)
        cptr, cpitch = _dev(coeffs, "coeffs")
        ptr, pitch = _dev(image, "image")
        if scratch is not None:
            _check_scratch(scratch, N.lib.dwt2d_workspace_bytes(W, H, levels), coeffs.device)
        N.check(N.lib.dwt2d_inverse_mallat(self._h, cptr, cpitch, W, H, levels, ptr, pitch,
                                           None if scratch is None else scratch.data_ptr(),
                                           _stream_handle(stream)))
        return image

    # -- host arrays (H2D + kernels + D2H inside the call) -------------
    def run_host(self, planes: Sequence[np.ndarray]) -> list[np.ndarray]:
        planes = [np.ascontiguousarray(p, dtype=np.float32) for p in planes]
        h2, w2 = planes[0].shape
        out = [np.empty_like(planes[0]) for _ in range(4)]
        N.check(N.lib.dwt2d_run_planar_host(self._h, N._P4(*[p.ctypes.data for p in planes]),
                                            N._P4(*[o.ctypes.data for o in out]), w2, h2))
        return out

    def forward_mallat_host(self, image: np.ndarray, levels: int, out: np.ndarray | None = None):
        image = np.ascontiguousarray(image, dtype=np.float32)
        H, W = image.shape
        if out is None:
            out = np.empty_like(image)
        N.check(N.lib.dwt2d_forward_mallat_host(self._h, image.ctypes.data, W, H, levels, out.ctypes.data))
        return out

    def inverse_mallat_host(self, coeffs: np.ndarray, levels: int, out: np.ndarray | None = None):
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float32)
        H, W = coeffs.shape
        if out is None:
            out = np.empty_like(coeffs)
        N.check(N.lib.dwt2d_inverse_mallat_host(self._h, coeffs.ctypes.data, W, H, levels, out.ctypes.data))
        return out


def workspace_bytes(width: int, height: int, levels: int) -> int:
    return int(N.lib.dwt2d_workspace_bytes(width, height, levels))
