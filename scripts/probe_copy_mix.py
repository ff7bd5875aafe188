"""Concurrent H2D + D2H with the host pipeline's copy shapes (16384^2 image,
16 bands): uploads of 64 MB bands on one stream while each band's detail
rows go down on another, as 2-D copies (HL: 8192 of 16384 columns; LH|HH:
whole rows) or as plain 1-D copies of the same byte count. Tells whether
2-D D2H copies share bandwidth worse with the uploads than 1-D ones."""
import sys
import time

import torch
from cuda.bindings import runtime as rt

W = H = 16384
B = 16
rows = H // B
n = W * H
himg = torch.empty(n, dtype=torch.float32).pin_memory()
hout = torch.empty(n, dtype=torch.float32).pin_memory()
dimg = torch.empty(n, dtype=torch.float32, device="cuda")
dout = torch.empty(n, dtype=torch.float32, device="cuda")
up = torch.cuda.Stream()
down = torch.cuda.Stream()
up2 = torch.cuda.Stream()
down2 = torch.cuda.Stream()
import ctypes
from pathlib import Path
zc = ctypes.CDLL(str(Path(__file__).resolve().parents[1] / "build/probe_zcopy.so"))
zc.zcopy2d_launch.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_longlong,
                              ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
CTAS = int(sys.argv[1]) if len(sys.argv) > 1 else 32
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost


def ck(r):
    if r[0] != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(r)


def run(mode):
    evs = [torch.cuda.Event() for _ in range(B)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for b in range(B):
        o = b * rows * W * 4
        us = up2 if (mode.endswith("x2") and b % 2) else up
        if mode.endswith("h2"):  # each band's upload split over two streams
            half = rows * W * 2
            ck(rt.cudaMemcpyAsync(dimg.data_ptr() + o, himg.data_ptr() + o, half, H2D, up.cuda_stream))
            ck(rt.cudaMemcpyAsync(dimg.data_ptr() + o + half, himg.data_ptr() + o + half, half, H2D, up2.cuda_stream))
            up.wait_stream(up2)
            us = up
        else:
            ck(rt.cudaMemcpyAsync(dimg.data_ptr() + o, himg.data_ptr() + o, rows * W * 4, H2D, us.cuda_stream))
        evs[b].record(us)
    w2, h2, hb = W // 2, H // 2, rows // 2
    for b in range(B):
        ds = down2 if (mode.endswith("x2") and b % 2) else down
        ds.wait_event(evs[b])
        y0 = b * hb
        if mode == "none":
            continue
        if mode.startswith("1d") and (mode.endswith("x2") or mode.endswith("h2")):
            o1 = (y0 * W) * 4
            ck(rt.cudaMemcpyAsync(hout.data_ptr() + o1, dout.data_ptr() + o1, hb * w2 * 4, D2H, ds.cuda_stream))
            o2 = ((h2 + y0) * W) * 4
            s2 = down2 if mode.endswith("h2") else ds
            if mode.endswith("h2"):
                s2.wait_event(evs[b])
            ck(rt.cudaMemcpyAsync(hout.data_ptr() + o2, dout.data_ptr() + o2, hb * W * 4, D2H, s2.cuda_stream))
            continue
        if mode == "2d":
            o1 = (y0 * W + w2) * 4
            ck(rt.cudaMemcpy2DAsync(hout.data_ptr() + o1, W * 4, dout.data_ptr() + o1, W * 4, w2 * 4, hb, D2H,
                                    down.cuda_stream))
            o2 = ((h2 + y0) * W) * 4
            ck(rt.cudaMemcpy2DAsync(hout.data_ptr() + o2, W * 4, dout.data_ptr() + o2, W * 4, W * 4, hb, D2H,
                                    down.cuda_stream))
        elif mode == "kernel":  # SM stores into pinned host memory (zero-copy)
            o1 = (y0 * W + w2) * 4
            assert zc.zcopy2d_launch(hout.data_ptr() + o1, W * 4, dout.data_ptr() + o1, W * 4, w2 * 4, hb, CTAS,
                                     down.cuda_stream) == 0
            o2 = ((h2 + y0) * W) * 4
            assert zc.zcopy2d_launch(hout.data_ptr() + o2, W * 4, dout.data_ptr() + o2, W * 4, W * 4, hb, CTAS,
                                     down.cuda_stream) == 0
        else:  # 1-D copies of the same byte count
            o1 = (y0 * W) * 4
            ck(rt.cudaMemcpyAsync(hout.data_ptr() + o1, dout.data_ptr() + o1, hb * w2 * 4, D2H, down.cuda_stream))
            o2 = ((h2 + y0) * W) * 4
            ck(rt.cudaMemcpyAsync(hout.data_ptr() + o2, dout.data_ptr() + o2, hb * W * 4, D2H, down.cuda_stream))
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


def both_big():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ck(rt.cudaMemcpyAsync(dimg.data_ptr(), himg.data_ptr(), n * 4, H2D, up.cuda_stream))
    ck(rt.cudaMemcpyAsync(hout.data_ptr(), dout.data_ptr(), n * 3, D2H, down.cuda_stream))
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


ts = sorted(both_big() for _ in range(5))
print(f"one 1 GiB H2D + one 768 MB D2H, concurrent: median {ts[2]:.2f} ms", flush=True)


# D2H alone through each mechanism (768 MB)
def d2h_only(mode):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if mode == "kernel":
        zc.zcopy2d_launch(hout.data_ptr(), W * 4, dout.data_ptr(), W * 4, W * 4, H * 3 // 4, CTAS, down.cuda_stream)
    else:
        ck(rt.cudaMemcpyAsync(hout.data_ptr(), dout.data_ptr(), n * 3, D2H, down.cuda_stream))
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


for mode in ["ce", "kernel", "ce", "kernel"]:
    ts = sorted(d2h_only(mode) for _ in range(5))
    print(f"D2H only {mode:6s} 768 MB median {ts[2]:7.2f} ms ({0.805306368e3 / ts[2]:.1f} GB/s)", flush=True)
hout.copy_(dout.cpu())
for mode in ["none", "1d", "1dx2", "1dh2", "1d", "1dx2", "1dh2"]:
    ts = sorted(run(mode) for _ in range(5))
    print(f"{mode:5s} median {ts[2]:7.2f} ms  min {ts[0]:7.2f} ms", flush=True)
