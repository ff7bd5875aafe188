"""Image-batch throughput on one GPU: n independent pyramids through
dwt2d_forward_mallat_batch (overlapping on library streams) vs one
forward_mallat per image on one stream, each captured once into a CUDA graph
and replayed (device time; eager calls of small images are host-bound),
CUDA events, median of 10:
    python scripts/probe_batch.py"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
for n, size, L in ((64, 512, 8), (64, 1024, 8), (16, 2048, 8), (8, 4096, 8)):
    imgs = [random_image(size, size, 1 + i, device="cuda") for i in range(n)]
    outs = [torch.empty_like(im) for im in imgs]

    def seq():
        for im, o in zip(imgs, outs):
            plan.forward_mallat(im, L, out=o)

    def bat():
        plan.forward_mallat_batch(imgs, L, outs=outs)

    res = {}
    st = torch.cuda.Stream()
    for name, fn in (("sequential", seq), ("batch", bat)):
        with torch.cuda.stream(st):
            fn()  # warm-up: workspaces in the stream-ordered pool
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                a.record()
                g.replay()
                b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        res[name] = statistics.median(ts)
    gpx = n * size * size / 1e9
    print(f"{n} x {size}^2, {L} levels: sequential {res['sequential']:.3f} ms ({gpx / res['sequential'] * 1e3:.1f} Gpixel/s), "
          f"batch {res['batch']:.3f} ms ({gpx / res['batch'] * 1e3:.1f} Gpixel/s)", flush=True)
