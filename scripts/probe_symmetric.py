"""Symmetric-extension pyramid timing under the crop switches (crop_tiles:
2 compiled crop kernel beside the fused kernel, 1 generic tile launch after
it, 0 one generic launch per sub-step; crop_core: positions per tile), with
the periodic pyramid for comparison:
    python scripts/probe_symmetric.py"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402


def med(plan, img, L, out, reps=10):
    plan.forward_mallat(img, L, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.forward_mallat(img, L, out=out)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


for n, L in ((4096, 1), (4096, 8), (16384, 8)):
    img = random_image(n, n, 1, device="cuda")
    out = torch.empty_like(img)
    per = med(dwt.Plan("cdf97", "nonseparable-lifting", optimized=True), img, L, out)
    print(f"{n} L{L} periodic {per:.4f} ms", flush=True)
    for tiles, core in [(2, 8), (2, 12), (2, 4), (1, 8), (0, 8)]:
        plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True, extension="symmetric")
        plan.tune(crop_tiles=tiles, crop_core=core)
        t = med(plan, img, L, out)
        print(f"{n} L{L} symmetric crop_tiles={tiles} core={core:2d} {t:.4f} ms ({t / per:.2f}x periodic)", flush=True)
