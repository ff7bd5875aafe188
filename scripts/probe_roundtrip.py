"""Forward level (polyconvolution, optimized) and inverse level at one size,
CUDA events, median of N: python scripts/probe_roundtrip.py --size 16384"""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--reps", type=int, default=15)
a = ap.parse_args()
n = a.size
img = random_image(n, n, 1, device="cuda")
back = torch.empty_like(img)
b = [torch.empty((n // 2, n // 2), device="cuda") for _ in range(4)]
fwd = dwt.Plan("cdf97", "nonseparable-polyconvolution", optimized=True)
inv = dwt.Plan("cdf97", "inverse-lifting")


def t(fn):
    fn()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


f = t(lambda: fwd.forward_level(img, b))
i = t(lambda: inv.inverse_level(b, back))
print(f"forward {f * 1e3:.1f} us  inverse {i * 1e3:.1f} us  ({8.0 * n * n / (i * 1e-3) / 1e9:.0f} GB/s)  "
      f"max |x - x'| {float((back - img).abs().max()):.2e}")
