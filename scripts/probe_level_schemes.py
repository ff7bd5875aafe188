"""Single forward level of every CDF 9/7 scheme variant at one size, timed
with CUDA events (median of N), for A/B runs of the run-time switches:
    DWT2D_TMA=0 python scripts/probe_level_schemes.py --size 16384"""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

SCHEMES = ["separable-convolution", "separable-lifting", "nonseparable-convolution",
           "nonseparable-polyconvolution", "nonseparable-lifting"]
ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--reps", type=int, default=15)
a = ap.parse_args()
n = a.size
img = random_image(n, n, 1, device="cuda")
bands = [torch.empty((n // 2, n // 2), device="cuda") for _ in range(4)]
for s in SCHEMES:
    for opt in (False, True):
        plan = dwt.Plan("cdf97", s, optimized=opt)
        plan.forward_level(img, bands)
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.forward_level(img, bands)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(f"{s:30s} {'opt ' if opt else 'base'} {ms * 1e3:9.1f} us  {8.0 * n * n / (ms * 1e-3) / 1e9:7.1f} GB/s",
              flush=True)
