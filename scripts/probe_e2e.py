"""End-to-end pyramid (pinned host image -> dwt2d_forward_mallat_host -> host
pyramid) at 16384^2, 8 levels, under host pipeline band sizes:
    python scripts/probe_e2e.py [--bands 0,512,256]"""
import argparse
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--levels", type=int, default=8)
ap.add_argument("--bands", default="0,2048,512,256")
a = ap.parse_args()
n = a.size
img = random_image(n, n, 1, device="cuda").cpu().pin_memory()
out = torch.empty_like(img).pin_memory()
hi, ho = img.numpy(), out.numpy()
for rows in [int(x) for x in a.bands.split(",")]:
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True).tune(host_band_rows=rows)
    plan.forward_mallat_host(hi, a.levels, ho)
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        plan.forward_mallat_host(hi, a.levels, ho)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    print(f"host_band_rows={rows:5d}: {t * 1e3:7.2f} ms  {n * n / t / 1e9:6.2f} Gpixel/s", flush=True)
