"""Run one pyramid level (or a whole pyramid) of the headline plan for
profiling under ncu: python scripts/prof_level.py [--size 16384] [--iters 3]
[--wavelet cdf97 --scheme nonseparable-lifting --optimized 1] [--pyramid 8]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--wavelet", default="cdf97")
ap.add_argument("--scheme", default="nonseparable-lifting")
ap.add_argument("--optimized", type=int, default=1)
ap.add_argument("--pyramid", type=int, default=0)
a = ap.parse_args()
plan = dwt.Plan(a.wavelet, a.scheme, optimized=bool(a.optimized))
img = random_image(a.size, a.size, 1, device="cuda")
if a.pyramid:
    out = torch.empty_like(img)
    for _ in range(a.iters):
        plan.forward_mallat(img, a.pyramid, out)
else:
    bands = [torch.empty((a.size // 2, a.size // 2), device="cuda") for _ in range(4)]
    for _ in range(a.iters):
        plan.forward_level(img, bands)
torch.cuda.synchronize()
print("ok", plan.info["key"])
