"""One forward 2-level pyramid of the headline plan at 16384^2 for profiling
the fused level-pair kernel under ncu: python scripts/prof_pair.py [--iters 3]"""
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
a = ap.parse_args()
plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
img = random_image(a.size, a.size, 1, device="cuda")
out = torch.empty_like(img)
for _ in range(a.iters):
    plan.forward_mallat(img, 2, out=out)
torch.cuda.synchronize()
print("ok")
