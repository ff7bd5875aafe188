"""A few symmetric-extension forward pyramids of the headline plan for a
launch list under ncu: python scripts/prof_symmetric.py [--size 16384] [--levels 8]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--levels", type=int, default=8)
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True, extension="symmetric")
img = random_image(a.size, a.size, 1, device="cuda")
out = torch.empty_like(img)
for _ in range(a.iters):
    plan.forward_mallat(img, a.levels, out=out)
torch.cuda.synchronize()
print("ok")
