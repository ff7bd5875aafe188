"""Symmetric-extension pyramid timing under the crop switches:
    python scripts/probe_symmetric.py  (DWT2D_CROP_TILES=0|1, DWT2D_CROP_CORE=n)"""
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1704_08657_b200 as dwt
from paper_1704_08657_b200.synth import random_image
for n, L in ((4096, 1), (16384, 8)):
    img = random_image(n, n, 1, device="cuda"); out = torch.empty_like(img)
    for setting in [("0", "8"), ("1", "8"), ("1", "4"), ("1", "12")]:
        os.environ["DWT2D_CROP_TILES"], os.environ["DWT2D_CROP_CORE"] = setting
        plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True, extension="symmetric")
        plan.forward_mallat(img, L, out=out); torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); plan.forward_mallat(img, L, out=out); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
        print(n, L, setting, round(statistics.median(ts), 4), flush=True)
