"""Wavefront pyramid probe: times forward_mallat (CUDA events, eager calls)
for a list of scheduler settings given as env assignments, e.g.

    python scripts/wave_probe.py "DWT2D_WAVEFRONT=0" "DWT2D_WAVE_LAG=3 DWT2D_WAVE_CHUNK_ROWS=8" --levels 8

Each setting is applied with os.environ before its calls (the library reads
these variables on every call)."""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

KNOBS = ["DWT2D_PAIR", "DWT2D_PAIR_DEEP", "DWT2D_PAIR_CHUNK_ROWS", "DWT2D_PDL", "DWT2D_LEVEL_CHUNK_ROWS", "DWT2D_WAVEFRONT", "DWT2D_WAVE_FROM", "DWT2D_WAVE_LAG", "DWT2D_WAVE_CHUNK_ROWS", "DWT2D_CHUNK_ROWS"]

ap = argparse.ArgumentParser()
ap.add_argument("settings", nargs="+")
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--levels", type=int, default=8)
ap.add_argument("--iters", type=int, default=30)
a = ap.parse_args()
plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
img = random_image(a.size, a.size, 1, device="cuda")
out = torch.empty_like(img)
scratch = torch.empty(dwt.workspace_bytes(a.size, a.size, a.levels) // 4 + 64, device="cuda")
ref = None
for s in a.settings:
    for k in KNOBS:
        os.environ.pop(k, None)
    for kv in s.split():
        k, v = kv.split("=")
        os.environ[k] = v
    for _ in range(3):
        plan.forward_mallat(img, a.levels, out=out, scratch=scratch)
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    same = bool(torch.equal(ref, out))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        plan.forward_mallat(img, a.levels, out=out, scratch=scratch)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    print(f"{s:60s} L={a.levels} {ms:.4f} ms  {a.size * a.size / ms / 1e6:.1f} Gpix/s  same={same}", flush=True)
