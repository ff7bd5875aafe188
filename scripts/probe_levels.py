"""Marginal cost of each pyramid level in production conditions: K
forward_mallat calls of L levels captured in one CUDA graph (PDL between
levels, no events inside), for L = 1..8; the difference between L and L-1
is what level L adds to the pyramid.

    python scripts/probe_levels.py [--size 16384] [--iters 50]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--max-levels", type=int, default=8)
ap.add_argument("--tune", default="", help="k=v,... plan tuning")
a = ap.parse_args()
plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
if a.tune:
    plan.tune(**{k: int(v) for k, v in (kv.split("=") for kv in a.tune.split(","))})
img = random_image(a.size, a.size, 1, device="cuda")
out = torch.empty_like(img)
st = torch.cuda.Stream()
scratch = torch.empty(dwt.workspace_bytes(a.size, a.size, a.max_levels) // 4 + 64, device="cuda")
prev = 0.0
for L in range(1, a.max_levels + 1):
    with torch.cuda.stream(st):
        for _ in range(3):
            plan.forward_mallat(img, L, out=out, scratch=scratch, stream=st.cuda_stream)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(a.iters):
            plan.forward_mallat(img, L, out=out, scratch=scratch, stream=st.cuda_stream)
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        t0.record(st)
        g.replay()
        t1.record(st)
    t1.synchronize()
    us = t0.elapsed_time(t1) / a.iters * 1e3
    print(f"levels {L}: {us:8.1f} us per pyramid  (+{us - prev:6.1f})", flush=True)
    prev = us
