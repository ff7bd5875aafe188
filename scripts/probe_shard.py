"""Per-step phases of the sharded strip pyramid (ring of `--world` virtual
ranks on one GPU, one stream each): push / interior / wait / border times
from CUDA events, and the whole pyramid from a graph of K pyramids.

    python scripts/probe_shard.py [--size 16384] [--world 1] [--levels 8]
"""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200 import strips as S  # noqa: E402
from paper_1704_08657_b200.native import Event  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--world", type=int, default=1)
ap.add_argument("--levels", type=int, default=8)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
Hs = a.size // a.world
img = random_image(a.size, a.size, 1, device="cuda")
strips = [img[r * Hs:(r + 1) * Hs] for r in range(a.world)]
outs = [torch.empty_like(s) for s in strips]
shards = [S.Shard(plan, a.size, Hs, a.levels, r, a.world) for r in range(a.world)]
S.connect_ring(shards)
streams = [torch.cuda.Stream() for _ in range(a.world)]
nsteps = shards[0].info()["steps"]
for _ in range(3):
    for sh, s, o, st in zip(shards, strips, outs, streams):
        sh.forward_mallat(s, out=o, stream=st)
try:
    torch.cuda.synchronize()
except Exception:
    for sh in shards:
        print("rank", sh.rank, sh.status(), sh.status_message())
    raise
evs = [[Event() for _ in range(1 + 4 * nsteps)] for _ in range(a.iters)]
for k in range(a.iters):
    for r, (sh, s, o, st) in enumerate(zip(shards, strips, outs, streams)):
        sh.forward_mallat(s, out=o, stream=st, events=evs[k] if r == 0 else None)
try:
    torch.cuda.synchronize()
except Exception:
    for sh in shards:
        print("rank", sh.rank, sh.status(), sh.status_message())
    raise
for e in range(nsteps):
    b = 1 + 4 * e
    ph = [statistics.mean(x[i].elapsed_ms(x[i + 1]) for x in evs) * 1e3 for i in (b - 1, b, b + 1, b + 2)]
    print(f"step {e}: push {ph[0]:8.2f} us  interior {ph[1]:8.2f}  wait {ph[2]:8.2f}  border {ph[3]:8.2f}")
g = torch.cuda.CUDAGraph()
st = streams[0]
with torch.cuda.graph(g, stream=st):
    for _ in range(a.iters):
        for sh, s, o in zip(shards, strips, outs):
            sh.forward_mallat(s, out=o, stream=st) if a.world == 1 else None
if a.world == 1:
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        t0.record(st)
        g.replay()
        t1.record(st)
    t1.synchronize()
    print(f"graph: {t0.elapsed_time(t1) / a.iters * 1e3:.1f} us per pyramid; "
          f"single-GPU forward_mallat for comparison below")
    full = torch.empty_like(img)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=st):
        for _ in range(a.iters):
            plan.forward_mallat(img, a.levels, out=full, stream=st.cuda_stream)
    with torch.cuda.stream(st):
        g2.replay()
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        t0.record(st)
        g2.replay()
        t1.record(st)
    t1.synchronize()
    print(f"graph: {t0.elapsed_time(t1) / a.iters * 1e3:.1f} us per single-GPU pyramid")
