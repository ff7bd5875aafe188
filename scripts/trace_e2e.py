"""Timeline of the host pipeline (dwt2d_forward_mallat_host) at 16384^2, 8
levels: timing events on its upload / compute / download streams (tuning
host_trace), printed to stderr by the library.
    python scripts/trace_e2e.py [--taper 0|1] [--levels-pipe 2]"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--taper", type=int, default=0)
ap.add_argument("--levels-pipe", type=int, default=0)
a = ap.parse_args()
n = a.size
img = random_image(n, n, 1, device="cuda").cpu().pin_memory()
out = torch.empty_like(img).pin_memory()
hi, ho = img.numpy(), out.numpy()
plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True).tune(host_taper=a.taper, host_levels=a.levels_pipe)
for _ in range(3):
    plan.forward_mallat_host(hi, 8, ho)
t0 = time.perf_counter()
plan.forward_mallat_host(hi, 8, ho)
print(f"wall {1e3 * (time.perf_counter() - t0):.2f} ms (untraced)", file=sys.stderr, flush=True)
plan.tune(host_trace=1)
t0 = time.perf_counter()
plan.forward_mallat_host(hi, 8, ho)
print(f"wall {1e3 * (time.perf_counter() - t0):.2f} ms (traced)", file=sys.stderr, flush=True)
