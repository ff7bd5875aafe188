"""Development probe (one B200): per program, the 16384^2 8-level pyramid
with the fused level pair (pair=1) against one launch per level (pair=0),
and single-level knob sweeps (chunk rows, bottom-up chunks, TMA staging).
L2 flushed before every run, CUDA events, median of 15.
    python scripts/probe_pair_programs.py [--sweep wavelet/scheme/opt|base]"""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

flush = None


def timed(fn, reps=15):
    global flush
    if flush is None:
        flush = torch.empty(128 << 20, device="cuda")
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweep", default="")
    ap.add_argument("--alt", action="store_true", help="bottom-up odd chunks on/off per program")
    a = ap.parse_args()
    n = 16384
    img = random_image(n, n, 1, device="cuda")
    if a.sweep:
        w, s, o = a.sweep.split("/")
        plan = dwt.Plan(w, s, optimized=o == "opt")
        bands = [torch.empty((n // 2, n // 2), device="cuda") for _ in range(4)]
        for tma in (1, 0):
            for alt in (1, 0):
                for chunk in (0, 16, 32, 64, 128):
                    plan.tune(tma=tma, alternate=alt, chunk_rows=chunk)
                    plan.forward_level(img, bands)
                    t = timed(lambda: plan.forward_level(img, bands))
                    print(f"{a.sweep} tma {tma} alternate {alt} chunk_rows {chunk:3d}: {t * 1e3:7.1f} us", flush=True)
        return
    if a.alt:
        bands = [torch.empty((n // 2, n // 2), device="cuda") for _ in range(4)]
        for s in ["separable-convolution", "separable-lifting", "nonseparable-convolution",
                  "nonseparable-polyconvolution", "nonseparable-lifting"]:
            for o in (False, True):
                plan = dwt.Plan("cdf97", s, optimized=o)
                res = {}
                for alt in (1, 0):
                    plan.tune(alternate=alt)
                    plan.forward_level(img, bands)
                    res[alt] = timed(lambda: plan.forward_level(img, bands))
                print(f"cdf97 {s} {'opt' if o else 'base'} 16384^2 level: alternate {res[1] * 1e3:.1f} us, "
                      f"top-down only {res[0] * 1e3:.1f} us", flush=True)
        return
    out = torch.empty_like(img)
    scratch = torch.empty(dwt.workspace_bytes(n, n, 8) // 4 + 64, device="cuda")
    for w, s, o in [("cdf97", "separable-convolution", True), ("cdf97", "nonseparable-polyconvolution", True),
                    ("cdf97", "separable-lifting", True), ("cdf97", "nonseparable-lifting", True),
                    ("cdf97", "separable-lifting", False), ("cdf97", "nonseparable-lifting", False)]:
        plan = dwt.Plan(w, s, optimized=o)
        res = {}
        for pair in (0, 1):
            plan.tune(pair=pair)
            plan.forward_mallat(img, 8, out=out, scratch=scratch)
            res[pair] = timed(lambda: plan.forward_mallat(img, 8, out=out, scratch=scratch))
        print(f"{w} {s} {'opt' if o else 'base'}: 8-level pyramid per-level {res[0] * 1e3:.1f} us, "
              f"pair {res[1] * 1e3:.1f} us", flush=True)


if __name__ == "__main__":
    main()
