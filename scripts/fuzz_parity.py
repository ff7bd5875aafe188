"""Randomised parity sweep on the GPU (development harness; the checkers are
the test infrastructure of tests/: the float64 restatement oracle/dwt_oracle
and the compiled reference oracle/_ref).

Each case draws a wavelet, scheme, optimized flag, lowering, extension,
level count, image size, seed and execution-policy switches, and checks
  1. composed lowering: the fused pyramid == the reference's float32
     pyramid (oracle/_ref, ref_pyramid_f32) bit for bit;
  2. the pyramid vs the float64 restatement: per-level error <= 1e-5 of the
     level input's peak;
  3. the pyramid under random chunk rows / level pair / TMA staging / chunk
     order switches == the default pyramid bit for bit (periodic), and the
     generic per-sub-step executor == the fused kernels bit for bit;
  4. forward then inverse pyramid (same wavelet and extension) returns the
     image within 5e-5 of its peak — periodic, or symmetric lifting schemes:
     with symmetric extension the convolution schemes are not inverted by
     inverse lifting at the borders in the reference's own semantics either
     (float64 restatement: 0.15-0.85 max error at 64x48);
  5. the host entry point (pinned-copy pipeline) == the device pyramid.
    python scripts/fuzz_parity.py --minutes 15 --seed 1 > profiles/r02_fuzz_parity.txt"""
import argparse
import os
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from oracle import dwt_oracle as O  # noqa: E402  (checker only)
from oracle import ref as R  # noqa: E402  (checker only)

WAVELETS = ["cdf53", "cdf97", "dd137"]
SCHEMES = O.SCHEMES

ap = argparse.ArgumentParser()
ap.add_argument("--minutes", type=float, default=10.0)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--max-side", type=int, default=768)
a = ap.parse_args()
rng = random.Random(a.seed)
dev = torch.device("cuda:0")
t_end = time.time() + 60 * a.minutes
counts = {"cases": 0, "ref_bit_exact": 0, "oracle": 0, "policy_bit_exact": 0, "generic_bit_exact": 0,
          "round_trip": 0, "host_equal": 0}
fails = []
reported = 0
worst, worst_tag = 0.0, ""


def plan(w, s, opt, ext, low, generic=False, **tune):
    if generic:
        os.environ["DWT2D_FORCE_GENERIC"] = "1"
    try:
        p = dwt.Plan(w, s, optimized=opt, extension=ext, lowering=low)
    finally:
        os.environ.pop("DWT2D_FORCE_GENERIC", None)
    if tune:
        p.tune(**tune)
    return p


while time.time() < t_end:
    w = rng.choice(WAVELETS)
    s = rng.choice(SCHEMES)
    opt = rng.random() < 0.5
    ext = "symmetric" if rng.random() < 0.3 else "periodic"
    low = rng.choice(["default", "composed"])
    L = rng.randint(1, 5)
    kmin = 3 if ext == "symmetric" else 1
    kmax = max(kmin, a.max_side >> L)
    W = (rng.randint(kmin, kmax)) << L
    H = (rng.randint(kmin, kmax)) << L
    seed = rng.randint(1, 10 ** 6)
    sym = ext == "symmetric"
    tag = f"{w}/{s}/{'opt' if opt else 'base'}/{low}/{ext} {W}x{H} L{L} seed {seed}"
    counts["cases"] += 1
    try:
        img = O.random_image(W, H, seed)
        x = torch.from_numpy(img).to(dev)
        p = plan(w, s, opt, ext, low)
        got = p.forward_mallat(x, L).cpu().numpy()
        if low == "composed" and R.available():
            ref = R.pyramid(w, s, img, L, optimized=opt, symmetric=sym)
            if not np.array_equal(got, ref):
                fails.append(f"REF {tag}: {int(np.sum(got != ref))} samples differ")
            else:
                counts["ref_bit_exact"] += 1
        truth = O.pyramid(w, s, img, L, opt, sym)
        e = max(O.level_errors(got, truth, img, L))
        if e > worst:
            worst, worst_tag = e, tag
        if e > 1e-5:
            fails.append(f"ORACLE {tag}: per-level error {e:.3e}")
        else:
            counts["oracle"] += 1
        if not sym:
            tune = {"chunk_rows": rng.choice([0, 1, 2, 3, 7, 16, 64]), "pair": rng.choice([0, 1, 2]),
                    "tma": rng.choice([0, 1, 2]), "alternate": rng.choice([0, 1, 2])}
            alt = plan(w, s, opt, ext, low, **tune).forward_mallat(x, L).cpu().numpy()
            if not np.array_equal(alt, got):
                fails.append(f"POLICY {tag} {tune}: {int(np.sum(alt != got))} samples differ")
            else:
                counts["policy_bit_exact"] += 1
        gen = plan(w, s, opt, ext, low, generic=True).forward_mallat(x, L).cpu().numpy()
        if not np.array_equal(gen, got):
            fails.append(f"GENERIC {tag}: {int(np.sum(gen != got))} samples differ")
        else:
            counts["generic_bit_exact"] += 1
        if not sym or "lifting" in s:
            inv = dwt.Plan(w, "inverse-lifting", extension=ext)
            back = inv.inverse_mallat(torch.from_numpy(got).to(dev), L).cpu().numpy()
            rt = float(np.max(np.abs(back.astype(np.float64) - img))) / (float(np.max(np.abs(img))) or 1.0)
            if rt > 5e-5:
                fails.append(f"ROUNDTRIP {tag}: {rt:.3e}")
            else:
                counts["round_trip"] += 1
        host = p.forward_mallat_host(img, L)
        if not np.array_equal(host, got):
            fails.append(f"HOST {tag}: {int(np.sum(host != got))} samples differ")
        else:
            counts["host_equal"] += 1
    except Exception as ex:  # noqa: BLE001
        fails.append(f"EXCEPTION {tag}: {type(ex).__name__}: {ex}")
    while reported < len(fails):
        print("FAIL " + fails[reported], flush=True)
        reported += 1
    if counts["cases"] % 25 == 0:
        print(f"... {counts} worst per-level error {worst:.3e} failures {len(fails)}", flush=True)

print(f"seed {a.seed}, {a.minutes} min: {counts}")
print(f"worst per-level error vs float64 oracle: {worst:.3e} (bar 1e-5) at {worst_tag}")
print(f"failures: {len(fails)}")
kinds = {}
for f in fails:
    kinds[f.split()[0]] = kinds.get(f.split()[0], 0) + 1
print(f"failures by check: {kinds}")
