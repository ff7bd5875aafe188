"""Randomised parity sweep of the row-strip sharded pyramid
(dwt2d_forward_mallat_sharded; virtual ranks sharing cuda:0, device-side
halo exchange through the ranks' exchange windows): random ring size,
program, level-pair policy, levels and strip geometry; the assembled strip
pyramids must equal the single-GPU pyramid bit for bit. Geometries whose
deepest strips are thinner than the level halo are rejected by the driver
(DWT2D_EINVAL) and counted separately.
    python scripts/fuzz_sharded.py --minutes 8 --seed 1"""
import argparse
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200 import strips as S  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

PROGRAMS = [("cdf97", "nonseparable-lifting", True), ("cdf97", "nonseparable-lifting", False),
            ("cdf97", "separable-lifting", True), ("cdf97", "separable-convolution", False),
            ("cdf97", "nonseparable-polyconvolution", True), ("cdf97", "nonseparable-convolution", True),
            ("cdf53", "separable-lifting", False), ("cdf53", "nonseparable-lifting", True),
            ("dd137", "nonseparable-lifting", True), ("dd137", "separable-lifting", False)]

ap = argparse.ArgumentParser()
ap.add_argument("--minutes", type=float, default=8.0)
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
rng = random.Random(a.seed)
t_end = time.time() + 60 * a.minutes
n = {"cases": 0, "bit_exact": 0, "rejected_thin": 0}
fails = []
while time.time() < t_end:
    w, s, opt = rng.choice(PROGRAMS)
    world = rng.choice([2, 3, 4, 5, 6, 8])
    L = rng.randint(1, 6)
    pair = rng.choice([0, 1, 2])
    W = rng.randint(4, 48) << L
    Hs = rng.randint(1, 24) << L
    seed = rng.randint(1, 10 ** 6)
    tag = f"{w}/{s}/{'opt' if opt else 'base'} world {world} {W}x{Hs}/rank L{L} pair {pair} seed {seed}"
    n["cases"] += 1
    plan = dwt.Plan(w, s, optimized=opt).tune(pair=pair)
    img = random_image(W, Hs * world, seed, device="cuda")
    strips = [img[r * Hs:(r + 1) * Hs].contiguous() for r in range(world)]
    try:
        outs = S.forward_mallat_sharded(plan, strips, L)
    except (ValueError, dwt.DwtError) as e:
        if "thinner" in str(e):
            n["rejected_thin"] += 1
            continue
        fails.append(f"ERROR {tag}: {e}")
        print("FAIL " + fails[-1], flush=True)
        continue
    full = plan.forward_mallat(img, L)
    torch.cuda.synchronize()
    if torch.equal(S.assemble_mallat(outs, L), full.cpu()):
        n["bit_exact"] += 1
    else:
        fails.append(f"DIFF {tag}")
        print("FAIL " + fails[-1], flush=True)
    del plan, outs, full, strips, img
print(f"seed {a.seed}, {a.minutes} min: {n}; failures {len(fails)}")
