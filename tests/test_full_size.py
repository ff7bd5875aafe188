"""Parity at BASELINE.json's full sizes through size-independent properties
(the float64 oracle cannot run 256-Mpixel or 4-Gpixel images in seconds):

* round trip: the 8-level forward pyramid (levels 1+2 fused, TMA-staged rows)
  followed by the inverse pyramid reproduces the image (float32 bar 5e-5);
* crop windows: the interior of a GPU level equals the float64 oracle on a
  crop of the image with a margin larger than the program's reach (the
  oracle's periodic wrap on the crop only reaches the margin);
* linearity: F(a x + y) = a F(x) + F(y) to float32 rounding;
* constant image: CDF 5/3 detail bands exactly zero (test_executor.cpp:198-211).

configs[3] (16384², 8 levels) and the per-GPU image of configs[4] (65536²).
"""
import numpy as np
import pytest
import torch

from oracle import dwt_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dwt():
    import paper_1704_08657_b200 as d
    return d


def _crop_check(plan, w, s, opt, img, bands, y0, x0, size=128, margin=16):
    """GPU level bands (planar, component grid) vs the oracle on a crop."""
    crop = img[2 * (y0 - margin):2 * (y0 + size + margin), 2 * (x0 - margin):2 * (x0 + size + margin)]
    truth = O.transform(w, s, O.split(crop.double().cpu().numpy()), opt)
    peak = float(crop.abs().max())
    err = 0.0
    for j in range(4):
        got = bands[j][y0:y0 + size, x0:x0 + size].double().cpu().numpy()
        ref = truth[j][margin:margin + size, margin:margin + size]
        err = max(err, float(np.max(np.abs(got - ref))))
    return err / peak


@pytest.mark.parametrize("n", [16384, 65536])
def test_full_size_round_trip_and_crops(dwt, n):
    from paper_1704_08657_b200.synth import random_image
    L = 8
    img = random_image(n, n, 1, device="cuda")
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    inv = dwt.Plan("cdf97", "inverse-lifting")
    coeffs = plan.forward_mallat(img, L)
    back = inv.inverse_mallat(coeffs, L)
    torch.cuda.synchronize()
    assert float((back - img).abs().max()) <= 5e-5
    del back, coeffs
    # level-1 crops: corners (periodic wrap) and interior
    bands = plan.forward_level(img)
    h2 = n // 2
    for (y0, x0) in [(16, 16), (h2 // 2, h2 // 3), (h2 - 144, h2 - 144)]:
        assert _crop_check(plan, "cdf97", "nonseparable-lifting", True, img, bands, y0, x0) <= 1e-5
    del bands
    torch.cuda.empty_cache()


def test_full_size_linearity(dwt):
    from paper_1704_08657_b200.synth import random_image
    n, L = 16384, 8
    x = random_image(n, n, 1, device="cuda")
    y = random_image(n, n, 2, device="cuda")
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    a = 0.5
    lhs = plan.forward_mallat(a * x + y, L)
    rhs = a * plan.forward_mallat(x, L) + plan.forward_mallat(y, L)
    torch.cuda.synchronize()
    # coefficients grow by up to ~130x over 8 levels (LL_8): relative bar
    assert float((lhs - rhs).abs().max()) <= 1e-5 * float(rhs.abs().max())


def test_full_size_constant_image_cdf53(dwt):
    n, L = 16384, 8
    img = torch.full((n, n), 0.375, device="cuda")
    for s in ["separable-lifting", "nonseparable-lifting"]:
        plan = dwt.Plan("cdf53", s, optimized=True)
        out = plan.forward_mallat(img, L).cpu().numpy()
        w = n >> L
        ll = out[:w, :w].copy()
        out[:w, :w] = 0.0
        assert np.count_nonzero(out) == 0, s  # every detail band exactly zero
        assert np.all(ll == np.float32(0.375)), s
