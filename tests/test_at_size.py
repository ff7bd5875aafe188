"""Parity at BASELINE.json's configuration sizes, with the production
run-time policy (the size-dependent switches — TMA staging at >= 512 MiB,
bottom-up chunks at >= 32 MiB, the fused level pair where level 1 is
staged — are all active at these sizes and at none of the small sizes of
test_gpu_parity.py).

* configs[1]: 4096^2, every CDF 9/7 scheme x {baseline, optimized}, one
  level, vs the float64 oracle over the whole image (SURVEY §8(c) metric);
  composed baselines bit for bit vs the reference's own float32 executor
  (oracle/_ref, reference test_executor.cpp:161-182, acceptance.cpp:160-198).
* configs[3]: the 16384^2 8-level pyramid as the bench runs it. Levels 1-4:
  oracle crop windows cut from the pyramid output itself (corners with the
  periodic wrap and interior points; a crop reproduces the level exactly
  beyond a margin of the level's reach). Levels 5-8 and
  LL_8: the whole level vs the float64 oracle run on the GPU's own LL_4.
  Plus: the fused level pair equals one launch per level bit for bit at this
  size and chunking.
* configs[2]: polyconvolution forward + inverse round trips, 1024^2 ..
  16384^2 (the sweep's numbers as assertions).
* configs[4]: the 65536^2 strip pyramid with 2/4/8 virtual ranks equals the
  single-GPU pyramid bit for bit (tests/test_sharded.py at 65536^2).
* the device LCG (synth.random_image, the input of every full-size test and
  the bench) equals the reference generator (random.hpp:13-37) bit for bit,
  for row bands starting at row0 != 0.
"""
import os

import numpy as np
import pytest
import torch

from oracle import dwt_oracle as O
from oracle import ref as R

pytestmark = pytest.mark.gpu

TOL = 1e-5
CPUS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def dwt():
    import paper_1704_08657_b200 as d
    return d


def _ref():
    if not R.available():
        pytest.skip("oracle/_ref not built")


# ------------------------------------------------------------- configs[1]

VARIANTS = [(s, o) for s in O.SCHEMES for o in (False, True)]


@pytest.fixture(scope="module")
def img4096(cuda):
    from paper_1704_08657_b200.synth import random_image
    return random_image(4096, 4096, 1, device="cuda")


@pytest.mark.parametrize("scheme,opt", VARIANTS)
def test_config1_4096_every_variant_vs_float64(dwt, img4096, scheme, opt):
    plan = dwt.Plan("cdf97", scheme, optimized=opt)
    got = [b.cpu().numpy() for b in plan.forward_level(img4096)]
    planes = O.split(img4096.cpu().numpy())
    truth = O.transform("cdf97", scheme, planes, opt)
    peak = float(max(np.max(np.abs(p)) for p in planes))
    err = max(float(np.max(np.abs(g.astype(np.float64) - t))) for g, t in zip(got, truth)) / peak
    assert err <= TOL, (scheme, opt, err)


@pytest.mark.parametrize("scheme", O.SCHEMES)
def test_config1_4096_composed_bit_exact_vs_reference(dwt, img4096, scheme):
    _ref()
    plan = dwt.Plan("cdf97", scheme, optimized=False, lowering="composed")
    planes_dev = [p.contiguous() for p in plan.forward_level(img4096)]  # warm: also the image path
    planes = O.split(img4096.cpu().numpy())
    got = [t.cpu().numpy() for t in plan.run([torch.from_numpy(p).cuda() for p in planes])]
    ref, _ = R.run("cdf97", scheme, planes, optimized=False, workers=CPUS)
    for j in range(4):
        assert np.array_equal(got[j], ref[j]), (scheme, j, int(np.sum(got[j] != ref[j])))
        # the image-input kernel (split fused into the loads) gives the same bits
        assert np.array_equal(planes_dev[j].cpu().numpy(), ref[j]), (scheme, j)


# ------------------------------------------------------------- configs[3]

N3, L3 = 16384, 8


@pytest.fixture(scope="module")
def pyr16k(dwt, cuda):
    from paper_1704_08657_b200.synth import random_image
    img = random_image(N3, N3, 1, device="cuda")
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    out8 = plan.forward_mallat(img, L3)
    torch.cuda.synchronize()
    return img, plan, out8


def _bands(mallat, W, H, level):
    """(LL or None, HL, LH, HH) views of `level` (1-based) in a Mallat buffer."""
    w, h = W >> (level - 1), H >> (level - 1)
    w2, h2 = w // 2, h // 2
    return (mallat[:h2, :w2], mallat[:h2, w2:w], mallat[h2:h, :w2], mallat[h2:h, w2:w])


def _crop_levels(img_np, level, y0, x0, size, margin):
    """Float64 oracle levels 1..level on the image crop whose level-`level`
    component window is [y0 - margin, y0 + size + margin) x (same in x),
    periodic wrap of the whole image for windows crossing its edges. Returns
    (bands of `level` on [margin, margin + size)^2, peak |level input|)."""
    f = 1 << level
    rows = np.arange((y0 - margin) * f, (y0 + size + margin) * f)
    cols = np.arange((x0 - margin) * f, (x0 + size + margin) * f)
    cur = np.take(np.take(img_np, rows, axis=0, mode="wrap"), cols, axis=1, mode="wrap").astype(np.float64)
    for _ in range(level):
        inp = cur
        res = O.transform("cdf97", "nonseparable-lifting", O.split(cur), True)
        cur = res[0]
    c = slice(margin, margin + size)
    peak = float(np.max(np.abs(inp[2 * margin:2 * (margin + size), 2 * margin:2 * (margin + size)])))
    return [r[c, c] for r in res], peak


@pytest.mark.parametrize("level", [1, 2, 3, 4])
def test_config3_pyramid_levels_1_to_4_crops(pyr16k, level):
    img, plan, out8 = pyr16k
    img_np = img.cpu().numpy()
    h2 = N3 >> level
    size, margin = 48, 16
    got_bands = _bands(out8, N3, N3, level)
    for (y0, x0) in [(0, 0), (h2 - size, h2 - size), (0, h2 - size // 2), (h2 // 2 + 7, h2 // 3 + 5)]:
        # windows crossing the image edge wrap (periodic): gather them the same way
        ys = np.arange(y0, y0 + size) % h2
        xs = np.arange(x0, x0 + size) % h2
        truth, peak = _crop_levels(img_np, level, y0, x0, size, margin)
        err = 0.0
        for j in (1, 2, 3):  # HL, LH, HH are stored at this level; LL feeds the next
            g = got_bands[j].cpu().numpy()[np.ix_(ys, xs)].astype(np.float64)
            err = max(err, float(np.max(np.abs(g - truth[j]))))
        assert err / peak <= TOL, (level, y0, x0, err / peak)


def test_config3_pyramid_levels_5_to_8_whole(dwt, pyr16k):
    img, plan, out8 = pyr16k
    out4 = plan.forward_mallat(img, 4)
    torch.cuda.synchronize()
    q = N3 >> 4
    # levels 1-4 of the 8-level pyramid are the 4-level pyramid's bits
    same = out8 == out4
    same[:q, :q] = True
    assert bool(same.all())
    cur = out4[:q, :q].double().cpu().numpy()  # the GPU's LL_4
    got = out8.cpu().numpy()
    for level in range(5, L3 + 1):
        peak = float(np.max(np.abs(cur)))
        res = O.transform("cdf97", "nonseparable-lifting", O.split(cur), True)
        bands = _bands(got, N3, N3, level)
        js = (0, 1, 2, 3) if level == L3 else (1, 2, 3)
        err = max(float(np.max(np.abs(bands[j].astype(np.float64) - res[j]))) for j in js)
        assert err / peak <= TOL, (level, err / peak)
        cur = res[0]


def test_config3_pair_equals_per_level_launches(dwt, pyr16k):
    img, plan, out8 = pyr16k
    per_level = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True).tune(pair=0)
    before = dwt.launch_count()
    b = per_level.forward_mallat(img, L3)
    torch.cuda.synchronize()
    assert dwt.launch_count() - before == L3
    assert torch.equal(out8, b)


def test_config3_host_pipeline_equals_device(dwt, pyr16k):
    """The e2e entry point (host image in, host pyramid out, transfers
    overlapped with level 1 by row bands) gives the device pyramid's bits."""
    img, plan, out8 = pyr16k
    host = plan.forward_mallat_host(img.cpu().numpy(), L3)
    assert np.array_equal(host, out8.cpu().numpy())


# ------------------------------------------------------------- configs[2]

@pytest.mark.parametrize("n", [1024, 2048, 4096, 8192, 16384])
@pytest.mark.parametrize("opt", [False, True])
def test_config2_polyconvolution_round_trip(dwt, cuda, n, opt):
    from paper_1704_08657_b200.synth import random_image
    img = random_image(n, n, 1, device="cuda")
    fwd = dwt.Plan("cdf97", "nonseparable-polyconvolution", optimized=opt)
    inv = dwt.Plan("cdf97", "inverse-lifting")
    back = inv.inverse_level(fwd.forward_level(img))
    torch.cuda.synchronize()
    err = float((back - img).abs().max())
    assert err <= 2e-5, (n, opt, err)  # measured 6e-6 (profiles/r01_configs.jsonl)


# ---------------------------------------------------------- device LCG

@pytest.fixture(scope="module")
def ref_image_16k():
    _ref()
    return R.random_image(N3, N3, 1)


@pytest.mark.parametrize("row0,rows", [(0, 64), (1, 3), (8191, 130), (12345, 1000), (N3 - 17, 17)])
def test_device_lcg_matches_reference_generator(ref_image_16k, cuda, row0, rows):
    from paper_1704_08657_b200.synth import random_image
    band = random_image(N3, N3, 1, row0=row0, rows=rows, device="cuda").cpu().numpy()
    assert np.array_equal(band, ref_image_16k[row0:row0 + rows])


def test_device_lcg_whole_16384_image(ref_image_16k, cuda):
    from paper_1704_08657_b200.synth import random_image
    img = random_image(N3, N3, 1, device="cuda")
    assert torch.equal(img, torch.from_numpy(ref_image_16k).to(cuda))
