"""GPU parity: the sm_100a level kernels against the CPU oracles.

Oracles (test infrastructure, oracle/):
  * oracle.dwt_oracle — float64 numpy restatement of the reference path
    (pinned against the compiled reference in test_oracle.py)
  * oracle.ref        — the compiled reference itself (oracle/_ref), float32
    and float64 executors

Tolerance (north star): per level, max |gpu - float64 truth|
over the bands written at that level divided by the peak |input| of the
level must be <= 1e-5. Composed lowerings use the reference's exact tap
tables, accumulation order and rounding, so they are additionally compared
bit for bit with the reference's float32 executor.
"""
import numpy as np
import pytest

from oracle import dwt_oracle as O
from oracle import ref as R

pytestmark = pytest.mark.gpu

WAVELETS = ["cdf53", "cdf97", "dd137"]
FORWARD = O.SCHEMES
TOL = 1e-5


def _plans():
    out = []
    for w in WAVELETS:
        for s in FORWARD:
            out.append((w, s, False))
            out.append((w, s, True))
        out.append((w, "inverse-lifting", False))
    return out


PLANS = _plans()


@pytest.fixture(scope="module")
def dwt():
    import paper_1704_08657_b200 as d
    return d


def _to_dev(planes, cuda):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(p, dtype=np.float32)).to(cuda) for p in planes]


def _err(got, truth, peak):
    return max(float(np.max(np.abs(g.astype(np.float64) - t))) for g, t in zip(got, truth)) / peak


# (w2, h2): vector path, odd widths (scalar path), tiny grids that wrap
# several times, a wide-and-short and a tall-and-narrow strip
SIZES = [(64, 48), (33, 17), (1, 1), (3, 2), (200, 6), (5, 130)]


@pytest.mark.parametrize("w,s,opt", PLANS)
def test_run_planar_matches_float64_oracle(dwt, cuda, w, s, opt):
    import torch
    plan = dwt.Plan(w, s, optimized=opt)
    scheme = O.make(w, s, opt)
    for (w2, h2) in SIZES:
        img = O.random_image(2 * w2, 2 * h2, 12345 + w2 * 7 + h2)
        planes = O.split(img)
        got = [t.cpu().numpy() for t in plan.run(_to_dev(planes, cuda))]
        torch.cuda.synchronize()
        truth = O.run(scheme, planes)
        peak = max(float(np.max(np.abs(p))) for p in planes) or 1.0
        e = _err(got, truth, peak)
        assert e <= TOL, f"{w}/{s}/opt={opt} {w2}x{h2}: err {e:.3e}"


@pytest.mark.parametrize("w,s,opt", [p for p in PLANS if not p[2]])
def test_composed_bit_exact_vs_reference_float32(dwt, cuda, w, s, opt):
    """Composed lowering == the reference float32 executor, bit for bit
    (same taps, same order, same product-then-sum rounding)."""
    if not R.available():
        pytest.skip("oracle/_ref not built")
    plan = dwt.Plan(w, s, optimized=opt, lowering="composed")
    for (w2, h2) in [(64, 48), (33, 17), (3, 2)]:
        img = O.random_image(2 * w2, 2 * h2, 99 + w2)
        planes = O.split(img)
        got = [t.cpu().numpy() for t in plan.run(_to_dev(planes, cuda))]
        ref, _ = R.run(w, s, planes, optimized=opt)
        for j in range(4):
            assert np.array_equal(got[j], ref[j]), (
                f"{w}/{s} {w2}x{h2} comp {j}: {int(np.sum(got[j] != ref[j]))} samples differ, "
                f"max {float(np.max(np.abs(got[j] - ref[j]))):.3e}")


@pytest.mark.parametrize("w,s,opt", [p for p in PLANS if p[1] != "inverse-lifting"])
def test_forward_level_from_image_equals_planar(dwt, cuda, w, s, opt):
    """polyphase split fused into the load gives the same bits as run() on
    pre-split planes."""
    import torch
    plan = dwt.Plan(w, s, optimized=opt)
    img = O.random_image(256, 96, 7)
    a = plan.forward_level(torch.from_numpy(img).to(cuda))
    b = plan.run(_to_dev(O.split(img), cuda))
    for j in range(4):
        assert torch.equal(a[j], b[j])


@pytest.mark.parametrize("w", WAVELETS)
def test_inverse_level_to_image(dwt, cuda, w):
    import torch
    inv = dwt.Plan(w, "inverse-lifting")
    planes = _to_dev(O.split(O.random_image(128, 64, 3)), cuda)
    img = inv.inverse_level(planes)
    ref = inv.run(planes)
    merged = O.merge([t.cpu().numpy() for t in ref])
    assert np.array_equal(img.cpu().numpy(), merged)


@pytest.mark.parametrize("w,s,opt", [(w, s, o) for w in WAVELETS for s in FORWARD for o in (False, True)])
def test_round_trip_every_scheme(dwt, cuda, w, s, opt):
    """forward(any scheme) then inverse lifting restores the planes
    (test_executor.cpp:279-299 periodic case)."""
    import torch
    fwd = dwt.Plan(w, s, optimized=opt)
    inv = dwt.Plan(w, "inverse-lifting")
    planes = _to_dev(O.split(O.random_image(128, 96, 404)), cuda)
    back = inv.run(fwd.run(planes))
    e = max(float((b - p).abs().max()) for b, p in zip(back, planes))
    assert e <= 2e-5 * (8 if w == "dd137" else 1), e


@pytest.mark.parametrize("w,s,opt", [("cdf97", "nonseparable-lifting", True),
                                     ("cdf97", "nonseparable-lifting", False),
                                     ("cdf97", "separable-lifting", False),
                                     ("cdf97", "nonseparable-polyconvolution", True),
                                     ("cdf97", "nonseparable-convolution", False),
                                     ("cdf97", "separable-convolution", True),
                                     ("cdf53", "separable-lifting", False),
                                     ("dd137", "nonseparable-lifting", True)])
def test_mallat_pyramid_per_level_tolerance(dwt, cuda, w, s, opt):
    """Multi-level against the float64 oracle pyramid with
    the per-level normalised error of §8(c)."""
    import torch
    W, H, L = 256, 192, 5
    img = O.random_image(W, H, 1)
    plan = dwt.Plan(w, s, optimized=opt)
    got = plan.forward_mallat(torch.from_numpy(img).to(cuda), L).cpu().numpy()
    truth = O.pyramid(w, s, img, L, opt)
    errs = O.level_errors(got, truth, img, L)
    assert max(errs) <= TOL, errs
    if R.available():
        ref32 = R.pyramid(w, s, img, L, optimized=opt)
        errs_ref = O.level_errors(ref32, truth, img, L)
        # the GPU is at least as close to float64 as the reference's own float path (x4 slack)
        assert max(errs) <= max(4 * max(errs_ref), 1e-6), (errs, errs_ref)


@pytest.mark.parametrize("w", WAVELETS)
def test_mallat_inverse_round_trip(dwt, cuda, w):
    import torch
    W, H, L = 512, 256, 6
    img = torch.from_numpy(O.random_image(W, H, 9)).to(cuda)
    fwd = dwt.Plan(w, "nonseparable-lifting", optimized=True)
    inv = dwt.Plan(w, "inverse-lifting")
    back = inv.inverse_mallat(fwd.forward_mallat(img, L), L)
    assert float((back - img).abs().max()) <= 5e-5


def test_host_entry_points_match_device(dwt, cuda):
    import torch
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    img = O.random_image(512, 256, 5)
    dev = plan.forward_mallat(torch.from_numpy(img).to(cuda), 4).cpu().numpy()
    host = plan.forward_mallat_host(img, 4)
    assert np.array_equal(dev, host)
    planes = O.split(img)
    a = plan.run_host(planes)
    b = [t.cpu().numpy() for t in plan.run(_to_dev(planes, cuda))]
    for j in range(4):
        assert np.array_equal(a[j], b[j])
    inv = dwt.Plan("cdf97", "inverse-lifting")
    back = inv.inverse_mallat_host(host, 4)
    assert float(np.max(np.abs(back - img))) <= 5e-5


@pytest.mark.parametrize("w,s,opt", [("cdf97", "nonseparable-lifting", True), ("cdf53", "separable-lifting", False),
                                     ("dd137", "nonseparable-lifting", True),
                                     ("cdf97", "nonseparable-convolution", False)])
def test_tma_staged_rows_bit_exact(dwt, cuda, w, s, opt, monkeypatch):
    """Input rows staged by TMA bulk copies (forced on every size with
    DWT2D_TMA=2) give the same bits as register prefetch: images narrower
    than one warp strip (several wraps per row), strips crossing the right
    edge, ragged chunks, pitched input views, pyramids."""
    import torch
    plan = dwt.Plan(w, s, optimized=opt)
    for W, H in [(64, 40), (256, 200), (2400, 96), (1024, 1024)]:
        base = torch.from_numpy(O.random_image(W + 64, H, 9)).to(cuda)
        for img in (base[:, :W].contiguous(), base[:, 32:32 + W]):  # dense and pitched
            for chunk in ["0", "5", "32"]:
                plan.tune(chunk_rows=int(chunk), tma=0)
                a = plan.forward_level(img)
                plan.tune(tma=2)
                b = plan.forward_level(img)
                for j in range(4):
                    assert torch.equal(a[j], b[j]), (W, H, chunk, j)
    img = torch.from_numpy(O.random_image(1024, 768, 5)).to(cuda)
    plan.tune(chunk_rows=0, tma=0)
    a = plan.forward_mallat(img, 5)
    plan.tune(tma=2)
    b = plan.forward_mallat(img, 5)
    assert torch.equal(a, b)


@pytest.mark.parametrize("w", ["cdf97", "cdf53", "dd137"])
def test_tma_staged_inverse_levels_bit_exact(dwt, cuda, w, monkeypatch):
    """Inverse levels with the four band planes staged by TMA (forced with
    DWT2D_TMA=2) give the same bits as register prefetch: narrow and wide
    levels, ragged chunks, inverse pyramids."""
    import torch
    inv = dwt.Plan(w, "inverse-lifting")
    for W, H in [(64, 40), (256, 200), (2400, 96), (1024, 1024)]:
        planes = _to_dev(O.split(O.random_image(W, H, 21)), cuda)
        for chunk in ["0", "5", "32"]:
            inv.tune(chunk_rows=int(chunk), tma=0)
            a = inv.inverse_level(planes)
            inv.tune(tma=2)
            b = inv.inverse_level(planes)
            assert torch.equal(a, b), (W, H, chunk)
    coeffs = dwt.Plan(w, "nonseparable-lifting", optimized=True).forward_mallat(
        torch.from_numpy(O.random_image(1024, 768, 5)).to(cuda), 5)
    inv.tune(chunk_rows=0, tma=0)
    a = inv.inverse_mallat(coeffs, 5)
    inv.tune(tma=2)
    b = inv.inverse_mallat(coeffs, 5)
    assert torch.equal(a, b)


@pytest.mark.parametrize("w,s,opt", [("cdf97", "nonseparable-lifting", True), ("cdf53", "separable-lifting", False),
                                     ("cdf97", "separable-lifting", True),
                                     ("cdf97", "nonseparable-polyconvolution", True),
                                     ("cdf97", "separable-convolution", True)])
def test_level_pair_bit_exact(dwt, cuda, w, s, opt, monkeypatch):
    """Levels 1 + 2 in one pass (LL_1 kept in registers, pair_engine.cuh;
    forced on every size with DWT2D_PAIR=2) give the same bits as one launch
    per level: narrow images (strips wrap), short images (chunks wrap
    periodically), ragged chunks, pitched input, 2..5 levels."""
    import torch
    plan = dwt.Plan(w, s, optimized=opt)
    assert plan.info["columns_per_lane"] == 4
    for W, H, L in [(1024, 768, 5), (256, 128, 3), (2400, 96, 2), (4096, 64, 2), (64, 64, 2)]:
        base = torch.from_numpy(O.random_image(W + 32, H, 13)).to(cuda)
        for img in (base[:, :W].contiguous(), base[:, 16:16 + W]):
            plan.tune(pair=0)
            a = plan.forward_mallat(img, L)
            plan.tune(pair=2)
            for chunk in [1, 3, 32]:
                plan.tune(pair_chunk_rows=chunk)
                before = dwt.launch_count()
                b = plan.forward_mallat(img, L)
                torch.cuda.synchronize()
                assert dwt.launch_count() - before == L - 1, (W, H, L)
                assert torch.equal(a, b), (W, H, L, chunk)


@pytest.mark.parametrize("w,s,opt", [("cdf97", "nonseparable-lifting", True), ("cdf97", "separable-lifting", False),
                                     ("dd137", "nonseparable-lifting", True), ("cdf53", "inverse-lifting", False)])
def test_bottom_up_chunks_bit_exact(dwt, cuda, w, s, opt, monkeypatch):
    """Odd chunks streaming bottom-up (DWT2D_ALTERNATE) produce the same bits
    as all-top-down streaming, for several chunk sizes incl. ragged ones."""
    import torch
    plan = dwt.Plan(w, s, optimized=opt)
    planes = _to_dev(O.split(O.random_image(256, 200, 4)), cuda)
    img = torch.from_numpy(O.random_image(256, 200, 4)).to(cuda)
    for chunk in ["3", "7", "16", "1000"]:
        plan.tune(chunk_rows=int(chunk), alternate=0)
        a = plan.run(planes)
        fa = plan.forward_level(img) if s != "inverse-lifting" else a
        plan.tune(alternate=2)  # also on this single-wave level
        b = plan.run(planes)
        fb = plan.forward_level(img) if s != "inverse-lifting" else b
        for j in range(4):
            assert torch.equal(a[j], b[j]), (chunk, j)
            assert torch.equal(fa[j], fb[j]), (chunk, j)


@pytest.mark.parametrize("taper", [0, 1])
@pytest.mark.parametrize("host_levels", [0, 1, 3])
@pytest.mark.parametrize("band_rows", ["0", "64", "96", "10000"])
def test_host_pipeline_bands_bit_exact(dwt, cuda, band_rows, host_levels, taper):
    """The pipelined host entry point (row bands uploaded while the first
    levels run band by band on earlier bands, compute bands trailing the
    upload bands by the bottom halo, LL tails computed early for band 0's
    periodic top halo) equals the device pyramid bit for bit, for several
    band splits incl. a ragged last band, 1, 2 or 3 pipelined levels, and
    tapered bands (short first and last bands)."""
    import torch
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True).tune(host_band_rows=int(band_rows),
                                                                           host_levels=host_levels,
                                                                           host_taper=taper)
    # H = 1026 / 1028: the default bands leave a 2-row remainder, which the
    # last band absorbs (a 2-row band would be thinner than its halo)
    # and deeper pyramids: exactly 3 levels, more levels, a single band, a
    # band count that leaves a remainder
    for W, H, L in [(256, 320, 3), (128, 96, 1), (128, 1026, 1), (128, 1028, 2), (64, 4100, 2), (128, 1024, 3),
                    (256, 512, 6), (96, 2048, 4), (64, 1312, 5)]:
        img = O.random_image(W, H, 21)
        dev = plan.forward_mallat(torch.from_numpy(img).to(cuda), L).cpu().numpy()
        host = plan.forward_mallat_host(img, L)
        assert np.array_equal(dev, host), (band_rows, W, H, L)


def test_host_entry_point_tiny_images(dwt, cuda):
    """Images shorter than one host-pipeline band and its halos go up whole
    (no band pipeline) and still equal the device pyramid bit for bit."""
    import torch
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    for W, H, L in [(8, 8, 3), (16, 4, 2), (64, 8, 1), (32, 16, 4)]:
        img = O.random_image(W, H, 5)
        dev = plan.forward_mallat(torch.from_numpy(img).to(cuda), L).cpu().numpy()
        host = plan.forward_mallat_host(img, L)
        assert np.array_equal(dev, host), (W, H, L)


def test_pitched_and_offset_views(dwt, cuda):
    """Row pitch != width and misaligned sub-views use the scalar path and
    agree with the dense vector path."""
    import torch
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    img = torch.from_numpy(O.random_image(200, 64, 11)).to(cuda)
    big = torch.zeros((64, 203), device=cuda)
    big[:, 1:201] = img
    view = big[:, 1:201]
    a = plan.forward_level(img)
    b = plan.forward_level(view)
    for j in range(4):
        assert torch.equal(a[j], b[j])


def test_validation_errors(dwt, cuda):
    import torch
    plan = dwt.Plan("cdf53", "separable-lifting")
    inv = dwt.Plan("cdf53", "inverse-lifting")
    with pytest.raises(ValueError):
        plan.forward_level(torch.zeros((6, 5), device=cuda))  # odd width
    with pytest.raises(ValueError):
        plan.forward_mallat(torch.zeros((12, 12), device=cuda), 3)  # 12 % 8 != 0
    with pytest.raises(ValueError):
        inv.forward_mallat(torch.zeros((16, 16), device=cuda), 1)  # inverse plan
    with pytest.raises(ValueError):
        plan.inverse_level([torch.zeros((4, 4), device=cuda)] * 4)  # forward plan
    with pytest.raises(ValueError):
        dwt.Plan("cdf53", "separable-lifting", workers=0)


def test_launch_count_and_native_library_loaded(dwt, cuda, monkeypatch):
    import torch
    from paper_1704_08657_b200 import native
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    img = torch.from_numpy(O.random_image(256, 256, 2)).to(cuda)
    before = dwt.launch_count()
    plan.forward_mallat(img, 8)  # level 8 is 1 component wide: no vector path, one launch per level
    torch.cuda.synchronize()
    assert dwt.launch_count() - before == 8
    maps = open("/proc/self/maps").read()
    assert str(native.LIB_PATH) in maps


# ---------------------------------------------------------------- symmetric
# extend_index's whole-sample symmetric rule applied to every intermediate of
# every step (image.hpp:21-25, executor.hpp:159-167), on the generic
# executor (one pass per sub-step).

SYM_SIZES = [(32, 24), (17, 9), (2, 3), (1, 1)]


@pytest.mark.parametrize("w,s,opt", PLANS)
def test_symmetric_matches_float64_oracle(dwt, cuda, w, s, opt):
    plan = dwt.Plan(w, s, optimized=opt, extension="symmetric")
    scheme = O.make(w, s, opt)
    for (w2, h2) in SYM_SIZES:
        planes = O.split(O.random_image(2 * w2, 2 * h2, 31 + w2))
        got = [t.cpu().numpy() for t in plan.run(_to_dev(planes, cuda))]
        truth = O.run(scheme, planes, symmetric=True)
        peak = max(float(np.max(np.abs(p))) for p in planes) or 1.0
        assert _err(got, truth, peak) <= TOL, (w, s, opt, w2, h2)


@pytest.mark.parametrize("w,s,opt", [p for p in PLANS if not p[2]])
def test_symmetric_composed_bit_exact_vs_reference(dwt, cuda, w, s, opt):
    if not R.available():
        pytest.skip("oracle/_ref not built")
    plan = dwt.Plan(w, s, optimized=opt, extension="symmetric", lowering="composed")
    for (w2, h2) in [(32, 24), (17, 9), (2, 3)]:
        planes = O.split(O.random_image(2 * w2, 2 * h2, 5 + h2))
        got = [t.cpu().numpy() for t in plan.run(_to_dev(planes, cuda))]
        ref, _ = R.run(w, s, planes, optimized=opt, symmetric=True)
        for j in range(4):
            assert np.array_equal(got[j], ref[j]), (w, s, w2, h2, j)


@pytest.mark.parametrize("w", WAVELETS)
def test_symmetric_reconstruction(dwt, cuda, w):
    """test_executor.cpp:300-326: with symmetric extension the lifting schemes
    reconstruct everywhere, the convolution family on the interior."""
    inv = dwt.Plan(w, "inverse-lifting", extension="symmetric")
    planes = _to_dev(O.split(O.random_image(64, 48, 404)), cuda)
    for s in FORWARD:
        back = inv.run(dwt.Plan(w, s, extension="symmetric").run(planes))
        margin = 0 if "lifting" in s else 8
        sl = (slice(margin, -margin or None), slice(margin, -margin or None))
        e = max(float((b[sl] - p[sl]).abs().max()) for b, p in zip(back, planes))
        assert e <= 5e-5 * (8 if w == "dd137" else 1), (s, e)


@pytest.mark.parametrize("w,s,opt", [("cdf97", "nonseparable-lifting", True), ("cdf97", "separable-convolution", False),
                                     ("cdf53", "nonseparable-polyconvolution", True),
                                     ("dd137", "nonseparable-lifting", False), ("cdf97", "inverse-lifting", False),
                                     ("dd137", "separable-lifting", True)])
@pytest.mark.parametrize("tiles", ["2", "1", "0"])
def test_symmetric_fused_with_border_crops_bit_exact(dwt, cuda, w, s, opt, tiles, monkeypatch):
    """Symmetric extension on the fused kernel + border crops equals the
    all-generic per-step symmetric executor bit for bit: planar run(),
    forward level from the image, inverse level to the image, incl. odd
    (scalar-path) widths, grids just above the crop threshold and levels too
    small for border bands (1 x 1 up to 23 x 300 components)."""
    import torch
    # compiled crop kernel beside the fused kernel's interior, one generic
    # tile launch, or one generic launch per sub-step
    fused = dwt.Plan(w, s, optimized=opt, extension="symmetric").tune(crop_tiles=int(tiles))
    monkeypatch.setenv("DWT2D_FORCE_GENERIC", "1")
    gen = dwt.Plan(w, s, optimized=opt, extension="symmetric")
    monkeypatch.delenv("DWT2D_FORCE_GENERIC")
    assert fused.info["generic"] == 0 and gen.info["generic"] == 1
    sizes = [(64, 48), (150, 101), (300, 40), (40, 300), (33, 33)]
    if tiles == "2":
        sizes += [(1, 1), (2, 3), (5, 4), (17, 9), (23, 300), (300, 7), (24, 24), (96, 13), (16, 12), (17, 13),
                  (15, 300), (300, 11)]
    for (w2, h2) in sizes:
        planes = _to_dev(O.split(O.random_image(2 * w2, 2 * h2, 7 + w2)), cuda)
        a, b = fused.run(planes), gen.run(planes)
        for j in range(4):
            assert torch.equal(a[j], b[j]), (w2, h2, j)
        if s == "inverse-lifting":
            ia, ib = fused.inverse_level(planes), gen.inverse_level(planes)
            assert torch.equal(ia, ib), (w2, h2)
        else:
            img = torch.from_numpy(O.random_image(2 * w2, 2 * h2, 3)).to(cuda)
            fa, fb = fused.forward_level(img), gen.forward_level(img)
            for j in range(4):
                assert torch.equal(fa[j], fb[j]), (w2, h2, j)


def test_symmetric_fused_pyramid_bit_exact(dwt, cuda, monkeypatch):
    import torch
    W, H, L = 1024, 768, 6
    img = torch.from_numpy(O.random_image(W, H, 11)).to(cuda)
    fused = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True, extension="symmetric")
    inv = dwt.Plan("cdf97", "inverse-lifting", extension="symmetric")
    monkeypatch.setenv("DWT2D_FORCE_GENERIC", "1")
    gen = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True, extension="symmetric")
    ginv = dwt.Plan("cdf97", "inverse-lifting", extension="symmetric")
    monkeypatch.delenv("DWT2D_FORCE_GENERIC")
    a, b = fused.forward_mallat(img, L), gen.forward_mallat(img, L)
    assert torch.equal(a, b)
    assert torch.equal(inv.inverse_mallat(a, L), ginv.inverse_mallat(b, L))


def test_symmetric_pyramid_and_inverse(dwt, cuda):
    import torch
    W, H, L = 128, 96, 4
    img = O.random_image(W, H, 2)
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True, extension="symmetric")
    got = plan.forward_mallat(torch.from_numpy(img).to(cuda), L)
    truth = O.pyramid("cdf97", "nonseparable-lifting", img, L, True, symmetric=True)
    assert max(O.level_errors(got.cpu().numpy(), truth, img, L)) <= TOL
    inv = dwt.Plan("cdf97", "inverse-lifting", extension="symmetric")
    back = inv.inverse_mallat(got, L)
    assert float((back.cpu() - torch.from_numpy(img)).abs().max()) <= 5e-5


@pytest.mark.parametrize("w,s,opt", [("cdf97", "nonseparable-lifting", True), ("cdf53", "separable-convolution", False),
                                     ("dd137", "inverse-lifting", False)])
def test_generic_executor_equals_fused_kernels(dwt, cuda, w, s, opt, monkeypatch):
    """Same tables, same order, same rounding: the generic per-sub-step
    executor and the fused single-pass kernel agree bit for bit (periodic)."""
    planes = _to_dev(O.split(O.random_image(96, 80, 17)), cuda)
    fused = dwt.Plan(w, s, optimized=opt)
    monkeypatch.setenv("DWT2D_FORCE_GENERIC", "1")
    gen = dwt.Plan(w, s, optimized=opt)
    assert gen.info["generic"] == 1 and fused.info["generic"] == 0
    a, b = fused.run(planes), gen.run(planes)
    for j in range(4):
        assert torch_equal(a[j], b[j])


def torch_equal(a, b):
    import torch
    return torch.equal(a, b)


def test_custom_definition_wavelet_on_gpu(dwt, cuda, tmp_path):
    """A definition-file wavelet of a new shape (generic executor) matches the
    reference executor on the same file, bit for bit (composed lowering)."""
    if not R.available():
        pytest.skip("oracle/_ref not built")
    f = tmp_path / "odd.txt"
    f.write_text("predict 0:-1/3 1:-1/3\nupdate -1:1/5 0:1/5\nscaling 1.25\n")
    planes = O.split(O.random_image(48, 40, 3))
    for s in FORWARD:
        plan = dwt.Plan(str(f), s)
        got = [t.cpu().numpy() for t in plan.run(_to_dev(planes, cuda))]
        ref, _ = R.run(str(f), s, planes)
        for j in range(4):
            assert np.array_equal(got[j], ref[j]), (s, j)


def test_symmetric_pyramid_in_a_cuda_graph(dwt, cuda):
    """The symmetric levels' crop kernel + fused kernel chain (side-stream
    fork/join for large levels, PDL with the fused kernel's wait at its end
    for small ones) captured in a CUDA graph and replayed equals eager calls
    and the per-step generic executor, also forward + inverse."""
    import torch
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True, extension="symmetric")
    inv = dwt.Plan("cdf97", "inverse-lifting", extension="symmetric")
    for (W, H, L) in [(2048, 1536, 7), (8192, 8192, 3)]:  # 8192^2: level 1 on the side-stream path
        img = torch.from_numpy(O.random_image(W, H, 17)).to(cuda)
        ref = plan.forward_mallat(img, L)
        back_ref = inv.inverse_mallat(ref, L)
        out = torch.zeros_like(img)
        back = torch.zeros_like(img)
        st = torch.cuda.Stream()
        scr = torch.empty(dwt.workspace_bytes(W, H, L) // 4 + 64, device=cuda)
        with torch.cuda.stream(st):
            plan.forward_mallat(img, L, out=out, scratch=scr, stream=st.cuda_stream)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            plan.forward_mallat(img, L, out=out, scratch=scr, stream=st.cuda_stream)
            inv.inverse_mallat(out, L, image=back, scratch=scr, stream=st.cuda_stream)
        for _ in range(3):
            out.zero_()
            back.zero_()
            torch.cuda.synchronize()
            with torch.cuda.stream(st):
                g.replay()
            torch.cuda.synchronize()
            assert torch.equal(out, ref) and torch.equal(back, back_ref), (W, H, L)
        assert float((back - img).abs().max()) <= 5e-5
