"""float64 execution (compile<double> / run<double>, reference
executor.hpp:52-238; the reference's equiv harness runs in double,
equiv.cpp:161-168): the generic GPU executor with float64 weights and
scales. Composed (baseline) programs and the inverse equal the reference's
own run<double> (oracle/_ref) bit for bit, periodic and symmetric; the
factored (optimized) programs, which the reference never executes, agree
with the float64 oracle restatement to 1e-12 of the input range; float64
levels round-trip to 1e-12."""
import numpy as np
import pytest

from oracle import dwt_oracle as O
from oracle import ref as R

pytestmark = pytest.mark.gpu

WAVELETS = ["cdf53", "cdf97", "dd137"]


def _planes(cuda, w2, h2, seed):
    import torch
    img = O.random_image(2 * w2, 2 * h2, seed).astype(np.float64)
    return img, [torch.from_numpy(np.ascontiguousarray(p)).to(cuda) for p in O.split(img)]


@pytest.mark.parametrize("wavelet", WAVELETS)
@pytest.mark.parametrize("symmetric", [False, True])
def test_float64_composed_bit_exact_vs_reference_run_double(cuda, wavelet, symmetric):
    if not R.available():
        pytest.skip("oracle/_ref not built")
    import paper_1704_08657_b200 as dwt
    ext = "symmetric" if symmetric else "periodic"
    for scheme in O.SCHEMES + ["inverse-lifting"]:
        plan = dwt.Plan(wavelet, scheme, optimized=False, extension=ext, lowering="composed")
        for (w2, h2) in [(40, 28), (33, 17), (8, 5)]:
            _, planes = _planes(cuda, w2, h2, 3 + w2)
            got = [t.cpu().numpy() for t in plan.run(planes)]
            ref, _ = R.run(wavelet, scheme, [p.cpu().numpy() for p in planes], optimized=False, symmetric=symmetric)
            for j in range(4):
                assert got[j].dtype == np.float64
                assert np.array_equal(got[j], ref[j]), (wavelet, scheme, ext, w2, h2, j)


@pytest.mark.parametrize("wavelet", WAVELETS)
def test_float64_factored_vs_float64_oracle(cuda, wavelet):
    import paper_1704_08657_b200 as dwt
    for scheme in O.SCHEMES:
        plan = dwt.Plan(wavelet, scheme, optimized=True)
        for symmetric in (False, True):
            plan = dwt.Plan(wavelet, scheme, optimized=True, extension="symmetric" if symmetric else "periodic")
            img, planes = _planes(cuda, 36, 20, 11)
            got = [t.cpu().numpy() for t in plan.run(planes)]
            truth = O.transform(wavelet, scheme, O.split(img), True, symmetric=symmetric)
            peak = float(np.max(np.abs(img)))
            err = max(float(np.max(np.abs(g - t))) for g, t in zip(got, truth)) / peak
            assert err <= 1e-12, (wavelet, scheme, symmetric, err)


@pytest.mark.parametrize("wavelet", WAVELETS)
def test_float64_level_round_trip(cuda, wavelet):
    import torch
    import paper_1704_08657_b200 as dwt
    img = torch.from_numpy(O.random_image(96, 64, 5).astype(np.float64)).to(cuda)
    base = torch.zeros((64, 96 + 32), dtype=torch.float64, device=cuda)
    base[:, 16:16 + 96] = img
    for view in (img, base[:, 16:16 + 96]):  # dense and pitched images
        for scheme in ("nonseparable-lifting", "separable-convolution"):
            fwd = dwt.Plan(wavelet, scheme, optimized=True)
            inv = dwt.Plan(wavelet, "inverse-lifting")
            bands = fwd.forward_level(view)
            assert all(b.dtype == torch.float64 for b in bands)
            back = inv.inverse_level(bands)
            torch.cuda.synchronize()
            assert float((back - img).abs().max()) <= 1e-12 * (8 if wavelet == "dd137" else 1), (wavelet, scheme)


def test_float64_needs_float64_tables(cuda):
    """Plans from bare float32 tables (dwt2d_plan_create_from_program
    without weights64) refuse float64 data instead of widening float
    weights; the built-in plans carry them."""
    import torch
    import paper_1704_08657_b200 as dwt
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    rows, taps = plan.tables()
    p2 = dwt.Plan.from_program(rows, taps, logical_steps=plan.info["logical_steps"], fma=True)
    _, planes = _planes(cuda, 16, 8, 1)
    with pytest.raises(dwt.DwtError):
        p2.run(planes)
    a = plan.run(planes)
    torch.cuda.synchronize()
    assert all(t.dtype == torch.float64 for t in a)
