"""Host side of the product (CPU only, no kernel launches): the C++ algebra
and lowering behind the C ABI, checked against the reference.

Plan creation runs the product's own C++ scheme builders, optimizer and
lowering; it needs the native library but no GPU.
"""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import dwt_oracle as O
from oracle import ref as R

GOLD = Path(__file__).parent / "golden"
WAVELETS = ["cdf53", "cdf97", "dd137"]


@pytest.fixture(scope="module")
def dwt():
    return pytest.importorskip("paper_1704_08657_b200.transform")


@pytest.fixture(scope="module")
def meta():
    return json.loads((GOLD / "reference_meta.json").read_text())


def test_describe_matches_reference_golden_file(dwt):
    # proj/tests/golden/describe_cdf53_nonseparable_lifting.txt, checked at test_io.cpp:223-233
    ref_golden = Path("/root/reference/proj/tests/golden/describe_cdf53_nonseparable_lifting.txt")
    text = dwt.Plan("cdf53", "nonseparable-lifting").describe()
    if ref_golden.exists():
        assert text == ref_golden.read_text()
    assert text.startswith("scheme: non-separable lifting\nid: nonseparable-lifting\nwavelet: cdf53\nsteps: 2\n")


@pytest.mark.parametrize("w", WAVELETS)
def test_describe_and_counts_match_reference(dwt, meta, w):
    for s in O.SCHEMES:
        for opt in (False, True):
            key = f"{w}|{s}|{int(opt)}"
            p = dwt.Plan(w, s, optimized=opt)
            assert p.describe() == meta["describe"][key]
            steps, ops = meta["counts"][key]
            info = p.info
            assert info["logical_steps"] == steps and info["operations"] == ops


def _ref_tables():
    gold = {}
    return gold


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("w", WAVELETS)
def test_composed_tables_equal_reference_compile(dwt, w):
    """The composed lowering hands the kernel exactly the reference's
    compile<float> tables: same rows, identity flags, scales, tap order and
    float weights (executor.hpp:52-103)."""
    combos = [(s, o) for s in O.SCHEMES for o in (False, True)] + [("inverse-lifting", False)]
    for s, opt in combos:
        rows, taps = dwt.Plan(w, s, optimized=opt, lowering="composed").tables()
        ref = R.taps(w, s, opt)
        flat_ref = [r for k in ref for r in k]
        assert len(rows) == len(flat_ref)
        for (ident, tb, te, sc), (rid, rsc, rtaps) in zip(rows, flat_ref):
            assert ident == rid
            if ident:
                continue
            assert np.float32(sc) == np.float32(rsc)
            mine = [(c, dm, dn, np.float32(wt)) for c, dm, dn, wt in taps[tb:te]]
            assert mine == [(c, dm, dn, np.float32(wt)) for c, dm, dn, wt in rtaps], (w, s, opt)


@pytest.mark.parametrize("w", WAVELETS)
def test_factored_tables_realize_paper_operation_count(dwt, w):
    """Optimized schemes run factor by factor: the multiply-adds per quad the
    kernel executes (non-unit taps) equal count_operations (paper Table 1)."""
    for s in O.SCHEMES:
        p = dwt.Plan(w, s, optimized=True)
        rows, taps = p.tables()
        fmas = 0
        for ident, tb, te, sc in rows:
            if ident:
                continue
            tl = taps[tb:te]
            # a leading unit self-tap is a copy, not an operation
            fmas += len(tl) - (1 if tl and tl[0][3] == 1.0 and tl[0][1] == 0 and tl[0][2] == 0 else 0)
        assert fmas <= p.info["taps_per_quad"]
        if s == "nonseparable-lifting":
            assert fmas == p.info["operations"], (w, fmas, p.info["operations"])


def test_plan_errors(dwt):
    with pytest.raises(ValueError):
        dwt.Plan("nope", "separable-lifting")
    with pytest.raises(ValueError):
        dwt.Plan("cdf53", "separable-lifting", workers=0)
    with pytest.raises(ValueError):
        dwt.Plan("cdf53", "inverse-lifting", optimized=True)
    with pytest.raises(ValueError):
        dwt.Plan("cdf53", "not-a-scheme")


def test_every_builtin_program_has_a_kernel(dwt):
    from paper_1704_08657_b200 import native
    keys = native.registry_keys()
    # the DD 13/7 non-separable convolutions (>200 taps/quad, 7x7 windows)
    # run on the generic executor: their unrolled fused bodies take cicc
    # over 30 minutes (gen_plans.cpp)
    heavy = {("dd137", s) for s in ("nonseparable-convolution", "nonseparable-polyconvolution")}
    assert len(keys) == 33 - 4
    for w in WAVELETS:
        for s in O.SCHEMES:
            for opt in (False, True):
                info = dwt.Plan(w, s, optimized=opt).info
                if (w, s) in heavy:
                    assert info["generic"] == 1 and info["columns_per_lane"] == 0
                else:
                    assert info["generic"] == 0 and info["columns_per_lane"] in (2, 4)


def test_program_tables_round_trip_through_the_abi(dwt):
    """compile() path of the C++ API: tables in, kernel found by fingerprint."""
    p = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    rows, taps = p.tables()
    q = dwt.Plan.from_program([(int(i), tb, te, sc) for i, tb, te, sc in rows], taps, logical_steps=4,
                              fma=True)
    assert q.info["fingerprint"] == p.info["fingerprint"]
    assert q.info["key"] == p.info["key"]


def test_definition_file_wavelet(dwt, tmp_path):
    """A definition file equal to cdf53 resolves to the cdf53 fused kernel; a
    new shape is parsed and planned on the generic GPU executor."""
    f = tmp_path / "mine.txt"
    f.write_text("# my wavelet\nname mine\npredict 0:-1/2 1:-1/2\nupdate -1:1/4 0:1/4\nscaling 1.0\n")
    p = dwt.Plan(str(f), "separable-lifting")
    assert p.info["fingerprint"] == dwt.Plan("cdf53", "separable-lifting").info["fingerprint"]
    assert p.info["generic"] == 0
    g = tmp_path / "odd.txt"
    g.write_text("predict 0:-1/3 1:-1/3\nupdate -1:1/5 0:1/5\n")
    q = dwt.Plan(str(g), "separable-lifting")
    assert q.info["generic"] == 1 and q.info["columns_per_lane"] == 0
    bad = tmp_path / "bad.txt"
    bad.write_text("update 0:1\n")
    with pytest.raises(ValueError):
        dwt.Plan(str(bad), "separable-lifting")


def test_symmetric_plans_use_the_fused_kernel(dwt):
    """symmetric extension: fused kernel + generic border crops (capi.cpp:
    run_symmetric); definition-file programs without an AOT kernel stay on
    the generic executor"""
    p = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True, extension="symmetric")
    assert p.info["generic"] == 0 and p.info["extension"] == 1
