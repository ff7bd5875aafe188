"""The oracle is pinned before it is trusted (CPU only).

* the numpy restatement (oracle/dwt_oracle.py) against the committed golden
  fixtures generated from the compiled reference (scripts/make_golden.py),
* against the compiled reference itself when oracle/_ref is built,
* the reference's known-answer tests for this path
  (test_executor.cpp:108-159, :198-211; test_algebra.cpp:220-252).
"""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import dwt_oracle as O
from oracle import ref as R

GOLD = Path(__file__).parent / "golden"
SCHEMES = O.SCHEMES


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD / "reference_outputs.npz")


@pytest.fixture(scope="module")
def meta():
    return json.loads((GOLD / "reference_meta.json").read_text())


def test_extend_index_frozen_examples():  # test_executor.cpp:108-123
    P, S = False, True
    assert O.extend_index(3, 8, P) == 3
    assert O.extend_index(-1, 8, P) == 7
    assert O.extend_index(8, 8, P) == 0
    assert O.extend_index(-9, 8, P) == 7
    assert O.extend_index(-1, 8, S) == 1
    assert O.extend_index(-2, 8, S) == 2
    assert O.extend_index(8, 8, S) == 6
    assert O.extend_index(9, 8, S) == 5
    assert O.extend_index(14, 8, S) == 0
    assert O.extend_index(15, 8, S) == 1
    assert O.extend_index(5, 1, S) == 0
    assert O.extend_index(5, 1, P) == 0
    with pytest.raises(ValueError):
        O.extend_index(0, 0, P)


def test_lcg_first_draw_and_golden_image(gold):  # test_executor.cpp:149-159
    first = (0x5851F42D4C957F2D + 0x14057B7EF767814F) & ((1 << 64) - 1)
    assert O.lcg_draws(1, 1)[0] == (first >> 11) * 2.0 ** -53
    assert np.array_equal(O.random_image(32, 24, 12345, np.float64), gold["img_32x24_seed12345_f64"])
    assert np.array_equal(O.random_image(32, 24, 12345, np.float32), gold["img_32x24_seed12345_f32"])


def test_split_merge():  # test_executor.cpp:125-147
    img = np.array([[1.0, 2.0], [3.0, 4.0]])
    p = O.split(img)
    assert [float(x[0, 0]) for x in p] == [1, 2, 3, 4]
    big = O.random_image(16, 12, 99, np.float64)
    assert np.array_equal(O.merge(O.split(big)), big)
    for bad in [(4, 3), (3, 4), (0, 0)]:
        with pytest.raises(ValueError):
            O.split(np.zeros(bad))


@pytest.mark.parametrize("w", ["cdf53", "cdf97", "dd137"])
def test_restatement_matches_reference_golden(gold, w):
    img = gold["img_32x24_seed12345_f64"]
    planes = O.split(img)
    for s in SCHEMES + ["inverse-lifting"]:
        for opt in ([False, True] if s != "inverse-lifting" else [False]):
            want = gold[f"{w}|{s}|{int(opt)}|f64"]
            got = np.stack(O.transform(w, s, planes, opt))
            dev = np.max(np.abs(got - want)) / max(np.max(np.abs(got)), np.max(np.abs(want)))
            assert dev < 1e-12, (w, s, opt, dev)  # test_executor.cpp:161-182 bound


def test_pyramid_restatement_matches_reference_golden(gold):
    img = gold["pyr_img_64x64_seed1_f32"]
    for w, s, o in [("cdf97", "nonseparable-lifting", True), ("cdf53", "separable-lifting", False)]:
        want = gold[f"pyr|{w}|{s}|{int(o)}|f64"]
        got = O.pyramid(w, s, img, 4, o)
        assert np.max(np.abs(got - want)) < 1e-11


def test_operation_counts_table(meta):  # test_algebra.cpp:227-243, paper Table 1
    for key, (steps, ops) in meta["counts"].items():
        w, s, o = key.split("|")
        sc = O.make(w, s, o == "1")
        assert len(sc.steps) == steps
        assert O.count_operations(sc) == ops, key
    pinned = {("cdf53", "separable-lifting", "0"): 16, ("cdf97", "separable-lifting", "0"): 32,
              ("cdf97", "nonseparable-lifting", "1"): 36, ("cdf53", "nonseparable-lifting", "1"): 18,
              ("dd137", "nonseparable-lifting", "1"): 50}
    for (w, s, o), ops in pinned.items():
        assert meta["counts"][f"{w}|{s}|{o}"][1] == ops


def test_constant_image_high_bands_vanish():  # test_executor.cpp:198-211
    planes = O.split(np.full((16, 16), 0.375))
    out = O.transform("cdf53", "separable-lifting", planes)
    assert all(np.all(out[j] == 0.0) for j in (1, 2, 3))
    assert np.all(out[0] == 0.375)


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("sym", [False, True])
def test_restatement_matches_live_reference(sym):
    img = O.random_image(40, 28, 777, np.float64)
    planes = O.split(img)
    for w in ["cdf53", "cdf97", "dd137"]:
        for s in SCHEMES:
            for opt in (False, True):
                a = O.transform(w, s, planes, opt, sym)
                b, bc = R.run(w, s, planes, optimized=opt, symmetric=sym)
                assert max(np.max(np.abs(x - y)) for x, y in zip(a, b)) < 1e-12
                assert bc == len(O.make(w, s, opt).steps)
