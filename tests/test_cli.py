"""The `dwt2d` CLI (paper_1704_08657_b200/bin/dwt2d, csrc/tools/dwt2d_cli.cpp)
against the reference CLI's contract: the ctest smoke checks of
proj/CMakeLists.txt:51-63 plus transform/bench on the GPU."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import dwt_oracle as O

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_1704_08657_b200" / "bin" / "dwt2d"


def run(*args, check=None):
    if not CLI.exists():
        pytest.skip("CLI not built")
    r = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=600)
    if check is not None:
        assert r.returncode == check, (r.returncode, r.stdout, r.stderr)
    return r


def test_cli_count():  # ctest cli_count
    r = run("count", "--wavelet", "cdf53", check=0)
    assert "cdf53,separable-lifting,baseline,4,16" in r.stdout
    assert r.stdout.splitlines()[0] == "wavelet,scheme,variant,steps,operations"
    assert "cdf97,nonseparable-lifting,optimized,4,36" in run("count", "--wavelet", "cdf97", check=0).stdout


def test_cli_describe():  # ctest cli_describe + golden file
    r = run("describe", "--wavelet", "cdf53", "--scheme", "nonseparable-lifting", check=0)
    assert "steps: 2" in r.stdout
    golden = Path("/root/reference/proj/tests/golden/describe_cdf53_nonseparable_lifting.txt")
    if golden.exists():
        assert r.stdout == golden.read_text()


def test_cli_odd_size_is_usage_error():  # ctest cli_odd_size (expect_usage_error.cmake)
    assert run("equiv", "--wavelet", "cdf53", "--size", "257").returncode == 2


def test_cli_usage_and_io_errors(tmp_path):
    assert run().returncode == 2
    assert run("frobnicate").returncode == 2
    assert run("count", "--bogus", "1").returncode == 2
    assert run("bench", "--precision", "64").returncode == 2
    assert run("transform", str(tmp_path / "missing.pgm"), "--out", str(tmp_path / "o")).returncode == 3
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P7 2 2 255\n")
    assert run("transform", str(bad), "--out", str(tmp_path / "o")).returncode == 3
    assert run("--help").returncode == 0


def _write_pgm(path, img8):
    h, w = img8.shape
    path.write_bytes(f"P5\n# test\n{w} {h}\n255\n".encode() + img8.astype(np.uint8).tobytes())


def _read_subbands(d, precision="32"):
    out = []
    for lab in ["ee", "oe", "eo", "oo"]:
        hdr = dict(l.split() for l in (d / f"{lab}.hdr").read_text().splitlines() if l.strip())
        assert hdr["precision"] == precision and hdr["component"] == lab
        dt = "<f4" if precision == "32" else "<f8"
        a = np.fromfile(d / f"{lab}.raw", dtype=dt).reshape(int(hdr["height"]), int(hdr["width"]))
        out.append(a)
    return out


@pytest.mark.gpu
def test_cli_equiv_passes_on_gpu():  # ctest cli_equiv
    r = run("equiv", "--wavelet", "cdf97", "--size", "64", "--seed", "7", check=0)
    assert "PASS" in r.stdout
    r = run("equiv", "--wavelet", "dd137", "--size", "64", "--extension", "symmetric", check=0)
    assert "PASS" in r.stdout
    # float64 (the default) at the reference's tolerances, float32 at 1e-5
    assert "device=B200-float64" in r.stdout and "tolerance 1e-12" in r.stdout
    r = run("equiv", "--wavelet", "cdf97", "--size", "64", "--precision", "32", check=0)
    assert "PASS" in r.stdout and "device=B200-float32" in r.stdout and "tolerance 1e-05" in r.stdout
    r = run("equiv", "--wavelet", "cdf97", "--size", "64", check=0)
    assert "PASS" in r.stdout and "tolerance 1e-09" in r.stdout


@pytest.mark.gpu
def test_cli_transform_matches_oracle(tmp_path):
    rng = np.random.default_rng(3)
    img8 = rng.integers(0, 256, size=(48, 64))
    pgm = tmp_path / "in.pgm"
    _write_pgm(pgm, img8)
    run("transform", pgm, "--out", tmp_path / "sb", "--wavelet", "cdf97", "--scheme", "nonseparable-lifting",
        "--optimize", "--precision", "32", check=0)
    got = _read_subbands(tmp_path / "sb")
    img = img8.astype(np.float64) / 255.0
    truth = O.transform("cdf97", "nonseparable-lifting", O.split(img.astype(np.float32).astype(np.float64)), True)
    assert max(float(np.max(np.abs(g - t))) for g, t in zip(got, truth)) <= 1e-5
    # the reference's default precision: float64 (dwt2d.cpp:121)
    run("transform", pgm, "--out", tmp_path / "sb64", "--wavelet", "cdf97", "--scheme", "nonseparable-lifting",
        "--optimize", check=0)
    got = _read_subbands(tmp_path / "sb64", "64")
    truth = O.transform("cdf97", "nonseparable-lifting", O.split(img), True)
    assert max(float(np.max(np.abs(g - t))) for g, t in zip(got, truth)) <= 1e-12
    run("transform", pgm, "--out", tmp_path / "pyr", "--levels", "3", check=0)
    assert (tmp_path / "pyr" / "level3" / "ee.raw").exists()


@pytest.mark.gpu
def test_cli_bench_csv(tmp_path):
    out = tmp_path / "b.csv"
    run("bench", "--wavelet", "cdf97", "--sizes", "256,512", "--repeats", "3", "--out", out, check=0)
    lines = out.read_text().splitlines()
    assert lines[0] == "scheme,wavelet,width,height,megapixels,precision,workers,seconds,throughput_gbps"
    assert len(lines) == 1 + 5 * 2
    for row in lines[1:]:
        f = row.split(",")
        assert len(f) == 9 and f[1] == "cdf97" and float(f[7]) > 0 and float(f[8]) > 0
