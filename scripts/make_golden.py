"""Generate tests/golden/ fixtures from the compiled reference (oracle/_ref).

Run in the build container (where /root/reference exists):
    python scripts/make_golden.py
Writes tests/golden/reference_outputs.npz: for every built-in wavelet, every
forward scheme (baseline and optimized) and inverse lifting, the reference's
float64 and float32 run() outputs on the LCG image random_image(32, 24, 12345)
(the fixture of the reference's own executor test, test_executor.cpp:162),
plus 4-level float64/float32 Mallat pyramids of random_image(64, 64, 1) for
cdf97 non-separable lifting (optimized) and cdf53 separable lifting, and the
reference's describe() text and (steps, operations) counts.
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import ref as R  # noqa: E402

SCHEMES = ["separable-convolution", "separable-lifting", "nonseparable-convolution",
           "nonseparable-polyconvolution", "nonseparable-lifting"]


def main():
    out = {}
    meta = {"counts": {}, "describe": {}}
    img64 = R.random_image(32, 24, 12345, np.float64)
    img32 = R.random_image(32, 24, 12345, np.float32)
    out["img_32x24_seed12345_f64"] = img64
    out["img_32x24_seed12345_f32"] = img32
    for w in ["cdf53", "cdf97", "dd137"]:
        combos = [(s, o) for s in SCHEMES for o in (False, True)] + [("inverse-lifting", False)]
        for s, o in combos:
            key = f"{w}|{s}|{int(o)}"
            d, _ = R.run(w, s, R.split(img64), optimized=o)
            f, _ = R.run(w, s, R.split(img32), optimized=o)
            out[key + "|f64"] = np.stack(d)
            out[key + "|f32"] = np.stack(f)
            if s != "inverse-lifting":
                meta["counts"][key] = list(R.count(w, s, o))
                meta["describe"][key] = R.describe(w, s, o)
    pimg = R.random_image(64, 64, 1, np.float32)
    out["pyr_img_64x64_seed1_f32"] = pimg
    for w, s, o in [("cdf97", "nonseparable-lifting", True), ("cdf53", "separable-lifting", False)]:
        key = f"pyr|{w}|{s}|{int(o)}"
        out[key + "|f64"] = R.pyramid(w, s, pimg.astype(np.float64), 4, optimized=o)
        out[key + "|f32"] = R.pyramid(w, s, pimg, 4, optimized=o)
    gdir = ROOT / "tests" / "golden"
    gdir.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(gdir / "reference_outputs.npz", **out)
    (gdir / "reference_meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
