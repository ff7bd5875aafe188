"""Measure every BASELINE.json config on one B200 (results -> profiles/).

  configs[0]  CDF 5/3 separable lifting 512^2 (reference CPU path): GPU time +
              the reference (oracle/_ref) on 1 and all host threads
  configs[1]  CDF 9/7, all five schemes x {baseline, optimized}, 4096^2,
              single level, device-resident, L2 flushed before every run
  configs[2]  CDF 9/7 non-separable polyconvolution forward + inverse round
              trip, 1024^2 .. 16384^2, with max round-trip error
  configs[3]  see bench.py (8-level 16384^2)
  configs[4]  CDF 9/7 non-separable lifting (optimized) at 65536^2 on one GPU
              (the per-GPU problem of the 8-GPU row-strip config), level 1
              and the 8-level pyramid

Timing: CUDA events around each transform on its stream, median of N runs,
a 512 MiB buffer rewritten between runs so every run starts from cold L2.
Throughput: the reference's traffic model, 2 * W * H * 4 bytes per level.
    python scripts/sweep_configs.py [--quick]
"""
import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

SCHEMES = ["separable-convolution", "separable-lifting", "nonseparable-convolution",
           "nonseparable-polyconvolution", "nonseparable-lifting"]
flush_buf = None


def flush():
    global flush_buf
    if flush_buf is None:
        flush_buf = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
    flush_buf.fill_(1.0)


def timed(fn, reps):
    ts = []
    for _ in range(reps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), min(ts)


def gbs(W, H, ms, levels=1):
    byts = sum(8.0 * (W >> l) * (H >> l) for l in range(levels))
    return byts / (ms * 1e-3) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02_configs.jsonl"))
    a = ap.parse_args()
    reps = 11 if a.quick else 101
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    lines = []

    def emit(d):
        d["peak_hbm_gbs"] = peak
        lines.append(d)
        print(json.dumps(d), flush=True)

    # configs[0]
    W = H = 512
    img = random_image(W, H, 1, device="cuda")
    plan = dwt.Plan("cdf53", "separable-lifting")
    bands = [torch.empty((H // 2, W // 2), device="cuda") for _ in range(4)]
    med, mn = timed(lambda: plan.forward_level(img, bands), reps)
    rec = {"config": 0, "workload": "cdf53 separable-lifting 512^2 forward, 1 level", "gpu_ms_median": med,
           "gpu_ms_min": mn, "gpu_gpix_s": W * H / (med * 1e-3) / 1e9, "gpu_gbs": gbs(W, H, med)}
    try:
        from oracle import ref as R
        import numpy as np
        from oracle import dwt_oracle as O
        himg = O.random_image(W, H, 1)
        planes = R.split(himg)
        for workers in (1, os.cpu_count()):
            R.run("cdf53", "separable-lifting", planes, workers=workers)
            ts = []
            for _ in range(7):
                t0 = time.perf_counter()
                R.run("cdf53", "separable-lifting", planes, workers=workers)
                ts.append(time.perf_counter() - t0)
            rec[f"reference_cpu_ms_workers{workers}"] = statistics.median(ts) * 1e3
        rec["host_cores"] = os.cpu_count()
    except Exception as e:  # noqa: BLE001
        rec["reference_cpu"] = f"unavailable: {e}"
    emit(rec)

    # configs[1]
    W = H = 4096
    img = random_image(W, H, 1, device="cuda")
    bands = [torch.empty((H // 2, W // 2), device="cuda") for _ in range(4)]
    for s in SCHEMES:
        for opt in (False, True):
            plan = dwt.Plan("cdf97", s, optimized=opt)
            plan.forward_level(img, bands)
            med, mn = timed(lambda: plan.forward_level(img, bands), reps)
            info = plan.info
            emit({"config": 1, "workload": f"cdf97 {s} {'optimized' if opt else 'baseline'} 4096^2 forward, 1 level",
                  "lowering": info["key"].split("/")[-1], "taps_per_quad": info["taps_per_quad"],
                  "paper_ops_per_quad": info["operations"], "substeps": info["substeps"],
                  "gpu_ms_median": med, "gpu_ms_min": mn, "gpu_gpix_s": W * H / (med * 1e-3) / 1e9,
                  "gpu_gbs": gbs(W, H, med), "frac_of_measured_copy": gbs(W, H, med) / peak})

    # symmetric extension: fused kernel + generic border
    # crops vs the all-generic per-step executor, headline scheme
    for n, levels in ((4096, 1), (16384, 8)):
        img = random_image(n, n, 1, device="cuda")
        out = torch.empty_like(img)
        res = {}
        for mode in ("fused", "generic"):
            if mode == "generic":
                os.environ["DWT2D_FORCE_GENERIC"] = "1"
            plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True, extension="symmetric")
            os.environ.pop("DWT2D_FORCE_GENERIC", None)
            plan.forward_mallat(img, levels, out=out)
            res[mode] = timed(lambda: plan.forward_mallat(img, levels, out=out), max(5, reps // 4))
        emit({"config": "symmetric", "workload": f"cdf97 nonseparable-lifting (optimized) symmetric extension "
                                                 f"{n}^2, {levels} level(s)",
              "gpu_ms_median": res["fused"][0], "gpu_ms_min": res["fused"][1],
              "gpu_gpix_s": n * n / (res["fused"][0] * 1e-3) / 1e9,
              "gpu_gbs": gbs(n, n, res["fused"][0], levels),
              "generic_executor_ms_median": res["generic"][0]})
        del img, out

    # configs[2]
    fwd = dwt.Plan("cdf97", "nonseparable-polyconvolution", optimized=True)
    inv = dwt.Plan("cdf97", "inverse-lifting")
    for n in ([1024, 4096] if a.quick else [1024, 2048, 4096, 8192, 16384]):
        img = random_image(n, n, 1, device="cuda")
        b = [torch.empty((n // 2, n // 2), device="cuda") for _ in range(4)]
        back = torch.empty_like(img)

        def rt():
            fwd.forward_level(img, b)
            inv.inverse_level(b, back)
        rt()
        err = float((back - img).abs().max())
        med, mn = timed(rt, max(5, reps // 4))
        emit({"config": 2, "workload": f"cdf97 nonseparable-polyconvolution (optimized) forward + inverse "
                                       f"lifting round trip {n}^2", "gpu_ms_median": med, "gpu_ms_min": mn,
              "gpu_gpix_s": n * n / (med * 1e-3) / 1e9, "gpu_gbs_16B_per_px": 16.0 * n * n / (med * 1e-3) / 1e9,
              "max_round_trip_error": err})
        del img, b, back
        torch.cuda.empty_cache()

    # configs[4] per-GPU problem at 65536^2
    if not a.quick:
        n = 65536
        plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
        img = random_image(n, n, 1, device="cuda")
        out = torch.empty_like(img)
        scratch = torch.empty(dwt.workspace_bytes(n, n, 8) // 4 + 64, device="cuda")
        plan.forward_mallat(img, 8, out=out, scratch=scratch)
        med, mn = timed(lambda: plan.forward_mallat(img, 8, out=out, scratch=scratch), 5)
        emit({"config": 4, "workload": "cdf97 nonseparable-lifting (optimized) 8-level pyramid 65536^2 (16 GiB) "
                                       "on one B200", "gpu_ms_median": med, "gpu_ms_min": mn,
              "gpu_gpix_s": n * n / (med * 1e-3) / 1e9, "pyramid_gbs": gbs(n, n, med, 8)})
        del img, out, scratch
        torch.cuda.empty_cache()
    Path(a.out).write_text("".join(json.dumps(l) + "\n" for l in lines))


if __name__ == "__main__":
    main()
