#!/usr/bin/env python3
"""Benchmark: CDF 9/7 forward 2-D DWT, Gpixel/s and HBM roofline on B200.

Workload (BASELINE.json configs[3], the north-star target): non-separable
lifting, optimized (paper's 36 ops/quad), CDF 9/7, float32, 8-level Mallat
pyramid of a 16384 x 16384 image per GPU. One step = one full 8-level
forward pyramid (8 fused level kernels) of the resident image.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): weak scaling, each rank transforms its
own 16384-row strip of a 16384 x (16384 N) image; rank 0 prints the line.

Timing: W untimed warm-up steps; the K timed steps are one CUDA graph
(events around the dominant kernel on every 8th pyramid) replayed between a
barrier + synchronize on both sides; CUDA events on the launching stream give
the step time and the dominant kernel's duration (a separate untimed graph
with an event after every level gives the per-level breakdown); max over
ranks. The image is
1 GiB, larger than the 126 MB L2, so the level-1 input always streams from
HBM (no explicit flush). nvidia-smi samples clocks during the timed region.

Metric and traffic model: pixels of the original image per second, and the
reference's own traffic model of 8 B per pixel per level (read + write
float32, proj/src/bench.cpp:84-85), i.e. 10.667 B per original pixel for 8
levels. roofline: the dominant launch — levels 1+2 fused in one pass
(pair_engine.cuh; 8 B/pixel/level for both levels) or level 1 alone — over
its measured duration vs the measured copy bandwidth in MEASURED_PEAKS.json.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WAVELET, SCHEME, OPTIMIZED = "cdf97", "nonseparable-lifting", True
SIZE, LEVELS = 16384, 8
METRIC = "CDF 9/7 2-D DWT Gpixel/s (ns/pixel) and achieved HBM GB/s vs peak, 1/2/4/8 GPU"
EVENT_STRIDE = 8  # timed pyramids per sampled dominant-kernel duration
# CPU baseline sample: a 16384 x 2048 row band of the same image, 8 levels
SAMPLE_ROWS = 2048


def workload_config(n):
    return {
        "workload": f"CDF 9/7 non-separable lifting (optimized, 36 ops/quad) forward 8-level Mallat "
                    f"pyramid, {SIZE}x{SIZE} float32 per GPU (BASELINE configs[3])",
        "wavelet": WAVELET, "scheme": SCHEME, "optimized": OPTIMIZED,
        "image": [SIZE, SIZE * n], "levels": LEVELS, "extension": "periodic",
        "parallelism": f"row-strips x{n}" if n > 1 else "single GPU",
        "l2": "inputs larger than L2 (1 GiB image per GPU vs 126 MB L2), no flush",
        "traffic_model": "8 B/pixel/level (reference bench.cpp:84-85)",
    }


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(name="ncu_level1_summary.json"):
    """dram bytes per launch of the dominant kernel from the committed ncu
    capture, if any."""
    p = ROOT / "profiles" / name
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return d.get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            time.sleep(0.1)
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for n, v in zip(names, r[2:6]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    n = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return n, rank, local


def cpu_reference(steps, warmup, workers=None):
    """Reference CPU implementation (oracle/_ref, compiled from the reference
    sources) on a bounded sample: a 16384 x SAMPLE_ROWS band, 8 levels."""
    from oracle import ref as R
    from oracle import dwt_oracle as O
    workers = workers or os.cpu_count() or 1
    img = O.random_image(SIZE, SAMPLE_ROWS, 1)
    times = []
    for i in range(warmup + steps):
        t = R.time_pyramid(WAVELET, SCHEME, img, LEVELS, optimized=OPTIMIZED, workers=workers, repeats=1)
        if i >= warmup:
            times.append(t)
    t = statistics.median(times)
    gpix = SIZE * SAMPLE_ROWS / t / 1e9
    return {"value": gpix, "unit": "Gpixel/s", "cores": workers, "kind": "reference",
            "sample": f"{SIZE}x{SAMPLE_ROWS} band of the LCG image, {LEVELS}-level Mallat loop over the "
                      f"reference compile/run API (oracle/_ref, reference sources, -O3), workers={workers}, "
                      f"median of {len(times)}", "seconds": t}


def run_reference_arm(args):
    n, rank, _ = dist_setup()
    if rank != 0:
        return 0
    cb = cpu_reference(args.steps, args.warmup)
    v = cb["value"]
    line = {
        "metric": METRIC, "value": v, "unit": "Gpixel/s", "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": cb["seconds"] * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference LCG image, seed 1)",
        "config": workload_config(n), "impl": "reference",
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": v, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


UP = DOWN = 2  # CDF 9/7 level reach in component rows (halo = 4 image rows each side)


def run_single(args, plan, img, out, dev):
    """N = 1: K pyramids (forward_mallat, the library's multi-level entry
    point) captured in one CUDA graph. The dominant kernel (levels 1+2 fused,
    or level 1) is bracketed by events on every EVENT_STRIDE-th pyramid of the
    timed graph (its mean duration is the roofline denominator); a second,
    untimed graph with an event after every level gives the breakdown."""
    import torch
    import paper_1704_08657_b200 as dwt
    from paper_1704_08657_b200.native import Event
    W = H = SIZE
    scratch = torch.empty(dwt.workspace_bytes(W, H, LEVELS) // 4 + 64, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(device=dev)

    def step(events=None):
        plan.forward_mallat(img, LEVELS, out=out, scratch=scratch, stream=stream.cuda_stream, events=events)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    stream.synchronize()

    def capture(event_sets):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for evs in event_sets:
                step(evs)
        return g

    # the dominant kernel's duration is sampled live inside the timed region on
    # every EVENT_STRIDE-th pyramid: an event node between two kernels breaks
    # their programmatic (PDL) overlap, ~7 us per pyramid if every step had one
    timed_events = [([Event(), Event()] + [None] * (LEVELS - 1)) if k % EVENT_STRIDE == 0 else None
                    for k in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if args.launch == "graph":
        launches0 = dwt.launch_count()
        graph = capture(timed_events)
        launches = dwt.launch_count() - launches0
        with torch.cuda.stream(stream):
            graph.replay()  # untimed replay warms the graph
        torch.cuda.synchronize()
        with ClockSampler(0 if dev.index is None else dev.index) as clk, torch.cuda.stream(stream):
            t0.record(stream)
            graph.replay()  # replays on the current stream (= `stream` here)
            t1.record(stream)
            t1.synchronize()
    else:  # eager: the library's calls as a user makes them (levels chained by PDL)
        torch.cuda.synchronize()
        launches0 = dwt.launch_count()
        with ClockSampler(0 if dev.index is None else dev.index) as clk, torch.cuda.stream(stream):
            t0.record(stream)
            for evs in timed_events:
                step(evs)
            t1.record(stream)
            t1.synchronize()
        launches = dwt.launch_count() - launches0
    torch.cuda.synchronize()
    ms_per_step = t0.elapsed_time(t1) / args.steps
    level1_ms = statistics.mean(e[0].elapsed_ms(e[1]) for e in timed_events if e is not None)

    # breakdown pass (not part of the timed region)
    nb = min(args.steps, 50)
    all_events = [[Event() for _ in range(LEVELS + 1)] for _ in range(nb)]
    g2 = capture(all_events)
    with torch.cuda.stream(stream):
        g2.replay()
    torch.cuda.synchronize()
    level_ms = [statistics.mean(e[l].elapsed_ms(e[l + 1]) for e in all_events) for l in range(LEVELS)]
    level_ms[0] = level1_ms
    return SIZE * SIZE / (ms_per_step * 1e-3) / 1e9, ms_per_step, level_ms, launches, clk


def run_sharded(args, plan, img, out, dev, n):
    """N > 1: each rank owns a 16384-row strip. The library's strip driver
    (dwt2d_forward_mallat_strip, C++) runs the pyramid: levels 1+2 as one
    fused pass from 12+12 halo rows, every later level from 4+4 rows, the
    rows coming from the ring neighbours through the exchange callback
    (NCCL batched send/recv). The timed region is K such pyramids; an
    untimed pass of the Python per-kernel path with events gives the
    per-kernel breakdown."""
    import torch
    import torch.distributed as dist
    import paper_1704_08657_b200 as dwt
    from paper_1704_08657_b200 import strips as S
    ex = S.HaloExchange()
    H, W = img.shape
    scratch = torch.empty(dwt.native.lib.dwt2d_strip_workspace_bytes(plan._h, W, H, LEVELS) // 4 + 64,
                          dtype=torch.float32, device=dev)

    def step():
        S.gpu_forward_mallat(plan, img, LEVELS, exchange=ex, out=out, scratch=scratch)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = dwt.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index or 0) as clk:
        t0.record()
        for _ in range(args.steps):
            step()
        t1.record()
        t1.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
    launches = dwt.launch_count() - launches0
    total = torch.tensor([t0.elapsed_time(t1)], device=dev)
    dist.all_reduce(total, op=dist.ReduceOp.MAX)
    ms_per_step = float(total.item()) / args.steps

    # breakdown (untimed): the same kernels through the Python strip path
    cur_events = []

    def timed(fn):
        def w(cur, top, bottom, out=None):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = fn(cur, top, bottom, out=out)
            e1.record()
            cur_events.append((e0, e1))
            return r
        return w

    pf = S.gpu_pair_fn(plan)
    pair = pf is not None and os.environ.get("DWT2D_PAIR", "1") != "0"
    nb = min(args.steps, 20)
    scratch_out = torch.empty_like(out)
    for _ in range(nb):
        S.forward_mallat_strips(timed(S.gpu_level_fn(plan)), img, LEVELS, UP, DOWN, ex, out=scratch_out,
                                pair_fn=timed(pf) if pair else None)
    torch.cuda.synchronize()
    per = LEVELS - 1 if pair else LEVELS  # kernels per pyramid
    kern_ms = [statistics.mean(cur_events[k * per + l][0].elapsed_time(cur_events[k * per + l][1])
                               for k in range(nb)) for l in range(per)]
    level_ms = [kern_ms[0], 0.0] + kern_ms[1:] if pair else kern_ms
    assert torch.equal(scratch_out, out), "strip driver and Python strip path disagree"
    return SIZE * SIZE * n / (ms_per_step * 1e-3) / 1e9, ms_per_step, level_ms, launches, clk


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--launch", default="graph", choices=["graph", "eager"],
                    help="timed region: one CUDA graph of K pyramids, or K eager library calls")
    ap.add_argument("--sharded", action="store_true",
                    help="run the N>1 strip path (halo exchange + strip kernels) even at N=1 (testing)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist
    import paper_1704_08657_b200 as dwt
    from paper_1704_08657_b200.synth import random_image

    # stdout carries exactly one JSON line (rank 0): everything else written
    # to fd 1 — e.g. the "NCCL version" banner printed when the first
    # communicator is created — goes to stderr
    json_out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    n, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = n > 1 or args.sharded
    if sharded:
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        if n == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)

    plan = dwt.Plan(WAVELET, SCHEME, optimized=OPTIMIZED)
    W = H = SIZE
    # this rank's strip: rows [rank*H, (rank+1)*H) of the W x (n*H) image
    img = random_image(W, H * n, 1, row0=rank * H, rows=H, device=dev)
    out = torch.empty_like(img)
    if sharded:
        value, ms_per_step, level_ms, launches_captured, clk = run_sharded(args, plan, img, out, dev, n)
    else:
        value, ms_per_step, level_ms, launches_captured, clk = run_single(args, plan, img, out, dev)
    pixels = W * H * n

    # end to end through the C ABI host entry point: pinned host image ->
    # H2D -> 8 levels -> D2H of the whole pyramid, synchronous per step
    host_img = img.cpu().pin_memory()
    host_out = torch.empty_like(host_img).pin_memory()
    if not sharded:
        hi, ho = host_img.numpy(), host_out.numpy()

        def e2e_step():
            plan.forward_mallat_host(hi, LEVELS, ho)
    else:
        from paper_1704_08657_b200 import strips as S
        ex = S.HaloExchange()
        dev_in, dev_out = torch.empty_like(img), torch.empty_like(img)

        def e2e_step():
            dev_in.copy_(host_img, non_blocking=True)
            S.gpu_forward_mallat(plan, dev_in, LEVELS, exchange=ex, out=dev_out)
            host_out.copy_(dev_out, non_blocking=True)
            torch.cuda.current_stream().synchronize()
    e2e_step()
    if sharded:
        dist.barrier()
    e2e_t = []
    for _ in range(args.e2e_steps):
        a = time.perf_counter()
        e2e_step()
        e2e_t.append(time.perf_counter() - a)
    e2e_s = statistics.median(e2e_t)
    if sharded:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    assert torch.equal(host_out.to(dev), out), "end-to-end entry point disagrees with device pyramid"

    if rank == 0:
        peak, peak_src = peaks()
        # the dominant kernel: level 1, or levels 1+2 fused in one pass
        # (pair_engine.cuh: one launch fewer per pyramid, the first event
        # pair then brackets both levels)
        fused12 = launches_captured == args.steps * (LEVELS - 1)
        l1_bytes = 8.0 * W * H * (1.25 if fused12 else 1.0)
        achieved = l1_bytes / (level_ms[0] * 1e-3) / 1e9
        kernel_desc = ("levels 1+2 fused (16384^2 -> LL_2 + 6 detail bands, LL_1 kept on chip), "
                       "8 B/pixel/level algorithmic" if fused12 else
                       "level 1 (16384^2 -> 4 x 8192^2), 8 B/pixel algorithmic")
        pyr_bytes = sum(8.0 * (W >> l) * (H >> l) for l in range(LEVELS))
        cpu = None
        if not args.no_cpu_baseline:
            try:
                cb = cpu_reference(steps=3, warmup=1)
                cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            except Exception as e:  # oracle not built on this box
                cpu = {"value": None, "unit": "Gpixel/s", "cores": 0, "kind": "reference",
                       "sample": f"unavailable: {e}"}
        line = {
            "metric": METRIC, "value": value, "unit": "Gpixel/s", "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference LCG random_image, seed 1, generated on device with jump-ahead)",
            "config": workload_config(n),
            "ns_per_pixel": ms_per_step * 1e6 / pixels,
            "pyramid_hbm_gbs_per_gpu": pyr_bytes / (ms_per_step * 1e-3) / 1e9,
            "levels_ms": [round(x, 5) for x in level_ms],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": ncu_traffic("ncu_pair_summary.json" if fused12 else "ncu_level1_summary.json"),
                         "algorithmic_bytes": l1_bytes,
                         "kernel": kernel_desc, "peak_source": peak_src},
            "e2e": {"value": pixels / e2e_s / 1e9, "unit": "Gpixel/s",
                    "h2d_bytes_per_step": int(W * H * 4), "d2h_bytes_per_step": int(W * H * 4),
                    "api": ("dwt2d_forward_mallat_host (C ABI), pinned host buffers" if not sharded else
                            "pinned host strip -> H2D -> dwt2d_forward_mallat_strip (C ABI strip "
                            "pyramid driver, NCCL halo callback) -> D2H, per rank")},
            "gpu_launches": int(launches_captured),
            "halo_exchange": ("NCCL batched send/recv per rank (ring): 12+12 image rows for the fused "
                              "levels 1+2, 4+4 rows for each later level" if sharded else None),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), file=json_out, flush=True)
    if sharded:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
