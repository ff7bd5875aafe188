"""BASELINE configs[1] (CDF 9/7, all five schemes x {baseline, optimized},
one forward level of a 4096^2 float32 image) as steady-state throughput:
back-to-back launches over 4 rotating input/output buffer sets (SURVEY
§8(d): "rotating >= 4 input/output buffer sets"), 32 launches captured in
one CUDA graph, median of 11 replays / 32. Each launch also pays the
write-back of an earlier launch's dirty outputs (the steady state of a
pipeline), but not a launch + event round trip of its own. Next to it: the
isolated cold-L2 time (buffer rewrite before each launch, events around
one launch), as scripts/sweep_configs.py measures.
    python scripts/probe_configs1_steady.py > profiles/r02_configs1_steady.jsonl"""
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1704_08657_b200 as dwt  # noqa: E402
from paper_1704_08657_b200.synth import random_image  # noqa: E402

SCHEMES = ["separable-convolution", "separable-lifting", "nonseparable-convolution",
           "nonseparable-polyconvolution", "nonseparable-lifting"]
W = H = 4096
SETS, ROUNDS = 4, 8
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
imgs = [random_image(W, H, 1 + k, device="cuda") for k in range(SETS)]
outs = [[torch.empty((H // 2, W // 2), device="cuda") for _ in range(4)] for _ in range(SETS)]
flush_buf = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
alg = 8.0 * W * H


def isolated(plan):
    ts = []
    for _ in range(21):
        flush_buf.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.forward_level(imgs[0], outs[0])
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def steady(plan):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for k in range(SETS):
            plan.forward_level(imgs[k], outs[k])
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(ROUNDS):
            for k in range(SETS):
                plan.forward_level(imgs[k], outs[k])
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(11):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / (SETS * ROUNDS))
    return statistics.median(ts)


for sch in SCHEMES:
    for opt in (False, True):
        plan = dwt.Plan("cdf97", sch, optimized=opt)
        ref = [t.clone() for t in (plan.forward_level(imgs[0], outs[0]) or outs[0])]
        iso = isolated(plan)
        st = steady(plan)
        same = all(torch.equal(a, b) for a, b in zip(ref, outs[0]))
        print(json.dumps({
            "config": 1, "workload": f"cdf97 {sch} {'optimized' if opt else 'baseline'} 4096^2 forward, 1 level",
            "steady_us": round(st * 1e3, 2), "steady_gbs": round(alg / (st * 1e-3) / 1e9, 1),
            "steady_frac_of_copy": round(alg / (st * 1e-3) / 1e9 / peak, 3),
            "isolated_cold_us": round(iso * 1e3, 2), "isolated_frac_of_copy": round(alg / (iso * 1e-3) / 1e9 / peak, 3),
            "graph_outputs_equal_eager": same, "peak_hbm_gbs": peak}), flush=True)
