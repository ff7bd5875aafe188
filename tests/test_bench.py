"""bench.py end to end on the GPU (the driver's contract): one JSON line on
stdout with the metric, the roofline of the dominant kernel, the e2e number
through the C ABI with host buffers, clocks and launch counts — at N = 1,
and at N = 2 through torchrun with two virtual ranks sharing cuda:0
(DWT2D_BENCH_VIRTUAL=1: the sharded path, IPC window exchange, per-rank
e2e with its bit check; times are meaningless there)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _json_line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_single_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
                        "--no-c4-reference", "--e2e-steps", "1"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _json_line(r.stdout)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["unit"] == "Gpixel/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["image"] == [16384, 16384] and d["config"]["levels"] == 8
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["achieved"] > 0 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 16384 * 16384 * 4
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"]
    assert len(d["levels_ms"]) == 8


@pytest.mark.gpu
def test_bench_two_virtual_ranks():
    env = dict(os.environ, DWT2D_BENCH_VIRTUAL="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--workload", "c3", "--e2e-steps", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _json_line(r.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["halo_exchange"]["bytes_per_rank_per_pyramid"] > 0
    assert d["cpu_baseline"] is None
