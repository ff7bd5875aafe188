"""Summarise one `ncu --set full` capture of a level kernel into a small JSON
(tracked under profiles/): DRAM bytes vs the 8 B/pixel algorithmic model,
time, occupancy, issue activity.

    python scripts/summarize_ncu.py gpurun_out/prof_level1.ncu-rep \
        --pixels 268435456 --command "..." > profiles/<name>.json
"""
import argparse
import csv
import io
import json
import subprocess

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "lts__t_sector_hit_rate.pct",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--pixels", type=int, required=True, help="input pixels of the captured launch")
    ap.add_argument("--command", default="")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    m = {n: {"unit": units[i], "value": vals[i]} for i, n in enumerate(head) if n in METRICS}
    rd = float(m["dram__bytes_read.sum"]["value"]) * SCALE[m["dram__bytes_read.sum"]["unit"]]
    wr = float(m["dram__bytes_write.sum"]["value"]) * SCALE[m["dram__bytes_write.sum"]["unit"]]
    alg = 8 * a.pixels
    out = {
        "kernel": vals[head.index("Kernel Name")],
        "command": a.command,
        "dram_bytes_per_launch": rd + wr,
        "dram_read_bytes": rd,
        "dram_write_bytes": wr,
        "algorithmic_bytes_per_launch": alg,
        "traffic_over_algorithmic": (rd + wr) / alg,
        "note": a.note,
        "metrics": m,
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
