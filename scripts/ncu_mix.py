"""Summaries of an ncu report (development only): key metrics, top stall
reasons, and the SASS instruction mix with stall samples.
    python scripts/ncu_mix.py report.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                                 text=True).stdout)))
h, v = raw[0], raw[2]
for k in ["gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread", "dram__bytes_read.sum",
          "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"]:
    if k in h:
        print(f"{k:60s} {v[h.index(k)]} {raw[1][h.index(k)]}")
st = sorted(((float(v[i]), k) for i, k in enumerate(h)
             if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio") and v[i]), reverse=True)
for x in st[:8]:
    print(f"  stall {x[1].split('stalled_')[1].split('_per')[0]:22s} {x[0]:.3f}")
src = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                                                 capture_output=True, text=True).stdout)))
hdr = [r for r in src if "Address" in r][0]
i0 = src.index(hdr) + 1
iS, iE, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
ops, ex = collections.Counter(), collections.Counter()
for r in src[i0:]:
    t = r[iSrc].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    try:
        ops[op] += int(r[iS])
        ex[op] += int(r[iE])
    except ValueError:
        pass
ts, te = sum(ops.values()) or 1, sum(ex.values()) or 1
for op, e in ex.most_common(16):
    print(f"  {op:10s} exec {e:11d} {100 * e / te:5.1f}%   stall samples {100 * ops[op] / ts:5.1f}%")
