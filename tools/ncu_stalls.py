#!/usr/bin/env python
"""Summarise an ncu --set full report: key raw metrics + warp-stall samples by reason and by
source line (needs -lineinfo). Usage: python tools/ncu_stalls.py report.ncu-rep [kernel-regex]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h = raw[0]
for row in raw[2:]:
    name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    print("==", name[:90])
    for k in KEYS:
        if k in h:
            print(f"   {k:60s} {raw[1][h.index(k)]:>10s} {row[h.index(k)]}")
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "cuda,sass"))))
hdr = next((r for r in src if r and r[0] == "Address" or (r and "Source" in r and "stall_lg" in r)), None)
if hdr is None:
    sys.exit(0)
i0 = src.index(hdr)
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
tot = collections.Counter()
by_line = collections.Counter()
for r in src[i0 + 1:]:
    if len(r) != len(hdr):
        continue
    for c in cols:
        try:
            v = float(r[hdr.index(c)] or 0)
        except ValueError:
            continue
        tot[c] += v
    try:
        by_line[r[hdr.index("Source")][:110]] += float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        pass
s = sum(tot.values()) or 1
print("stall reasons (share of samples):")
for c, v in tot.most_common(10):
    print(f"   {c:25s} {100 * v / s:5.1f}%")
print("top source lines by samples:")
for l, v in by_line.most_common(25):
    print(f"   {v:8.0f}  {l}")

# instruction counts per source line
ie = hdr.index("Instructions Executed") if "Instructions Executed" in hdr else None
if ie is not None:
    cnt = collections.Counter()
    for r in src[i0 + 1:]:
        if len(r) == len(hdr):
            try:
                cnt[r[hdr.index("Source")][:110]] += float(r[ie] or 0)
            except ValueError:
                pass
    tot = sum(cnt.values()) or 1
    print(f"warp instructions executed by source line (total {tot:.3e}):")
    for l, v in cnt.most_common(30):
        print(f"   {100 * v / tot:5.1f}%  {l.strip()}")
