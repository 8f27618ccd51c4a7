#!/usr/bin/env python
"""Summarise an ncu launch list (gpu__time_duration.sum per launch) for the last timed device
dade_search step of a bench run: kernel, duration and share of the step. Usage: launch_shares.py launches.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(r for r in rows if "Kernel Name" in r)
i0 = rows.index(h)
kn, mv = h.index("Kernel Name"), h.index("Metric Value")
seq = [(r[kn], float(r[mv].replace(",", ""))) for r in rows[i0 + 1:] if len(r) == len(h)]
# steps are separated by the torch fill kernel (the untimed L2 flush); the last timed DEVICE step
# is the last one with a single k_rotate (the e2e steps after it rotate + probe in two halves)
steps, cur = [], []
for k, v in seq:
    if "FillFunctor" in k:
        if cur:
            steps.append(cur)
        cur = []
    else:
        cur.append((k, v))
steps.append(cur)
step = [s for s in steps if sum("k_rotate" in k for k, _ in s) == 1 and any("k_scan" in k for k, _ in s)][-1]
tot = sum(v for _, v in step)
print(f"| kernel | duration (us) | share of step |")
print(f"|---|---|---|")
for k, v in step:
    name = k.split("(")[0].replace("dade::", "").replace("<unnamed>::", "")
    print(f"| `{name}` | {v / 1e3:.1f} | {100 * v / tot:.1f}% |")
print(f"| **total (serialised, cold cache)** | {tot / 1e3:.1f} | 100% |")
