#!/usr/bin/env python
"""Summarise an ncu launch list (gpu__time_duration.sum per launch) for the LAST dade_search
step of a bench run: kernel, launches, total and share of the step. Usage: launch_shares.py launches.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(r for r in rows if "Kernel Name" in r)
i0 = rows.index(h)
kn, mv = h.index("Kernel Name"), h.index("Metric Value")
seq = [(r[kn], float(r[mv].replace(",", ""))) for r in rows[i0 + 1:] if len(r) == len(h)]
# the last step = everything after the last torch fill kernel (the untimed L2 flush)
last_fill = max(i for i, (k, _) in enumerate(seq) if "FillFunctor" in k)
step = [(k, v) for k, v in seq[last_fill + 1:] if "FillFunctor" not in k]
tot = sum(v for _, v in step)
print(f"| kernel | duration (us) | share of step |")
print(f"|---|---|---|")
for k, v in step:
    name = k.split("(")[0].replace("dade::", "").replace("<unnamed>::", "")
    print(f"| `{name}` | {v / 1e3:.1f} | {100 * v / tot:.1f}% |")
print(f"| **total (serialised, cold cache)** | {tot / 1e3:.1f} | 100% |")
