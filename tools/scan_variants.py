#!/usr/bin/env python
"""Time dade_search on the bench workload for each k_scan tuning variant (DADE_SCAN_VARIANT).
Usage: python tools/scan_variants.py [--config c2] [--nprobe 8] [--variants 0,1,2]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from datagen import synth  # noqa: E402
from paper_2404_16322_b200 import Index, build  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--nprobe", type=int, default=8)
ap.add_argument("--variants", default="0,1,2,3,4,5")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--var", default="DADE_SCAN_VARIANT", help="environment variable the values are assigned to")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--nlist", type=int, default=0)
a = ap.parse_args()
build.build()
cfg = synth.config(a.config)
if a.n:
    cfg = cfg.scaled(n=a.n, nlist=a.nlist or max(1, a.n // 244))
m = synth.model(cfg)
X = torch.from_numpy(synth.base(cfg, m, workers=min(16, os.cpu_count() or 1))).cuda()
Q = torch.from_numpy(synth.queries(cfg, m=m)).cuda()
Qc = torch.from_numpy(synth.cal_queries(cfg, m=m)).cuda()
ix = Index(cfg.d)
ix.fit_rotation(X)
ix.build_ivf(X, cfg.nlist, kmeans_iters=10)
ix.calibrate(X, Qc, cfg.k, n_neg=cfg.n_neg, nprobe_neg=cfg.nprobe_neg, seed=0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for v in a.variants.split(","):
    os.environ[a.var] = v
    for _ in range(3):
        ix.search(Q, cfg.k, a.nprobe, cfg.delta_d, 0.005)
    sc, tot = [], []
    for _ in range(a.reps):
        flush.fill_(1.0)
        _, _, st = ix.search(Q, cfg.k, a.nprobe, cfg.delta_d, 0.005, stats=True)
        sc.append(st["ms_scan"]); tot.append(st["ms_total"])
    sc.sort(); tot.sort()
    print(f"{a.var}={v}: scan median {sc[len(sc)//2]:.4f} ms min {sc[0]:.4f}  total median {tot[len(tot)//2]:.4f} ms", flush=True)
