#!/usr/bin/env python
"""Build the bench workload, then run ONE dade_search between cudaProfilerStart/Stop so that
`ncu --profile-from-start off` captures exactly the kernels of one search step.
Usage: python tools/profile_search.py [--config c2] [--nprobe 8]"""
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
ap.add_argument("--alpha", type=float, default=0.005)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--nlist", type=int, default=0)
ap.add_argument("--opt", default="", help="OPTION=VALUE (dade_set_option) set just before the profiled search")
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
for _ in range(3):
    ix.search(Q, cfg.k, a.nprobe, cfg.delta_d, a.alpha)
if a.opt:
    k_, v_ = a.opt.split("=", 1)
    ix.set_option(k_, int(v_))
torch.cuda.synchronize()
torch.cuda.profiler.start()
ix.search(Q, cfg.k, a.nprobe, cfg.delta_d, a.alpha)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled one search:", a.config, "nprobe", a.nprobe)
