#!/usr/bin/env python
"""Where the end-to-end time of a host-buffer search goes (bench workload, CUDA events, L2 flushed
before each measurement): H2D of the queries alone, D2H of the results alone, the device-buffer
search, the same search cut into c device chunks, and dade_search_host at c pipeline chunks.
Usage: python tools/e2e_breakdown.py [--config c2] [--nprobe 8] [--reps 10]"""
import argparse
import json
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
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
build.build()
cfg = synth.config(a.config)
m = synth.model(cfg)
X = torch.from_numpy(synth.base(cfg, m, workers=min(16, os.cpu_count() or 1))).cuda()
Qn = synth.queries(cfg, m=m)
Q = torch.from_numpy(Qn).cuda()
Qc = torch.from_numpy(synth.cal_queries(cfg, m=m)).cuda()
st = torch.cuda.current_stream()
ix = Index(cfg.d, 0, st)
ix.fit_rotation(X)
ix.build_ivf(X, cfg.nlist, kmeans_iters=10)
ix.calibrate(X, Qc, cfg.k, n_neg=cfg.n_neg, nprobe_neg=cfg.nprobe_neg, seed=0)
del X
K, dd, nq = cfg.k, cfg.delta_d, cfg.nq
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
Qh = torch.from_numpy(Qn).pin_memory()
ih = torch.empty((nq, K), dtype=torch.int64).pin_memory()
dh = torch.empty((nq, K), dtype=torch.float32).pin_memory()
ids = torch.empty((nq, K), dtype=torch.int64, device="cuda")
dists = torch.empty((nq, K), dtype=torch.float32, device="cuda")
Qtmp = torch.empty_like(Q)


def timeit(fn):
    ts = []
    for r in range(a.reps + 3):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1))
    return round(sorted(ts)[len(ts) // 2], 4)


def dev_chunks(c):
    def f():
        for i in range(c):
            q0, q1 = nq * i // c, nq * (i + 1) // c
            ix.search(Q[q0:q1], K, a.nprobe, dd, 0.005, ids=ids[q0:q1], dists=dists[q0:q1])
    return f


def host_chunks(c, prep=1):
    def f():
        ix.set_option("host_chunks", c)
        ix.set_option("host_prep_chunks", prep)
        ix.search_host(Qh, K, a.nprobe, dd, 0.005, ids=ih, dists=dh)
    return f


out = {"config": cfg.name, "nprobe": a.nprobe, "nq": nq,
       "h2d_ms": timeit(lambda: Qtmp.copy_(Qh, non_blocking=True)),
       "d2h_ms": timeit(lambda: (ih.copy_(ids, non_blocking=True), dh.copy_(dists, non_blocking=True))),
       "search_ms": timeit(dev_chunks(1))}
for c in (2, 4):
    out[f"search_{c}dev_chunks_ms"] = timeit(dev_chunks(c))
for c in (1, 2, 4):
    out[f"search_host_{c}_ms"] = timeit(host_chunks(c))
for pc in (2, 3, 4):
    out[f"search_host_prep{pc}_ms"] = timeit(host_chunks(1, pc))
out["h2d_GBps"] = round(Qh.numel() * 4 / out["h2d_ms"] / 1e6, 1)
print(json.dumps(out), flush=True)

# per-size stage times (library events) and the host cost of issuing one search call
import time  # noqa: E402
ix.set_timing(True)
for n in (nq, nq // 2, nq // 4):
    stages = []
    for r in range(a.reps + 3):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ix.search(Q[:n], K, a.nprobe, dd, 0.005, ids=ids[:n], dists=dists[:n])
        t_issue = (time.perf_counter() - t0) * 1e3
        torch.cuda.synchronize()
        if r >= 3:
            stages.append(dict(ix.get_timing(), issue_ms=t_issue))
    med = {k: round(sorted(s[k] for s in stages)[len(stages) // 2], 4) for k in stages[0]}
    print(json.dumps({"nq": n, **med}), flush=True)
ix.set_timing(False)
