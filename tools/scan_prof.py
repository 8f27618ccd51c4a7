#!/usr/bin/env python
"""Where a query's latency chain goes inside k_scan: builds a separate library with
-DDADE_SCAN_PROF (per-phase clock64 cycles summed over warps; the product library has none of
it), runs the bench workload's search and prints cycles per query and events per query per phase.
Usage: python tools/scan_prof.py [--config c2] [--nprobe 8] [--nq 10000]"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PROF_LIB = os.environ.get("DADE_PROF_LIB", os.path.join(ROOT, "exp_libs", "libdade_prof.so"))


def build_prof():
    from paper_2404_16322_b200 import build as B
    os.makedirs(os.path.dirname(PROF_LIB), exist_ok=True)
    B.build(extra=["-DDADE_SCAN_PROF"], out=PROF_LIB)


PHASES = ["query_start", "tile_wait", "round_full", "round_drain", "epoch_end", "stage1", "results", "exit"]

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--nprobe", type=int, default=8)
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--no-build", action="store_true")
    a = ap.parse_args()
    if not a.no_build:
        build_prof()
    os.environ["DADE_LIB"] = PROF_LIB
    import torch
    from datagen import synth
    from paper_2404_16322_b200 import Index
    from paper_2404_16322_b200.dade import lib
    cfg = synth.config(a.config)
    m = synth.model(cfg)
    X = torch.from_numpy(synth.base(cfg, m, workers=min(16, os.cpu_count() or 1))).cuda()
    nq = a.nq or cfg.nq
    Q = torch.from_numpy(synth.queries(cfg, n=nq, m=m)).cuda()
    Qc = torch.from_numpy(synth.cal_queries(cfg, m=m)).cuda()
    ix = Index(cfg.d)
    ix.fit_rotation(X)
    ix.build_ivf(X, cfg.nlist, kmeans_iters=10)
    ix.calibrate(X, Qc, cfg.k, n_neg=cfg.n_neg, nprobe_neg=cfg.nprobe_neg, seed=0)
    del X
    L = lib()
    f = L.dade_scan_prof_read
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = (ctypes.c_ulonglong * 16)()
    for _ in range(3):
        ix.search(Q, cfg.k, a.nprobe, cfg.delta_d, 0.005)
    torch.cuda.synchronize()
    f(buf, 1)
    ix.set_timing(True)
    ix.search(Q, cfg.k, a.nprobe, cfg.delta_d, 0.005)
    t = ix.get_timing()
    torch.cuda.synchronize()
    f(buf, 1)
    cyc, cnt = list(buf)[:8], list(buf)[8:]
    tot = sum(cyc)
    out = {"config": cfg.name, "nq": nq, "nprobe": a.nprobe, "scan_ms": round(t["scan"], 4),
           "warp_cycles_total": tot,
           "phases": {ph: {"share": round(c / tot, 4), "cycles_per_query": round(c / nq, 1),
                           "events_per_query": round(n / nq, 2), "cycles_per_event": round(c / max(n, 1), 1)}
                      for ph, c, n in zip(PHASES, cyc, cnt)}}
    print(json.dumps(out, indent=1), flush=True)
