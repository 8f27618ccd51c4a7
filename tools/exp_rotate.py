#!/usr/bin/env python
"""Rotation timing (a1 database rows, a4 queries): builds a one-list IVF over n random rows (the
layout write is the rotation of every row, gathered in list order) and times build_ivf and
prepare (query rotation + a one-centroid probe) with CUDA events. DADE_LIB selects the library
(A/B against an older build). Prints one JSON line per (n, D).
Usage: python tools/exp_rotate.py [--shapes 10000000x96,1000000x128] [--nq 10000] [--reps 5]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2404_16322_b200 import Index, build
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="10000000x96,1000000x128,1000000x960")
    ap.add_argument("--nq", type=int, default=10000)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    if "DADE_LIB" not in os.environ:
        build.build()
    g = torch.Generator(device="cuda").manual_seed(0)
    for shp in a.shapes.split(","):
        n, D = (int(v) for v in shp.split("x"))
        X = torch.randn((n, D), device="cuda", generator=g) * 40.0 + 100.0
        Q = torch.randn((a.nq, D), device="cuda", generator=g) * 40.0 + 100.0
        R, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((D, D)))
        ix = Index(D)
        ix.set_rotation(np.full(D, 100.0), R, np.ones(D))
        c0 = X[:1].clone()

        def timed(fn):
            ts = []
            for r in range(a.reps + 1):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                if r:
                    ts.append(e0.elapsed_time(e1))
            ts.sort()
            return ts[len(ts) // 2]

        t_build = timed(lambda: ix.build_ivf(X, 1, centroids=c0))
        t_prep = timed(lambda: ix.prepare(Q, 1))
        print(json.dumps({"lib": os.environ.get("DADE_LIB", "product"), "n": n, "D": D, "nq": a.nq,
                          "build_ivf_ms": round(t_build, 3), "prepare_ms": round(t_prep, 4)}), flush=True)
        del X, Q, ix
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
