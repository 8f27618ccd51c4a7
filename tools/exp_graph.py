#!/usr/bin/env python
"""NEXT-4 measurement: HNSW base-layer refinement with and without the DCO (the paper's HNSW vs
HNSW-BSA-p comparison, on a synthetic stand-in). Builds the IVF (for the graph's
candidate pools), the graph (dade_build_graph: pools from IVF searches at nprobe_pool lists, HNSW's
heuristic to M0 = 32), calibrates with K = ef for each ef, and reports per ef: recall@10 against
the exact top-10, QPS (CUDA events, L2 flushed), dims read per tested node and pruned fraction —
alpha = 0 (plain refinement) and alpha = 0.005.
Usage: python tools/exp_graph.py [--config c2] [--n 200000] [--nlist 1024] [--nq 10000]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from datagen import synth
    from paper_2404_16322_b200 import Index, build
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--nlist", type=int, default=1024)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--nprobe-pool", type=int, default=8)
    ap.add_argument("--efs", default="16,32,64,128")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    build.build()
    cfg = synth.config(a.config).scaled(n=a.n, nlist=a.nlist, nq=a.nq)
    m = synth.model(cfg)
    X = torch.from_numpy(synth.base(cfg, m, workers=min(16, os.cpu_count() or 1))).cuda()
    Q = torch.from_numpy(synth.queries(cfg, m=m)).cuda()
    Qc = torch.from_numpy(synth.cal_queries(cfg, m=m)).cuda()
    ix = Index(cfg.d)
    ix.fit_rotation(X)
    ix.build_ivf(X, cfg.nlist, kmeans_iters=10)
    t0 = time.time()
    ix.build_graph(X, M0=32, P=64, nprobe_pool=a.nprobe_pool)
    torch.cuda.synchronize()
    t_graph = time.time() - t0
    gt, _ = ix.bruteforce_knn(X, Q, 10)
    gt = gt.cpu().numpy()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for ef in [int(e) for e in a.efs.split(",")]:
        ix.calibrate(X, Qc, ef, n_neg=cfg.n_neg, nprobe_neg=cfg.nprobe_neg, seed=0)
        for alpha in (0.0, 0.005):
            ids, d, st = ix.graph_search(Q, 10, ef, cfg.delta_d, alpha, stats=True)
            found = ids.cpu().numpy()
            rc = sum(len(set(f.tolist()) & set(g.tolist())) for f, g in zip(found, gt)) / (10 * len(gt))
            ts = []
            for _ in range(a.reps):
                flush.fill_(1.0)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ix.graph_search(Q, 10, ef, cfg.delta_d, alpha)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            ms = ts[len(ts) // 2]
            print(json.dumps({"config": cfg.name, "n": cfg.n, "nq": cfg.nq, "ef": ef, "alpha": alpha,
                              "recall@10": round(rc, 5), "qps": round(cfg.nq / (ms / 1e3), 1), "ms": round(ms, 4),
                              "tested_per_query": st["tested"] / cfg.nq, "expansions_per_query": st["n_epochs"] / cfg.nq,
                              "dims_per_tested": round(st["dims_scanned"] / st["tested"], 2),
                              "pruned_frac": round(sum(st["pruned_at_step"]) / st["tested"], 4),
                              "graph_build_s": round(t_graph, 1)}), flush=True)


if __name__ == "__main__":
    main()
