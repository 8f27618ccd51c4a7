#!/usr/bin/env python
"""NEXT-2: evaluation features of the paper, run on the built GPU path through the
public API.

  significance  — the Exp-2 analogue (Fig. 6: target recall r swept 0.9 … 0.999):
                  recall@K of the DADE search against exact IVF at the same nprobe, the fraction of
                  dimensions read (scan rate) and the search time, per r = 1 − α.
  approx        — the Exp-7 / Table III analogue (R27): recall@100 of a flat scan
                  ranked by the d = 32 estimate, PCA-partial vs Rand-partial vs BSA-res
                  (`dade_estimate_knn`), 1,000 queries, exact top-100 from dade_bruteforce_knn.
  preprocessing — the Exp-3 analogue: time of fit_rotation (PCA), build_ivf
                  (k-means + assignment + layout) and calibrate, and the extra space the method
                  keeps (R, μ: D² + D doubles; the calibration table).

Usage: python tools/experiments.py significance [--config c2] [--nprobe 8]
       python tools/experiments.py approx [--config c2] [--d 32]
       python tools/experiments.py preprocessing [--config c2]
Prints one JSON object per line (results also summarised in profiles/)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from datagen import synth  # noqa: E402
from paper_2404_16322_b200 import Index, build  # noqa: E402


def recall(found, truth, K):
    return sum(len(set(f[:K].tolist()) & set(g[:K].tolist())) for f, g in zip(found, truth)) / (K * len(found))


def setup(cfg):
    m = synth.model(cfg)
    X = torch.from_numpy(synth.base(cfg, m, workers=min(16, os.cpu_count() or 1))).cuda()
    Q = torch.from_numpy(synth.queries(cfg, m=m)).cuda()
    Qc = torch.from_numpy(synth.cal_queries(cfg, m=m)).cuda()
    ix = Index(cfg.d)
    t = {}
    torch.cuda.synchronize(); t0 = time.time()
    ix.fit_rotation(X); torch.cuda.synchronize(); t["fit_rotation_s"] = time.time() - t0; t0 = time.time()
    ix.build_ivf(X, cfg.nlist, kmeans_iters=10); torch.cuda.synchronize(); t["build_ivf_s"] = time.time() - t0
    t0 = time.time()
    ix.calibrate(X, Qc, cfg.k, n_neg=cfg.n_neg, nprobe_neg=cfg.nprobe_neg, seed=0)
    torch.cuda.synchronize(); t["calibrate_s"] = time.time() - t0
    return ix, X, Q, t


def cmd_significance(a):
    cfg = synth.config(a.config)
    ix, X, Q, _ = setup(cfg)
    K, dd = cfg.k, cfg.delta_d
    ei, _ = ix.search(Q, K, a.nprobe, dd, 0.0)                     # exact IVF at the same nprobe
    ei = ei.cpu().numpy()
    for r in (0.9, 0.95, 0.99, 0.995, 0.999, 1.0):
        alpha = 1.0 - r
        for _ in range(2):
            ix.search(Q, K, a.nprobe, dd, alpha)
        gi, _, st = ix.search(Q, K, a.nprobe, dd, alpha, stats=True)
        out = {"experiment": "significance", "config": cfg.name, "nprobe": a.nprobe, "target_recall_r": r,
               "recall_vs_exact_ivf": round(recall(gi.cpu().numpy(), ei, K), 5),
               "scan_rate": round(st["dims_scanned"] / max(1, st["tested"] * cfg.d), 4),
               "search_ms": round(st["ms_total"], 4), "scan_ms": round(st["ms_scan"], 4)}
        print(json.dumps(out), flush=True)


def cmd_preprocessing(a):
    cfg = synth.config(a.config)
    ix, X, Q, t = setup(cfg)
    cal = ix.get_calibration()
    out = {"experiment": "preprocessing", "config": cfg.name, "n": cfg.n, "D": cfg.d, "nlist": cfg.nlist,
           **{k: round(v, 3) for k, v in t.items()},
           "rotation_bytes": 8 * (cfg.d * cfg.d + 2 * cfg.d),
           "calibration_table_bytes": 8 * (len(cal["m1"]) + int(np.asarray(cal["v"]).size)),
           "base_bytes": 4 * cfg.n * cfg.d}
    print(json.dumps(out), flush=True)


def cmd_approx(a):
    cfg = synth.config(a.config)
    m = synth.model(cfg)
    X = torch.from_numpy(synth.base(cfg, m, workers=min(16, os.cpu_count() or 1))).cuda()
    Q = torch.from_numpy(synth.queries(cfg, n=1000, m=m)).cuda()
    K = 100
    out = {"experiment": "approx", "config": cfg.name, "n": cfg.n, "D": cfg.d, "d": a.d, "nq": 1000, "K": K}
    ix = Index(cfg.d)
    ix.fit_rotation(X)
    ix.build_ivf(X, cfg.nlist, kmeans_iters=1)     # the flat scan ignores the lists
    gt = ix.bruteforce_knn(X, Q, K)[0].cpu().numpy()
    for est, col in (("partial", "PCA"), ("residual", "BSA-res")):
        ix.estimate_knn(Q[:8], a.d, K, est)
        torch.cuda.synchronize(); t0 = time.time()
        ids, _ = ix.estimate_knn(Q, a.d, K, est)
        torch.cuda.synchronize()
        out[col] = round(recall(ids.cpu().numpy(), gt, K), 4)
        out[col + "_scan_ms"] = round(1e3 * (time.time() - t0), 2)
    mean, _, lam = ix.get_rotation()
    ix.close()
    ir = Index(cfg.d)
    ir.set_rotation(mean, synth.haar_basis(cfg.d, np.random.default_rng(12345)).T.copy(), lam)
    ir.build_ivf(X, cfg.nlist, kmeans_iters=1)
    out["Rand"] = round(recall(ir.estimate_knn(Q, a.d, K, "partial")[0].cpu().numpy(), gt, K), 4)
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["significance", "preprocessing", "approx"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--nprobe", type=int, default=8)
    ap.add_argument("--d", type=int, default=32)
    a = ap.parse_args()
    build.build()
    {"significance": cmd_significance, "preprocessing": cmd_preprocessing, "approx": cmd_approx}[a.cmd](a)


if __name__ == "__main__":
    main()
