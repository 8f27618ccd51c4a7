#!/usr/bin/env python
"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every
kernel family of the library once — PCA moments, rotation, the tcgen05 filter GEMMs (d_hat
writer k_l2_tc and the fused k_probe_tc path), the fp64 certification selects, calibration
features, k_scan with one and four warps per query (TMA/mbarrier ring, shared-memory survivor
ring, the G > 1 epoch merge), the decision-log build, the BSA-res scan, the Exp-7 estimate scan
and the shard merge. Prints one line per stage; sizes are kept small because the sanitizer
serialises and instruments every access.
Usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from datagen import synth  # noqa: E402
from paper_2404_16322_b200 import Index, build  # noqa: E402


def main():
    build.build()
    cfg = synth.config("c2", n=100_000, nlist=256, nq=200, n_cal=64)
    X = torch.from_numpy(synth.base(cfg)).cuda()
    Q = torch.from_numpy(synth.queries(cfg)).cuda()
    Qc = torch.from_numpy(synth.cal_queries(cfg)).cuda()
    ix = Index(cfg.d)
    ix.fit_rotation(X)
    print("fit_rotation ok", flush=True)
    ix.build_ivf(X, cfg.nlist, kmeans_iters=2)
    print("build_ivf ok", flush=True)
    ix.calibrate(X, Qc, cfg.k, n_neg=20, nprobe_neg=8, seed=0)
    print("calibrate ok", flush=True)
    for G in (1, 4):
        ix.set_option("scan_warps", G)
        i, d, st = ix.search(Q, cfg.k, 8, 16, 0.005, stats=True)
        print(f"search G={G} ok tested={st['tested']}", flush=True)
    ix.set_option("scan_warps", 0)
    ix.search(Q, cfg.k, 8, 32, 0.005)
    ix.search(Q, cfg.k, 8, 48 if cfg.d % 48 == 0 else 64, 0.005)
    print("search dd=32/64 ok", flush=True)
    ix.search_log(Q[:50].contiguous(), cfg.k, 8, 16, 0.005)
    print("search_log ok", flush=True)
    ix.search_method(Q, cfg.k, 8, 16, "bsa_res", 8.0)
    ix.search_method(Q, cfg.k, 8, 16, "adsampling", 2.1)
    print("search_method ok", flush=True)
    for path in (1, 2):  # d_hat matrix + k_select_gmin, fused k_probe_tc + k_probe_finish
        ix.set_option("knn_path", path)
        ix.probe(Q, 8)
        ix.bruteforce_knn(X[:20000].contiguous(), Q[:64].contiguous(), 10)
        print(f"probe/knn path={path} ok", flush=True)
    ix.set_option("knn_path", 0)
    ix.estimate_knn(Q[:64].contiguous(), 32, 10, "partial")
    ix.estimate_knn(Q[:64].contiguous(), 32, 10, "residual")
    print("estimate ok", flush=True)
    ids, dists = ix.search(Q, cfg.k, 8, 16, 0.0)
    ix.merge_topk(torch.stack([ids, ids]), torch.stack([dists, dists]))
    print("merge ok", flush=True)
    Qh = synth.queries(cfg)
    ix.search_host(Qh, cfg.k, 8, 16, 0.005)
    print("search_host ok", flush=True)
    torch.cuda.synchronize()
    print("SANITIZE RUN DONE", flush=True)


if __name__ == "__main__":
    main()
