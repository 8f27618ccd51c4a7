#!/usr/bin/env python
"""A/B timing of k_scan across library builds (experiment libs from tools/build_variant.py or the
product library) on one workload. The index is built once with the product library and saved
(/tmp/dade_exp_<cfg>.idx); every library then loads it in its own subprocess, so all variants
search the identical layout and calibration.

Usage: python tools/exp_scan.py --config c4 --nprobe 8 LIB[=ENV:V,ENV2:V] ...
(DADE_EXP_OPTS:scan_order:2 sets dade_set_option values in the child)
Prints one JSON line per library: scan ms (median / min of --reps, L2 flushed), total ms, scan
rate, recall@10 vs exact IVF at the same nprobe."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def prepare(a):
    import numpy as np
    import torch
    from datagen import synth
    from paper_2404_16322_b200 import Index, build
    build.build()
    cfg = synth.config(a.config)
    if a.n:
        cfg = cfg.scaled(n=a.n, nlist=a.nlist or max(1, a.n // 244))
    path = f"/tmp/dade_exp_{cfg.name}_{cfg.n}.idx"
    m = synth.model(cfg)
    Q = synth.queries(cfg, m=m)
    np.save(path + ".q.npy", Q)
    if os.path.exists(path):
        return path
    X = torch.from_numpy(synth.base(cfg, m, workers=min(16, os.cpu_count() or 1))).cuda()
    Qc = torch.from_numpy(synth.cal_queries(cfg, m=m)).cuda()
    ix = Index(cfg.d)
    ix.fit_rotation(X)
    ix.build_ivf(X, cfg.nlist, kmeans_iters=10)
    ix.calibrate(X, Qc, cfg.k, n_neg=cfg.n_neg, nprobe_neg=cfg.nprobe_neg, seed=0)
    ix.save(path)
    return path


def child(a, path):
    import numpy as np
    import torch
    from datagen import synth
    from paper_2404_16322_b200 import Index
    cfg = synth.config(a.config)
    Q = torch.from_numpy(np.load(path + ".q.npy")).cuda()
    ix = Index(cfg.d)
    ix.load(path)
    for kv in filter(None, os.environ.get("DADE_EXP_OPTS", "").split(",")):
        k_, v_ = kv.split(":")
        ix.set_option(k_, int(v_))
    K, dd = cfg.k, cfg.delta_d
    ei, _ = ix.search(Q, K, a.nprobe, dd, 0.0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for _ in range(3):
        ix.search(Q, K, a.nprobe, dd, 0.005)
    sc, tot = [], []
    st = None
    for _ in range(a.reps):
        flush.fill_(1.0)
        i, d, st = ix.search(Q, K, a.nprobe, dd, 0.005, stats=True)
        sc.append(st["ms_scan"]); tot.append(st["ms_total"])
    sc.sort(); tot.sort()
    ii, ee = i.cpu().numpy(), ei.cpu().numpy()
    rc = sum(len(set(f[:10].tolist()) & set(g[:10].tolist())) for f, g in zip(ii, ee)) / (10 * len(ii))
    print(json.dumps({"lib": os.environ.get("DADE_LIB", "product"), "env": a.env, "config": cfg.name,
                      "nprobe": a.nprobe, "scan_ms_med": round(sc[len(sc) // 2], 4), "scan_ms_min": round(sc[0], 4),
                      "total_ms_med": round(tot[len(tot) // 2], 4),
                      "scan_rate": round(st["dims_scanned"] / (st["tested"] * cfg.d), 4),
                      "recall_vs_exact_ivf": round(rc, 5), "n_epochs": st["n_epochs"]}), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--nprobe", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--nlist", type=int, default=0)
    ap.add_argument("--child", default="")
    ap.add_argument("--env", default="")
    ap.add_argument("libs", nargs="*")
    a = ap.parse_args()
    if a.child:
        child(a, a.child)
        sys.exit(0)
    path = prepare(a)
    for spec in a.libs or ["product"]:
        lib, _, envs = spec.partition("=")
        env = dict(os.environ)
        if lib != "product":
            env["DADE_LIB"] = os.path.abspath(lib)
        for kv in filter(None, envs.split(",")):
            k, v = kv.split(":", 1)
            env[k] = v
        cmd = [sys.executable, __file__, "--config", a.config, "--nprobe", str(a.nprobe), "--reps", str(a.reps),
               "--child", path, "--env", envs]
        if a.n:
            cmd += ["--n", str(a.n), "--nlist", str(a.nlist)]
        subprocess.run(cmd, env=env)
