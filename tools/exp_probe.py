#!/usr/bin/env python
"""A/B timing of the probe (a5) paths on a saved bench index (tools/exp_scan.py saves it):
knn_path 1 (d_hat matrix + group-minima select), 2 (fused filter, no d_hat), 3 (group minima
only + exact re-rank of in-window groups), and probe_passes 1 / 3. Prints one JSON line per
setting: probe ms (CUDA events, L2 flushed) and the whole-search stage split; checks that every
path returns the same probes.
Usage: python tools/exp_probe.py --config c4 --nprobe 8"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    sys.argv = [a for a in sys.argv]
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--nprobe", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import exp_scan
    from datagen import synth
    from paper_2404_16322_b200 import Index
    path = exp_scan.prepare(argparse.Namespace(config=a.config, n=0, nlist=0))
    cfg = synth.config(a.config)
    Q = torch.from_numpy(np.load(path + ".q.npy")).cuda()
    ix = Index(cfg.d)
    ix.load(path)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ref = None
    for path_opt in (0, 1, 2, 3):
        for passes in (1, 3):
            ix.set_option("knn_path", path_opt)
            ix.set_option("probe_passes", passes)
            try:
                pr = ix.probe(Q, a.nprobe)
            except Exception as e:  # a path may not apply to this shape
                print(json.dumps({"knn_path": path_opt, "passes": passes, "error": str(e)[:120]}), flush=True)
                continue
            same = None
            if ref is None:
                ref = pr.clone()
            else:
                same = bool(torch.equal(ref, pr))
            ts, sc = [], []
            for _ in range(3):
                ix.probe(Q, a.nprobe)
            for _ in range(a.reps):
                flush.fill_(1.0)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ix.probe(Q, a.nprobe)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
                flush.fill_(1.0)
                _, _, st = ix.search(Q, cfg.k, a.nprobe, cfg.delta_d, 0.005, stats=True)
                sc.append(st["ms_total"])
            ts.sort(); sc.sort()
            print(json.dumps({"config": cfg.name, "knn_path": path_opt, "passes": passes, "same_probes": same,
                              "probe_ms_med": round(ts[len(ts) // 2], 4),
                              "search_ms_med": round(sc[len(sc) // 2], 4)}), flush=True)


if __name__ == "__main__":
    main()
