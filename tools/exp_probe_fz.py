#!/usr/bin/env python
"""A/B timing of the probe (a5) filter paths on a bench-shaped centroid set, without building the
database: centroids = the first nlist rows of the config's synthetic base (the same mixture the
k-means centroids summarise), queries = the config's queries. knn_path 1 (d_hat matrix + group
minima), 2 (fused filter of probe_tc.cu), 4 (throughput fused filter, fp16 operands), 5 (the same,
tf32). Prints one JSON line per path: probe ms (CUDA events on the library's stream, L2 flushed
between runs, median of --reps) and whether the probes equal path 1's.
Usage: python tools/exp_probe_fz.py --config c4 [--nprobe 8] [--paths 1,4,5]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from datagen import synth
    from paper_2404_16322_b200 import Index, build
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--nprobe", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--paths", default="1,2,4,5")
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--seed-stride", default="", help="comma list of DADE_OPT_FZ_SEED_STRIDE values (path 4)")
    ap.add_argument("--gmin-ratio", default="", help="comma list of DADE_OPT_GMIN_RATIO values (path 0)")
    ap.add_argument("--chunk-mb", default="", help="comma list of DADE_OPT_DHAT_CHUNK_MB values (path 1)")
    ap.add_argument("--h16", action="store_true", help="also time path 1 with the fp16-operand d_hat writer (DADE_OPT_DHAT_H16)")
    ap.add_argument("--debug", type=int, default=0, help="fz_debug option (1/2: pipeline-only launch first)")
    ap.add_argument("--fz", default="", help="comma list of S:G:cps[:cpc[:rows[:cols]]] overrides for paths 4/5, e.g. 4:1:1,12:2:1")
    a = ap.parse_args()
    build.build()
    cfg = synth.config(a.config)
    m = synth.model(cfg)
    nrows = cfg.nlist + 1000
    X = synth.base(cfg, m, rows=slice(0, nrows), workers=min(16, os.cpu_count() or 1))
    Q = synth.queries(cfg, m=m, n=a.nq or None)
    Xd = torch.from_numpy(X).cuda()
    Qd = torch.from_numpy(Q).cuda()
    ix = Index(cfg.d)
    ix.fit_rotation(Xd)
    ix.build_ivf(Xd, cfg.nlist, centroids=Xd[:cfg.nlist].contiguous())
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    ref = None
    if a.debug:
        ix.set_option("fz_debug", a.debug)
    runs = [(int(p), None) for p in a.paths.split(",")]
    runs += [(4, tuple(int(v) for v in f.split(":"))) for f in a.fz.split(",") if f]
    runs += [(1, ("dhat_h16", 1)), (1, ("dhat_h16", 2)), (1, ("dhat_h16", 3))] if a.h16 else []  # 2: 128 x 256 tiles
    runs += [(1, ("chunk_mb", int(v))) for v in a.chunk_mb.split(",") if v]
    runs += [(0, ("gmin_ratio", int(v))) for v in a.gmin_ratio.split(",") if v]
    runs += [(4, ("seed_stride", int(v))) for v in a.seed_stride.split(",") if v]
    for path, fz in runs:
        ix.set_option("knn_path", path)
        ix.set_option("gmin_ratio", fz[1] if fz and fz[0] == "gmin_ratio" else 1)
        ix.set_option("fz_seed_stride", fz[1] if fz and fz[0] == "seed_stride" else 0)
        ix.set_option("dhat_h16", fz[1] if fz and fz[0] == "dhat_h16" else 0)
        if fz and fz[0] == "chunk_mb":
            ix.set_option("dhat_chunk_mb", fz[1])
        elif fz and fz[0] in ("gmin_ratio", "seed_stride", "dhat_h16"):
            pass
        else:
            ix.set_option("dhat_chunk_mb", 0)
            for nm, val in zip(("fz_stages", "fz_groups", "fz_cps", "fz_cpc", "fz_rows", "fz_cols"),
                               (tuple(fz) + (0,) * 6)[:6] if fz else (0,) * 6):
                ix.set_option(nm, val)
        try:
            pr = ix.probe(Qd, a.nprobe)
        except Exception as e:  # an override that does not fit shared memory / TMEM: report, go on
            print(json.dumps({"config": cfg.name, "knn_path": path, "fz": fz, "error": str(e)[:120]}), flush=True)
            continue
        same = None
        if ref is None:
            ref = pr.clone()
        else:
            same = bool(torch.equal(ref, pr))
        for _ in range(3):
            ix.probe(Qd, a.nprobe)
        ts = []
        for _ in range(a.reps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ix.probe(Qd, a.nprobe)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        D, C, nq = cfg.d, cfg.nlist, Q.shape[0]
        print(json.dumps({"config": cfg.name, "nq": nq, "nlist": C, "D": D, "nprobe": a.nprobe, "knn_path": path, "fz": fz,
                          "same_probes_as_first": same, "probe_ms_med": round(ts[len(ts) // 2], 4),
                          "probe_ms_min": round(ts[0], 4),
                          "filter_tflops_at_med": round(2 * nq * C * D / (ts[len(ts) // 2] / 1e3) / 1e12, 1)}),
              flush=True)


if __name__ == "__main__":
    main()
