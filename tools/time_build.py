import sys, time, torch
sys.path.insert(0, '/root/repo')
from datagen import synth
from paper_2404_16322_b200 import Index
for name in ("c2", "c3"):
    cfg = synth.config(name)
    m = synth.model(cfg)
    X = torch.from_numpy(synth.base(cfg, m, workers=16)).cuda()
    ix = Index(cfg.d)
    ix.fit_rotation(X)
    torch.cuda.synchronize(); t = time.time()
    ix.build_ivf(X, cfg.nlist, kmeans_iters=10)
    torch.cuda.synchronize(); print(name, "build_ivf s", time.time() - t, flush=True)
