import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from datagen import synth
from paper_2404_16322_b200 import Index
cfg = synth.config("c2"); m = synth.model(cfg)
X = synth.base(cfg, m); Q = synth.queries(cfg, m=m)[:20]
ix = Index(cfg.d); Xd = torch.from_numpy(X).cuda()
ix.fit_rotation(Xd); ix.build_ivf(Xd, cfg.nlist, kmeans_iters=10)
off, row_id, assign, C = ix.get_ivf()
C = C.astype(np.float64); Qd = Q.astype(np.float64)
mu = C.mean(0).astype(np.float32).astype(np.float64)
Cc = C - mu; Qc = Qd - mu
gamma = 2 * (3 * 128 + 16) * 2**-23
bmax = (Cc**2).sum(1).max()
for q, qc in zip(Qd, Qc):
    d = ((C - q)**2).sum(1)
    S = gamma * ((qc**2).sum() + bmax)
    cnt = []
    for s in range(4):
        ds = np.sort(d[s*1024:(s+1)*1024]); t = ds[7]
        cnt.append(int((ds <= t + 2*S).sum()))
    print(f"dk={np.sort(d)[7]:.1f} d0={np.sort(d)[0]:.1f} |qc|2={(qc**2).sum():.0f} bmax={bmax:.0f} S={S:.2f} win {cnt}")
