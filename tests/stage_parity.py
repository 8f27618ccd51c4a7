"""Stage-isolated oracle parity helpers: the oracle runs its own search (O5) on
the artefacts the GPU built — rotation (μ, R, λ), IVF (centroids, lists) and calibration table —
so a full-size search can be checked query by query without the oracle rebuilding a 10M-row
index; and per-candidate decisions of the GPU's decision log are compared with the oracle's.

Tolerance (R21): a decision may differ only where the oracle's closest call
|m1·P_d + β'_d − τ| / (|m1·P_d| + |β'_d| + τ) is ≤ BAND = 1e-5 — the north_star's distance
tolerance, which covers the fp32 storage of x̃ and q̃, the fp32 block sums, the fp32 m1 / β' and
the GPU's fp32 τ. A difference inside the band can change τ for the rest of that query's
candidate stream, so the rest of such a query is not compared; such queries must stay rare.
No method arithmetic here beyond calling the oracle."""
import numpy as np

from oracle import dade_oracle as O

BAND = 1e-5


class LazyRotated:
    """x̃ rows on demand: `obj[ids - id_base]` = O.rotate(X[rows], μ, R) (fp64), so the oracle can
    search a 10M-row base without materialising all of x̃."""

    def __init__(self, X, mean, R):
        self.X, self.mean, self.R = X, mean, R
        self.shape = X.shape

    def __getitem__(self, rows):
        return O.rotate(self.X[rows], self.mean, self.R)


def oracle_index_from_gpu(ix, X, id_base=0, with_cal=True):
    """The oracle's index dict built from the GPU index's own artefacts (dade_get_rotation /
    dade_get_ivf / dade_get_calibration) over the raw base X of this shard."""
    mean, R, lam = ix.get_rotation()
    off, row_id, assign, cent = ix.get_ivf()
    idx = {"centroids": cent, "assign": assign, "off": off, "row_id": row_id, "mean": mean, "R": R,
           "cal": ix.get_calibration() if with_cal else None, "id_base": id_base, "lam": lam,
           "Xr": LazyRotated(X, mean, R)}
    return idx


def compare_decisions(glog, ocands, band=BAND):
    """glog: GPU decision log, int array [n, 3] (query, id, dims read). ocands: the oracle's
    st["candidates"] (per query, epoch by epoch in stream order: query, id, dims, closest call).
    Asserts every tested candidate appears exactly once on both sides and that, per query, the
    first candidate whose dims differ (if any) lies inside the band. Returns (flagged queries,
    per-query dims dict of the compared part)."""
    glog = np.asarray(glog, np.int64)
    oq, oi, od, om = (np.concatenate(c) for c in zip(*ocands)) if ocands else (np.zeros(0),) * 4
    gkey = glog[:, 0] * (1 << 32) + glog[:, 1]
    okey = oq.astype(np.int64) * (1 << 32) + oi.astype(np.int64)
    assert len(np.unique(gkey)) == len(gkey), "a candidate was logged twice"
    assert len(gkey) == len(okey), (len(gkey), len(okey))
    order = np.argsort(gkey)
    gk, gd = gkey[order], glog[order, 2]
    pos = np.searchsorted(gk, okey)
    assert np.all(pos < len(gk)) and np.array_equal(gk[np.minimum(pos, len(gk) - 1)], okey), \
        "tested candidate sets differ"
    gdo = gd[pos]                                            # GPU dims in the oracle's stream order
    flagged = {}
    diff = gdo != od
    for q in np.unique(oq[diff]):
        first = np.nonzero(diff & (oq == q))[0][0]
        assert om[first] <= band, (int(q), int(oi[first]), int(od[first]), int(gdo[first]), float(om[first]))
        flagged[int(q)] = int(oi[first])
    return flagged, oq, od, gdo


def step_histogram(q, dims, D, delta_d, exclude=()):
    """pruned_at_step counts (index s = pruned at d = s·Δd) over the candidates of queries not in
    `exclude` (dims == D: survived)."""
    keep = ~np.isin(q, list(exclude)) if len(exclude) else np.ones(len(q), bool)
    d = dims[keep]
    h = np.zeros(D // delta_d, np.int64)
    pr = d[d < D] // delta_d
    np.add.at(h, pr, 1)
    return h
