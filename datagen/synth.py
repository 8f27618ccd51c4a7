"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no PCA, no distances, no
pruning): it only draws the input arrays (base vectors, queries, calibration
queries) whose shapes, spectra and value distributions imitate the paper's
datasets (Table II), following the recipes that
BASELINE.json's `configs` state and SURVEY.md §8(d) fixes where a config
leaves freedom. The real datasets are absent from the container; these
synthetic stand-ins replace them (DESIGN.md §"Input recipe").

Random streams: SeedSequence([seed, stream]) with
  0 = model (Haar basis, centres), 1 = base (chunk c -> [seed, 1, c]),
  2 = queries, 3 = calibration queries, 4 = held-out calibration queries.
"""
from __future__ import annotations

import dataclasses
import numpy as np

CHUNK = 1 << 17  # rows per base chunk (independent seed per chunk)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int            # base vectors
    d: int            # dimension D
    nq: int           # search queries
    n_cal: int        # calibration queries
    nlist: int        # IVF lists (1 = flat)
    nprobes: tuple    # nprobe sweep
    k: int            # K
    delta_d: int      # Δd
    n_comp: int       # mixture components (0 = single Gaussian)
    spectrum: float   # λ_i ∝ i^-spectrum
    lam_total: float  # Σλ (within-component)
    centre_std: float # centre ~ N(0, centre_std² I)  (ignored by "sift")
    kind: str         # "mix" | "sift" | "gist" | "deep"
    n_neg: int = 50   # Label-1 calibration pairs per calibration query
    nprobe_neg: int = 0  # negatives drawn from this many probed lists (0 = whole base)
    seed: int = 0

    def scaled(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs[0..4]; constants marked "proposed" in SURVEY §8(d).
CONFIGS = {
    # configs[0]: flat, 10k x 128, 20-component mixture, centres ~N(0,4I), λ_i ∝ 1/i (Σλ = D)
    "c1": Config("c1", 10_000, 128, 100, 100, 1, (1,), 10, 32, 20, 1.0, 128.0, 2.0, "mix",
                 n_neg=50, nprobe_neg=0),
    # configs[1]: SIFT-shaped 1M x 128, integer-valued [0,255], 256 components
    "c2": Config("c2", 1_000_000, 128, 10_000, 1_000, 4096, (16, 24, 32, 48, 64, 96, 128, 192, 256),
                 10, 16, 256, 1.0, 128.0 * 144.0, 0.0, "sift", n_neg=50, nprobe_neg=16),
    # configs[2]: GIST-shaped 1M x 960, single Gaussian λ_i ∝ i^-1.5, min-max to [0,1]
    "c3": Config("c3", 1_000_000, 960, 1_000, 1_000, 4096, (16, 24, 32, 48, 64, 96, 128),
                 100, 32, 0, 1.5, 960.0, 0.0, "gist", n_neg=50, nprobe_neg=16),
    # configs[3]: Deep-shaped 10M x 96, 1024 components, L2-normalised
    "c4": Config("c4", 10_000_000, 96, 10_000, 1_000, 16384, (32, 48, 64, 96, 128, 192, 256),
                 10, 16, 1024, 1.0, 96 * 0.25, 1.0, "deep", n_neg=50, nprobe_neg=32),
    # configs[4]: 100M x 256, 4096 components, λ_i ∝ i^-1.2
    "c5": Config("c5", 100_000_000, 256, 10_000, 1_000, 65536, (32, 64, 128),
                 100, 32, 4096, 1.2, 256.0, 2.0, "mix", n_neg=50, nprobe_neg=64),
}


def config(name: str, **overrides) -> Config:
    return CONFIGS[name].scaled(**overrides) if overrides else CONFIGS[name]


def _rng(cfg: Config, *stream) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([cfg.seed, *stream])))


def haar_basis(d: int, rng: np.random.Generator) -> np.ndarray:
    """Haar-random orthogonal matrix: QR of a Gaussian, column signs fixed by diag(R)."""
    g = rng.standard_normal((d, d))
    q, r = np.linalg.qr(g)
    return q * np.sign(np.diag(r))[None, :]


@dataclasses.dataclass
class Model:
    basis: np.ndarray      # D x D orthogonal (columns = principal directions of the within spectrum)
    sqrt_lam: np.ndarray   # D
    centres: np.ndarray    # n_comp x D (empty for single Gaussian)


def model(cfg: Config) -> Model:
    rng = _rng(cfg, 0)
    d = cfg.d
    basis = haar_basis(d, rng)
    lam = np.arange(1, d + 1, dtype=np.float64) ** (-cfg.spectrum)
    lam *= cfg.lam_total / lam.sum()
    sl = np.sqrt(lam)
    if cfg.kind == "sift":
        z = rng.standard_normal((cfg.n_comp, d))
        centres = 60.0 + 3.0 * (z * sl[None, :]) @ basis.T
    elif cfg.n_comp > 0:
        centres = cfg.centre_std * rng.standard_normal((cfg.n_comp, d))
    else:
        centres = np.zeros((0, d))
    return Model(basis, sl, centres)


def _draw(cfg: Config, m: Model, rng: np.random.Generator, n: int) -> np.ndarray:
    """n raw float64 rows from the config's generative model (before post-processing)."""
    g = rng.standard_normal((n, cfg.d))
    x = (g * m.sqrt_lam[None, :]) @ m.basis.T
    if cfg.n_comp > 0:
        comp = rng.integers(0, cfg.n_comp, size=n)
        x += m.centres[comp]
    return x


def _post(cfg: Config, x: np.ndarray, minmax=None) -> np.ndarray:
    if cfg.kind == "sift":
        x = np.clip(np.rint(x), 0.0, 255.0)          # round-half-even, clip to [0,255]
    elif cfg.kind == "deep":
        x = x / np.linalg.norm(x, axis=1, keepdims=True)
    elif cfg.kind == "gist":
        lo, hi = minmax
        x = np.clip((x - lo) / (hi - lo), 0.0, 1.0)
    return np.ascontiguousarray(x, dtype=np.float32)


_MINMAX: dict = {}


def _gist_minmax(cfg: Config, m: Model):
    """Global scalar min / max of the raw base (one pass; cached per config: the model is a
    deterministic function of the config)."""
    if cfg not in _MINMAX:
        lo, hi = np.inf, -np.inf
        for c in range((cfg.n + CHUNK - 1) // CHUNK):
            n = min(CHUNK, cfg.n - c * CHUNK)
            x = _draw(cfg, m, _rng(cfg, 1, c), n)
            lo, hi = min(lo, x.min()), max(hi, x.max())
        _MINMAX[cfg] = (lo, hi)
    return _MINMAX[cfg]


def _chunk(args):
    cfg, m, c, minmax = args
    n = min(CHUNK, cfg.n - c * CHUNK)
    return _post(cfg, _draw(cfg, m, _rng(cfg, 1, c), n), minmax)


def base(cfg: Config, m: Model | None = None, rows: slice | None = None, workers: int = 0) -> np.ndarray:
    """Base vectors S (n x D float32, row-major). `rows` selects a contiguous id range
    (e.g. one shard) without generating the rest (chunk c is seeded [seed, 1, c]).
    `workers` > 1 draws chunks in parallel processes (identical result: chunks are independent)."""
    m = m or model(cfg)
    lo_id, hi_id = (0, cfg.n) if rows is None else (rows.start or 0, rows.stop)
    minmax = _gist_minmax(cfg, m) if cfg.kind == "gist" else None
    out = np.empty((hi_id - lo_id, cfg.d), dtype=np.float32)
    chunks = list(range(lo_id // CHUNK, (hi_id + CHUNK - 1) // CHUNK))

    def put(c, x):
        c0 = c * CHUNK
        a, b = max(lo_id, c0), min(hi_id, c0 + x.shape[0])
        out[a - lo_id:b - lo_id] = x[a - c0:b - c0]

    if workers > 1 and len(chunks) > 1:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(workers) as pool:
            for c, x in zip(chunks, pool.imap(_chunk, [(cfg, m, c, minmax) for c in chunks])):
                put(c, x)
    else:
        for c in chunks:
            put(c, _chunk((cfg, m, c, minmax)))
    return out


def queries(cfg: Config, n: int | None = None, stream: int = 2, m: Model | None = None) -> np.ndarray:
    """Queries from the same distribution (stream 2 = search, 3 = calibration, 4 = held-out)."""
    m = m or model(cfg)
    n = cfg.nq if n is None else n
    minmax = _gist_minmax(cfg, m) if cfg.kind == "gist" else None
    return _post(cfg, _draw(cfg, m, _rng(cfg, stream), n), minmax)


def cal_queries(cfg: Config, n: int | None = None, m: Model | None = None) -> np.ndarray:
    return queries(cfg, cfg.n_cal if n is None else n, stream=3, m=m)


def heldout_queries(cfg: Config, n: int, m: Model | None = None) -> np.ndarray:
    return queries(cfg, n, stream=4, m=m)
