"""Shared helpers: graph builders for the BASELINE.json configs (scaled) and
parity metrics."""
import numpy as np

import paper_1708_07271_b200 as P
from oracle import pyoracle as O

SEED = 0x170807271

# BASELINE.json configs (n, mean degree, p_ref, p_copy, R); C4 is the social model.
CONFIGS = {
    1: dict(kind="copy", n=1 << 20, deg=12.0, p_ref=0.7, p_copy=0.8, R=3),
    2: dict(kind="copy", n=1 << 24, deg=20.0, p_ref=0.7, p_copy=0.8, R=3),
    3: dict(kind="copy", n=1 << 26, deg=24.0, p_ref=0.7, p_copy=0.8, R=3),
    4: dict(kind="social", n=1 << 25, R=0),
    5: dict(kind="copy", n=1 << 27, deg=16.0, p_ref=0.7, p_copy=0.8, R=3),
}


def make_graph(cfg: int, n: int = 0, seed_offset: int = 0) -> P.CsrGraph:
    c = CONFIGS[cfg]
    n = n or c["n"]
    if c["kind"] == "social":
        return P.CsrGraph.social(n, seed=SEED + cfg + seed_offset)
    return P.CsrGraph.copy_model(n, c["deg"], c["p_ref"], c["p_copy"], seed=SEED + cfg + seed_offset)


def bv_params(cfg: int, **kw) -> P.BvParams:
    p = P.BvParams(max_ref=CONFIGS[cfg]["R"])
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def csr_from_rows(rows):
    n = len(rows)
    ro = np.zeros(n + 1, dtype=np.uint64)
    ro[1:] = np.cumsum([len(r) for r in rows])
    cols = np.asarray([c for r in rows for c in r], dtype=np.uint32)
    return P.CsrGraph.from_arrays(n, ro, cols)


def oracle_csr(g: P.CsrGraph) -> O.Csr:
    return O.Csr.from_arrays(g.n, g.row_offsets, g.columns)


def x_uniform(n: int, seed: int = 1) -> np.ndarray:
    """x ~ U[0,1): (u64 >> 11) * 2^-53."""
    rng = np.random.default_rng(seed)
    return (rng.integers(0, 2**64, size=n, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0**-53


def max_rel_err(y, want) -> float:
    y = np.asarray(y, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    denom = np.abs(want)
    err = np.abs(y - want)
    zero = denom == 0
    if np.any(err[zero] != 0):
        return float("inf")  # empty rows must be exactly 0
    if np.all(zero):
        return 0.0
    return float(np.max(err[~zero] / denom[~zero]))
