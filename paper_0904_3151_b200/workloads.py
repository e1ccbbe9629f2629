"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference publishes no dataset for this path; these generators are the
pinned interpretation recorded in SURVEY.md Appendix C (all use
``np.random.default_rng(seed)`` and produce float32 rows, or uint64 words for
config 2).  Every generator takes a scale knob so that tests can draw a
CPU-oracle-sized instance with the same shape and value distribution.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class BuildConfig:
    """Parameters of one build configuration (see BASELINE.json ``configs``)."""
    name: str
    epsilon: float          # radius in the config's metric
    metric: str             # "cosine" or "euclidean"
    length: int
    blocks: int
    mismatch: int
    replicates: int
    seed: int = 0


CONFIGS = {
    "cfg1": BuildConfig("cfg1", 0.1, "cosine", 32, 8, 2, 1),
    "cfg2": BuildConfig("cfg2", 0.0, "hamming", 64, 8, 2, 1),
    "cfg3": BuildConfig("cfg3", 0.05, "cosine", 48, 12, 3, 3),
    "cfg4": BuildConfig("cfg4", 0.08, "cosine", 64, 16, 2, 1),
    "cfg5": BuildConfig("cfg5", 0.15, "euclidean", 64, 16, 3, 2),
}


def _normalise64(x: np.ndarray) -> np.ndarray:
    return x / np.linalg.norm(x, axis=1, keepdims=True)


def cfg1_points(n: int = 20_000, dim: int = 64, clusters: int = 200,
                seed: int = 0) -> np.ndarray:
    """Config 1: Gaussian clusters (centres N(0,I), sigma 0.1), L2-normalised."""
    rng = np.random.default_rng(seed)
    centres = rng.standard_normal((clusters, dim))
    lab = rng.integers(0, clusters, n)
    x = centres[lab] + 0.1 * rng.standard_normal((n, dim))
    return _normalise64(x).astype(np.float32)


def cfg2_words(n_base: int = 10_000_000, n_planted: int = 500_000,
               seed: int = 0) -> np.ndarray:
    """Config 2: uniform 64-bit strings plus planted partners at Hamming 0-2.

    Partners are copies of distinct random sources with h ~ U{0,1,2} distinct
    random bit flips, appended after the base rows.  Returns uint64[n, 1].
    """
    rng = np.random.default_rng(seed)
    w = rng.integers(0, 2**64, size=n_base, dtype=np.uint64)
    src = rng.choice(n_base, n_planted, replace=False)
    h = rng.integers(0, 3, n_planted)
    partners = w[src].copy()
    for i in np.nonzero(h > 0)[0]:
        pos = rng.choice(64, int(h[i]), replace=False)
        flip = np.uint64(0)
        for p in pos:
            flip |= np.uint64(1) << np.uint64(int(p))
        partners[i] ^= flip
    return np.concatenate([w, partners]).reshape(-1, 1)


def cfg3_points(n: int = 1_600_000, dim: int = 384, planted_rows: int | None = None,
                seed: int = 0) -> np.ndarray:
    """Config 3: |N(0,1)|^2 entries, planted near-duplicate groups, normalised.

    The first ``planted_rows`` rows (5% of n by default) form groups of size
    U{2..10}; every member is ``base + N(0, 0.02^2)`` noise added *before*
    normalisation (no clipping).  Normalisation is in float32.
    """
    rng = np.random.default_rng(seed)
    if planted_rows is None:
        planted_rows = n // 20
    raw = rng.standard_normal((n, dim), dtype=np.float32)
    np.square(raw, out=raw)
    row = 0
    while row < planted_rows:
        g = min(int(rng.integers(2, 11)), planted_rows - row)
        if g < 2:
            break
        base = raw[row].copy()
        raw[row:row + g] = base + 0.02 * rng.standard_normal((g, dim), dtype=np.float32)
        row += g
    raw /= np.linalg.norm(raw, axis=1, keepdims=True)
    return raw


def cfg4_points(n: int = 4_000_000, dim: int = 128, largest: int = 50_000,
                subset: int | None = None, seed: int = 0, labels: bool = False):
    """Config 4: rank-size Zipf(1.2) clusters (sigma 0.05) plus N(0,I) singletons.

    Cluster r has floor(largest * r^-1.2) members (kept when >= 2); rows are
    normalised in float64, permuted, optionally row-subsampled, cast to f32.
    ``labels=True`` also returns each row's cluster rank (0 = largest, -1 =
    singleton); the random stream is the same either way.
    """
    rng = np.random.default_rng(seed)
    ranks = np.arange(1, 100_000, dtype=np.float64)
    sizes = np.floor(largest * ranks ** -1.2).astype(np.int64)
    sizes = sizes[sizes >= 2]
    m = int(sizes.sum())
    if m > n:
        raise ValueError("planted rows exceed n")
    centres = rng.standard_normal((sizes.size, dim))
    x = np.empty((n, dim), dtype=np.float64)
    x[:m] = (centres[np.repeat(np.arange(sizes.size), sizes)]
             + 0.05 * rng.standard_normal((m, dim)))
    x[m:] = rng.standard_normal((n - m, dim))
    x = _normalise64(x)
    perm = rng.permutation(n)
    x = x[perm]
    lab = None
    if labels:
        lab = np.full(n, -1, dtype=np.int64)
        lab[:m] = np.repeat(np.arange(sizes.size), sizes)
        lab = lab[perm]
    if subset is not None:
        sel = np.sort(rng.choice(n, subset, replace=False))
        x = x[sel]
        lab = lab[sel] if labels else None
    x = x.astype(np.float32)
    return (x, lab) if labels else x


def cfg5_points(n: int = 20_000_000, dim: int = 128, clusters: int = 1_000_000,
                seed: int = 0, labels: bool = False):
    """Config 5: Gaussian clusters (sigma 0.05) normalised per 2^20-row block.
    ``labels=True`` also returns each row's cluster id (same random stream)."""
    rng = np.random.default_rng(seed)
    centres = rng.standard_normal((clusters, dim), dtype=np.float32)
    out = np.empty((n, dim), dtype=np.float32)
    labs = np.empty(n, dtype=np.int64) if labels else None
    for lo in range(0, n, 1 << 20):
        rows = min(1 << 20, n - lo)
        lab = rng.integers(0, clusters, rows)
        blk = centres[lab] + 0.05 * rng.standard_normal((rows, dim), dtype=np.float32)
        blk /= np.linalg.norm(blk, axis=1, keepdims=True)
        out[lo:lo + rows] = blk
        if labels:
            labs[lo:lo + rows] = lab
    return (out, labs) if labels else out


def planted_clusters(n, dim, clusters, cluster_size, spread, seed):
    """Tight clusters on the unit sphere plus a diffuse N(0,I) background.

    Same distribution as the reference test fixture (tests/conftest.py:42-57):
    unit centres repeated ``cluster_size`` times plus ``spread`` jitter, then
    Gaussian background rows; float32.
    """
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((clusters, dim))
    centers /= np.linalg.norm(centers, axis=1, keepdims=True)
    planted = np.repeat(centers, cluster_size, axis=0)
    planted = planted + spread * rng.standard_normal(planted.shape)
    background = rng.standard_normal((n - clusters * cluster_size, dim))
    return np.vstack([planted, background]).astype(np.float32)


def restricted_subset(labels: np.ndarray, clusters, extra: int = 20_000,
                      seed: int = 4321) -> np.ndarray:
    """Sorted row subset S for restricted-subset parity:
    every member of the given clusters plus ``extra`` seeded random rows.
    The Hamming pair set is a pairwise predicate, so (pairs of the full
    build) restricted to S x S must equal the pairs enumerated on pool[S]."""
    rng = np.random.default_rng(seed)
    n = labels.shape[0]
    pick = rng.choice(n, min(extra, n), replace=False)
    members = np.nonzero(np.isin(labels, np.asarray(list(clusters), dtype=np.int64)))[0]
    return np.unique(np.concatenate([members, pick])).astype(np.int64)


def largest_clusters(labels: np.ndarray, count: int) -> list:
    """Ids of the ``count`` most populous clusters (ties: smaller id first)."""
    lab = labels[labels >= 0]
    sizes = np.bincount(lab)
    order = np.argsort(-sizes, kind="stable")
    return [int(c) for c in order[:count]]
