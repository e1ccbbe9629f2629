"""Exhaustive ground truth on the GPU: the same entry
points and results as the reference's ``exact`` module (exact.py:57-173),
computed by ``eg_bf_cosine_candidates`` (tcgen05 fp16 screen with a
certified margin) + ``eg_verify`` (exact fp64 distances) and ``eg_bf_hamming``
(all-pairs XOR/popcount).  The reference refuses more than 50,000 rows by
default (``limit``, exact.py:27-33); the GPU versions keep that default so
they behave the same, and pass ``limit=None`` to measure recall at full scale
(e.g. the 1.6M rows of config 3).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native, engine
from .bitpool import BitStringPool
from .edges import EdgeList
from .hamming_join import PairSet
from .lsh import VectorDataset

__all__ = ["ErrorReport", "brute_force_cosine", "brute_force_hamming", "measure_errors"]

_DEFAULT_LIMIT = 50_000


@dataclass(frozen=True)
class ErrorReport:
    """Set differences between an approximate result and the exact edge set
    (exact.py:30-49)."""
    true_edge_count: int
    missing_count: int
    false_candidate_count: int
    missing_ratio: float
    per_replicate: tuple[int, ...] | None = None


def _check_limit(n: int, limit) -> None:
    if limit is not None and n > limit:
        raise ValueError(
            f"{n} rows exceed the exhaustive-comparison limit of {limit}; "
            "raise `limit` explicitly if this is intentional")


def _candidates(fn, cap0: int, dev):
    """Run a capacity-bounded enumerator; grow the buffer once if needed."""
    cap = max(int(cap0), 1024)
    while True:
        keys = torch.empty(cap, dtype=torch.int64, device=dev)
        cnt = fn(keys, cap)
        if cnt <= cap:
            return keys[:cnt]
        cap = int(cnt)


def brute_force_cosine(data, epsilon: float, *, limit=_DEFAULT_LIMIT, block_rows: int = 1024,
                       device=None) -> EdgeList:
    """Exact cosine-radius edges by all-pairs comparison (exact.py:57-95).

    ``block_rows`` is accepted for compatibility (the result does not depend
    on it).  Distances are the exact fp64 filter distances of eg_verify; the
    edge set equals the reference's except for pairs within ~1e-15 of
    ``epsilon`` (the reference's BLAS product has its own rounding)."""
    rows = data.vectors if isinstance(data, VectorDataset) else data
    if isinstance(rows, torch.Tensor):
        n = int(rows.shape[0])
    else:
        rows = np.asarray(rows)
        n = int(rows.shape[0]) if rows.ndim else 0
    _check_limit(n, limit)
    dev = engine.require_device(device)
    with torch.cuda.device(dev):
        x = engine.as_device_rows(rows, dev)
        if n < 2:
            return EdgeList()
        norms = engine.validate_rows(x)
        lib = _native.lib()
        dim = int(x.shape[1])
        ws = engine._ws(lib.eg_bf_cosine_workspace(n, dim), dev)
        st = engine._stream(dev)

        def run(keys, cap):
            cnt = engine.ctypes_i64(0)
            _native.check(lib.eg_bf_cosine_candidates(
                engine._p(x), int(x.dtype == torch.float64), n, dim, engine._p(norms),
                float(epsilon), engine._p(keys), cap, engine.ctypes_addr(cnt), engine._p(ws),
                ws.numel(), st), "brute_force_cosine")
            return int(cnt.value)

        keys = _candidates(run, 4 * n, dev)
        engine.sort_pair_keys(keys, n)
        ek, ed = engine.verify(x, norms, keys, _native.METRIC_COSINE, float(epsilon))
        return EdgeList(engine.keys_to_pairs(ek.cpu().numpy()), ed.cpu().numpy())


def brute_force_hamming(pool: BitStringPool, d: int, *, limit=_DEFAULT_LIMIT,
                        block_rows: int = 256, device=None) -> PairSet:
    """Exact d-neighbour pairs by exhaustive XOR-popcount (exact.py:98-121)."""
    n = pool.count
    _check_limit(n, limit)
    if d < 0:
        raise ValueError("d must be non-negative")
    if n < 2:
        return PairSet(np.empty((0, 2), dtype=np.int64), assume_normalized=True)
    dev = engine.require_device(device)
    with torch.cuda.device(dev):
        words = np.ascontiguousarray(pool.words)
        codes = torch.from_numpy(words.view(np.int64)).to(dev)
        lib = _native.lib()
        ws = engine._ws(lib.eg_bf_hamming_workspace(), dev)
        st = engine._stream(dev)

        def run(keys, cap):
            cnt = engine.ctypes_i64(0)
            _native.check(lib.eg_bf_hamming(engine._p(codes), n, int(words.shape[1]), int(d),
                                            engine._p(keys), cap, engine.ctypes_addr(cnt),
                                            engine._p(ws), ws.numel(), st),
                          "brute_force_hamming")
            return int(cnt.value)

        keys = _candidates(run, 4 * n, dev)
        engine.sort_pair_keys(keys, n)
        return PairSet(engine.keys_to_pairs(keys.cpu().numpy()), assume_normalized=True)


def _pair_array(obj) -> np.ndarray:
    if isinstance(obj, np.ndarray):
        return obj.reshape(-1, 2).astype(np.int64, copy=False)
    if isinstance(obj, PairSet):
        return obj.array
    if isinstance(obj, EdgeList):
        return obj.pairs
    for attr in ("pairs", "edge_list"):
        inner = getattr(obj, attr, None)
        if inner is not None:
            return _pair_array(inner)
    raise TypeError(f"cannot read pairs from {type(obj).__name__}")


def _pair_keys(pairs: np.ndarray) -> np.ndarray:
    if pairs.size and int(pairs.max()) >= 1 << 31:
        raise ValueError("indices above 2**31 are not supported here")
    return (pairs[:, 0] << np.int64(32)) | pairs[:, 1]


def measure_errors(approx, exact) -> ErrorReport:
    """Missing/extra accounting of an approximate edge set against the exact
    one (exact.py:146-173): host set arithmetic on sorted int64 keys."""
    a = _pair_keys(_pair_array(approx))
    e = _pair_keys(_pair_array(exact))
    missing = int(np.setdiff1d(e, a).size)
    extra = int(np.setdiff1d(a, e).size)
    true_count = int(e.size)
    attribution = getattr(approx, "per_replicate_new", None)
    if attribution is None:
        attribution = getattr(getattr(approx, "stats", None), "per_replicate_new", None)
    return ErrorReport(true_edge_count=true_count, missing_count=missing,
                       false_candidate_count=extra,
                       missing_ratio=missing / true_count if true_count else 0.0,
                       per_replicate=tuple(attribution) if attribution is not None else None)
