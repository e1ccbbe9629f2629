"""All-pairs Hamming joins by the multiple sorting method (mirrors
hamming_join.py).

``enumerate_pairs`` and ``grouped_radix_sort`` run on the GPU through the C
ABI (``eg_msm_pairs`` / ``eg_grouped_sort`` + ``eg_sort_pair_keys``); the
result is the reference's exact pair set, sorted by ``(i, j)``.
"""

from __future__ import annotations

import logging
import math

import numpy as np
import torch

from . import engine
from .bitpool import BitStringPool, block_mask_bits, block_partition, validate_mask

__all__ = ["PairSet", "SortScratch", "enumerate_pairs", "grouped_radix_sort", "mask_count"]

logger = logging.getLogger(__name__)


class PairSet:
    """Set of index pairs ``(i, j)``, ``i < j``, stored sorted and unique
    (hamming_join.py:152-213)."""

    __slots__ = ("array",)

    def __init__(self, pairs, *, assume_normalized: bool = False):
        arr = np.asarray(pairs, dtype=np.int64)
        if arr.size == 0:
            arr = arr.reshape(0, 2)
        if arr.ndim != 2 or arr.shape[1] != 2:
            raise ValueError("pairs must have shape (m, 2)")
        if not assume_normalized:
            lo, hi = arr.min(axis=1), arr.max(axis=1)
            if np.any(lo == hi):
                raise ValueError("self-pairs are not allowed")
            arr = np.unique(np.column_stack([lo, hi]), axis=0)
        self.array = arr

    @classmethod
    def from_pairs(cls, pairs) -> "PairSet":
        return cls(np.array(list(pairs), dtype=np.int64).reshape(-1, 2))

    def to_set(self) -> set[tuple[int, int]]:
        return {(int(i), int(j)) for i, j in self.array}

    def __len__(self) -> int:
        return self.array.shape[0]

    def __iter__(self):
        for i, j in self.array:
            yield int(i), int(j)

    def __contains__(self, pair) -> bool:
        i, j = sorted((int(pair[0]), int(pair[1])))
        lo = np.searchsorted(self.array[:, 0], i, side="left")
        hi = np.searchsorted(self.array[:, 0], i, side="right")
        return bool(np.any(self.array[lo:hi, 1] == j))

    def __eq__(self, other) -> bool:
        if not isinstance(other, PairSet):
            return NotImplemented
        return self.array.shape == other.array.shape and bool(np.array_equal(self.array, other.array))

    def __repr__(self) -> str:  # pragma: no cover
        return f"PairSet({len(self)} pairs)"


class SortScratch:
    """API-compatibility shim for the reference's CPU sort scratch
    (hamming_join.py:216-242).  The GPU path sizes its own workspaces from
    the torch caching allocator, so this only keeps the validation."""

    def __init__(self, capacity: int, chunk_bits: int = 16):
        if capacity < 1:
            raise ValueError("capacity must be positive")
        if not (1 <= chunk_bits <= 24):
            raise ValueError("chunk_bits must be in [1, 24]")
        self.capacity = capacity
        self.chunk_bits = chunk_bits

    def check(self, n: int, chunk_bits: int) -> None:
        if n > self.capacity:
            raise ValueError(f"scratch sized for {self.capacity} rows, got {n}")
        if chunk_bits != self.chunk_bits:
            raise ValueError(f"scratch built for chunk_bits={self.chunk_bits}, got {chunk_bits}")


def mask_count(k: int, d: int) -> int:
    if d < 0 or k < 0 or d > k:
        raise ValueError(f"need 0 <= d <= k, got d={d}, k={k}")
    return math.comb(k, d)


def _codes_on_device(pool: BitStringPool, dev):
    w = np.ascontiguousarray(pool.words).view(np.int64)
    return torch.from_numpy(w).to(dev).reshape(1, pool.count, pool.word_count)


def grouped_radix_sort(pool: BitStringPool, mask, chunk_bits: int = 16,
                       scratch: SortScratch | None = None, *, device=None):
    """``(perm, group_bounds)`` with equal masked keys contiguous
    (hamming_join.py:275-297): the reference's own permutation (first-seen
    buckets of chunk_bits-wide counting passes, last chunk first), computed
    on the GPU by eg_grouped_sort."""
    if pool.count == 0:
        raise ValueError("pool is empty")
    if scratch is None:
        scratch = SortScratch(pool.count, chunk_bits)
    scratch.check(pool.count, chunk_bits)
    mask = validate_mask(mask, pool.block_count)
    dev = engine.require_device(device)
    codes = _codes_on_device(pool, dev)
    perm, bounds = engine.grouped_sort(codes[0], pool.length, pool.block_bounds,
                                       block_mask_bits(mask), chunk_bits)
    return perm.cpu().numpy().astype(np.int64), bounds.cpu().numpy()


def warn_oversized(largest: int, n: int, oversized_fraction: float):
    """Same trigger and message shape as hamming_join.py:341-344, 365-368."""
    if n > 16 and largest > oversized_fraction * n:
        logger.warning("largest equal-key group holds %d of %d rows; the block "
                       "parameters look too coarse for this pool", largest, n)


def enumerate_pairs(pool: BitStringPool, d: int, chunk_bits: int = 16,
                    scratch: SortScratch | None = None, oversized_fraction: float = 0.25,
                    *, device=None) -> PairSet:
    """All ``(i, j)``, ``i < j``, with Hamming distance <= d
    (hamming_join.py:300-375), computed by the sm_100a MSM kernels."""
    n = pool.count
    if n == 0:
        raise ValueError("pool is empty")
    k = pool.block_count
    if not (0 <= d < k <= pool.length):
        raise ValueError(f"need 0 <= d < k <= length, got d={d}, k={k}, length={pool.length}")
    if scratch is None:
        scratch = SortScratch(n, chunk_bits)
    scratch.check(n, chunk_bits)
    dev = engine.require_device(device)
    codes = _codes_on_device(pool, dev)
    keys, info = engine.msm_candidates(codes, pool.length, k, d,
                                       oversized_fraction=oversized_fraction,
                                       block_bounds=pool.block_bounds)
    if info["reference_blocks"]:   # else the plan ruled the warning out on the reference blocks
        warn_oversized(info["max_group"], n, oversized_fraction)
    engine.sort_pair_keys(keys, n)
    return PairSet(engine.edges_to_host(keys, None)[0], assume_normalized=True)
