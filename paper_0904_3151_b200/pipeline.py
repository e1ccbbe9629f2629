"""End-to-end eps-graph construction (mirrors pipeline.py).

``build_graph`` runs the whole reference pipeline (pipeline.py:242-354) on
one B200:

    row stats (validation + fp64 norms)        eg_row_stats
    projection of all replicates at once       eg_project
    every (replicate, mask) unit               eg_msm_pairs   (MSM sort,
        groups, pair enumeration, canonical-mask and first-witness rules:
        the output is already the deduplicated candidate set)
    candidate sort by (i, j)                   eg_sort_pair_keys
    exact verify + stable compaction           eg_verify

Host work is limited to drawing the Gaussian directions with numpy (the
reference's own call), scalar parameter math, and the boundary conversion
of the final uint64 pair keys to the reference's int64 ``(m, 2)`` layout.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native, engine
from .bitpool import BitStringPool
from .edges import EdgeList
from .errors import DataError
from .hamming_join import PairSet, enumerate_pairs, warn_oversized
from .lsh import VectorDataset, center_normalize, collision_prob
from .tuning import MsmParams, missing_edge_bound

__all__ = [
    "CandidateSet", "GraphStats", "NeighborGraph", "build_graph", "build_graph_device",
    "build_graph_hamming", "build_graph_lsh_only", "dedup_across_replicates", "filter_exact",
]


@dataclass
class CandidateSet:
    """Union of per-replicate pair sets with first-witness provenance
    (pipeline.py:47-63); ``pairs`` ordered by replicate, then (i, j)."""
    pairs: np.ndarray
    per_replicate_raw: tuple
    per_replicate_new: tuple

    def __len__(self) -> int:
        return self.pairs.shape[0]


@dataclass
class GraphStats:
    """Build counters (pipeline.py:66-84).  ``timings`` keeps the reference
    keys (project_s, enumerate_s, dedup_s, filter_s, total_s), measured with
    CUDA events; dedup is fused into enumeration on the GPU (dedup_s = 0)."""
    candidate_count: int
    edge_count: int
    false_candidate_count: int
    per_replicate_raw: tuple
    per_replicate_new: tuple
    achieved_bound: float
    timings: dict = field(default_factory=dict)


@dataclass
class NeighborGraph:
    node_count: int
    params: MsmParams
    edge_list: EdgeList
    stats: GraphStats

    @property
    def edges(self):
        return self.edge_list.as_tuples()

    @property
    def edge_count(self) -> int:
        return len(self.edge_list)


_METRICS = {"cosine": _native.METRIC_COSINE, "euclidean": _native.METRIC_EUCLIDEAN}


def _metric_id(metric: str) -> int:
    try:
        return _METRICS[metric]
    except KeyError:
        raise ValueError(f"metric must be 'cosine' or 'euclidean', got {metric!r}") from None


def lsh_radius(params: MsmParams, metric: str) -> float:
    """Cosine radius the LSH parameters are tuned for.  For 'euclidean' the
    params carry the Euclidean radius and unit rows are assumed, mapped by
    cosine_radius_from_euclidean (lsh.py:218-222)."""
    if metric == "euclidean":
        return params.epsilon * params.epsilon / 2.0
    return params.epsilon


def build_graph_device(x: torch.Tensor, params: MsmParams, *, metric: str = "cosine",
                       units=None, norms: torch.Tensor | None = None, codes=None,
                       blocks: int | None = None):
    """Build with rows already resident on the device.

    Returns a dict of device tensors (``keys`` sorted uint64 pair keys,
    ``dist`` float64) plus counters and per-stage CUDA-event timings.
    ``units`` (optional) restricts the (replicate, mask) units to these
    indices (sharding); ``codes`` lets a caller pass pre-gathered codes.
    ``blocks`` is the block count the units use (default: ``eg_msm_plan``'s
    choice; the pair set is the same for every count).
    """
    dev = x.device
    n = x.shape[0]
    mid = _metric_id(metric)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    bad = None
    fix = None
    reps = list(range(1, params.replicates + 1))
    flags_ready = None
    if norms is None and codes is None:
        # one pass over the rows: norms + flags fused into the projection
        codes, norms, bad, fix = engine.project_rows(x, params.length, params.seed, reps)
    else:
        if norms is None:
            norms, bad = engine.row_stats_async(x)
        if codes is None:
            codes, fix = engine.project_codes(x, norms, params.length, params.seed, reps)
    if bad is not None:
        # the flags travel to pinned host memory behind the projection; they
        # are checked before any unit runs (zero-norm / NaN rows share the
        # all-zero code and would form one giant group), after the plan's own
        # synchronisation when it makes one
        bad_host = torch.empty(bad.shape, dtype=bad.dtype, pin_memory=True)
        bad_host.copy_(bad, non_blocking=True)
        bad = bad_host
        flags_ready = torch.cuda.Event()
        flags_ready.record()
    ev[1].record()
    if blocks is None:
        blocks = engine.plan_blocks(codes, params.length, params.blocks, params.mismatch)
    if flags_ready is not None:
        flags_ready.synchronize()
        engine.raise_bad_rows(bad)
    keys, info = engine.msm_candidates(
        codes, params.length, params.blocks, params.mismatch, blocks=blocks,
        select=None if units is None else (lambda total: units))
    ev[2].record()
    engine.sort_pair_keys(keys, n)
    ev[3].record()
    ekeys, edist = engine.verify(x, norms, keys, mid, params.epsilon)
    ev[4].record()
    return {
        "keys": ekeys, "dist": edist, "candidates": keys, "codes": codes, "norms": norms,
        "info": info, "fixups": fix, "events": ev,
    }


def _bounds(length: int, k: int) -> np.ndarray:
    from .bitpool import block_partition
    return block_partition(length, k)


def _event_timings(ev, t_host):
    torch.cuda.synchronize()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(ev) - 1)]
    return {
        "project_s": ms[0] / 1e3,
        "enumerate_s": ms[1] / 1e3,
        "dedup_s": 0.0,
        "sort_s": ms[2] / 1e3,
        "filter_s": ms[3] / 1e3,
        "total_s": t_host,
    }


def build_graph(data, params: MsmParams, *, threads: int | None = None, chunk_bits: int = 16,
                normalize: bool = False, max_pool_bytes: int = 1 << 30,
                metric: str = "cosine", device=None, devices=None) -> NeighborGraph:
    """Construct the eps-neighbour graph (pipeline.py:242-354) on B200s.

    Arguments follow the reference; ``threads`` and ``max_pool_bytes`` are
    accepted for compatibility (all replicate pools stay resident in HBM and
    the result is identical for any value), ``chunk_bits`` is validated.
    New: ``metric`` ('cosine' | 'euclidean'), ``device`` (one GPU) and
    ``devices`` (a count or a list of CUDA devices: the units are sharded
    over them, distributed.build_on_devices; same result for any list).
    ``data`` may also be a torch tensor (CPU, pinned, or on a device).
    """
    t0 = time.perf_counter()
    if not (1 <= chunk_bits <= 24):
        raise ValueError("chunk_bits must be in [1, 24]")
    _metric_id(metric)
    if isinstance(data, VectorDataset):
        rows = data.vectors
    else:
        rows = data
    if normalize:
        rows = center_normalize(rows.cpu().numpy() if isinstance(rows, torch.Tensor) else rows).vectors
    if devices is not None:
        from .distributed import _device_list, build_on_devices
        devs = _device_list(devices)
        engine.require_device(devs[0])
        if len(rows) == 0:
            raise DataError("cannot build a graph over an empty dataset")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.device(devs[0]):
            ev[0].record()
        out = build_on_devices(rows, params, metric, devs)
        n = len(rows)
        info = out["info"]
        with torch.cuda.device(devs[0]):
            ev[1].record()
            ev[1].synchronize()
            pairs, dist = engine.edges_to_host(out["keys"], out["dist"])
        timings = {"project_s": 0.0, "enumerate_s": ev[0].elapsed_time(ev[1]) / 1e3,
                   "dedup_s": 0.0, "sort_s": 0.0, "filter_s": 0.0}
    else:
        dev = engine.require_device(device)
        with torch.cuda.device(dev):
            x = engine.as_device_rows(rows, dev)
            n = x.shape[0]
            if n == 0:
                raise DataError("cannot build a graph over an empty dataset")
            out = build_graph_device(x, params, metric=metric)
            info = out["info"]
            pairs, dist = engine.edges_to_host(out["keys"], out["dist"])
            timings = _event_timings(out["events"], 0.0)
    if info.get("reference_blocks", info["blocks"] == params.blocks):
        # else the plan ruled the warning out on the reference blocks
        warn_oversized(info["max_group"], n, 0.25)
    edges = EdgeList(pairs, dist)
    timings["total_s"] = time.perf_counter() - t0
    cand = info["emitted"]
    stats = GraphStats(
        candidate_count=cand,
        edge_count=len(edges),
        false_candidate_count=cand - len(edges),
        per_replicate_raw=info["raw"],
        per_replicate_new=info["new"],
        achieved_bound=missing_edge_bound(params.length, params.mismatch,
                                          collision_prob(lsh_radius(params, metric)),
                                          params.replicates),
        timings=timings)
    return NeighborGraph(node_count=n, params=params, edge_list=edges, stats=stats)


def filter_exact(data, candidates, epsilon: float, block_pairs: int = 1 << 20, *,
                 metric: str = "cosine", device=None) -> EdgeList:
    """Keep exactly the candidates within ``epsilon`` (pipeline.py:183-223).

    ``block_pairs`` is accepted for compatibility (the GPU verifies all
    candidates in one pass; results do not depend on it)."""
    if isinstance(candidates, CandidateSet):
        pairs = candidates.pairs
    elif isinstance(candidates, PairSet):
        pairs = candidates.array
    else:
        pairs = np.asarray(candidates, dtype=np.int64).reshape(-1, 2)
    if isinstance(data, torch.Tensor):
        rows = data
    else:
        # the reference validates through as_dataset (pipeline.py:197): list
        # input is accepted, a non-finite row raises DataError
        rows = data.vectors if isinstance(data, VectorDataset) else VectorDataset(data).vectors
    n = rows.shape[0]
    if pairs.size and (pairs.min() < 0 or pairs.max() >= n):
        raise IndexError("candidate index out of range")
    if pairs.shape[0] == 0:
        return EdgeList()
    dev = engine.require_device(device)
    with torch.cuda.device(dev):
        x = engine.as_device_rows(rows, dev)
        norms, nonfinite, _ = engine.row_stats(x)
        if nonfinite != -1:
            raise DataError(f"row {nonfinite} has a non-finite entry")
        keys = torch.from_numpy(engine.pairs_to_keys(pairs)).to(dev)
        engine.sort_pair_keys(keys, n)
        ek, ed = engine.verify(x, norms, keys, _metric_id(metric), epsilon)
        return EdgeList(engine.keys_to_pairs(ek.cpu().numpy()), ed.cpu().numpy())


def dedup_across_replicates(pools, raw, d: int, *, device=None) -> CandidateSet:
    """First-witness merge of per-replicate pair sets (pipeline.py:109-146):
    a pair of replicate h survives iff its Hamming distance exceeds d in
    every earlier pool; computed by ``eg_first_witness`` on the device."""
    if len(pools) != len(raw):
        raise ValueError("one raw pair set per pool is required")
    if len({(p.count, p.length) for p in pools}) > 1:
        raise ValueError("pools must share count and length")
    dev = engine.require_device(device)
    with torch.cuda.device(dev):
        dpools = [torch.from_numpy(np.ascontiguousarray(p.words).view(np.int64)).to(dev)
                  for p in pools]
        pieces, raw_counts, new_counts = [], [], []
        W = pools[0].word_count if pools else 1
        for h, pairs in enumerate(raw):
            arr = pairs.array if isinstance(pairs, PairSet) else np.asarray(pairs, np.int64)
            arr = arr.reshape(-1, 2)
            raw_counts.append(arr.shape[0])
            if arr.shape[0] and h > 0:
                keys = torch.from_numpy(engine.pairs_to_keys(arr)).to(dev)
                keep = engine.first_witness(keys, dpools[:h], W, d)
                kept = engine.compact_keys(keys, keep)
                arr = engine.keys_to_pairs(kept.cpu().numpy())
            new_counts.append(arr.shape[0])
            if arr.shape[0]:
                pieces.append(arr)
    pairs = np.vstack(pieces) if pieces else np.empty((0, 2), dtype=np.int64)
    return CandidateSet(pairs=pairs, per_replicate_raw=tuple(raw_counts),
                        per_replicate_new=tuple(new_counts))


def _max_feasible_length(p: float, gamma: float, replicates: int, fallback: int) -> int:
    """Largest length whose d=0 bound stays within gamma (pipeline.py:357-380)."""
    from .errors import InfeasibleError
    if p == 0.0:
        return fallback
    target = -math.expm1(math.log(gamma) / replicates)
    if target <= 0.0:
        return fallback
    length = max(1, math.floor(math.log(target) / math.log1p(-p)))
    while length > 1 and missing_edge_bound(length, 0, p, replicates) > gamma:
        length -= 1
    while missing_edge_bound(length + 1, 0, p, replicates) <= gamma:
        length += 1
    if missing_edge_bound(length, 0, p, replicates) > gamma:
        raise InfeasibleError(
            f"even a single bit misses too much: bound at length=1 is "
            f"{missing_edge_bound(1, 0, p, replicates):.3e} > gamma={gamma}")
    return length


def build_graph_lsh_only(data, epsilon: float, gamma: float, *, replicates: int = 300,
                         seed: int = 0, threads: int | None = None, chunk_bits: int = 16,
                         normalize: bool = False, device=None) -> NeighborGraph:
    """d = 0, k = 1 baseline (pipeline.py:383-408): one empty mask per
    replicate, i.e. a full-key grouping sort per unit."""
    rows = data.vectors if isinstance(data, VectorDataset) else data
    if len(rows) == 0:
        raise DataError("cannot build a graph over an empty dataset")
    p = collision_prob(epsilon)
    fallback = 2 * math.ceil(math.log2(max(len(rows), 2)))
    length = _max_feasible_length(p, gamma, replicates, fallback)
    params = MsmParams(epsilon=epsilon, gamma=gamma, length=length, mismatch=0, blocks=1,
                       replicates=replicates, seed=seed)
    return build_graph(data, params, threads=threads, chunk_bits=chunk_bits,
                       normalize=normalize, device=device)


def build_graph_hamming(pool: BitStringPool, d: int, chunk_bits: int = 16, *,
                        device=None) -> PairSet:
    """Exact d-neighbour pairs of a pool (pipeline.py:411-430)."""
    if d < 0:
        raise ValueError("d must be non-negative")
    n = pool.count
    if d >= pool.length:
        ii, jj = np.triu_indices(n, k=1)
        return PairSet(np.column_stack([ii, jj]).astype(np.int64), assume_normalized=True)
    working = pool if d < pool.block_count else pool.partitioned(max(1, min(2 * d, pool.length)))
    return enumerate_pairs(working, d, chunk_bits=chunk_bits, device=device)
