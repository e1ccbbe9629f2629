"""Multi-GPU build: one process per GPU, torch.distributed (NCCL) plumbing.

Sharding: every output pair has exactly one owning
(replicate, mask) unit -- the canonical-mask rule inside a replicate and the
first-witness rule across replicates -- so units can be split across ranks
with disjoint outputs and no cross-rank dedup.

    1. rows are split into equal shards; each rank projects its shard and
       computes its row norms and bad-row flags in the same pass
       (eg_project_rows); the flags are MIN-reduced over the ranks;
    2. codes and norms are all-gathered over NVLink (NCCL all_gather);
    3. rank 0 plans the block count on the gathered codes (eg_msm_plan) and
       broadcasts it (8 bytes), units are
       assigned cyclically (unit u -> rank u % world), each rank
       runs eg_msm_pairs on its units, sorts and verifies its candidates
       (rows are resident on every rank for the verify gathers);
    4. per-rank sorted edge runs are gathered to rank 0 only and merged
       there (merge path, log2(ranks) rounds; eg_merge_runs).

The collective/merge logic is written against a small ``ops`` interface so
the same code runs with the CUDA ops (``DeviceOps``) and, in tests, with the
CPU oracle over gloo.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as tdist

from . import engine


def my_units(total: int, world: int, rank: int):
    """Cyclic unit assignment: balanced to within one unit per rank."""
    return list(range(rank, total, world))


def row_shard(n: int, world: int, rank: int):
    per = -(-n // world)
    lo = min(n, rank * per)
    return lo, min(n, lo + per), per


class DeviceOps:
    """CUDA implementations of the per-rank stages."""

    def norms(self, x):
        return engine.validate_rows(x)

    def project(self, x, norms, params):
        codes, _ = engine.project_codes(x, norms, params.length, params.seed,
                                        list(range(1, params.replicates + 1)))
        return codes

    def project_rows(self, x, params):
        """Norms, bad-row flags and codes of a row shard in one pass over
        the rows (eg_project_rows); no host sync."""
        codes, norms, bad, _ = engine.project_rows(x, params.length, params.seed,
                                                   list(range(1, params.replicates + 1)))
        return codes, norms, bad

    def raise_bad(self, bad):
        engine.raise_bad_rows(bad)

    def plan(self, codes, params):
        """Block count of the units (deterministic in the codes, so every
        rank holding the gathered codes picks the same one)."""
        return engine.plan_blocks(codes, params.length, params.blocks, params.mismatch)

    def unit_count(self, blocks, mismatch):
        """Units per replicate of a plan code (block count or design)."""
        return engine.unit_count(blocks, mismatch)

    def candidates(self, codes, params, units, blocks):
        return engine.msm_candidates(codes, params.length, params.blocks, params.mismatch,
                                     blocks=blocks, select=lambda total: units)

    def sort(self, keys, n):
        return engine.sort_pair_keys(keys, n)

    def verify(self, x, norms, keys, metric, eps):
        from .pipeline import _metric_id
        return engine.verify(x, norms, keys, _metric_id(metric), eps)

    def merge_runs(self, keys, dists, offsets):
        """Concatenated sorted per-rank runs (run r = keys[offsets[r]:
        offsets[r+1]]) -> one sorted run, distances carried (eg_merge_runs:
        log2(runs) merge-path rounds instead of a re-sort)."""
        m = keys.numel()
        if m <= 1 or len(offsets) <= 2:
            return keys, dists
        from . import _native
        lib = _native.lib()
        keys = keys.contiguous()
        vals = dists.contiguous().view(torch.int64)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        ws = engine._ws(lib.eg_merge_runs_workspace(m, 1), keys.device)
        _native.check(lib.eg_merge_runs(keys.data_ptr(), vals.data_ptr(), off.ctypes.data,
                                        len(offsets) - 1, ws.data_ptr(), ws.numel(),
                                        engine._stream(keys.device)), "merge_runs")
        return keys, vals.view(torch.float64)


def _all_gather_rows(t: torch.Tensor, per: int, world: int) -> torch.Tensor:
    """All-gather equal-size row shards (dim 0 padded to ``per``)."""
    pad = per - t.shape[0]
    if pad:
        t = torch.cat([t, t.new_zeros((pad,) + tuple(t.shape[1:]))])
    out = t.new_empty((per * world,) + tuple(t.shape[1:]))
    tdist.all_gather_into_tensor(out, t.contiguous())
    return out


def gather_codes(codes_shard, norms_shard, n, world, rank):
    """(reps, n_r, W) shards -> (reps, n, W) full codes + full norms, in ONE
    all-gather: each rank packs its rows as [codes of every replicate |
    norm bits] (int64), so the collective latency is paid once."""
    lo, hi, per = row_shard(n, world, rank)
    reps, nr, W = codes_shard.shape
    packed = torch.cat([codes_shard.permute(1, 0, 2).reshape(nr, reps * W),
                        norms_shard.contiguous().view(torch.int64).reshape(nr, 1)], dim=1)
    full = _all_gather_rows(packed, per, world)[:n]
    codes = full[:, :reps * W].reshape(n, reps, W).permute(1, 0, 2).contiguous()
    norms = full[:, reps * W].contiguous().view(torch.float64)
    return codes, norms


def global_bad_rows(bad_local: torch.Tensor, row0: int) -> torch.Tensor:
    """(first non-finite row, first zero-norm row) of the whole pool from
    every rank's shard flags (-1 = none): MIN over ranks of the global row
    indices, so all ranks see the reference's first offending row."""
    big = torch.iinfo(torch.int64).max
    g = torch.where(bad_local >= 0, bad_local + row0, torch.full_like(bad_local, big))
    if tdist.is_available() and tdist.is_initialized() and tdist.get_world_size() > 1:
        tdist.all_reduce(g, op=tdist.ReduceOp.MIN)
    return torch.where(g == big, torch.full_like(g, -1), g)


def gather_edges(keys, dists, world, rank, ops, n):
    """Per-rank sorted edge runs -> merged sorted edges on rank 0 only: the
    run lengths are all-gathered (8 bytes per rank), the runs themselves go
    to rank 0 alone (one gather, keys and distance bits together), and rank
    0 merges the sorted runs (ops.merge_runs) instead of re-sorting."""
    cnt = torch.tensor([keys.numel()], dtype=torch.int64, device=keys.device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    tdist.all_gather(counts, cnt)
    counts = [int(c.item()) for c in counts]
    mx = max(counts) if counts else 0
    if mx == 0:
        return (keys[:0], dists[:0]) if rank == 0 else (None, None)
    kd = torch.stack([keys, dists.contiguous().view(torch.int64)], dim=1)
    kp = torch.cat([kd, kd.new_zeros((mx - keys.numel(), 2))])
    parts = [kp.new_empty((mx, 2)) for _ in range(world)] if rank == 0 else None
    tdist.gather(kp, gather_list=parts, dst=0)
    if rank != 0:
        return None, None
    ks = torch.cat([parts[r][:counts[r], 0] for r in range(world)]).contiguous()
    ds = torch.cat([parts[r][:counts[r], 1] for r in range(world)]).contiguous()
    offsets = [0]
    for c in counts:
        offsets.append(offsets[-1] + c)
    return ops.merge_runs(ks, ds.view(torch.float64), offsets)


def broadcast_int(value, rank: int, device) -> int:
    """Rank 0's integer to every rank (one 8-byte broadcast)."""
    t = torch.tensor([int(value) if rank == 0 else 0], dtype=torch.int64, device=device)
    if tdist.is_available() and tdist.is_initialized() and tdist.get_world_size() > 1:
        tdist.broadcast(t, src=0)
    return int(t.item())


def build_step(x, params, metric: str, world: int, rank: int, ops=None,
               force_dist: bool = False):
    """One full build of ``x`` (resident rows) on ``world`` ranks.

    Returns a dict with rank 0's merged ``keys``/``dist`` (None on other
    ranks) and this rank's counters.  ``force_dist`` runs the sharded code
    path (collectives included) even for a single rank (tests)."""
    ops = ops or DeviceOps()
    n = x.shape[0]
    if world == 1 and not force_dist:
        from .pipeline import build_graph_device
        out = build_graph_device(x, params, metric=metric)
        return {"keys": out["keys"], "dist": out["dist"], "info": out["info"],
                "candidates": out["candidates"], "codes": out["codes"]}
    lo, hi, per = row_shard(n, world, rank)
    xs = x[lo:hi]
    if hasattr(ops, "project_rows"):
        # one pass over the shard (norms + flags fused into the projection);
        # the flags are agreed over the ranks so every rank raises the same
        # error instead of one rank leaving the collectives
        codes_s, norms_s, bad_s = ops.project_rows(xs, params)
        bad = global_bad_rows(bad_s, lo)
        codes, norms = gather_codes(codes_s, norms_s, n, world, rank)
        ops.raise_bad(bad)
    else:
        norms_s = ops.norms(xs)
        codes_s = ops.project(xs, norms_s, params)
        codes, norms = gather_codes(codes_s, norms_s, n, world, rank)
    # one plan (rank 0), one 8-byte broadcast: every rank runs the same units
    blocks = broadcast_int(ops.plan(codes, params) if rank == 0 else 0, rank, codes.device)
    units = my_units(params.replicates * ops.unit_count(blocks, params.mismatch), world, rank)
    keys, info = ops.candidates(codes, params, units, blocks)
    info = dict(info, plan=blocks)
    keys = ops.sort(keys, n)
    ek, ed = ops.verify(x, norms, keys, metric, params.epsilon)
    mk, md = gather_edges(ek, ed, world, rank, ops, n)
    return {"keys": mk, "dist": md, "info": info}


def hamming_step(codes, params, world: int, rank: int):
    """Config 2: enumerate_pairs over resident words, units sharded."""
    n = codes.shape[1]
    keys, info = engine.msm_candidates(codes, params.length, params.blocks, params.mismatch,
                                       select=lambda total: my_units(total, world, rank))
    engine.sort_pair_keys(keys, n)
    if world > 1:
        dummy = torch.zeros(keys.numel(), dtype=torch.float64, device=keys.device)
        keys, _ = gather_edges(keys, dummy, world, rank, DeviceOps(), n)
        if rank != 0:
            keys = None
    return {"keys": keys, "dist": None, "info": info}


def last_counts(res):
    if not res:
        return None
    info = res.get("info") or {}
    keys = res.get("keys")
    return {"candidates": info.get("emitted"), "raw": info.get("raw"), "new": info.get("new"),
            "edges": int(keys.numel()) if keys is not None else None,
            "max_group": info.get("max_group"), "blocks": info.get("blocks"),
            "plan": info.get("plan"), "units": info.get("units")}


# ------------------------------------------------ one process, many devices
def _device_list(devices):
    if isinstance(devices, int):
        if devices < 1:
            raise ValueError("devices must be >= 1")
        return [torch.device("cuda", i) for i in range(devices)]
    out = []
    for d in devices:
        dev = torch.device("cuda", d) if isinstance(d, int) else torch.device(d)
        if dev.type != "cuda" or dev.index is None:
            raise ValueError(f"devices must name CUDA devices with an index, got {d!r}")
        out.append(dev)
    if not out:
        raise ValueError("devices must not be empty")
    return out


def build_on_devices(rows, params, metric: str, devices):
    """The sharded build of ``build_step`` driven from ONE process over
    several devices (``build_graph(..., devices=)``): row
    shards projected on their devices, codes and norms gathered by peer
    copies, the block count planned once, (replicate, mask) units dealt
    cyclically over the shards, each shard's candidates sorted and verified
    on its device, and the sorted edge runs merged on the first device.

    ``devices`` is a count or a list of CUDA devices; a device may appear
    more than once (its shards then run one after another on it), which is
    how one GPU exercises the multi-device path.  Every pair has exactly one
    owning unit and a per-pair-deterministic distance, so the result is the
    same for any device list (the mirror of the reference's thread-count
    contract, tests/test_pipeline.py:130-135)."""
    from concurrent.futures import ThreadPoolExecutor

    from .pipeline import _metric_id
    devs = _device_list(devices)
    world = len(devs)
    distinct = list(dict.fromkeys(devs))
    n = rows.shape[0]
    reps_ids = list(range(1, params.replicates + 1))

    def on(dev, fn):
        with torch.cuda.device(dev):
            out = fn()
            torch.cuda.current_stream(dev).synchronize()
            return out

    def run(fn_by_shard):
        """fn_by_shard(s) for every shard, shards of one device in order,
        devices concurrently (ctypes and torch release the GIL)."""
        results = [None] * world

        def work(dev):
            for s in range(world):
                if devs[s] == dev:
                    results[s] = on(dev, lambda: fn_by_shard(s))
        with ThreadPoolExecutor(max_workers=len(distinct)) as ex:
            list(ex.map(work, distinct))
        return results

    # rows on every device (one H2D per device from host memory, else a peer copy)
    src = rows if isinstance(rows, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(rows))
    if src.device.type == "cpu" and not src.is_pinned() and len(distinct) > 1:
        src = src.pin_memory()
    xs = {}

    def put(dev):
        xs[dev] = on(dev, lambda: engine.as_device_rows(src, dev))
    with ThreadPoolExecutor(max_workers=len(distinct)) as ex:
        list(ex.map(put, distinct))

    # 1. projection of the row shards (norms and bad-row flags in the same pass)
    shards = [row_shard(n, world, s) for s in range(world)]
    proj = run(lambda s: engine.project_rows(xs[devs[s]][shards[s][0]:shards[s][1]],
                                             params.length, params.seed, reps_ids))
    # first offending row over all shards (reference order: non-finite, then zero norm)
    flags = []
    for s, (codes_s, norms_s, bad_s, _) in enumerate(proj):
        b = bad_s.cpu().tolist()
        flags.append([v + shards[s][0] if v >= 0 else -1 for v in b])
    from .errors import DataError
    nonfinite = [f[0] for f in flags if f[0] >= 0]
    zero = [f[1] for f in flags if f[1] >= 0]
    if nonfinite:
        raise DataError(f"row {min(nonfinite)} has a non-finite entry")
    if zero:
        raise DataError(f"row {min(zero)} has zero norm and cannot be projected")

    # 2. codes and norms of all rows on every device (peer copies)
    full = {}

    def gather(dev):
        def f():
            codes = torch.cat([p[0].to(dev, non_blocking=True) for p in proj], dim=1)
            norms = torch.cat([p[1].to(dev, non_blocking=True) for p in proj])
            return codes, norms
        full[dev] = on(dev, f)
    with ThreadPoolExecutor(max_workers=len(distinct)) as ex:
        list(ex.map(gather, distinct))

    # 3. one plan (deterministic in the codes) for every shard
    blocks = on(devs[0], lambda: engine.plan_blocks(full[devs[0]][0], params.length,
                                                    params.blocks, params.mismatch))
    ops = DeviceOps()
    total_units = params.replicates * engine.unit_count(blocks, params.mismatch)

    def shard_build(s):
        dev = devs[s]
        codes, norms = full[dev]
        units = my_units(total_units, world, s)
        if not units:
            empty = torch.empty(0, dtype=torch.int64, device=dev)
            return empty, empty.to(torch.float64), None
        keys, info = ops.candidates(codes, params, units, blocks)
        keys = ops.sort(keys, n)
        ek, ed = engine.verify(xs[dev], norms, keys, _metric_id(metric), params.epsilon)
        return ek, ed, info
    parts = run(shard_build)

    # 4. merge the sorted per-shard edge runs on the first device
    def merge():
        dev = devs[0]
        ks = torch.cat([p[0].to(dev) for p in parts])
        ds = torch.cat([p[1].to(dev) for p in parts])
        offsets = [0]
        for p in parts:
            offsets.append(offsets[-1] + p[0].numel())
        return ops.merge_runs(ks, ds, offsets)
    keys, dist = on(devs[0], merge)
    infos = [p[2] for p in parts if p[2] is not None]
    reps = params.replicates
    info = {
        "emitted": sum(i["emitted"] for i in infos),
        "max_group": max([i["max_group"] for i in infos] or [0]),
        "raw": tuple(sum(i["raw"][h] for i in infos) for h in range(reps)),
        "new": tuple(sum(i["new"][h] for i in infos) for h in range(reps)),
        "blocks": blocks,
        "reference_blocks": all(i.get("reference_blocks", False) for i in infos) and bool(infos),
        "devices": [str(d) for d in devs],
    }
    return {"keys": keys, "dist": dist, "info": info}
