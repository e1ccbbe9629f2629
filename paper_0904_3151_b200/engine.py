"""Device-side stages of the build: thin wrappers over the C ABI.

Each function takes/returns torch CUDA tensors (PyTorch is used only for
device memory and streams) and calls one ``eg_*`` entry point on the current
stream.  Workspaces come from the torch caching allocator.
"""

from __future__ import annotations

import itertools
import math
import threading
from math import comb

import numpy as np
import torch

from . import _native
from ._native import check
from .errors import DataError

_capacity_hint: dict = {}


def require_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_0904_3151_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _ws(nbytes: int, dev) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)


def _p(t) -> int:
    return t.data_ptr() if t is not None else 0


def as_device_rows(data, dev):
    """(n, D) float rows on ``dev``: float32 stays float32, everything else
    becomes float64 (the reference casts to float64, lsh.py:160)."""
    if isinstance(data, torch.Tensor):
        t = data
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        t = t.to(dev, non_blocking=True).contiguous()
    else:
        arr = np.asarray(data)
        if arr.dtype != np.float32:
            arr = np.asarray(arr, dtype=np.float64)
        arr = np.ascontiguousarray(arr)
        t = torch.from_numpy(arr).to(dev, non_blocking=True)
    if t.dim() != 2:
        raise DataError("vectors must form a 2-D array")
    return t


def row_stats_async(x: torch.Tensor):
    """fp64 row norms + device flags (first non-finite row, first zero-norm
    row; 2^64-1 when none), without synchronising."""
    n, dim = x.shape
    norms = torch.empty(n, dtype=torch.float64, device=x.device)
    bad = torch.empty(2, dtype=torch.int64, device=x.device)
    check(_native.lib().eg_row_stats(_p(x), int(x.dtype == torch.float64), n, dim, _p(norms),
                                     _p(bad), _stream(x.device)), "row_stats")
    return norms, bad


def raise_bad_rows(bad):
    """Reference error shapes: lsh.py:55-56, then lsh.py:121-125."""
    nonfinite, zero = (int(v) for v in bad.cpu().tolist())
    if nonfinite != -1:
        raise DataError(f"row {nonfinite} has a non-finite entry")
    if zero != -1:
        raise DataError(f"row {zero} has zero norm and cannot be projected")


def row_stats(x: torch.Tensor):
    norms, bad = row_stats_async(x)
    nonfinite, zero = (int(v) for v in bad.cpu().tolist())
    return norms, nonfinite, zero


def validate_rows(x: torch.Tensor):
    norms, bad = row_stats_async(x)
    raise_bad_rows(bad)
    return norms


def directions(length: int, dim: int, seed: int, replicate_id: int) -> np.ndarray:
    """Gaussian directions of one replicate, drawn on the host with the same
    numpy call as the reference (lsh.py:116-118, 142-146).  Column-blocked
    draws from one generator are a seamless stream, so one ``(length, dim)``
    draw equals the reference's blocked draws."""
    ss = np.random.SeedSequence([int(seed), int(replicate_id)])
    return np.random.Generator(np.random.PCG64(ss)).standard_normal((length, dim))


_dir_cache: dict = {}


def device_directions(length: int, dim: int, seed: int, replicate_ids, dev):
    """Directions of the replicates and their norms, resident on ``dev``
    (drawn once per (length, dim, seed, replicates, device) and kept: the
    draw is deterministic, so repeated builds reuse the device copy)."""
    key = (length, dim, int(seed), tuple(int(h) for h in replicate_ids), str(dev))
    hit = _dir_cache.get(key)
    if hit is None:
        r = np.concatenate([directions(length, dim, seed, h) for h in replicate_ids], axis=0)
        rnorm = np.sqrt(np.einsum("ij,ij->i", r, r))
        hit = (torch.from_numpy(np.ascontiguousarray(r)).to(dev),
               torch.from_numpy(rnorm).to(dev))
        if len(_dir_cache) >= 8:
            _dir_cache.pop(next(iter(_dir_cache)))
        _dir_cache[key] = hit
    return hit


def project_rows(x: torch.Tensor, length: int, seed: int, replicate_ids):
    """Row norms + bad-row flags + packed codes in one pass over the rows
    (``eg_project_rows``); returns (codes, norms, bad, fixups), no sync."""
    dev = x.device
    n, dim = x.shape
    reps = len(replicate_ids)
    W = max(1, -(-length // 64))
    r_d, rn_d = device_directions(length, dim, seed, replicate_ids, dev)
    codes = torch.empty((reps, n, W), dtype=torch.int64, device=dev)
    norms = torch.empty(n, dtype=torch.float64, device=dev)
    bad = torch.empty(2, dtype=torch.int64, device=dev)
    lib = _native.lib()
    ws = _ws(lib.eg_project_workspace(n, dim, length, reps), dev)
    fix = torch.zeros(1, dtype=torch.int64, device=dev)
    check(lib.eg_project_rows(_p(x), int(x.dtype == torch.float64), n, dim, _p(norms), _p(bad),
                              _p(r_d), _p(rn_d), length, reps, _p(codes), _p(ws), ws.numel(),
                              _p(fix), _stream(dev)), "project_rows")
    return codes, norms, bad, fix


def project_codes(x: torch.Tensor, norms: torch.Tensor, length: int, seed: int,
                  replicate_ids) -> tuple[torch.Tensor, torch.Tensor]:
    """Packed codes ``(r, n, W)`` uint64 for the given replicate ids, plus a
    device counter of band entries recomputed exactly (no host sync)."""
    dev = x.device
    n, dim = x.shape
    reps = len(replicate_ids)
    W = max(1, -(-length // 64))
    r_d, rn_d = device_directions(length, dim, seed, replicate_ids, dev)
    codes = torch.empty((reps, n, W), dtype=torch.int64, device=dev)
    lib = _native.lib()
    ws = _ws(lib.eg_project_workspace(n, dim, length, reps), dev)
    fix = torch.zeros(1, dtype=torch.int64, device=dev)
    check(lib.eg_project(_p(x), int(x.dtype == torch.float64), n, dim, _p(norms), _p(r_d),
                         _p(rn_d), length, reps, _p(codes), _p(ws), ws.numel(),
                         _p(fix), _stream(dev)), "project")
    return codes, fix


def masks_for(k: int, d: int):
    """Lexicographic d-subsets of range(k) (hamming_join.py:333)."""
    return list(itertools.combinations(range(k), d))


DESIGN_BASE = 10000   # plan codes >= this name a covering design: BASE + 100 v + m


def plan_design(plan: int, d: int):
    """(block count, ordered masked-block bitmasks of one replicate's units,
    is_design) of a plan code: a block count k' (the complete family of
    d-subsets, reference order) or DESIGN_BASE + 100 v + m (the library's
    covering design C(v, m, d), eg_msm_design).  A pure function of its
    arguments, memoised: it runs between the plan and the first unit kernel,
    where host time is device idle time."""
    hit = _plan_cache.get((plan, d))
    if hit is None:
        v, masks, is_design = _plan_design(int(plan), int(d))
        masks.setflags(write=False)
        hit = _plan_cache[(plan, d)] = (v, masks, is_design)
    return hit


_plan_cache: dict = {}


def _plan_design(plan: int, d: int):
    if plan < DESIGN_BASE:
        bits = []
        for m in masks_for(plan, d):
            b = 0
            for blk in m:
                b |= 1 << blk
            bits.append(b)
        return plan, np.asarray(bits, dtype=np.uint64), False
    v, m = divmod(plan - DESIGN_BASE, 100)
    lib = _native.lib()
    count = lib.eg_msm_design(v, m, d, None, 0)
    if count <= 0:
        raise ValueError(f"no covering design C({v}, {m}, {d}) in the library's table")
    out = np.zeros(count, dtype=np.uint64)
    lib.eg_msm_design(v, m, d, out.ctypes.data, count)
    return v, out, True


def unit_count(plan: int, d: int) -> int:
    """Units per replicate of a plan code."""
    if plan < DESIGN_BASE:
        return comb(plan, max(0, d))
    return len(plan_design(plan, d)[1])


def units_for(replicates, k: int, d: int):
    """(replicate index, block bitmask) for every unit, in reference order
    (``k``: a block count or a design's plan code)."""
    key = (tuple(int(h) for h in replicates), int(k), int(d))
    hit = _units_cache.get(key)
    if hit is None:
        _, family, _ = plan_design(k, d)
        reps = np.repeat(np.asarray(key[0], dtype=np.int32), len(family))
        bits = np.tile(family, len(reps) // max(1, len(family)))
        reps.setflags(write=False)
        bits.setflags(write=False)
        if len(_units_cache) >= 64:
            _units_cache.clear()
        hit = _units_cache[key] = (reps, bits)
    return hit


_units_cache: dict = {}
_xrep_scratch: dict = {}


def msm_plan(codes: torch.Tensor, length: int, k: int, d: int,
             oversized_fraction: float = 0.25) -> int:
    """Block count the MSM units run with (``eg_msm_plan``).

    The emitted pair set does not depend on it (hamming_join.py:300-375), so
    the library picks the count with the lowest modelled cost on a sample
    of replicate 0's codes; it returns ``k`` itself whenever the reference's
    oversized-group warning could fire on the reference blocks, so
    ``max_group`` keeps the reference's meaning where it matters."""
    reps, n, W = codes.shape
    if n == 0:
        return k
    lib = _native.lib()
    ws = _ws(lib.eg_msm_plan_workspace(length, k, d), codes.device)
    out = ctypes.c_int32(k)
    cost = (ctypes.c_double * 2)()
    check(lib.eg_msm_plan(_p(codes), n, length, k, d, float(oversized_fraction),
                          ctypes.addressof(out), ctypes.addressof(cost), _p(ws), ws.numel(),
                          _stream(codes.device)), "msm_plan")
    _last_plan.update(k=k, chosen=int(out.value), cost_ms=float(cost[0]), ref_ms=float(cost[1]))
    return int(out.value)


_last_plan: dict = {}


def msm_pairs(codes: torch.Tensor, length: int, block_bounds, d: int, unit_reps, unit_masks,
              capacity: int | None = None, full_codes: torch.Tensor | None = None,
              design=None):
    """Run the MSM units; returns (keys tensor, counts dict).

    ``design`` (covering-design units): the ordered family of masked block
    sets the unit masks are members of (eg_msm_pairs_design).

    ``full_codes`` (strings longer than the kernels' EG_MAX_LENGTH bits):
    ``codes`` is then a prefix view of them; the units emit the pairs within
    Hamming d on the prefix (a superset), which are filtered by the full
    codes' Hamming distance before the cross-replicate rule (also on the
    full codes)."""
    dev = codes.device
    reps, n, W = codes.shape
    k = len(block_bounds) - 1
    if length > _native.MAX_LENGTH or k > _native.MAX_BLOCKS:
        raise ValueError(f"eg_msm_pairs runs on <= {_native.MAX_LENGTH} bits and <= "
                         f"{_native.MAX_BLOCKS} blocks (msm_candidates maps larger ones)")
    lib = _native.lib()
    bb = np.ascontiguousarray(block_bounds, dtype=np.int32)
    ur = np.ascontiguousarray(unit_reps, dtype=np.int32)
    um = np.ascontiguousarray(unit_masks, dtype=np.uint64)
    dm = None if design is None else np.ascontiguousarray(design, dtype=np.uint64)
    hint_key = (n, length, k, d, reps, len(ur), full_codes is not None)
    if capacity is None:
        capacity = _capacity_hint.get(hint_key)
        if capacity is None:
            # cold call: a sampled upper bound of the output (eg_msm_estimate_
            # pairs) sizes the buffer, so the rerun below stays exceptional
            capacity = max(1 << 16, 2 * n)
            if n >= 1 << 16:
                capacity = max(capacity, int(estimate_pairs(codes, d)[1]))
    ws = _ws(lib.eg_msm_workspace(n, length, reps), dev)
    counts = (ctypes_i64 * (2 * reps + 2))()
    # cross-replicate rule in a separate streaming pass (and always when the
    # prefix pairs still need the full-code filter)
    defer = reps > 1 or full_codes is not None
    reruns = 0
    # buffers of the cross-replicate pass, made before the units run: the
    # device idles between eg_msm_pairs' final synchronisation and the next
    # launch for as long as the host takes to get there
    xkeep = xnewc = xnewc_host = None
    if reps > 1 and full_codes is None:
        # per-(device, thread) scratch kept between calls (stream-ordered reuse)
        skey = (str(dev), threading.get_ident())
        hit = _xrep_scratch.get(skey)
        if hit is None or hit[0].numel() < max(capacity, 1) or hit[1].numel() != reps:
            hit = (torch.empty(max(capacity, 1), dtype=torch.uint8, device=dev),
                   torch.empty(reps, dtype=torch.int64, device=dev),
                   torch.empty(reps, dtype=torch.int64, pin_memory=True))
            if len(_xrep_scratch) >= 16:
                _xrep_scratch.clear()
            _xrep_scratch[skey] = hit
        xkeep, xnewc, xnewc_host = hit
    while True:
        out = torch.empty(max(capacity, 1), dtype=torch.int64, device=dev)
        rtag = torch.empty(max(capacity, 1), dtype=torch.int16, device=dev) if defer else None
        rc = lib.eg_msm_pairs_design(_p(codes), n, length, reps, bb.ctypes.data, k, d,
                                     ur.ctypes.data, um.ctypes.data, len(ur),
                                     None if dm is None else dm.ctypes.data,
                                     0 if dm is None else len(dm), _p(out), _p(rtag), capacity,
                                     ctypes_addr(counts), _p(ws), ws.numel(), _stream(dev))
        if rc == _native.EG_ERR_CAPACITY:
            # the exact total is known now: one more pass with that capacity
            capacity = int(counts[0])
            reruns += 1
            del out, rtag
            continue
        check(rc, "msm_pairs")
        break
    total = int(counts[0])
    _capacity_hint[hint_key] = max(1 << 16, int(total * 1.25) + 1024)
    raw = tuple(int(counts[2 + h]) for h in range(reps))
    keys = out[:total]
    xcodes = codes
    if full_codes is not None:
        # prefix pairs -> pairs within d on the full codes (per replicate)
        xcodes = full_codes
        tag = rtag[:total] if reps > 1 else None
        keep = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
        rawc = torch.empty(reps, dtype=torch.int64, device=dev)
        check(lib.eg_hamming_filter_async(_p(keys), _p(tag), total, _p(full_codes), n,
                                          full_codes.shape[2], d, reps, _p(keep), _p(rawc),
                                          _stream(dev)), "hamming_filter")
        sel = keep[:total].bool()
        keys = keys[sel]
        if reps > 1:
            rtag = rtag[:total][sel]
        total = int(keys.numel())
        raw = tuple(int(v) for v in rawc.tolist())
    if reps > 1:
        if xkeep is not None and xkeep.numel() >= max(total, 1):
            keep, newc, newc_host = xkeep, xnewc, xnewc_host
        else:
            keep = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
            newc = torch.empty(reps, dtype=torch.int64, device=dev)
            newc_host = torch.empty(reps, dtype=torch.int64, pin_memory=True)
        # Few droppable pairs and a small set: drop them IN PLACE (key ~0)
        # and sort the whole array at once -- the dropped keys end up behind
        # the sum(new) survivors, so no compaction pass and no host round
        # trip between the units, the filter and the sort.
        in_place = (full_codes is None and 1 < total <= (1 << 24)
                    and 5 * sum(raw[1:]) <= 2 * total)
        check(lib.eg_xrep_filter_async(_p(keys), _p(rtag), total, _p(xcodes), n,
                                       xcodes.shape[2], d, reps,
                                       None if in_place else _p(keep), _p(newc),
                                       _stream(dev)), "xrep_filter")
        # the counts reach pinned host memory behind the filter; the
        # synchronisation below (or the compaction's) makes them readable
        newc_host.copy_(newc, non_blocking=True)
        if in_place:
            sort_pair_keys(keys, n)
            torch.cuda.current_stream(dev).synchronize()
            new = tuple(int(v) for v in newc_host.tolist())
            keys = keys[:sum(new)]
            keys._eg_sorted = True      # sort_pair_keys(keys, n) is a no-op on this tensor
        else:
            keys = compact_keys(keys, keep[:total])
            new = tuple(int(v) for v in newc_host.tolist())
    elif full_codes is not None:
        new = raw
    else:
        new = tuple(int(counts[2 + reps + h]) for h in range(reps))
    info = {
        "emitted": int(keys.numel()),
        "max_group": int(counts[1]),
        "raw": raw,
        "new": new,
        "capacity": capacity,
        "reruns": reruns,
    }
    return keys, info


def msm_view(codes: torch.Tensor, length: int, k: int, d: int):
    """(codes view, its length, block count to plan from, full codes or None)
    the kernels run on.  The answer {(i, j): Hamming <= d} does not depend
    on the blocks (hamming_join.py:300-375), so k > EG_MAX_BLOCKS runs with
    at most EG_MAX_BLOCKS blocks, and strings longer than EG_MAX_LENGTH bits
    are enumerated on their first EG_MAX_LENGTH bits (pairs within d there
    are a superset of the answer) and filtered by the full codes."""
    if d >= _native.MAX_BLOCKS:
        raise NotImplementedError(
            f"mismatch d={d}: the enumeration needs a partition into more than d <= "
            f"{_native.MAX_BLOCKS - 1} blocks")
    reps, n, W = codes.shape
    if length <= _native.MAX_LENGTH and k <= _native.MAX_BLOCKS:
        return codes, length, k, None
    lv = min(length, _native.MAX_LENGTH)
    wv = -(-lv // 64)
    view = codes[:, :, :wv].contiguous() if W > wv else codes
    kv = max(d + 1, min(k, _native.MAX_BLOCKS, lv))
    return view, lv, kv, (codes if lv < length else None)


def plan_blocks(codes: torch.Tensor, length: int, k: int, d: int,
                oversized_fraction: float = 0.25) -> int:
    """Block count of the units (eg_msm_plan on the kernels' view)."""
    view, lv, kv, _ = msm_view(codes, length, k, d)
    return msm_plan(view, lv, kv, d, oversized_fraction)


def msm_candidates(codes: torch.Tensor, length: int, k: int, d: int, *, blocks: int | None = None,
                   select=None, oversized_fraction: float = 0.25, block_bounds=None):
    """All (replicate, mask) units of the planned block count (or
    ``blocks``), optionally restricted by ``select(total_units) -> indices``
    (sharding): (candidate keys, info).  info["reference_blocks"] says
    whether the units ran on the reference's own blocks (``block_bounds``
    when given, else the standard partition) -- only then is
    info["max_group"] the reference's largest group."""
    from .bitpool import block_partition
    view, lv, kv, full = msm_view(codes, length, k, d)
    plan = blocks or msm_plan(view, lv, kv, d, oversized_fraction)
    kk, family, is_design = plan_design(plan, d)
    same = kk == k and not is_design and full is None and lv == length
    bounds = block_bounds if (same and block_bounds is not None) else block_partition(lv, kk)
    ureps, umasks = units_for(range(codes.shape[0]), plan, d)
    if select is not None:
        sel = np.asarray(select(len(ureps)), dtype=np.int64)
        ureps, umasks = ureps[sel], umasks[sel]
    keys, info = msm_pairs(view, lv, bounds, d, ureps, umasks, full_codes=full,
                           design=family if is_design else None)
    info["blocks"] = kk
    info["plan"] = plan
    info["units"] = int(len(ureps))
    info["reference_blocks"] = same
    return keys, info


def estimate_pairs(codes: torch.Tensor, d: int):
    """(point estimate, ~4-sigma upper bound) of the raw pairs the MSM units
    emit over all replicates of ``codes`` (eg_msm_estimate_pairs)."""
    reps, n, W = codes.shape
    est = (ctypes.c_double * 2)()
    ws = _ws(4096, codes.device)
    check(_native.lib().eg_msm_estimate_pairs(_p(codes), n, W, reps, d, ctypes.addressof(est),
                                              _p(ws), ws.numel(), _stream(codes.device)),
          "msm_estimate_pairs")
    return float(est[0]), float(est[1])


def sort_pair_keys(keys: torch.Tensor, n: int) -> torch.Tensor:
    m = keys.numel()
    if getattr(keys, "_eg_sorted", False):     # msm_pairs' in-place path sorted it already
        return keys
    if m > 1:
        lib = _native.lib()
        ws = _ws(lib.eg_sort_workspace(m, 0), keys.device)
        check(lib.eg_sort_pair_keys(_p(keys), m, n, _p(ws), ws.numel(), _stream(keys.device)),
              "sort_pair_keys")
    return keys


def sort_keys(keys: torch.Tensor, key_bits: int = 64, vals: torch.Tensor | None = None):
    m = keys.numel()
    if m > 1:
        lib = _native.lib()
        ws = _ws(lib.eg_sort_workspace(m, int(vals is not None)), keys.device)
        check(lib.eg_sort_keys(_p(keys), _p(vals), m, key_bits, _p(ws), ws.numel(),
                               _stream(keys.device)), "sort_keys")
    return keys, vals


def verify(x: torch.Tensor, norms: torch.Tensor, keys: torch.Tensor, metric: int, eps: float):
    """Exact filter of sorted candidate keys -> (edge keys, distances)."""
    dev = x.device
    n, dim = x.shape
    m = keys.numel()
    out_k = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    out_d = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
    if m == 0:
        return out_k[:0], out_d[:0]
    lib = _native.lib()
    ws = _ws(lib.eg_verify_workspace(m), dev)
    cnt = ctypes_i64(0)
    rc = lib.eg_verify(_p(x), int(x.dtype == torch.float64), n, dim, _p(norms), _p(keys), m,
                       metric, float(eps), _p(out_k), _p(out_d), ctypes_addr(cnt), _p(ws),
                       ws.numel(), _stream(dev))
    if rc == _native.EG_ERR_ARG:
        raise IndexError("candidate index out of range")
    check(rc, "verify")
    c = int(cnt.value)
    return out_k[:c], out_d[:c]


def first_witness(keys: torch.Tensor, pools, W: int, d: int) -> torch.Tensor:
    """keep[p] = Hamming > d in every pool of ``pools`` (device word arrays)."""
    dev = keys.device
    m = keys.numel()
    keep = torch.ones(max(m, 1), dtype=torch.uint8, device=dev)
    if m == 0 or not pools:
        return keep[:m]
    ptrs = torch.tensor([p.data_ptr() for p in pools], dtype=torch.int64, device=dev)
    check(_native.lib().eg_first_witness(_p(keys), m, _p(ptrs), len(pools), W, d, _p(keep),
                                         _stream(dev)), "first_witness")
    return keep[:m]


def compact_keys(keys: torch.Tensor, flags: torch.Tensor) -> torch.Tensor:
    m = keys.numel()
    out = torch.empty(max(m, 1), dtype=torch.int64, device=keys.device)
    if m == 0:
        return out[:0]
    lib = _native.lib()
    ws = _ws(lib.eg_compact_workspace(m), keys.device)
    cnt = ctypes_i64(0)
    check(lib.eg_compact_keys(_p(keys), _p(flags), m, _p(out), ctypes_addr(cnt), _p(ws),
                              ws.numel(), _stream(keys.device)), "compact")
    return out[:int(cnt.value)]


def grouped_sort(codes_1: torch.Tensor, length: int, block_bounds, mask_bits: int,
                 chunk_bits: int = 16):
    """(perm int32 tensor, bounds int64 tensor): the reference's
    grouped_radix_sort permutation (first-seen buckets, chunk_bits-wide
    passes) and its equal-key run offsets."""
    dev = codes_1.device
    n, W = codes_1.shape
    k = len(block_bounds) - 1
    lib = _native.lib()
    bb = np.ascontiguousarray(block_bounds, dtype=np.int32)
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    bounds = torch.empty(n + 1, dtype=torch.int64, device=dev)
    ws = _ws(lib.eg_grouped_sort_workspace(n, chunk_bits), dev)
    g = ctypes_i64(0)
    check(lib.eg_grouped_sort(_p(codes_1), n, length, bb.ctypes.data, k, mask_bits, chunk_bits,
                              _p(perm), _p(bounds), ctypes_addr(g), _p(ws), ws.numel(),
                              _stream(dev)), "grouped_sort")
    return perm, bounds[:int(g.value) + 1]


def edges_to_host(keys: torch.Tensor, dist: torch.Tensor | None):
    """Device edge keys (+ distances) -> host int64 (m, 2) pairs and float64
    distances, the boundary layout (edges.py:12-55).  The (i, j) split runs
    on the device and both arrays land in pinned host memory (torch's
    caching host allocator: repeated builds reuse the pinned blocks), in
    2^27-edge chunks."""
    m = int(keys.numel())
    if m == 0:
        return np.empty((0, 2), np.int64), np.empty(0, np.float64)
    ph = torch.empty((m, 2), dtype=torch.int64, pin_memory=True)
    dh = torch.empty(m, dtype=torch.float64, pin_memory=True) if dist is not None else None
    step = 1 << 27
    for lo in range(0, m, step):
        k = keys[lo:lo + step]
        ph[lo:lo + k.numel()].copy_(torch.stack((k >> 32, k & 0xFFFFFFFF), dim=1),
                                    non_blocking=True)
    if dh is not None:
        dh.copy_(dist, non_blocking=True)
    torch.cuda.current_stream(keys.device).synchronize()
    return ph.numpy(), (dh.numpy() if dh is not None else None)


def keys_to_pairs(keys_host: np.ndarray) -> np.ndarray:
    """uint64 (i << 32 | j) keys -> int64 (m, 2) pairs (boundary format)."""
    k = keys_host.view(np.uint64)
    out = np.empty((k.shape[0], 2), dtype=np.int64)
    out[:, 0] = (k >> np.uint64(32)).astype(np.int64)
    out[:, 1] = (k & np.uint64(0xFFFFFFFF)).astype(np.int64)
    return out


def pairs_to_keys(pairs: np.ndarray) -> np.ndarray:
    p = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    return ((p[:, 0].astype(np.uint64) << np.uint64(32)) | p[:, 1].astype(np.uint64)).view(np.int64)


import ctypes  # noqa: E402

ctypes_i64 = ctypes.c_int64


def ctypes_addr(obj) -> int:
    return ctypes.addressof(obj)


def log2_ceil(v: int) -> int:
    return max(0, math.ceil(math.log2(max(v, 1))))
