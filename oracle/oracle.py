"""CPU oracle for the eps-graph build path -- TEST INFRASTRUCTURE ONLY.

This module restates the reference algorithm (``epsgraph`` 0.1.0,
``/root/reference/pkg/src/epsgraph``) on the CPU: a plain-C core
(``oracle/epsgraph_oracle.c``, loaded through ctypes) plus numpy glue.  It is
the checker that the CUDA product path is compared against.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (the ``cpu_baseline`` leg and
``--impl reference``) may import it; the product package never does.

Parity of the oracle itself is pinned by the fixtures in ``tests/golden/``,
which were produced by running the reference package in the build container
(``tests/golden/make_golden.py``) and are checked by
``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import itertools
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libepsgraph_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C restatement (gcc, -ffp-contract=off, OpenMP)."""
    src = os.path.join(_HERE, "epsgraph_oracle.c")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(src)):
        return _LIB_PATH
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    P = ctypes.c_void_p
    i64, i32 = ctypes.c_int64, ctypes.c_int32
    lib.or_project_words.argtypes = [P, i64, i32, P, i32, P, i32]
    lib.or_project_words.restype = ctypes.c_int
    lib.or_first_nonfinite.argtypes = [P, i64, i32]
    lib.or_first_nonfinite.restype = i64
    lib.or_grouped_radix_sort.argtypes = [P, i64, i32, i32, P, i32, P, i32, i32, P, P]
    lib.or_grouped_radix_sort.restype = i64
    lib.or_enumerate_pairs.argtypes = [P, i64, i32, i32, P, i32, i32, i32, i32,
                                       ctypes.POINTER(ctypes.POINTER(i64)),
                                       ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.or_enumerate_pairs.restype = ctypes.c_int
    lib.or_free.argtypes = [P]
    lib.or_first_witness.argtypes = [P, i64, P, i32, i32, i32, P]
    lib.or_cosine_dist.argtypes = [P, i64, i32, P, i64, P, i32]
    lib.or_bf_hamming_digest.argtypes = [P, P, i64, i32, i32, P, i32]
    lib.or_bf_hamming_digest.restype = None
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------- projection

def directions(length: int, dim: int, seed: int, replicate_id: int) -> np.ndarray:
    """Gaussian directions of one replicate (lsh.py:116-118, 142-146).

    The reference draws them in column blocks from one generator; the stream
    is seamless, so one ``(length, dim)`` draw is identical.
    """
    ss = np.random.SeedSequence([int(seed), int(replicate_id)])
    rng = np.random.Generator(np.random.PCG64(ss))
    return rng.standard_normal((length, dim))


def project_words(x, length: int, seed: int, replicate_id: int,
                  threads: int = 0) -> np.ndarray:
    """Packed sign bits of one replicate (lsh.py:128-147). x is cast to f64."""
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, dim = x.shape
    r = np.ascontiguousarray(directions(length, dim, seed, replicate_id))
    W = max(1, -(-length // 64))
    words = np.zeros((n, W), dtype=np.uint64)
    rc = lib.or_project_words(_ptr(x), n, dim, _ptr(r), length, _ptr(words), threads)
    assert rc == 0
    return words


def block_partition(length: int, k: int) -> np.ndarray:
    """bitpool.py:44-69."""
    if k < 1 or k > length:
        raise ValueError(f"block count {k} outside [1, {length}]")
    base, rem = divmod(length, k)
    sizes = np.full(k, base, dtype=np.int64)
    sizes[:rem] += 1
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


# ---------------------------------------------------------------- enumerate

def grouped_radix_sort(words, length, bounds, mask, chunk_bits=16):
    """hamming_join.py:275-297 -- reproduces the reference perm exactly."""
    lib = _load()
    words = np.ascontiguousarray(words, dtype=np.uint64)
    n, W = words.shape
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    k = len(bounds) - 1
    m = np.ascontiguousarray(sorted(mask), dtype=np.int32)
    perm = np.empty(n, dtype=np.int64)
    gb = np.empty(n + 1, dtype=np.int64)
    ng = lib.or_grouped_radix_sort(_ptr(words), n, W, length, _ptr(bounds), k,
                                   _ptr(m) if m.size else None, m.size,
                                   chunk_bits, _ptr(perm), _ptr(gb))
    if ng < 0:
        raise ValueError("bad arguments")
    return perm, gb[:ng + 1].copy()


def enumerate_pairs(words, length, bounds, d, chunk_bits=16, threads=0):
    """hamming_join.py:300-375. Returns (pairs int64[m,2] sorted, max_group)."""
    lib = _load()
    words = np.ascontiguousarray(words, dtype=np.uint64)
    n, W = words.shape
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    k = len(bounds) - 1
    if n == 0:
        raise ValueError("pool is empty")
    if not (0 <= d < k <= length):
        raise ValueError(f"need 0 <= d < k <= length, got d={d}, k={k}, length={length}")
    out = ctypes.POINTER(ctypes.c_int64)()
    cnt = ctypes.c_int64()
    big = ctypes.c_int64()
    rc = lib.or_enumerate_pairs(_ptr(words), n, W, length, _ptr(bounds), k, d,
                                chunk_bits, threads, ctypes.byref(out),
                                ctypes.byref(cnt), ctypes.byref(big))
    if rc != 0:
        raise RuntimeError(f"oracle enumerate failed ({rc})")
    m = cnt.value
    if m:
        arr = np.ctypeslib.as_array(out, shape=(m, 2)).copy()
    else:
        arr = np.empty((0, 2), dtype=np.int64)
    lib.or_free(ctypes.cast(out, ctypes.c_void_p))
    return arr, int(big.value)


def brute_force_hamming(words, d):
    """exact.py:99-121 restated: all (i<j) with popcount(xor) <= d."""
    words = np.asarray(words, dtype=np.uint64)
    n = words.shape[0]
    chunks = []
    for lo in range(0, n, 256):
        diff = words[lo:lo + 256, None, :] ^ words[None, lo:, :]
        dist = np.bitwise_count(diff).sum(axis=2, dtype=np.int64)
        ii, jj = np.nonzero(dist <= d)
        keep = jj > ii
        if keep.any():
            chunks.append(np.column_stack([ii[keep] + lo, jj[keep] + lo]))
    if not chunks:
        return np.empty((0, 2), dtype=np.int64)
    return np.vstack(chunks).astype(np.int64)


def bf_hamming_digest(words, ids, d, threads=0):
    """exact.py:99-121 in digest form (see or_bf_hamming_digest): (count,
    sum of mix(key) mod 2^64, xor of mix(key)) over all pairs a < b of the
    rows with popcount(xor) <= d, keys built from the global ``ids``."""
    words = np.ascontiguousarray(words, dtype=np.uint64)
    if words.ndim == 1:
        words = words.reshape(-1, 1)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    out = np.zeros(3, dtype=np.uint64)
    _load().or_bf_hamming_digest(_ptr(words), _ptr(ids), words.shape[0], words.shape[1], d,
                                 _ptr(out), threads)
    return int(out[0]), int(out[1]), int(out[2])


def mix_digest(keys) -> tuple:
    """The same digest over uint64 pair keys (i << 32 | j), numpy side."""
    z = np.asarray(keys).view(np.uint64).copy()
    z ^= z >> np.uint64(30)
    z *= np.uint64(0xbf58476d1ce4e5b9)
    z ^= z >> np.uint64(27)
    z *= np.uint64(0x94d049bb133111eb)
    z ^= z >> np.uint64(31)
    return int(z.size), int(z.sum(dtype=np.uint64)), int(np.bitwise_xor.reduce(z)) if z.size else 0


def first_witness(pairs, earlier_words, d):
    """pipeline.py:109-146: keep pairs whose Hamming > d in all earlier pools."""
    lib = _load()
    pairs = np.ascontiguousarray(pairs, dtype=np.int64).reshape(-1, 2)
    keep = np.ones(pairs.shape[0], dtype=np.uint8)
    if not earlier_words or pairs.shape[0] == 0:
        return keep.astype(bool)
    arrs = [np.ascontiguousarray(w, dtype=np.uint64) for w in earlier_words]
    W = arrs[0].shape[1]
    ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    lib.or_first_witness(_ptr(pairs), pairs.shape[0], ctypes.cast(ptrs, ctypes.c_void_p),
                         len(arrs), W, d, _ptr(keep))
    return keep.astype(bool)


# ------------------------------------------------------------------- filter

def cosine_dist(x, pairs, threads=0):
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.float64)
    pairs = np.ascontiguousarray(pairs, dtype=np.int64).reshape(-1, 2)
    dist = np.empty(pairs.shape[0], dtype=np.float64)
    if pairs.shape[0]:
        lib.or_cosine_dist(_ptr(x), x.shape[0], x.shape[1], _ptr(pairs),
                           pairs.shape[0], _ptr(dist), threads)
    return dist


def filter_exact(x, pairs, epsilon, threads=0):
    """pipeline.py:183-223 -> (pairs sorted by (i,j), distances)."""
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if pairs.size and (pairs.min() < 0 or pairs.max() >= np.asarray(x).shape[0]):
        raise IndexError("candidate index out of range")
    dist = cosine_dist(x, pairs, threads)
    keep = dist <= epsilon
    p, dd = pairs[keep], dist[keep]
    order = np.lexsort((p[:, 1], p[:, 0]))
    return p[order], dd[order]


# -------------------------------------------------------------------- build

@dataclass
class OracleGraph:
    pairs: np.ndarray
    distances: np.ndarray
    candidate_count: int
    per_replicate_raw: tuple
    per_replicate_new: tuple
    codes: list = field(default_factory=list)
    timings: dict = field(default_factory=dict)


def build_graph(x, epsilon, length, mismatch, blocks, replicates, seed=0,
                threads=0, keep_codes=False, metric="cosine"):
    """pipeline.py:242-354 restated (cosine; euclidean mapped per lsh.py:218)."""
    import time
    t0 = time.perf_counter()
    x64 = np.ascontiguousarray(x, dtype=np.float64)
    if metric == "euclidean":
        epsilon = epsilon * epsilon / 2.0
    bounds = block_partition(length, blocks)
    codes, raw, new, pieces = [], [], [], []
    t_proj = t_enum = 0.0
    for h in range(replicates):
        ta = time.perf_counter()
        w = project_words(x64, length, seed, h + 1, threads)
        tb = time.perf_counter()
        pr, _ = enumerate_pairs(w, length, bounds, mismatch, 16, threads)
        tc = time.perf_counter()
        t_proj += tb - ta
        t_enum += tc - tb
        raw.append(pr.shape[0])
        keep = first_witness(pr, codes, mismatch)
        pr = pr[keep]
        new.append(pr.shape[0])
        pieces.append(pr)
        codes.append(w)
    cand = np.vstack(pieces) if pieces else np.empty((0, 2), np.int64)
    tf = time.perf_counter()
    p, dd = filter_exact(x64, cand, epsilon, threads)
    t1 = time.perf_counter()
    return OracleGraph(p, dd, cand.shape[0], tuple(raw), tuple(new),
                       codes if keep_codes else [],
                       {"project_s": t_proj, "enumerate_s": t_enum,
                        "filter_s": t1 - tf, "total_s": t1 - t0})


def pair_digest(pairs) -> str:
    """Order-sensitive sha256 of an int64 (m,2) pair array."""
    import hashlib
    a = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1, 2))
    return hashlib.sha256(a.tobytes()).hexdigest()


def words_digest(words) -> str:
    import hashlib
    a = np.ascontiguousarray(np.asarray(words, dtype=np.uint64))
    return hashlib.sha256(a.tobytes()).hexdigest()


def masks(k, d):
    return list(itertools.combinations(range(k), d))


def collision_prob(epsilon):
    return math.acos(1.0 - epsilon) / math.pi
