"""Full-scale parity fixtures made by running the REFERENCE package itself.

Build container only (the reference tree does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_full.py cfg3 [cfg2 cfg4_10 cfg5_2m cfg4_full cfg5_full]

Each config writes ``tests/golden/full/<name>.json``: sha256 digests of the
reference's exact int64 arrays (codes, per-replicate raw pair sets, the
candidate union, the edge set) plus counts, so the GPU tests can compare at
the real configuration shapes without shipping the arrays.  Edge parity is
exact except for pairs whose distance lies within 1e-6 of epsilon
(BASELINE.json north_star): those "band" pairs are listed explicitly with
their reference distances, and ``edges_core_sha256`` is the digest of the
edge set with the band pairs removed.

Inputs come from ``paper_0904_3151_b200.workloads`` (seeded generators,
SURVEY.md App. C).  Where the full configuration is not CPU-feasible for the
reference (config 4 at n=4M: 1.4e9 edges; config 5 at n=20M: ~4 h), the
fixture pins (a) the reference's codes on the full input (config 4) or on a
1M-row sample via the reference's own ``rows=`` mode (config 5,
lsh.py:128-138), and (b) the restricted-subset answer of SURVEY.md 8(c):
``enumerate_pairs`` on pool[S] for a seeded row subset S of whole clusters
plus random rows, the union/first-witness over replicates, and
``filter_exact`` on it.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import epsgraph as ref  # noqa: E402  (the reference package)
from epsgraph.lsh import _project_words  # noqa: E402

from paper_0904_3151_b200 import workloads  # noqa: E402

OUT = os.path.join(HERE, "full")
BAND = 1e-6


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sorted_pairs(p: np.ndarray) -> np.ndarray:
    p = np.asarray(p, dtype=np.int64).reshape(-1, 2)
    order = np.lexsort((p[:, 1], p[:, 0]))
    return np.ascontiguousarray(p[order])


def distances(x: np.ndarray, pairs: np.ndarray) -> np.ndarray:
    """filter_exact's formula (pipeline.py:203-214) for every pair."""
    x64 = x.astype(np.float64, copy=False)
    norms = np.sqrt(np.einsum("ij,ij->i", x64, x64))
    out = np.empty(pairs.shape[0], dtype=np.float64)
    for lo in range(0, pairs.shape[0], 1 << 20):
        i, j = pairs[lo:lo + (1 << 20), 0], pairs[lo:lo + (1 << 20), 1]
        d = 1.0 - np.einsum("ij,ij->i", x64[i], x64[j]) / (norms[i] * norms[j])
        out[lo:lo + i.shape[0]] = np.clip(d, 0.0, 2.0)
    return out


def edge_record(x, cand_pairs, eps, edges):
    """Digests of an edge set plus its 1e-6 band (see module docstring)."""
    cand = sorted_pairs(cand_pairs)
    dist = distances(x, cand)
    band = np.abs(dist - eps) <= BAND
    ep = edges.pairs.astype(np.int64)
    core = ep
    if band.any():
        bkeys = set(map(tuple, cand[band].tolist()))
        core = np.array([p for p in ep.tolist() if tuple(p) not in bkeys],
                        dtype=np.int64).reshape(-1, 2)
    return {
        "candidate_count": int(cand.shape[0]),
        "candidates_sha256": digest(cand),
        "edge_count": int(ep.shape[0]),
        "edges_sha256": digest(ep),
        "edges_core_sha256": digest(core),
        "distance_sum": float(np.sum(edges.distances)),
        "band": {"pairs": cand[band].tolist(), "dist": dist[band].tolist()},
    }


def reference_pieces(x, length, k, d, reps, seed=0):
    """project -> enumerate_pairs per replicate (threads over replicates, as
    build_graph does, pipeline.py:316-327) -> dedup_across_replicates."""
    x64 = np.ascontiguousarray(x, dtype=np.float64)

    def one(h):
        t0 = time.perf_counter()
        words = _project_words(x64, ref.ProjectionSpec(length, seed, h))
        pool = ref.BitStringPool(words, length).partitioned(k)
        raw = ref.enumerate_pairs(pool, d)
        print(f"  replicate {h}: {raw.array.shape[0]} raw pairs, "
              f"{time.perf_counter() - t0:.1f}s", flush=True)
        return pool, raw

    with ThreadPoolExecutor(max_workers=reps) as ex:
        res = list(ex.map(one, range(1, reps + 1)))
    pools = [p for p, _ in res]
    raws = [r for _, r in res]
    cand = ref.dedup_across_replicates(pools, raws, d)
    return pools, raws, cand


def build_config(name, x, eps_cos, length, k, d, reps, extra=None):
    t0 = time.perf_counter()
    ref.build_graph(x[:64], ref.MsmParams(eps_cos, 1e-6, length, d, k, reps, 0), threads=1)
    pools, raws, cand = reference_pieces(x, length, k, d, reps)
    edges = ref.filter_exact(x, cand, eps_cos)
    rec = {
        "n": int(x.shape[0]), "dim": int(x.shape[1]), "epsilon_cos": eps_cos,
        "length": length, "blocks": k, "mismatch": d, "replicates": reps,
        "codes_sha256": [digest(p.words) for p in pools],
        "raw_sha256": [digest(r.array) for r in raws],
        "per_replicate_raw": list(cand.per_replicate_raw),
        "per_replicate_new": list(cand.per_replicate_new),
    }
    rec.update(edge_record(x, cand.pairs, eps_cos, edges))
    rec["reference_wall_s"] = time.perf_counter() - t0
    if extra:
        rec.update(extra)
    return rec


def subset_record(x, S, eps_cos, length, k, d, reps):
    """Reference answer on pool[S]; pair indices are global
    row ids (S is sorted, so the remap keeps i < j and the order)."""
    xs = np.ascontiguousarray(x[S])
    pools, raws, cand = reference_pieces(xs, length, k, d, reps)
    edges = ref.filter_exact(xs, cand, eps_cos)
    g_cand = S[cand.pairs]
    g_edges = ref.EdgeList(S[edges.pairs], edges.distances) if len(edges) else edges
    rec = {
        "rows": int(S.shape[0]), "rows_sha256": digest(S),
        "codes_sha256": [digest(p.words) for p in pools],
        "raw_sha256": [digest(S[r.array]) for r in raws],
        "per_replicate_raw": list(cand.per_replicate_raw),
        "per_replicate_new": list(cand.per_replicate_new),
    }
    rec.update(edge_record(x, g_cand, eps_cos, g_edges))
    return rec


def gen_cfg2():
    words = workloads.cfg2_words()
    pool = ref.BitStringPool(words, 64).partitioned(8)
    ref.enumerate_pairs(ref.BitStringPool(words[:100], 64).partitioned(8), 2)
    t0 = time.perf_counter()
    pairs = ref.enumerate_pairs(pool, 2).array
    return {"n": int(words.shape[0]), "blocks": 8, "mismatch": 2,
            "count": int(pairs.shape[0]), "pairs_sha256": digest(pairs),
            "reference_wall_s": time.perf_counter() - t0}


def gen_cfg3():
    return build_config("cfg3", workloads.cfg3_points(), 0.05, 48, 12, 3, 3)


def gen_cfg4_10():
    x = workloads.cfg4_points(4_000_000, subset=400_000)
    return build_config("cfg4_10", x, 0.08, 64, 16, 2, 1,
                        {"generator": "cfg4_points(4_000_000, subset=400_000)"})


def gen_cfg5_2m():
    x = workloads.cfg5_points(2_000_000, clusters=100_000)
    return build_config("cfg5_2m", x, 0.15 * 0.15 / 2.0, 64, 16, 3, 2,
                        {"generator": "cfg5_points(2_000_000, clusters=100_000)",
                         "metric": "euclidean", "epsilon": 0.15})


def gen_cfg4_full():
    x, lab = workloads.cfg4_points(labels=True)
    t0 = time.perf_counter()
    words = _project_words(np.ascontiguousarray(x, dtype=np.float64),
                           ref.ProjectionSpec(64, 0, 1))
    rec = {"n": int(x.shape[0]), "codes_sha256": [digest(words)],
           "codes_wall_s": time.perf_counter() - t0}
    S = workloads.restricted_subset(lab, [3, 4, 5])
    rec["subset_mid"] = {"clusters": [3, 4, 5], "extra": 20_000, "seed": 4321}
    rec["subset_mid"].update(subset_record(x, S, 0.08, 64, 16, 2, 1))
    big = workloads.restricted_subset(lab, [0, 1, 2])
    rec["subset_big"] = {"clusters": [0, 1, 2], "extra": 20_000, "seed": 4321,
                         "rows": int(big.shape[0]), "rows_sha256": digest(big)}
    return rec


def gen_cfg5_full():
    x, lab = workloads.cfg5_points(labels=True)
    rng = np.random.default_rng(99)
    sample = np.sort(rng.choice(x.shape[0], 1_000_000, replace=False))
    xs = np.ascontiguousarray(x[sample], dtype=np.float64)
    t0 = time.perf_counter()
    codes = [_project_words(xs, ref.ProjectionSpec(64, 0, h)) for h in (1, 2)]
    rec = {"n": int(x.shape[0]), "code_sample": {"rows": 1_000_000, "seed": 99,
                                                 "rows_sha256": digest(sample)},
           "codes_sample_sha256": [digest(c) for c in codes],
           "codes_wall_s": time.perf_counter() - t0}
    cl = workloads.largest_clusters(lab, 3)
    S = workloads.restricted_subset(lab, cl)
    rec["subset"] = {"clusters": cl, "extra": 20_000, "seed": 4321}
    rec["subset"].update(subset_record(x, S, 0.15 * 0.15 / 2.0, 64, 16, 3, 2))
    # a wider subset: the 3,000 most populous clusters (~100k rows) plus the
    # same 20k random rows
    cl = workloads.largest_clusters(lab, 3000)
    S = workloads.restricted_subset(lab, cl)
    rec["subset_wide"] = {"clusters_top": 3000, "extra": 20_000, "seed": 4321}
    rec["subset_wide"].update(subset_record(x, S, 0.15 * 0.15 / 2.0, 64, 16, 3, 2))
    return rec


GENS = {"cfg2": gen_cfg2, "cfg3": gen_cfg3, "cfg4_10": gen_cfg4_10, "cfg5_2m": gen_cfg5_2m,
        "cfg4_full": gen_cfg4_full, "cfg5_full": gen_cfg5_full}


def main(names):
    os.makedirs(OUT, exist_ok=True)
    for name in names:
        t0 = time.perf_counter()
        rec = GENS[name]()
        rec["numpy"] = np.__version__
        rec["reference"] = ref.__version__
        with open(os.path.join(OUT, f"{name}.json"), "w") as f:
            json.dump(rec, f, indent=1, sort_keys=True)
        print(name, "done", f"{time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(GENS))
