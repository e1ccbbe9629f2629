"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container only (the reference tree does not exist on the
GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

It writes small ``.npz`` files plus ``manifest.json`` next to this script.
Large outputs are stored as sha256 digests of the exact int64 arrays (and
counts), which stay size-independent.  The inputs come from
``paper_0904_3151_b200.workloads`` (seeded), so tests can regenerate them.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import epsgraph as ref  # noqa: E402  (the reference package)
from epsgraph.lsh import _project_words  # noqa: E402

from paper_0904_3151_b200 import workloads  # noqa: E402

FIG2_STRINGS = [
    "1011111100111110", "1101011101110001", "1100100011011100",
    "0100000101111101", "1010001011101010", "1111001110010111",
    "0000000100111110", "0101100101111000", "1101100011011110",
    "1001001110010111",
]


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def pool_from_bits(bits, k):
    return ref.BitStringPool.from_bits(bits.astype(np.uint8)).partitioned(k)


def gen_fig2(manifest):
    bits = np.array([[int(c) for c in s] for s in FIG2_STRINGS], dtype=np.uint8)
    pool = pool_from_bits(bits, 4)
    out = {"words": pool.words}
    for d in range(4):
        out[f"pairs_d{d}"] = ref.enumerate_pairs(pool, d).array
    np.savez_compressed(os.path.join(HERE, "fig2.npz"), **out)
    manifest["fig2"] = {"length": 16, "k": 4,
                        "pairs_d2": out["pairs_d2"].tolist()}


def gen_random_pools(manifest):
    """Enumeration and grouping on seeded random pools (cf. the reference's
    brute-force equivalence suites, tests/test_hamming_join.py:124-156)."""
    rng = np.random.default_rng(20261020)
    cases = []
    arrays = {}
    lengths = [8, 16, 24, 33, 48, 64, 70, 100, 128]
    for c in range(48):
        length = int(lengths[c % len(lengths)])
        k = int(rng.integers(1, min(length, 16) + 1))
        d = int(rng.integers(0, k))
        n = int(rng.integers(2, 400))
        density = float(rng.choice([0.1, 0.3, 0.5]))
        if c % 7 == 3:           # duplicate-heavy pool
            base = (rng.random((max(2, n // 8), length)) < density)
            bits = base[rng.integers(0, base.shape[0], n)]
        else:
            bits = rng.random((n, length)) < density
        pool = pool_from_bits(bits, k)
        pairs = ref.enumerate_pairs(pool, d).array
        brute = ref.brute_force_hamming(pool, d).array
        assert np.array_equal(pairs, brute)
        arrays[f"words_{c}"] = pool.words
        arrays[f"pairs_{c}"] = pairs
        mask = tuple(sorted(rng.choice(k, size=min(d, k), replace=False).tolist()))
        perm, gb = ref.grouped_radix_sort(pool, mask)
        arrays[f"perm_{c}"] = perm
        arrays[f"gbounds_{c}"] = gb
        cases.append({"case": c, "n": n, "length": length, "k": k, "d": d,
                      "mask": list(mask), "count": int(pairs.shape[0])})
    np.savez_compressed(os.path.join(HERE, "random_pools.npz"), **arrays)
    manifest["random_pools"] = cases


def gen_projection(manifest):
    """Packed sign bits, float32 and float64 inputs (lsh.py:128-172)."""
    rng = np.random.default_rng(777)
    cases = []
    arrays = {}
    specs = [(64, 2, 96, 0, 1), (50, 7, 100, 2, 4), (10, 13, 257, 6, 2),
             (200, 64, 32, 0, 1), (300, 8, 24, 7, 3), (150, 384, 48, 0, 2),
             (100, 128, 64, 0, 1), (40, 5, 130, 11, 9)]
    for c, (n, dim, length, seed, rep) in enumerate(specs):
        if c % 2 == 0:
            x = rng.standard_normal((n, dim)).astype(np.float32)
        else:
            x = rng.standard_normal((n, dim))
        words = ref.project(x, ref.ProjectionSpec(length, seed, rep)).words
        arrays[f"x_{c}"] = x
        arrays[f"words_{c}"] = words
        cases.append({"case": c, "n": n, "dim": dim, "length": length,
                      "seed": seed, "replicate_id": rep,
                      "dtype": str(x.dtype)})
    np.savez_compressed(os.path.join(HERE, "projection.npz"), **arrays)
    manifest["projection"] = cases


def graph_record(g, with_arrays=True):
    rec = {
        "candidate_count": g.stats.candidate_count,
        "edge_count": g.stats.edge_count,
        "false_candidate_count": g.stats.false_candidate_count,
        "per_replicate_raw": list(g.stats.per_replicate_raw),
        "per_replicate_new": list(g.stats.per_replicate_new),
        "achieved_bound": g.stats.achieved_bound,
        "pairs_sha256": digest(g.edge_list.pairs.astype(np.int64)),
        "distance_sum": float(np.sum(g.edge_list.distances)),
    }
    return rec


def gen_small_build(manifest):
    """build_graph on the reference test fixture (tests/test_pipeline.py:36-44)."""
    x = workloads.planted_clusters(300, 8, 6, 20, 0.03, 21)
    params = ref.MsmParams(epsilon=0.05, gamma=1e-3, length=24, mismatch=2,
                           blocks=4, replicates=4, seed=7)
    g = ref.build_graph(x, params, threads=1)
    pools = [ref.project(x, ref.ProjectionSpec(24, 7, h)).partitioned(4)
             for h in range(1, 5)]
    raw = [ref.enumerate_pairs(p, 2) for p in pools]
    merged = ref.dedup_across_replicates(pools, raw, 2)
    cand = ref.brute_force_hamming(pools[0], 6)
    filt = ref.filter_exact(x, cand, 0.05)
    arrays = {"x": x, "edges": g.edge_list.pairs, "dist": g.edge_list.distances,
              "merged": merged.pairs, "filter_cand": cand.array,
              "filter_edges": filt.pairs, "filter_dist": filt.distances}
    for h, r in enumerate(raw):
        arrays[f"raw_{h}"] = r.array
        arrays[f"codes_{h}"] = pools[h].words
    lsh = ref.build_graph_lsh_only(x, 0.05, 1e-3, replicates=50)
    arrays["lsh_edges"] = lsh.edge_list.pairs
    np.savez_compressed(os.path.join(HERE, "small_build.npz"), **arrays)
    rec = graph_record(g)
    rec["params"] = {"epsilon": 0.05, "length": 24, "mismatch": 2, "blocks": 4,
                     "replicates": 4, "seed": 7}
    rec["merged_raw"] = list(merged.per_replicate_raw)
    rec["merged_new"] = list(merged.per_replicate_new)
    rec["lsh_only"] = {"length": lsh.params.length,
                       "candidate_count": lsh.stats.candidate_count,
                       "per_replicate_new_sum": int(sum(lsh.stats.per_replicate_new))}
    manifest["small_build"] = rec


def gen_config(manifest, name, x, cfg, keep_arrays=False):
    params = ref.MsmParams(epsilon=cfg["epsilon"], gamma=1e-6,
                           length=cfg["length"], mismatch=cfg["mismatch"],
                           blocks=cfg["blocks"], replicates=cfg["replicates"],
                           seed=cfg.get("seed", 0))
    ref.build_graph(x[:50], params, threads=1)   # JIT warm-up
    t0 = time.perf_counter()
    g = ref.build_graph(x, params, threads=os.cpu_count())
    wall = time.perf_counter() - t0
    rec = graph_record(g)
    rec["params"] = cfg
    rec["n"] = int(x.shape[0])
    rec["wall_s"] = wall
    codes = [_project_words(np.ascontiguousarray(x, dtype=np.float64),
                            ref.ProjectionSpec(cfg["length"], cfg.get("seed", 0), h + 1))
             for h in range(cfg["replicates"])]
    rec["codes_sha256"] = [digest(c) for c in codes]
    if keep_arrays:
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                            edges=g.edge_list.pairs.astype(np.int32),
                            dist=g.edge_list.distances)
    manifest[name] = rec
    print(name, rec["edge_count"], rec["candidate_count"], f"{wall:.1f}s", flush=True)


def gen_hamming_config(manifest, name, words, k, d):
    pool = ref.BitStringPool(words, 64).partitioned(k)
    t0 = time.perf_counter()
    pairs = ref.enumerate_pairs(pool, d).array
    wall = time.perf_counter() - t0
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), pairs=pairs)
    manifest[name] = {"n": int(words.shape[0]), "k": k, "d": d,
                      "count": int(pairs.shape[0]), "pairs_sha256": digest(pairs),
                      "wall_s": wall}
    print(name, pairs.shape[0], f"{wall:.1f}s", flush=True)


def gen_exact(manifest):
    """The reference's exhaustive oracle (exact.py:57-121) on seeded inputs:
    brute_force_cosine on a cfg1-shaped and a cfg3-shaped sample,
    brute_force_hamming on a cfg2-shaped pool and a random 48-bit pool."""
    out = {}
    meta = {}
    cases = {
        "cos_cfg1": (workloads.cfg1_points(3_000, clusters=60), 0.1),
        "cos_cfg3": (workloads.cfg3_points(6_000, planted_rows=600), 0.05),
    }
    for name, (x, eps) in cases.items():
        e = ref.brute_force_cosine(x, eps)
        out[f"{name}_pairs"] = e.pairs
        out[f"{name}_dist"] = e.distances
        meta[name] = {"n": int(x.shape[0]), "eps": eps, "edges": int(len(e.pairs)),
                      "pairs_sha256": digest(e.pairs)}
    words = workloads.cfg2_words(20_000, 1_000)
    pool = ref.BitStringPool(words, 64)
    p = ref.brute_force_hamming(pool, 2)
    out["ham_cfg2_pairs"] = p.array
    meta["ham_cfg2"] = {"n": int(words.shape[0]), "d": 2, "pairs": int(len(p.array)),
                        "pairs_sha256": digest(p.array)}
    rng = np.random.default_rng(21)
    bits = (rng.random((4_000, 48)) < 0.5).astype(np.uint8)
    bits[2_000:2_400] = bits[:400]
    flip = rng.integers(0, 48, size=400)
    bits[np.arange(2_000, 2_400), flip] ^= 1
    pool = ref.BitStringPool.from_bits(bits)
    out["ham_rand_words"] = pool.words
    for d in (0, 1, 3, 6):
        p = ref.brute_force_hamming(pool, d)
        out[f"ham_rand_d{d}_pairs"] = p.array
        meta[f"ham_rand_d{d}"] = {"pairs": int(len(p.array)), "pairs_sha256": digest(p.array)}
    np.savez_compressed(os.path.join(HERE, "exact.npz"), **out)
    manifest["exact"] = meta


def gen_io(manifest):
    """Edge files written by the reference's io.write_edges (io.py:145-158):
    special distances, values at %.9f rounding boundaries, random ones,
    large indices and Euclidean-scale distances; the bytes are the fixture."""
    import tempfile
    rng = np.random.default_rng(31)
    special = [0.0, 2.0, 1.0, 0.123456789123, 5e-10, 1.5e-9, 2.5e-9, 0.0000000015,
               0.9999999995, 1.9999999995, 0.1234567885, 0.1234567895, 1e-300, 5e-324,
               12345.678901234, 1e9, 3.0000000005, 7.25, 0.5, 0.05]
    m = 4000
    d = np.concatenate([np.array(special), rng.random(m) * 2.0,
                        rng.random(200) * 1e4, np.round(rng.random(200) * 2, 9),
                        np.round(rng.random(200) * 2, 10) + 5e-10])
    i = np.sort(rng.integers(0, 4_000_000_000, d.size))
    j = i + rng.integers(1, 1000, d.size)
    pairs = np.stack([i, j], axis=1).astype(np.int64)
    order = np.lexsort((pairs[:, 1], pairs[:, 0]))
    pairs, d = pairs[order], d[order]
    keep = np.ones(len(pairs), dtype=bool)
    keep[1:] = np.any(pairs[1:] != pairs[:-1], axis=1)
    pairs, d = pairs[keep], d[keep]
    edges = ref.EdgeList(pairs, d)
    meta = {"epsilon": 0.05, "nodes": 1600000, "normalize": False, "tag": "golden"}
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "e.txt")
        ref.write_edges(path, edges, meta)
        blob = open(path, "rb").read()
    np.savez_compressed(os.path.join(HERE, "io_edges.npz"), pairs=pairs, dist=d,
                        text=np.frombuffer(blob, dtype=np.uint8))
    manifest["io_edges"] = {"edges": int(len(pairs)), "bytes": len(blob),
                            "sha256": hashlib.sha256(blob).hexdigest(), "meta": meta}


def gen_estimate(manifest):
    """The reference's estimate_output_size (tuning.py:190-229) on seeded
    cfg1- and cfg3-shaped samples."""
    out = {}
    for name, x, eps, pairs, seed in [
            ("cfg1", workloads.cfg1_points(5_000, clusters=50), 0.1, 20_000, 0),
            ("cfg3", workloads.cfg3_points(20_000, planted_rows=4_000), 0.05, 50_000, 3),
            ("tiny", workloads.cfg1_points(40, clusters=2), 0.3, 7, 1)]:
        e = ref.estimate_output_size(x, eps, sample_pairs=pairs, seed=seed)
        out[name] = {"eps": eps, "sample_pairs": pairs, "seed": seed, "hits": e.hits,
                     "total_pairs": e.total_pairs, "estimate_s": e.estimate_s,
                     "ci": [e.ci_low, e.ci_high]}
    manifest["estimate"] = out


def main():
    manifest = {"numpy": np.__version__, "reference": ref.__version__}
    gen_fig2(manifest)
    gen_random_pools(manifest)
    gen_projection(manifest)
    gen_small_build(manifest)
    gen_exact(manifest)
    gen_io(manifest)
    gen_estimate(manifest)
    # Config 1 at full size (809,648 edges).
    gen_config(manifest, "cfg1", workloads.cfg1_points(),
               {"epsilon": 0.1, "length": 32, "blocks": 8, "mismatch": 2,
                "replicates": 1})
    # Config 2 at reduced size: same generator, 200k base + 10k planted.
    gen_hamming_config(manifest, "cfg2_small",
                       workloads.cfg2_words(200_000, 10_000), 8, 2)
    # Config 3 shape at n=20k (first 5% planted), full D/params.
    gen_config(manifest, "cfg3_small", workloads.cfg3_points(20_000),
               {"epsilon": 0.05, "length": 48, "blocks": 12, "mismatch": 3,
                "replicates": 3}, keep_arrays=True)
    # Config 4 shape: Zipf clusters capped at 2000, n=60k.
    gen_config(manifest, "cfg4_small",
               workloads.cfg4_points(60_000, largest=2_000),
               {"epsilon": 0.08, "length": 64, "blocks": 16, "mismatch": 2,
                "replicates": 1})
    # Config 5 shape (euclidean 0.15 -> cosine 0.15^2/2), n=40k, 2k clusters.
    gen_config(manifest, "cfg5_small",
               workloads.cfg5_points(40_000, clusters=2_000),
               {"epsilon": 0.15 * 0.15 / 2.0, "length": 64, "blocks": 16,
                "mismatch": 3, "replicates": 2})
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] in ("exact", "io", "estimate"):   # one family only
        path = os.path.join(HERE, "manifest.json")
        with open(path) as f:
            manifest = json.load(f)
        {"exact": gen_exact, "io": gen_io, "estimate": gen_estimate}[sys.argv[1]](manifest)
        with open(path, "w") as f:
            json.dump(manifest, f, indent=1, sort_keys=True)
    else:
        main()
