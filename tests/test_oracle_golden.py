"""Pin the CPU oracle against fixtures produced by the reference itself.

The oracle (oracle/epsgraph_oracle.c) is the checker for the CUDA path, so
before it is trusted it must reproduce the reference's own outputs: packed
projection bits, the exact grouped-sort permutation, enumerate_pairs,
first-witness dedup, the exact filter and whole builds (digests).
"""

import numpy as np
import pytest

from conftest import FIG2_CLOSE_PAIRS, golden
from paper_0904_3151_b200 import workloads


def test_fig2_pool(oracle):
    g = golden("fig2")
    bounds = oracle.block_partition(16, 4)
    for d in range(4):
        pairs, _ = oracle.enumerate_pairs(g["words"], 16, bounds, d)
        np.testing.assert_array_equal(pairs, g[f"pairs_d{d}"])
    pairs, _ = oracle.enumerate_pairs(g["words"], 16, bounds, 2)
    assert {tuple(p) for p in pairs.tolist()} == FIG2_CLOSE_PAIRS


def test_block_partition_kats(oracle):
    # bitpool.py:44-69 known answers (reference tests/test_bitpool.py:21-25)
    assert oracle.block_partition(16, 4).tolist() == [0, 4, 8, 12, 16]
    assert oracle.block_partition(10, 3).tolist() == [0, 4, 7, 10]
    assert oracle.block_partition(7, 7).tolist() == list(range(8))
    assert oracle.block_partition(5, 1).tolist() == [0, 5]


def test_random_pools_enumerate_and_grouping(oracle, manifest):
    g = golden("random_pools")
    for case in manifest["random_pools"]:
        c = case["case"]
        words = g[f"words_{c}"]
        bounds = oracle.block_partition(case["length"], case["k"])
        pairs, _ = oracle.enumerate_pairs(words, case["length"], bounds, case["d"])
        np.testing.assert_array_equal(pairs, g[f"pairs_{c}"], err_msg=str(case))
        # the grouped sort reproduces the reference permutation bit-for-bit
        perm, gb = oracle.grouped_radix_sort(words, case["length"], bounds, case["mask"])
        np.testing.assert_array_equal(perm, g[f"perm_{c}"])
        np.testing.assert_array_equal(gb, g[f"gbounds_{c}"])


def test_random_pools_threads_invariant(oracle, manifest):
    g = golden("random_pools")
    for case in manifest["random_pools"][:10]:
        c = case["case"]
        bounds = oracle.block_partition(case["length"], case["k"])
        a, _ = oracle.enumerate_pairs(g[f"words_{c}"], case["length"], bounds, case["d"], threads=1)
        b, _ = oracle.enumerate_pairs(g[f"words_{c}"], case["length"], bounds, case["d"], threads=4)
        np.testing.assert_array_equal(a, b)


def test_projection_bits(oracle, manifest):
    g = golden("projection")
    for case in manifest["projection"]:
        c = case["case"]
        words = oracle.project_words(g[f"x_{c}"], case["length"], case["seed"],
                                     case["replicate_id"])
        np.testing.assert_array_equal(words, g[f"words_{c}"], err_msg=str(case))


def test_small_build(oracle, manifest):
    g = golden("small_build")
    rec = manifest["small_build"]
    p = rec["params"]
    res = oracle.build_graph(g["x"], p["epsilon"], p["length"], p["mismatch"],
                             p["blocks"], p["replicates"], p["seed"], keep_codes=True)
    for h in range(p["replicates"]):
        np.testing.assert_array_equal(res.codes[h], g[f"codes_{h}"])
    assert res.per_replicate_raw == tuple(rec["per_replicate_raw"])
    assert res.per_replicate_new == tuple(rec["per_replicate_new"])
    assert res.candidate_count == rec["candidate_count"]
    np.testing.assert_array_equal(res.pairs, g["edges"])
    np.testing.assert_allclose(res.distances, g["dist"], rtol=0, atol=1e-12)


def test_dedup_and_filter(oracle):
    g = golden("small_build")
    codes = [g[f"codes_{h}"] for h in range(4)]
    pieces = []
    for h in range(4):
        raw = g[f"raw_{h}"]
        pieces.append(raw[oracle.first_witness(raw, codes[:h], 2)])
    np.testing.assert_array_equal(np.vstack(pieces), g["merged"])
    p, dd = oracle.filter_exact(g["x"], g["filter_cand"], 0.05)
    np.testing.assert_array_equal(p, g["filter_edges"])
    np.testing.assert_allclose(dd, g["filter_dist"], rtol=0, atol=1e-12)


def test_filter_rejects_bad_indices(oracle):
    x = np.ones((4, 3), dtype=np.float32)
    with pytest.raises(IndexError):
        oracle.filter_exact(x, np.array([[0, 4]]), 0.1)


@pytest.mark.slow
def test_cfg1_build_digest(oracle, manifest):
    rec = manifest["cfg1"]
    x = workloads.cfg1_points()
    res = oracle.build_graph(x, 0.1, 32, 2, 8, 1, 0, threads=0, keep_codes=True)
    assert oracle.words_digest(res.codes[0]) == rec["codes_sha256"][0]
    assert res.candidate_count == rec["candidate_count"]
    assert res.pairs.shape[0] == rec["edge_count"]
    assert oracle.pair_digest(res.pairs) == rec["pairs_sha256"]
    assert abs(float(res.distances.sum()) - rec["distance_sum"]) < 1e-6


def test_cfg2_small(oracle, manifest):
    rec = manifest["cfg2_small"]
    words = workloads.cfg2_words(200_000, 10_000)
    pairs, _ = oracle.enumerate_pairs(words, 64, oracle.block_partition(64, 8), 2, threads=0)
    assert pairs.shape[0] == rec["count"]
    assert oracle.pair_digest(pairs) == rec["pairs_sha256"]


@pytest.mark.slow
def test_cfg3_small_build(oracle, manifest):
    rec = manifest["cfg3_small"]
    x = workloads.cfg3_points(20_000)
    res = oracle.build_graph(x, 0.05, 48, 3, 12, 3, 0, threads=0, keep_codes=True)
    for h in range(3):
        assert oracle.words_digest(res.codes[h]) == rec["codes_sha256"][h]
    assert res.per_replicate_raw == tuple(rec["per_replicate_raw"])
    assert res.per_replicate_new == tuple(rec["per_replicate_new"])
    assert oracle.pair_digest(res.pairs) == rec["pairs_sha256"]


def test_bf_hamming_digest_matches_pair_list(oracle):
    """The digest form of the exhaustive Hamming join (used for the config-4
    full-scale restriction) agrees with the pinned pair list."""
    g = golden("exact")
    words = g["ham_rand_words"]
    ids = np.arange(words.shape[0], dtype=np.int64) * 3 + 5     # any increasing ids
    for d in (0, 1, 3):
        pairs = g[f"ham_rand_d{d}_pairs"]
        keys = (ids[pairs[:, 0]].astype(np.uint64) << np.uint64(32)) | ids[pairs[:, 1]].astype(np.uint64)
        assert oracle.bf_hamming_digest(words, ids, d) == oracle.mix_digest(keys)


def _full_fixture(name):
    import json
    import os
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "full", f"{name}.json")) as f:
        return json.load(f)


@pytest.mark.slow
def test_oracle_cfg4_ten_percent_vs_reference(oracle):
    """The C oracle pinned against the reference's own config-4 answer at a
    10% row sample (400k rows, 13.9M edges; tests/golden/full)."""
    rec = _full_fixture("cfg4_10")
    x = workloads.cfg4_points(4_000_000, subset=400_000)
    g = oracle.build_graph(x, 0.08, 64, 2, 16, 1, 0, keep_codes=True)
    assert oracle.words_digest(g.codes[0]) == rec["codes_sha256"][0]
    assert list(g.per_replicate_raw) == rec["per_replicate_raw"]
    assert g.candidate_count == rec["candidate_count"]
    assert not rec["band"]["pairs"]
    assert oracle.pair_digest(g.pairs) == rec["edges_sha256"]
    assert abs(float(np.sum(g.distances)) - rec["distance_sum"]) <= 1e-12 * len(g.distances)


@pytest.mark.slow
def test_oracle_cfg4_full_subset_vs_reference(oracle):
    """SURVEY.md 8(c) restriction at full config 4: the oracle's
    enumerate_pairs on pool[S] equals the reference's (whole clusters 3-5 +
    20k random rows of the n=4M input)."""
    rec = _full_fixture("cfg4_full")["subset_mid"]
    x, lab = workloads.cfg4_points(labels=True)
    S = workloads.restricted_subset(lab, rec["clusters"], rec["extra"], rec["seed"])
    assert oracle.words_digest(S) == rec["rows_sha256"]
    w = oracle.project_words(x[S], 64, 0, 1)
    assert oracle.words_digest(w) == rec["codes_sha256"][0]
    pairs, _ = oracle.enumerate_pairs(w, 64, oracle.block_partition(64, 16), 2)
    assert oracle.pair_digest(S[pairs]) == rec["raw_sha256"][0]
