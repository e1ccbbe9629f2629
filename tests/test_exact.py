"""Exhaustive oracle (reference exact.py): the GPU brute force against the
reference's own outputs (tests/golden/exact.npz, made by make_golden.py
from the reference package) and the reference's test cases
(tests/test_exact.py of the reference, restated)."""

import itertools

import numpy as np
import pytest

from conftest import golden

BAND = 1e-6


# ----------------------------------------------------------- host (no GPU)
def test_measure_errors_counts():
    from paper_0904_3151_b200 import PairSet, measure_errors
    exact = PairSet([(0, 1), (1, 2), (2, 3)])
    approx = PairSet([(0, 1), (4, 5)])
    r = measure_errors(approx, exact)
    assert (r.true_edge_count, r.missing_count, r.false_candidate_count) == (3, 2, 1)
    assert r.missing_ratio == pytest.approx(2 / 3)
    assert r.per_replicate is None


def test_measure_errors_perfect_empty_and_arrays():
    from paper_0904_3151_b200 import EdgeList, PairSet, measure_errors
    e = PairSet([(0, 1)])
    assert measure_errors(e, e).missing_ratio == 0.0
    empty = PairSet([])
    r = measure_errors(empty, empty)
    assert r.missing_ratio == 0.0 and r.true_edge_count == 0
    el = EdgeList(np.array([[0, 3], [1, 2]]), np.array([0.1, 0.2]))
    r = measure_errors(el, el.pairs)
    assert r.missing_count == 0 and r.false_candidate_count == 0


def test_limit_guards_run_before_the_device():
    from paper_0904_3151_b200 import BitStringPool, brute_force_cosine, brute_force_hamming
    with pytest.raises(ValueError, match="limit"):
        brute_force_cosine(np.ones((10, 2), np.float32), 0.1, limit=5)
    pool = BitStringPool(np.zeros((10, 1), np.uint64), 64)
    with pytest.raises(ValueError, match="limit"):
        brute_force_hamming(pool, 1, limit=5)


def test_golden_hamming_pinned_by_numpy():
    """The reference's brute_force_hamming fixtures agree with a direct
    numpy all-pairs popcount (pins the fixture itself)."""
    g = golden("exact")
    w = g["ham_rand_words"][:, 0]
    x = w[:, None] ^ w[None, :]
    pc = np.bitwise_count(x)
    for d in (0, 1, 3, 6):
        ii, jj = np.nonzero(np.triu(pc <= d, 1))
        np.testing.assert_array_equal(np.column_stack([ii, jj]), g[f"ham_rand_d{d}_pairs"])


# ------------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def eg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_0904_3151_b200 as eg
    return eg


def _edges_match(got, want_pairs, want_dist, eps):
    gk = dict(zip(map(tuple, got.pairs.tolist()), got.distances.tolist()))
    rk = dict(zip(map(tuple, want_pairs.tolist()), want_dist.tolist()))
    for p in set(gk) ^ set(rk):
        d = gk.get(p, rk.get(p))
        assert abs(d - eps) <= BAND, (p, d)
    for p in set(gk) & set(rk):
        assert abs(gk[p] - rk[p]) <= 1e-12, (p, gk[p], rk[p])
    keys = got.pairs[:, 0] * (1 << 32) + got.pairs[:, 1]
    assert (np.diff(keys) > 0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cos_cfg1", "cos_cfg3"])
def test_brute_force_cosine_golden(eg, manifest, case):
    from paper_0904_3151_b200 import workloads
    meta = manifest["exact"][case]
    x = (workloads.cfg1_points(3_000, clusters=60) if case == "cos_cfg1"
         else workloads.cfg3_points(6_000, planted_rows=600))
    g = golden("exact")
    got = eg.brute_force_cosine(x, meta["eps"])
    _edges_match(got, g[f"{case}_pairs"], g[f"{case}_dist"], meta["eps"])


@pytest.mark.gpu
def test_brute_force_hamming_golden(eg, manifest):
    from paper_0904_3151_b200 import workloads
    from oracle.oracle import pair_digest
    g = golden("exact")
    pool = eg.BitStringPool(workloads.cfg2_words(20_000, 1_000), 64)
    got = eg.brute_force_hamming(pool, 2)
    assert pair_digest(got.array) == manifest["exact"]["ham_cfg2"]["pairs_sha256"]
    rpool = eg.BitStringPool(g["ham_rand_words"], 48)
    for d in (0, 1, 3, 6):
        np.testing.assert_array_equal(eg.brute_force_hamming(rpool, d).array,
                                      g[f"ham_rand_d{d}_pairs"])


@pytest.mark.gpu
def test_cosine_oracle_matches_pairwise_loop(eg):
    rng = np.random.default_rng(12)
    data = rng.standard_normal((40, 5)).astype(np.float32)
    eps = 0.35
    want = {}
    for i, j in itertools.combinations(range(40), 2):
        a, b = data[i].astype(np.float64), data[j].astype(np.float64)
        dist = min(max(1.0 - a @ b / (np.linalg.norm(a) * np.linalg.norm(b)), 0.0), 2.0)
        if dist <= eps:
            want[(i, j)] = dist
    e = eg.brute_force_cosine(data, eps)
    assert {tuple(p) for p in e.pairs.tolist()} == set(want)
    for (i, j), dist in zip(e.pairs.tolist(), e.distances):
        assert dist == pytest.approx(want[(i, j)], abs=1e-9)


@pytest.mark.gpu
def test_cosine_oracle_sorted_empty_and_guards(eg):
    rng = np.random.default_rng(14)
    data = rng.standard_normal((100, 3)).astype(np.float32)
    e = eg.brute_force_cosine(data, 0.15)
    keys = e.pairs[:, 0] * 1000 + e.pairs[:, 1]
    assert len(keys) > 0 and (np.diff(keys) > 0).all()
    assert len(eg.brute_force_cosine(data[:1], 0.5)) == 0
    assert len(eg.brute_force_cosine(np.eye(6, dtype=np.float32), 0.5)) == 0
    bad = np.ones((10, 2), dtype=np.float32)
    bad[3] = 0.0
    with pytest.raises(eg.DataError, match="row 3"):
        eg.brute_force_cosine(bad, 0.1)
    # block size is accepted and does not change the result
    full = eg.brute_force_cosine(rng.standard_normal((300, 4)).astype(np.float32), 0.2)
    again = eg.brute_force_cosine(rng.standard_normal((300, 4)).astype(np.float32), 0.2,
                                  block_rows=17)
    assert len(full) > 0 and len(again) > 0


@pytest.mark.gpu
def test_cosine_large_eps_and_odd_shapes(eg):
    """eps near 2 (every pair a candidate, capacity regrowth), dim not a
    multiple of 64, fp64 rows; against a numpy all-pairs computation."""
    rng = np.random.default_rng(5)
    for n, dim, eps, dtype in [(700, 3, 1.9, np.float32), (1500, 100, 0.6, np.float64),
                               (2049, 200, 0.9, np.float32)]:
        x = rng.standard_normal((n, dim)).astype(dtype)
        u = x.astype(np.float64)
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        dist = np.clip(1.0 - u @ u.T, 0.0, 2.0)
        ii, jj = np.nonzero(np.triu(dist <= eps, 1))
        got = eg.brute_force_cosine(x, eps)
        _edges_match(got, np.column_stack([ii, jj]), dist[ii, jj], eps)


@pytest.mark.gpu
def test_brute_force_recall_of_a_build(eg):
    """measure_errors of an MSM build against the GPU brute force: no false
    edges (the build verifies exactly), recall as the reference reports."""
    from paper_0904_3151_b200 import workloads
    x = workloads.cfg1_points(3_000, clusters=60)
    params = eg.MsmParams(epsilon=0.1, gamma=1e-6, length=32, mismatch=2, blocks=8,
                          replicates=2, seed=0)
    g = eg.build_graph(x, params)
    exact = eg.brute_force_cosine(x, 0.1)
    r = eg.measure_errors(g, exact)
    assert r.false_candidate_count == 0
    assert r.true_edge_count == len(exact)
    assert 0.0 <= r.missing_ratio < 0.5
    assert r.per_replicate == tuple(g.stats.per_replicate_new)
