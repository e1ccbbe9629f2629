"""CUDA path vs the pinned oracle / reference fixtures (needs a B200).

Every comparison goes through the package's public API, which calls the
C ABI of libepsgraph_b200.so.  Integer outputs (codes, pair sets, counts)
must be bit-exact; distances agree to 1e-12 (fp64, different summation
order) and edge sets must be identical except for pairs within 1e-6 of eps.
"""

import logging

import numpy as np
import pytest

from conftest import FIG2_CLOSE_PAIRS, golden, pack_bits

pytestmark = pytest.mark.gpu

DIST_TOL = 1e-12
BAND = 1e-6


@pytest.fixture(scope="module")
def eg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_0904_3151_b200 as eg
    from paper_0904_3151_b200 import _native
    _native.lib()
    return eg


def pairs_equal_except_band(got_pairs, got_dist, ref_pairs, ref_dist, eps, dist_tol=DIST_TOL):
    gk = {tuple(p): d for p, d in zip(got_pairs.tolist(), got_dist.tolist())}
    rk = {tuple(p): d for p, d in zip(ref_pairs.tolist(), ref_dist.tolist())}
    for p in set(gk) ^ set(rk):
        d = gk.get(p, rk.get(p))
        assert abs(d - eps) <= BAND, (p, d)
    for p in set(gk) & set(rk):
        assert abs(gk[p] - rk[p]) <= dist_tol, (p, gk[p], rk[p])


# ------------------------------------------------------------- enumeration

def test_fig2_pool(eg):
    g = golden("fig2")
    pool = eg.BitStringPool(g["words"], 16).partitioned(4)
    for d in range(4):
        got = eg.enumerate_pairs(pool, d)
        np.testing.assert_array_equal(got.array, g[f"pairs_d{d}"])
    assert eg.enumerate_pairs(pool, 2).to_set() == FIG2_CLOSE_PAIRS


def test_random_pools_match_reference(eg, manifest):
    g = golden("random_pools")
    for case in manifest["random_pools"]:
        c = case["case"]
        pool = eg.BitStringPool(g[f"words_{c}"], case["length"]).partitioned(case["k"])
        got = eg.enumerate_pairs(pool, case["d"])
        np.testing.assert_array_equal(got.array, g[f"pairs_{c}"], err_msg=str(case))


def test_grouped_sort_reference_permutation(eg, manifest):
    """grouped_radix_sort returns the reference's exact permutation and group
    bounds (first-seen counting passes, hamming_join.py:52-82, 275-297)."""
    g = golden("random_pools")
    for case in manifest["random_pools"]:
        c = case["case"]
        pool = eg.BitStringPool(g[f"words_{c}"], case["length"]).partitioned(case["k"])
        perm, bounds = eg.grouped_radix_sort(pool, case["mask"])
        np.testing.assert_array_equal(perm, g[f"perm_{c}"], err_msg=str(case))
        np.testing.assert_array_equal(bounds, g[f"gbounds_{c}"], err_msg=str(case))


@pytest.mark.parametrize("chunk_bits", [1, 5, 8, 16, 24])
def test_grouped_sort_chunk_bits_vs_oracle(eg, oracle, manifest, chunk_bits):
    """Every chunk width gives the oracle's permutation (the order depends on
    chunk_bits; the grouping does not)."""
    g = golden("random_pools")
    for case in manifest["random_pools"][:20]:
        c = case["case"]
        pool = eg.BitStringPool(g[f"words_{c}"], case["length"]).partitioned(case["k"])
        perm, bounds = eg.grouped_radix_sort(pool, case["mask"], chunk_bits=chunk_bits)
        wp, wb = oracle.grouped_radix_sort(pool.words, pool.length, pool.block_bounds,
                                           case["mask"], chunk_bits)
        np.testing.assert_array_equal(perm, wp, err_msg=str(case))
        np.testing.assert_array_equal(bounds, wb, err_msg=str(case))


def test_duplicates_and_oversized_warning(eg, caplog):
    bits = np.zeros((64, 16), dtype=np.uint8)
    pool = eg.BitStringPool.from_bits(bits).partitioned(4)
    with caplog.at_level(logging.WARNING, logger="paper_0904_3151_b200"):
        got = eg.enumerate_pairs(pool, 1)
    assert len(got) == 64 * 63 // 2
    assert any("group" in r.message for r in caplog.records)


def test_d_zero_duplicates(eg):
    strings = ["1010", "0101", "1010", "1111", "0101", "1010"]
    pool = eg.BitStringPool.from_bits(np.array([[int(c) for c in s] for s in strings])).partitioned(2)
    assert eg.enumerate_pairs(pool, 0).to_set() == {(0, 2), (0, 5), (2, 5), (1, 4)}


def test_single_row_and_validation(eg):
    pool = eg.BitStringPool.from_bits(np.array([[1, 0, 1, 0, 1, 0, 1, 0]])).partitioned(2)
    assert len(eg.enumerate_pairs(pool, 1)) == 0
    with pytest.raises(ValueError):
        eg.enumerate_pairs(pool, 2)
    with pytest.raises(ValueError):
        eg.enumerate_pairs(pool, -1)
    empty = eg.BitStringPool(np.zeros((0, 1), np.uint64), 8).partitioned(2)
    with pytest.raises(ValueError):
        eg.enumerate_pairs(empty, 1)


@pytest.mark.parametrize("n,length,k,d,density", [
    (3000, 64, 8, 2, 0.5),
    (5000, 48, 12, 3, 0.5),
    (4000, 128, 16, 3, 0.5),      # two words
    (2500, 256, 32, 2, 0.5),      # four words, max length
    (3000, 70, 7, 2, 0.3),        # unequal blocks across a word boundary
    (4000, 20, 20, 4, 0.5),       # one bit per block
    (6000, 24, 4, 1, 0.1),        # skewed bits: big groups
])
def test_random_pools_vs_oracle(eg, oracle, n, length, k, d, density):
    rng = np.random.default_rng(n + length + k + d)
    base = (rng.random((n // 3, length)) < density).astype(np.uint8)
    bits = base[rng.integers(0, base.shape[0], n)]
    flip = rng.random(bits.shape) < 0.02
    bits = bits ^ flip.astype(np.uint8)
    words = pack_bits(bits)
    pool = eg.BitStringPool(words, length).partitioned(k)
    got = eg.enumerate_pairs(pool, d)
    want, _ = oracle.enumerate_pairs(words, length, pool.block_bounds, d)
    np.testing.assert_array_equal(got.array, want)


def test_spill_path_giant_group(eg, oracle):
    # 5000 rows sharing most bits -> buckets far above shared-memory capacity
    rng = np.random.default_rng(5)
    n, length = 6000, 64
    base = rng.integers(0, 2**63, dtype=np.int64).astype(np.uint64)
    words = np.full((n, 1), base, dtype=np.uint64)
    flips = rng.integers(0, 64, size=(n, 3))
    for j in range(3):
        sel = rng.random(n) < 0.5
        words[sel, 0] ^= (np.uint64(1) << flips[sel, j].astype(np.uint64))
    words[5000:, 0] = rng.integers(0, 2**63, size=1000, dtype=np.int64).astype(np.uint64)
    pool = eg.BitStringPool(words, length).partitioned(8)
    for d in (1, 2):
        got = eg.enumerate_pairs(pool, d)
        want, _ = oracle.enumerate_pairs(words, length, pool.block_bounds, d)
        np.testing.assert_array_equal(got.array, want)


def test_medium_tier_bucket(eg, oracle):
    # one key group of ~3000 rows: bucket above the small tier (2048), inside
    # the medium tier (4096); plus background rows
    rng = np.random.default_rng(9)
    n = 5000
    base = np.uint64(int(rng.integers(0, 2**63)))
    words = np.full((n, 1), base, dtype=np.uint64)
    flip = rng.integers(0, 64, size=n).astype(np.uint64)
    sel = rng.random(n) < 0.7
    words[sel, 0] ^= np.uint64(1) << flip[sel]
    words[3000:, 0] = rng.integers(0, 2**63, size=n - 3000, dtype=np.int64).astype(np.uint64)
    pool = eg.BitStringPool(words, 64).partitioned(8)
    for d in (1, 2):
        got = eg.enumerate_pairs(pool, d)
        want, _ = oracle.enumerate_pairs(words, 64, pool.block_bounds, d)
        np.testing.assert_array_equal(got.array, want)


def test_hamming_builder_variants(eg, oracle):
    rng = np.random.default_rng(31)
    bits = (rng.random((200, 32)) < 0.5).astype(np.uint8)
    pool = eg.BitStringPool.from_bits(bits).partitioned(4)
    for d in (0, 1, 3):
        np.testing.assert_array_equal(eg.build_graph_hamming(pool, d).array,
                                      oracle.brute_force_hamming(pool.words, d))
    one = eg.BitStringPool.from_bits((rng.random((60, 16)) < 0.5).astype(np.uint8))
    np.testing.assert_array_equal(eg.build_graph_hamming(one, 2).array,
                                  oracle.brute_force_hamming(one.words, 2))
    assert len(eg.build_graph_hamming(one, 16)) == 60 * 59 // 2


# --------------------------------------------------------------- projection

def test_projection_bits_match_reference(eg, manifest):
    g = golden("projection")
    for case in manifest["projection"]:
        c = case["case"]
        pool = eg.project(g[f"x_{c}"], eg.ProjectionSpec(case["length"], case["seed"],
                                                          case["replicate_id"]))
        np.testing.assert_array_equal(pool.words, g[f"words_{c}"], err_msg=str(case))


def test_projection_vs_oracle_large(eg, oracle):
    from paper_0904_3151_b200 import workloads
    x = workloads.cfg3_points(30_000, planted_rows=3000)
    for rep in (1, 2):
        got = eg.project(x, eg.ProjectionSpec(48, 0, rep)).words
        want = oracle.project_words(x, 48, 0, rep)
        np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("simt", ["0", "1"])
def test_projection_fixup_overflow_path(eg, oracle, native_options, simt):
    """A tiny band-list capacity forces the overflow recompute (bitmap path on
    the tensor cores, full recompute on the SIMT path): codes still exact."""
    from paper_0904_3151_b200 import workloads
    native_options(fixup_cap=64, project_path=1 if simt == "1" else 0)
    x = workloads.cfg3_points(6_000, planted_rows=600)
    got = eg.project(x, eg.ProjectionSpec(48, 0, 1)).words
    np.testing.assert_array_equal(got, oracle.project_words(x, 48, 0, 1))


def test_projection_validation(eg):
    with pytest.raises(eg.DataError, match="row 1"):
        eg.project(np.array([[1.0, 1.0], [0.0, 0.0]], dtype=np.float32), eg.ProjectionSpec(8))
    with pytest.raises(eg.DataError, match="row 1"):
        eg.project(np.array([[1.0, 2.0], [np.nan, 0.0]], dtype=np.float32), eg.ProjectionSpec(8))
    with pytest.raises(eg.DataError):
        eg.project(np.zeros((0, 4), dtype=np.float32), eg.ProjectionSpec(8))


def test_sign_convention(eg):
    data = np.array([[1.0, 2.0], [-1.0, -2.0], [2.0, 4.0]], dtype=np.float32)
    bits = eg.project(data, eg.ProjectionSpec(length=96)).to_bits()
    assert np.all(bits[0] != bits[1])
    np.testing.assert_array_equal(bits[0], bits[2])


def test_long_projection(eg, oracle):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((7, 5))
    got = eg.project(x, eg.ProjectionSpec(length=3000, seed=4, replicate_id=2)).words
    np.testing.assert_array_equal(got, oracle.project_words(x, 3000, 4, 2))


# -------------------------------------------------------------------- build

def test_small_build_matches_reference(eg, manifest):
    g = golden("small_build")
    rec = manifest["small_build"]
    p = rec["params"]
    params = eg.MsmParams(epsilon=p["epsilon"], gamma=1e-3, length=p["length"],
                          mismatch=p["mismatch"], blocks=p["blocks"],
                          replicates=p["replicates"], seed=p["seed"])
    graph = eg.build_graph(g["x"], params)
    assert graph.stats.per_replicate_raw == tuple(rec["per_replicate_raw"])
    assert graph.stats.per_replicate_new == tuple(rec["per_replicate_new"])
    assert graph.stats.candidate_count == rec["candidate_count"]
    assert graph.stats.edge_count == rec["edge_count"]
    np.testing.assert_array_equal(graph.edge_list.pairs, g["edges"])
    np.testing.assert_allclose(graph.edge_list.distances, g["dist"], rtol=0, atol=DIST_TOL)
    assert abs(graph.stats.achieved_bound - rec["achieved_bound"]) <= 1e-12 * rec["achieved_bound"]
    again = eg.build_graph(g["x"], params, threads=3)
    assert again.edge_list == graph.edge_list      # bit-exact, per-pair deterministic


def test_dedup_and_filter_match_reference(eg):
    g = golden("small_build")
    pools = [eg.BitStringPool(g[f"codes_{h}"], 24).partitioned(4) for h in range(4)]
    raw = [eg.PairSet(g[f"raw_{h}"], assume_normalized=True) for h in range(4)]
    merged = eg.dedup_across_replicates(pools, raw, 2)
    np.testing.assert_array_equal(merged.pairs, g["merged"])
    edges = eg.filter_exact(g["x"], g["filter_cand"], 0.05)
    np.testing.assert_array_equal(edges.pairs, g["filter_edges"])
    np.testing.assert_allclose(edges.distances, g["filter_dist"], rtol=0, atol=DIST_TOL)
    with pytest.raises(IndexError):
        eg.filter_exact(g["x"], np.array([[0, 400]]), 0.1)


def test_lsh_only_matches_reference(eg, manifest):
    g = golden("small_build")
    graph = eg.build_graph_lsh_only(g["x"], 0.05, 1e-3, replicates=50)
    rec = manifest["small_build"]["lsh_only"]
    assert graph.params.length == rec["length"]
    assert graph.stats.candidate_count == rec["candidate_count"]
    np.testing.assert_array_equal(graph.edge_list.pairs, g["lsh_edges"])


def test_lsh_only_default_300_replicates(eg, oracle):
    """build_graph_lsh_only's default replicates=300 (pipeline.py:383-408;
    the reference's test_acceptance.py calls it so): replicate tags wider
    than 8 bits, counts and edges equal to the oracle's d=0, k=1 build."""
    g = golden("small_build")
    graph = eg.build_graph_lsh_only(g["x"], 0.05, 1e-3)
    assert graph.params.replicates == 300
    ref = oracle.build_graph(g["x"], 0.05, graph.params.length, 0, 1, 300, 0)
    assert graph.stats.per_replicate_raw == ref.per_replicate_raw
    assert graph.stats.per_replicate_new == ref.per_replicate_new
    np.testing.assert_array_equal(graph.edge_list.pairs, ref.pairs)


def test_bad_rows_rejected_before_enumeration(eg):
    """Many zero / NaN rows share the all-zero code: the DataError must come
    before the units run (no giant-group enumeration)."""
    import time
    params = eg.MsmParams(0.05, 1e-3, 32, 2, 8, 2, 0)
    x = np.random.default_rng(3).standard_normal((200_000, 16)).astype(np.float32)
    x[1000:150_000] = 0.0
    t0 = time.perf_counter()
    with pytest.raises(eg.DataError, match="row 1000 has zero norm"):
        eg.build_graph(x, params)
    x[1000:150_000] = np.nan
    with pytest.raises(eg.DataError, match="row 1000 has a non-finite entry"):
        eg.build_graph(x, params)
    assert time.perf_counter() - t0 < 30


def test_build_edge_cases(eg):
    params = eg.MsmParams(0.05, 1e-3, 24, 2, 4, 2, 7)
    with pytest.raises(eg.DataError):
        eg.build_graph(np.zeros((0, 4), dtype=np.float32), params)
    one = eg.build_graph(np.ones((1, 4), dtype=np.float32), params)
    assert one.edge_count == 0 and one.node_count == 1
    x = np.ones((5, 3), dtype=np.float32)
    x[3] = 0
    with pytest.raises(eg.DataError, match="row 3"):
        eg.build_graph(x, params)


@pytest.mark.parametrize("env", [{}, {"project_path": 3}, {"project_path": 1},
                                 {"fixup_force_seq": 1}, {"project_path": 2}])
def test_fused_norms_and_flags(eg, oracle, native_options, env):
    """eg_project_rows: norms accumulated inside the tensor-core projection
    are bit-identical to k_row_stats' (unfused and SIMT paths), codes equal
    the oracle's, and the bad-row flags give the reference's errors."""
    import torch
    from paper_0904_3151_b200 import engine, workloads
    native_options(**env)
    x = workloads.cfg3_points(5_000, planted_rows=500)
    xd = torch.from_numpy(x).cuda()
    codes, norms, bad, _ = engine.project_rows(xd, 48, 0, [1, 2])
    ref_norms, _ = engine.row_stats_async(xd)
    assert torch.equal(norms, ref_norms)
    np.testing.assert_allclose(norms.cpu().numpy(),
                               np.sqrt((x.astype(np.float64) ** 2).sum(axis=1)), rtol=1e-14)
    assert bad.cpu().tolist() == [-1, -1]
    got = codes.cpu().numpy().view(np.uint64)
    np.testing.assert_array_equal(got[0], oracle.project_words(x, 48, 0, 1))
    np.testing.assert_array_equal(got[1], oracle.project_words(x, 48, 0, 2))
    params = eg.MsmParams(0.05, 1e-3, 48, 3, 12, 2, 0)
    for bad_row, val in [(4321, np.nan), (777, 0.0), (130, np.inf)]:
        y = x.copy()
        y[bad_row] = val
        with pytest.raises(eg.DataError, match=f"row {bad_row}"):
            eg.build_graph(y, params)


def _config_build(eg, oracle, manifest, name, x, metric="cosine"):
    rec = manifest[name]
    p = rec["params"]
    eps = p["epsilon"]
    if metric == "euclidean":
        eps = float(np.sqrt(2.0 * eps))
    params = eg.MsmParams(epsilon=eps, gamma=1e-6, length=p["length"], mismatch=p["mismatch"],
                          blocks=p["blocks"], replicates=p["replicates"], seed=0)
    graph = eg.build_graph(x, params, metric=metric)
    assert graph.stats.per_replicate_raw == tuple(rec["per_replicate_raw"])
    assert graph.stats.per_replicate_new == tuple(rec["per_replicate_new"])
    assert graph.stats.candidate_count == rec["candidate_count"]
    if metric == "cosine":
        assert oracle.pair_digest(graph.edge_list.pairs) == rec["pairs_sha256"]
    else:
        ref = oracle.build_graph(x, p["epsilon"], p["length"], p["mismatch"], p["blocks"],
                                 p["replicates"], 0)
        # Euclidean on fp32-normalised rows agrees with the cosine route to
        # ~1e-7 (|x| = 1 only to fp32 precision): identical edge sets except
        # within the 1e-6 band, distances equal to 1e-6.
        d_cos = graph.edge_list.distances ** 2 / 2.0
        pairs_equal_except_band(graph.edge_list.pairs, d_cos, ref.pairs, ref.distances,
                                p["epsilon"], dist_tol=BAND)
    return graph


def test_cfg1_full(eg, oracle, manifest):
    from paper_0904_3151_b200 import workloads
    x = workloads.cfg1_points()
    graph = _config_build(eg, oracle, manifest, "cfg1", x)
    assert graph.edge_count == 809_648
    pool = eg.project(x, eg.ProjectionSpec(32, 0, 1))
    assert oracle.words_digest(pool.words) == manifest["cfg1"]["codes_sha256"][0]


def test_cfg2_small(eg, oracle, manifest):
    from paper_0904_3151_b200 import workloads
    words = workloads.cfg2_words(200_000, 10_000)
    got = eg.build_graph_hamming(eg.BitStringPool(words, 64).partitioned(8), 2)
    assert len(got) == manifest["cfg2_small"]["count"]
    assert oracle.pair_digest(got.array) == manifest["cfg2_small"]["pairs_sha256"]


def test_cfg3_small(eg, oracle, manifest):
    from paper_0904_3151_b200 import workloads
    _config_build(eg, oracle, manifest, "cfg3_small", workloads.cfg3_points(20_000))


def test_cfg4_small(eg, oracle, manifest):
    from paper_0904_3151_b200 import workloads
    _config_build(eg, oracle, manifest, "cfg4_small", workloads.cfg4_points(60_000, largest=2_000))


def test_cfg5_small_euclidean(eg, oracle, manifest):
    from paper_0904_3151_b200 import workloads
    _config_build(eg, oracle, manifest, "cfg5_small",
                  workloads.cfg5_points(40_000, clusters=2_000), metric="euclidean")


def _tc_tau(dim, tf32):
    """Relative band of the tensor-core projection (project_tc.cuh tc_tau,
    project_h16.cuh h16_tau)."""
    if tf32:
        mmas = 3.0 * ((dim + 7) // 8)
        return 2.0 * (mmas * 2.0 ** -22 + 3.0 * 2.0 ** -20) + dim * 2.0 ** -52
    mmas = 3.0 * ((dim + 15) // 16)
    return 2.0 * (mmas + 3.0) * 2.0 ** -22 + dim * 2.0 ** -52


@pytest.mark.parametrize("tf32", [False, True])
@pytest.mark.parametrize("n,dim,length,reps", [(20000, 384, 48, 3), (7000, 100, 64, 2),
                                               (5000, 128, 64, 1), (3000, 64, 32, 1)])
def test_tc_projection_error_band(eg, oracle, native_options, n, dim, length, reps, tf32):
    """The tensor-core projection's raw accumulator (kind::f16 2-term fp16
    splits by default, kind::tf32 3xTF32 with project_path=2) stays well
    inside the certified band it uses to decide signs; signs equal the
    oracle."""
    import torch
    from paper_0904_3151_b200 import _native, engine
    native_options(project_path=2 if tf32 else 0)
    rng = np.random.default_rng(n + dim)
    x = rng.standard_normal((n, dim)).astype(np.float32)
    x[: n // 4] = np.abs(x[: n // 4])          # skewed rows like config 3
    dev = torch.device("cuda", 0)
    xd = torch.from_numpy(x).to(dev)
    cols = length * reps
    dump = torch.zeros((n, cols), dtype=torch.float32, device=dev)
    lib = _native.lib()
    lib.eg_debug_set_tc_dump(dump.data_ptr())
    try:
        norms = engine.validate_rows(xd)
        codes, _ = engine.project_codes(xd, norms, length, 0, list(range(1, reps + 1)))
        torch.cuda.synchronize()
    finally:
        lib.eg_debug_set_tc_dump(None)
    acc = dump.cpu().numpy().astype(np.float64)
    r = np.concatenate([engine.directions(length, dim, 0, h) for h in range(1, reps + 1)])
    exact = x.astype(np.float64) @ r.T
    scale = np.linalg.norm(x.astype(np.float64), axis=1)[:, None] * np.linalg.norm(r, axis=1)[None, :]
    ratio = np.abs(acc - exact) / scale
    tau = _tc_tau(dim, tf32)
    print(f"tc band: max err/(|x||r|) = {ratio.max():.3e}, tau = {tau:.3e}, "
          f"in-band share = {np.mean(np.abs(exact) <= tau * scale):.2e}")
    assert ratio.max() < tau / 2, (ratio.max(), tau)
    for h in range(reps):
        want = oracle.project_words(x, length, 0, h + 1)
        np.testing.assert_array_equal(codes[h].cpu().numpy().view(np.uint64), want)


@pytest.mark.parametrize("env", [{"msm_streams": 1}, {"msm_streams": 1, "sort_path": 1}])
def test_msm_launch_variants(eg, oracle, manifest, native_options, env):
    """The single-stream schedule gives the same pair sets as the default
    two-stream overlap."""
    from paper_0904_3151_b200 import workloads
    native_options(**env)
    words = workloads.cfg2_words(200_000, 10_000)
    got = eg.build_graph_hamming(eg.BitStringPool(words, 64).partitioned(8), 2)
    assert oracle.pair_digest(got.array) == manifest["cfg2_small"]["pairs_sha256"]
    g = golden("random_pools")
    for case in manifest["random_pools"][:16]:
        c = case["case"]
        pool = eg.BitStringPool(g[f"words_{c}"], case["length"]).partitioned(case["k"])
        np.testing.assert_array_equal(eg.enumerate_pairs(pool, case["d"]).array, g[f"pairs_{c}"])


def test_sharded_path_over_nccl_single_rank(eg, oracle):
    """The multi-GPU code path (row-sharded projection, NCCL all-gathers of
    codes/norms, unit ownership, edge gather + device merge) on one rank."""
    import socket
    import torch
    import torch.distributed as tdist
    from paper_0904_3151_b200 import distributed, workloads
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                             world_size=1, device_id=torch.device("cuda", 0))
    try:
        x = workloads.cfg1_points(6000, clusters=60)
        params = eg.MsmParams(0.1, 1e-6, 32, 2, 8, 2, 0)
        res = distributed.build_step(torch.from_numpy(x).cuda(), params, "cosine", 1, 0,
                                     force_dist=True)
        ref = oracle.build_graph(x, 0.1, 32, 2, 8, 2, 0)
        from paper_0904_3151_b200 import engine
        pairs = engine.keys_to_pairs(res["keys"].cpu().numpy())
        np.testing.assert_array_equal(pairs, ref.pairs)
        np.testing.assert_allclose(res["dist"].cpu().numpy(), ref.distances, rtol=0, atol=1e-12)
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("blocks", [4, 5, 7, 9, 16, 48, 10604, 10804, 11105, 11106, 11406])
def test_forced_block_counts_same_pairs(eg, oracle, manifest, native_options, blocks):
    """The pair set does not depend on the units' partition
    (hamming_join.py:300-375): every forced k' > d -- and every covering
    design of the library's table (plan codes 10000 + 100 v + m, first-member
    ownership) -- reproduces the reference-k pairs, per-replicate raw/new
    counts and edges."""
    native_options(msm_blocks=blocks)
    rng = np.random.default_rng(blocks)
    n, length, k, d = 5000, 48, 12, 3
    base = (rng.random((n // 3, length)) < 0.3).astype(np.uint8)
    bits = base[rng.integers(0, base.shape[0], n)] ^ (rng.random((n, length)) < 0.02)
    words = pack_bits(bits.astype(np.uint8))
    pool = eg.BitStringPool(words, length).partitioned(k)
    got = eg.enumerate_pairs(pool, d)
    want, _ = oracle.enumerate_pairs(words, length, pool.block_bounds, d)
    np.testing.assert_array_equal(got.array, want)
    g = golden("small_build")
    rec = manifest["small_build"]
    pp = rec["params"]
    v = blocks if blocks < 10000 else (blocks - 10000) // 100
    if pp["mismatch"] < v <= pp["length"]:
        params = eg.MsmParams(epsilon=pp["epsilon"], gamma=1e-3, length=pp["length"],
                              mismatch=pp["mismatch"], blocks=pp["blocks"],
                              replicates=pp["replicates"], seed=pp["seed"])
        graph = eg.build_graph(g["x"], params)
        np.testing.assert_array_equal(graph.edge_list.pairs, g["edges"])
        assert graph.stats.per_replicate_raw == tuple(rec["per_replicate_raw"])
        assert graph.stats.per_replicate_new == tuple(rec["per_replicate_new"])
        assert graph.stats.candidate_count == rec["candidate_count"]


def test_block_plan_auto_large_pool(eg, oracle):
    """Auto plan on a pool above the planning threshold (skewed bits, planted
    near-duplicates): whatever k' the plan picks, pairs equal the oracle's."""
    from paper_0904_3151_b200 import engine
    rng = np.random.default_rng(11)
    n, length, k, d = 120_000, 48, 12, 3
    p1 = rng.uniform(0.05, 0.95, length)
    bits = (rng.random((n, length)) < p1).astype(np.uint8)
    src = rng.integers(0, n, n // 20)
    dst = rng.integers(0, n, n // 20)
    bits[dst] = bits[src] ^ (rng.random((len(src), length)) < 0.03)
    words = pack_bits(bits)
    pool = eg.BitStringPool(words, length).partitioned(k)
    got = eg.enumerate_pairs(pool, d)
    assert engine._last_plan["chosen"] > d
    want, _ = oracle.enumerate_pairs(words, length, pool.block_bounds, d)
    np.testing.assert_array_equal(got.array, want)


def test_block_plan_keeps_reference_when_oversized(eg, caplog):
    """Where the reference would warn about an oversized group, the plan
    keeps the reference blocks, so the warning (and max_group) match."""
    from paper_0904_3151_b200 import engine
    rng = np.random.default_rng(5)
    n, length = 70_000, 32
    bits = (rng.random((n, length)) < 0.5).astype(np.uint8)
    bits[: n // 3] = bits[0]                   # a third of the rows identical
    pool = eg.BitStringPool(pack_bits(bits), length).partitioned(8)
    with caplog.at_level(logging.WARNING, logger="paper_0904_3151_b200"):
        codes_pairs = eg.enumerate_pairs(pool, 1)
    assert engine._last_plan.get("chosen", 8) == 8
    assert any("group" in r.message for r in caplog.records)
    assert len(codes_pairs) >= (n // 3) * (n // 3 - 1) // 2


@pytest.mark.parametrize("plan,length,d", [(10703, 100, 2), (10905, 100, 2), (11304, 64, 2),
                                           (10906, 130, 4), (11207, 64, 4)])
def test_design_units_wide_codes(eg, oracle, native_options, plan, length, d):
    """Covering-design units on 2- and 3-word codes and for d = 2 and 4."""
    native_options(msm_blocks=plan)
    rng = np.random.default_rng(plan)
    n = 6000
    base = (rng.random((n // 4, length)) < 0.4).astype(np.uint8)
    bits = base[rng.integers(0, base.shape[0], n)] ^ (rng.random((n, length)) < 0.012)
    words = pack_bits(bits.astype(np.uint8))
    pool = eg.BitStringPool(words, length).partitioned(8)
    got = eg.enumerate_pairs(pool, d)
    want, _ = oracle.enumerate_pairs(words, length, pool.block_bounds, d)
    assert len(want) > 1000
    np.testing.assert_array_equal(got.array, want)


@pytest.mark.parametrize("blocks", [4, 5, 6, 10604, 10705])
def test_coarse_blocks_all_tiers_deterministic(eg, oracle, native_options, blocks):
    """Coarse forced block counts on skewed bits send buckets through every
    tier (small, pair-heavy -> medium, giant -> tiles); the pair set must
    equal the oracle's and be identical run to run."""
    native_options(msm_blocks=blocks)
    rng = np.random.default_rng(blocks + 100)
    n, length, k, d = 50_000, 48, 12, 3
    bits = (rng.random((n, length)) < 0.8).astype(np.uint8)
    words = pack_bits(bits)
    pool = eg.BitStringPool(words, length).partitioned(k)
    first = eg.enumerate_pairs(pool, d).array
    again = eg.enumerate_pairs(pool, d).array
    np.testing.assert_array_equal(first, again)
    want, _ = oracle.enumerate_pairs(words, length, pool.block_bounds, d)
    np.testing.assert_array_equal(first, want)


@pytest.mark.parametrize("tf32", ["0", "1"])
def test_projection_extreme_magnitudes(eg, oracle, native_options, tf32):
    """Rows outside the fp16 range of the kind::f16 split: entries >= 2^15
    (the row goes to the exact fix-up whole), rows of tiny magnitude (fp16
    subnormals: the absolute floor of the band) and mixed-scale rows --
    codes still bit-exact with the oracle."""
    native_options(project_path=2 if tf32 == "1" else 0)
    rng = np.random.default_rng(7)
    x = rng.standard_normal((4000, 96)).astype(np.float32)
    x[:500] *= np.float32(1e5)                         # fp16 overflow
    x[500:1000] *= np.float32(1e-6)                    # fp16 subnormal range
    x[1000:1500, ::3] *= np.float32(3e4)               # mixed scales
    x[1500:1600] = np.abs(x[1500:1600]) * np.float32(1e-30)
    for rep in (1, 2):
        got = eg.project(x, eg.ProjectionSpec(64, 3, rep)).words
        np.testing.assert_array_equal(got, oracle.project_words(x, 64, 3, rep))


@pytest.mark.parametrize("classic", ["0", "1"])
def test_radix_sort_kernels(eg, native_options, classic):
    """Onesweep (decoupled look-back) and classic LSD passes: pair-key sort
    and key-value sort equal numpy's stable sort on ragged sizes, including
    skewed digits (long look-back chains) and keys with equal halves."""
    import torch
    from paper_0904_3151_b200 import engine
    native_options(sort_path=int(classic))
    rng = np.random.default_rng(3)
    dev = torch.device("cuda", 0)
    for m in (1, 2, 2047, 2048, 2049, 100_003, 1_500_000):
        n = 1 << 21
        i = rng.integers(0, n, m)
        j = rng.integers(0, n, m)
        if m > 1000:
            i[: m // 3] = 7                     # one digit value dominates
        keys = (i.astype(np.int64) << 32) | j
        t = torch.from_numpy(keys.copy()).to(dev)
        engine.sort_pair_keys(t, n)
        np.testing.assert_array_equal(t.cpu().numpy(), np.sort(keys))
        vals = torch.arange(m, dtype=torch.int32, device=dev)
        t = torch.from_numpy(keys.copy()).to(dev)
        engine.sort_keys(t, 64, vals)
        order = np.argsort(keys, kind="stable")
        np.testing.assert_array_equal(t.cpu().numpy(), keys[order])
        np.testing.assert_array_equal(vals.cpu().numpy(), order.astype(np.int32))


# --------------------------------------------------------------- boundary

@pytest.mark.parametrize("plan", [0, 10804])
def test_build_graph_devices_invariance(eg, native_options, plan):
    """build_graph(devices=...) shards the units over the listed devices
    (one process); the edge list is bit-identical for any device list
    (mirror of the reference's thread-count contract,
    tests/test_pipeline.py:130-135).  A repeated device runs its shards one
    after another, which exercises the sharded path on one GPU.  plan =
    10804: the units of the covering design C(8,4,3), dealt over the shards."""
    import torch
    from paper_0904_3151_b200 import workloads
    if plan:
        native_options(msm_blocks=plan)
    x = workloads.cfg3_points(30_000, planted_rows=3_000)
    params = eg.MsmParams(0.05, 1e-6, 48, 3, 12, 3, 0)
    one = eg.build_graph(x, params)
    lists = [[0, 0], [0, 0, 0]]
    if torch.cuda.device_count() > 1:
        lists.append(torch.cuda.device_count())
    for devs in lists:
        many = eg.build_graph(x, params, devices=devs)
        assert many.edge_list == one.edge_list, devs
        assert many.stats.per_replicate_raw == one.stats.per_replicate_raw
        assert many.stats.per_replicate_new == one.stats.per_replicate_new
        assert many.stats.candidate_count == one.stats.candidate_count
    bad = x.copy()
    bad[20_001] = 0.0
    with pytest.raises(eg.DataError, match="row 20001 has zero norm"):
        eg.build_graph(bad, params, devices=[0, 0, 0])


@pytest.mark.parametrize("length,k,d", [(300, 10, 2), (257, 70, 1), (200, 100, 2), (520, 8, 3)])
def test_long_strings_and_many_blocks(eg, oracle, length, k, d):
    """No length / block-count caps: strings longer than the kernels' 256
    bits run on their first 256 bits and are filtered by the full codes,
    k > 64 runs with at most 64 blocks; pair sets equal the oracle's
    enumerate_pairs at the reference k (hamming_join.py:300-375)."""
    rng = np.random.default_rng(length + k)
    n = 3000
    base = (rng.random((n // 4, length)) < 0.5).astype(np.uint8)
    bits = base[rng.integers(0, base.shape[0], n)]
    flips = rng.random((n, length)) < (1.5 / length)
    bits = bits ^ flips.astype(np.uint8)
    words = pack_bits(bits)
    pool = eg.BitStringPool(words, length).partitioned(k)
    got = eg.enumerate_pairs(pool, d).array
    want, _ = oracle.enumerate_pairs(words, length, pool.block_bounds, d)
    np.testing.assert_array_equal(got, want)
    assert got.shape[0] > n // 4


def test_lsh_only_long_strings(eg, oracle):
    """build_graph_lsh_only at a small epsilon picks a length above 256 bits
    (pipeline.py:357-408); the build equals the oracle's."""
    from paper_0904_3151_b200 import workloads
    x = workloads.cfg1_points(1_000, clusters=10)
    g = eg.build_graph_lsh_only(x, 0.001, 1e-3)
    assert g.params.length > 256 and g.params.replicates == 300
    ref = oracle.build_graph(x, 0.001, g.params.length, 0, 1, 300, 0)
    assert g.stats.per_replicate_raw == ref.per_replicate_raw
    assert g.stats.per_replicate_new == ref.per_replicate_new
    np.testing.assert_array_equal(g.edge_list.pairs, ref.pairs)


def test_output_estimate_sizes_cold_calls(eg):
    """The sampled output estimate (eg_msm_estimate_pairs) bounds the MSM
    output of a cold call, so the capacity is right the first time (no
    rerun of the units)."""
    import torch
    from paper_0904_3151_b200 import engine, workloads
    engine._capacity_hint.clear()
    x = workloads.cfg5_points(300_000, clusters=15_000)
    params = eg.MsmParams(0.15, 1e-6, 64, 3, 16, 2, 0)
    out = eg.build_graph_device(torch.from_numpy(x).cuda(), params, metric="euclidean")
    info = out["info"]
    assert info["reruns"] == 0
    est, hi = engine.estimate_pairs(out["codes"], 3)
    raw = sum(info["raw"])
    assert 0.5 * raw <= est <= 2.0 * raw
    assert hi >= raw


@pytest.mark.parametrize("runs", [1, 2, 3, 8, 13])
def test_merge_runs_kernel(eg, runs):
    """eg_merge_runs (merge path): sorted runs of ragged sizes (some empty)
    with payloads -> one sorted run, payloads following their keys."""
    import torch
    from paper_0904_3151_b200.distributed import DeviceOps
    rng = np.random.default_rng(runs)
    sizes = rng.integers(0, 50_000, runs)
    sizes[0] = 0 if runs > 2 else sizes[0]
    allk = rng.choice(1 << 40, int(sizes.sum()), replace=False).astype(np.int64)
    parts, offs = [], [0]
    for r, sz in enumerate(sizes):
        parts.append(np.sort(allk[offs[-1]:offs[-1] + sz]))
        offs.append(offs[-1] + int(sz))
    keys = np.concatenate(parts) if parts else np.empty(0, np.int64)
    dist = (keys.astype(np.float64) * 0.5)
    k, d = DeviceOps().merge_runs(torch.from_numpy(keys).cuda(), torch.from_numpy(dist).cuda(),
                                  offs)
    order = np.argsort(keys, kind="stable")
    np.testing.assert_array_equal(k.cpu().numpy(), keys[order])
    np.testing.assert_array_equal(d.cpu().numpy(), dist[order])
