"""Host-side logic and the C ABI surface (no GPU needed)."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

import paper_0904_3151_b200 as eg
from paper_0904_3151_b200 import _native, engine


def header_symbols():
    with open(os.path.join(ROOT, "include", "epsgraph_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(eg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    _native.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert _native.lib().eg_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    params = eg.MsmParams(0.1, 1e-3, 16, 1, 4, 1)
    with pytest.raises(RuntimeError, match="CUDA"):
        eg.build_graph(np.random.rand(10, 4).astype(np.float32), params)
    pool = eg.BitStringPool.from_bits(np.zeros((4, 8), np.uint8)).partitioned(2)
    with pytest.raises(RuntimeError, match="CUDA"):
        eg.enumerate_pairs(pool, 1)


def test_block_partition_kats():
    assert eg.block_partition(16, 4).tolist() == [0, 4, 8, 12, 16]
    assert eg.block_partition(10, 3).tolist() == [0, 4, 7, 10]
    assert eg.block_partition(7, 7).tolist() == list(range(8))
    assert eg.block_partition(5, 1).tolist() == [0, 5]
    with pytest.raises(ValueError):
        eg.block_partition(3, 4)


def test_bit_layout_kat():
    bits = np.zeros((1, 130), dtype=np.uint8)
    bits[0, [0, 63, 64, 129]] = 1
    w = eg.BitStringPool.from_bits(bits).words[0]
    assert int(w[0]) == (1 | (1 << 63)) and int(w[1]) == 1 and int(w[2]) == 2


def test_kept_word_mask_kat():
    bounds = eg.block_partition(16, 4)
    assert int(eg.kept_word_mask(16, bounds, (1,))[0]) == 0xFF0F
    assert int(eg.kept_word_mask(16, bounds, ())[0]) == 0xFFFF


def test_units_are_lexicographic_masks():
    reps, bits = engine.units_for([0, 1], 4, 2)
    masks = [tuple(b for b in range(4) if int(m) >> b & 1) for m in bits[:6]]
    assert masks == [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
    assert reps.tolist() == [0] * 6 + [1] * 6


def test_canonical_mask_rule_matches_first_witness():
    """The O(1) rule in msm.cuh (lexicographically first d-subset containing
    the differing blocks) equals the reference's first-collision search over
    masks in combination order (hamming_join.py:130-141)."""
    import itertools
    rng = np.random.default_rng(0)
    for k, d in [(4, 2), (8, 2), (12, 3), (16, 3), (6, 0), (5, 4)]:
        masks = list(itertools.combinations(range(k), d))
        for _ in range(200):
            nd = int(rng.integers(0, d + 1))
            delta = set(rng.choice(k, nd, replace=False).tolist())
            first = next(m for m in masks if delta <= set(m))
            fill = [b for b in range(k) if b not in delta][:d - nd]
            assert tuple(sorted(delta | set(fill))) == first


def test_design_table_covers_every_subset():
    """Every covering design of the library's table (eg_msm_design): members
    mask m of the v blocks, and every t-subset of the blocks lies inside a
    member -- so every pair differing in <= t blocks shares a masked key in
    some unit, and the first such member owns it exactly once."""
    import itertools
    found = 0
    for t in (2, 3, 4):
        for v in range(t + 2, 17):
            for m in range(t + 1, v):
                try:
                    vv, fam, is_design = engine.plan_design(engine.DESIGN_BASE + 100 * v + m, t)
                except ValueError:
                    continue
                found += 1
                fam = [int(f) for f in fam]
                assert vv == v and is_design and len(fam) == engine.unit_count(
                    engine.DESIGN_BASE + 100 * v + m, t)
                assert len(fam) < len(list(itertools.combinations(range(v), t)))
                assert all(bin(f).count("1") == m and f < (1 << v) for f in fam)
                for c in itertools.combinations(range(v), t):
                    s = sum(1 << b for b in c)
                    owners = [q for q, f in enumerate(fam) if f & s == s]
                    assert owners, (v, m, t, c)
    assert found >= 20
    reps, bits = engine.units_for([0, 1], engine.DESIGN_BASE + 804, 3)
    assert len(bits) == 28 and reps.tolist() == [0] * 14 + [1] * 14
    assert (bits[:14] == bits[14:]).all()


def test_pair_key_round_trip():
    pairs = np.array([[0, 1], [5, 9], [2**31, 2**32 - 1]], dtype=np.int64)
    np.testing.assert_array_equal(engine.keys_to_pairs(engine.pairs_to_keys(pairs)), pairs)


def test_pairset_and_edgelist():
    ps = eg.PairSet([(5, 2), (2, 5), (1, 3)])
    assert ps.array.tolist() == [[1, 3], [2, 5]]
    assert (5, 2) in ps and (1, 2) not in ps
    with pytest.raises(ValueError):
        eg.PairSet([(3, 3)])
    e = eg.EdgeList.from_rows([(3, 4, 0.5), (1, 2, 0.25)])
    assert e.pairs.tolist() == [[1, 2], [3, 4]]
    assert e == eg.EdgeList(np.array([[1, 2], [3, 4]]), np.array([0.25, 0.5]))


def test_params_validation():
    with pytest.raises(ValueError):
        eg.MsmParams(1.5, 0.1, 16, 1, 4, 1)
    with pytest.raises(ValueError):
        eg.MsmParams(0.1, 0.0, 16, 1, 4, 1)
    with pytest.raises(ValueError):
        eg.MsmParams(0.1, 0.1, 16, 4, 4, 1)
    with pytest.raises(ValueError):
        eg.MsmParams(0.1, 0.1, 16, 1, 4, 0)


def test_achieved_bound_matches_reference(manifest):
    for name in ("small_build", "cfg1", "cfg3_small", "cfg4_small"):
        rec = manifest[name]
        p = rec["params"]
        got = eg.missing_edge_bound(p["length"], p["mismatch"], eg.collision_prob(p["epsilon"]),
                                    p["replicates"])
        assert math.isclose(got, rec["achieved_bound"], rel_tol=1e-12)


def test_min_replicates_ladder():
    # reference tests/test_tuning.py:118-122 known answers
    assert [eg.min_replicates(50, d, 0.1, 1e-6) for d in range(8)] == \
        [2674, 402, 117, 48, 25, 15, 10, 7]


def test_dataset_validation_host():
    with pytest.raises(eg.DataError, match="row 1"):
        eg.VectorDataset(np.array([[1.0, 2.0], [np.nan, 0.0]], dtype=np.float32))
    with pytest.raises(eg.DataError):
        eg.VectorDataset(np.zeros(4))


def test_workload_generators_shapes():
    from paper_0904_3151_b200 import workloads
    assert workloads.cfg1_points(100).shape == (100, 64)
    w = workloads.cfg2_words(1000, 50)
    assert w.shape == (1050, 1) and w.dtype == np.uint64
    x = workloads.cfg3_points(1000)
    assert x.shape == (1000, 384) and x.dtype == np.float32
    np.testing.assert_allclose(np.linalg.norm(x, axis=1), 1.0, rtol=1e-5)


def test_library_reads_no_environment():
    """Path choices come from eg_set_option only: no product source reads
    the environment (the statically linked CUDA runtime's own getenv aside)."""
    for path in _native.sources():
        with open(path) as f:
            assert "getenv" not in f.read(), path


def test_options_api_validates_names():
    lib = _native.lib()
    assert lib.eg_set_option(b"no_such_option", 1) == _native.EG_ERR_ARG
    assert lib.eg_set_option(b"project_path", 9) == _native.EG_ERR_ARG
    assert lib.eg_set_option(b"msm_streams", 1) == _native.EG_OK
    lib.eg_reset_options()
    with _native.options(sort_path=1):
        pass
    import pytest
    with pytest.raises(ValueError):
        with _native.options(bogus=1):
            pass
