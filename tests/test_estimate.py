"""Output-size estimate (reference tuning.py:175-229) against the
reference's own results on seeded inputs (manifest "estimate", made by
make_golden.py)."""

import numpy as np
import pytest


def _inputs(name):
    from paper_0904_3151_b200 import workloads
    return {"cfg1": lambda: workloads.cfg1_points(5_000, clusters=50),
            "cfg3": lambda: workloads.cfg3_points(20_000, planted_rows=4_000),
            "tiny": lambda: workloads.cfg1_points(40, clusters=2)}[name]()


@pytest.mark.parametrize("name", ["cfg1", "cfg3", "tiny"])
def test_wilson_interval_matches_reference(manifest, name):
    from paper_0904_3151_b200.tuning import wilson_interval
    g = manifest["estimate"][name]
    lo, hi = wilson_interval(g["hits"], g["sample_pairs"])
    assert [lo * g["total_pairs"], hi * g["total_pairs"]] == pytest.approx(g["ci"], rel=1e-12)


def test_estimate_argument_checks():
    from paper_0904_3151_b200 import estimate_output_size
    with pytest.raises(ValueError, match="two vectors"):
        estimate_output_size(np.ones((1, 3), np.float32), 0.1)
    with pytest.raises(ValueError, match="sample_pairs"):
        estimate_output_size(np.ones((4, 3), np.float32), 0.1, sample_pairs=0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg1", "cfg3", "tiny"])
def test_estimate_output_size_matches_reference(manifest, name):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_0904_3151_b200 as eg
    g = manifest["estimate"][name]
    e = eg.estimate_output_size(_inputs(name), g["eps"], sample_pairs=g["sample_pairs"],
                                seed=g["seed"])
    assert (e.hits, e.total_pairs, e.sampled_pairs) == (g["hits"], g["total_pairs"],
                                                        g["sample_pairs"])
    assert e.estimate_s == pytest.approx(g["estimate_s"], rel=1e-12)
    assert [e.ci_low, e.ci_high] == pytest.approx(g["ci"], rel=1e-12)
