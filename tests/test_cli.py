"""CLI (reference cli.py) and auto_params (tuning.py:232-297) against the
reference's own outputs (tests/golden/make_golden_cli.py)."""

import contextlib
import hashlib
import io
import json
import os

import pytest

from conftest import GOLDEN

CLI = os.path.join(GOLDEN, "cli")


@pytest.fixture(scope="module")
def fx():
    with open(os.path.join(CLI, "cli.json")) as f:
        return json.load(f)


def run(argv):
    from paper_0904_3151_b200 import cli
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    out = buf.getvalue().strip()
    return rc, (json.loads(out) if out else None)


def test_auto_params_match_reference(fx):
    from paper_0904_3151_b200 import tuning
    for case in fx["auto_params"]:
        est = None
        if case["est"] is not None:
            s, lo, hi = case["est"]
            n = case["n"]
            est = tuning.OutputEstimate(1000, 10, n * (n - 1) // 2, s, lo, hi)
        if case.get("infeasible"):
            with pytest.raises(tuning.InfeasibleError):
                tuning.auto_params_detailed(case["n"], case["eps"], case["gamma"], est)
            continue
        p, r = tuning.auto_params_detailed(case["n"], case["eps"], case["gamma"], est)
        assert [p.length, p.mismatch, p.blocks, p.replicates] == case["params"], case
        got = [r.collision_p, r.initial_length, r.halved, r.q_gamma, r.replicate_cap,
               r.cap_applied, r.achieved_bound]
        assert got[1:6] == case["report"][1:6]
        assert got[0] == pytest.approx(case["report"][0], rel=1e-15)
        assert got[6] == case["report"][6]      # bit-identical (edge-file metadata)


def test_usage_errors_exit_1(tmp_path):
    assert run([])[0] == 1
    assert run(["build"])[0] == 1
    assert run(["bench", "x", "--epsilon-list", "a,b", "--sizes", "1"])[0] == 1
    data = os.path.join(CLI, "cfg1_3000.epgd")
    rc, _ = run(["build", data, "-o", str(tmp_path / "e.txt"), "--epsilon", "0.1",
                 "--lsh-only", "--length", "8"])
    assert rc == 1
    rc, _ = run(["bench", data, "--epsilon-list", "0.1", "--sizes", "1"])
    assert rc == 1
    rc, _ = run(["bench", data, "--epsilon-list", "0.1", "--sizes", "10,99999"])
    assert rc == 1


def test_missing_file_is_data_error(tmp_path):
    assert run(["build", str(tmp_path / "nope.epgd"), "-o", str(tmp_path / "e"),
                "--epsilon", "0.1"])[0] == 2


def _sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["build_overrides", "build_auto", "build_partial",
                                  "build_lsh_only", "build_normalize"])
def test_build_command_matches_reference(fx, tmp_path, name):
    """Same JSON record (minus timings) and byte-identical edge file as the
    reference's `epsgraph build`, through the GPU build."""
    case = fx["cases"][name]
    argv = list(case["argv"])
    out = str(tmp_path / "e.txt")
    argv[argv.index("-o") + 1] = out
    argv[1] = os.path.join(CLI, "cfg1_3000.epgd")
    rc, rec = run(argv)
    assert rc == case["rc"] == 0
    rec["stats"].pop("timings")
    want = case["record"]
    for key in ("input", "output"):
        rec.pop(key), want.pop(key)
    assert rec == want
    assert _sha(out) == case["edges_sha256"]


@pytest.mark.gpu
def test_build_devices_flag_same_bytes(fx, tmp_path):
    case = fx["cases"]["build_overrides"]
    argv = list(case["argv"])
    out = str(tmp_path / "e.txt")
    argv[argv.index("-o") + 1] = out
    argv[1] = os.path.join(CLI, "cfg1_3000.epgd")
    rc, _ = run(argv + ["--devices", "0,0"])
    assert rc == 0
    assert _sha(out) == case["edges_sha256"]


@pytest.mark.gpu
def test_estimate_bench_and_errors(fx, tmp_path):
    data = os.path.join(CLI, "cfg1_3000.epgd")
    rc, rec = run(["estimate", data, "--epsilon", "0.1"])
    want = fx["cases"]["estimate"]["record"]
    rec.pop("input"), want.pop("input")
    assert rc == 0 and rec == want
    rc, rec = run(["bench", data, "--epsilon-list", "0.1", "--sizes", "1000,3000"])
    assert rc == 0
    for r, w in zip(rec["rows"], fx["cases"]["bench"]["record"]["rows"]):
        assert {k: r[k] for k in ("size", "epsilon", "params", "edges", "candidates")} == \
            {k: w[k] for k in ("size", "epsilon", "params", "edges", "candidates")}
    rc, _ = run(["build", os.path.join(CLI, "bad.csv"), "-o", str(tmp_path / "e"),
                 "--epsilon", "0.1"])
    assert rc == fx["cases"]["bad_data"]["rc"] == 2
