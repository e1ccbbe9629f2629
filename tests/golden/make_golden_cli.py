"""CLI fixtures made by running the REFERENCE command line (cli.py) itself.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_cli.py

Writes tests/golden/cli/: the dataset file, and cli.json with each
command's JSON record (timings dropped) and the sha256 of the edge files it
wrote; plus auto_params cases (tuning.py:232-297) for the host tests.
"""
import contextlib
import hashlib
import io
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import epsgraph as ref  # noqa: E402
from epsgraph import cli as refcli  # noqa: E402

from paper_0904_3151_b200 import workloads  # noqa: E402

OUT = os.path.join(HERE, "cli")


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = refcli.main(argv)
    rec = json.loads(buf.getvalue()) if buf.getvalue().strip() else None
    if rec and "stats" in rec:
        rec["stats"].pop("timings", None)
    if rec and "rows" in rec:
        for r in rec["rows"]:
            r.pop("seconds", None)
            r.pop("seconds_per_10k_pairs", None)
            r.pop("stages", None)
    return rc, rec


def sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def main():
    os.makedirs(OUT, exist_ok=True)
    x = workloads.cfg1_points(3000, clusters=30)
    data = os.path.join(OUT, "cfg1_3000.epgd")
    ref.write_dataset(data, x)
    bad = x.copy()
    bad[17, 3] = float("nan")
    badp = os.path.join(OUT, "bad.csv")
    import numpy as np
    np.savetxt(badp, bad[:40], delimiter=",")
    cases = {}
    with tempfile.TemporaryDirectory() as td:
        e = os.path.join(td, "e.txt")
        for name, argv in {
            "build_overrides": ["build", data, "-o", e, "--epsilon", "0.1", "--length", "32",
                                "--mismatch", "2", "--blocks", "8", "--replicates", "2"],
            "build_auto": ["build", data, "-o", e, "--epsilon", "0.1"],
            "build_partial": ["build", data, "-o", e, "--epsilon", "0.1", "--length", "24"],
            "build_lsh_only": ["build", data, "-o", e, "--epsilon", "0.05", "--lsh-only"],
            "build_normalize": ["build", data, "-o", e, "--epsilon", "0.1", "--normalize",
                                "--length", "32", "--mismatch", "2", "--blocks", "8",
                                "--replicates", "1"],
        }.items():
            rc, rec = run(argv)
            cases[name] = {"argv": argv[2:3] and argv, "rc": rc, "record": rec,
                           "edges_sha256": sha(e)}
        rc, rec = run(["estimate", data, "--epsilon", "0.1"])
        cases["estimate"] = {"rc": rc, "record": rec}
        rc, rec = run(["bench", data, "--epsilon-list", "0.1", "--sizes", "1000,3000"])
        cases["bench"] = {"rc": rc, "record": rec}
        rc, _ = run(["build", badp, "-o", e, "--epsilon", "0.1"])
        cases["bad_data"] = {"rc": rc}
        rc, _ = run(["build", data, "-o", e, "--epsilon", "0.1", "--lsh-only", "--length", "8"])
        cases["conflict"] = {"rc": rc}
    auto = []
    for n, eps, gamma, est in [(20_000, 0.1, 1e-6, None), (1_600_000, 0.05, 1e-6, None),
                               (4_000_000, 0.08, 1e-3, (1.0e9, 0.9e9, 1.1e9)),
                               (500, 0.3, 1e-2, (2.0, 0.0, 3.0)), (10, 0.01, 0.5, None),
                               (100_000, 0.02, 1e-4, (5e5, 4e5, 6e5))]:
        e_obj = None
        if est is not None:
            e_obj = ref.tuning.OutputEstimate(sampled_pairs=1000, hits=10,
                                              total_pairs=n * (n - 1) // 2, estimate_s=est[0],
                                              ci_low=est[1], ci_high=est[2])
        try:
            p, r = ref.tuning.auto_params_detailed(n, eps, gamma, e_obj)
            auto.append({"n": n, "eps": eps, "gamma": gamma, "est": est,
                         "params": [p.length, p.mismatch, p.blocks, p.replicates],
                         "report": [r.collision_p, r.initial_length, r.halved, r.q_gamma,
                                    r.replicate_cap, r.cap_applied, r.achieved_bound]})
        except ref.InfeasibleError:
            auto.append({"n": n, "eps": eps, "gamma": gamma, "est": est, "infeasible": True})
    with open(os.path.join(OUT, "cli.json"), "w") as f:
        json.dump({"cases": cases, "auto_params": auto}, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
