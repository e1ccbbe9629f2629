"""Multi-rank host logic over gloo (world_size 2, CPU).

The per-rank compute is stubbed with the CPU oracle (test infrastructure);
what is under test is paper_0904_3151_b200.distributed: row sharding of the
projection, the all-gather of codes and norms, cyclic (replicate, mask) unit
ownership with disjoint outputs, and the gather + merge of per-rank sorted
edge runs on rank 0.  The result must equal the single-process oracle build.
"""

import itertools
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleOps:
    """CPU stand-ins for DeviceOps, built on the oracle."""

    def __init__(self, orc, x_full, blocks=None):
        self.orc = orc
        self.x = np.asarray(x_full)
        self.blocks = blocks

    def norms(self, xs):
        return torch.from_numpy(np.sqrt((xs.numpy().astype(np.float64) ** 2).sum(axis=1)))

    def project(self, xs, norms, params):
        codes = [self.orc.project_words(xs.numpy(), params.length, params.seed, h + 1)
                 for h in range(params.replicates)]
        return torch.from_numpy(np.stack(codes).view(np.int64))

    def project_rows(self, xs, params):
        """Fused stage of DeviceOps: codes, norms, (non-finite, zero) flags."""
        v = xs.numpy().astype(np.float64)
        ss = (v ** 2).sum(axis=1)
        nonfin = np.flatnonzero(~np.isfinite(ss))
        zero = np.flatnonzero(ss == 0.0)
        bad = torch.tensor([int(nonfin[0]) if nonfin.size else -1,
                            int(zero[0]) if zero.size else -1], dtype=torch.int64)
        return self.project(xs, None, params), torch.from_numpy(np.sqrt(ss)), bad

    def raise_bad(self, bad):
        from paper_0904_3151_b200 import engine
        engine.raise_bad_rows(bad)

    def plan(self, codes, params):
        # the block count is a cost knob: any k' > d gives the same pairs
        return self.blocks or params.blocks

    def unit_count(self, blocks, mismatch):
        from paper_0904_3151_b200 import engine
        return engine.unit_count(blocks, mismatch)

    def candidates(self, codes, params, units, blocks):
        """Pairs owned by `units`: owner = (replicate, first member of the
        plan's family whose masked blocks contain the differing blocks) --
        for a block count that is the canonical mask; the rule the CUDA
        kernels implement."""
        from paper_0904_3151_b200 import engine
        orc = self.orc
        words = [c.numpy().view(np.uint64) for c in codes]
        blocks, family, _ = engine.plan_design(blocks, params.mismatch)
        family = [int(f) for f in family]
        bounds = orc.block_partition(params.length, blocks)
        blk = np.zeros(params.length, dtype=np.int64)
        for b in range(blocks):
            blk[bounds[b]:bounds[b + 1]] = b
        mine = set(units)
        keys = []
        for h in range(params.replicates):
            pairs, _ = orc.enumerate_pairs(words[h], params.length, bounds, params.mismatch)
            keep = orc.first_witness(pairs, words[:h], params.mismatch)
            for (i, j) in pairs[keep]:
                x = int(words[h][i, 0] ^ words[h][j, 0])
                delta = 0
                for t in range(params.length):
                    if x >> t & 1:
                        delta |= 1 << int(blk[t])
                owner = next(q for q, f in enumerate(family) if f & delta == delta)
                unit = h * len(family) + owner
                if unit in mine:
                    keys.append((int(i) << 32) | int(j))
        return torch.tensor(keys, dtype=torch.int64), {}

    def sort(self, keys, n):
        return torch.sort(keys).values

    def verify(self, x, norms, keys, metric, eps):
        k = keys.numpy().view(np.uint64)
        pairs = np.stack([(k >> np.uint64(32)).astype(np.int64),
                          (k & np.uint64(0xffffffff)).astype(np.int64)], axis=1)
        d = self.orc.cosine_dist(self.x, pairs)
        keep = d <= eps
        return keys[torch.from_numpy(keep)], torch.from_numpy(d[keep])

    def merge_runs(self, keys, dists, offsets):
        """k-way merge of the sorted runs (heapq), like eg_merge_runs."""
        import heapq
        runs = []
        for r in range(len(offsets) - 1):
            a, b = offsets[r], offsets[r + 1]
            k = keys[a:b].tolist()
            assert k == sorted(k), "rank runs must arrive sorted"
            runs.append(list(zip(k, dists[a:b].tolist())))
        merged = list(heapq.merge(*runs))
        return (torch.tensor([m[0] for m in merged], dtype=torch.int64),
                torch.tensor([m[1] for m in merged], dtype=torch.float64))


def _worker(rank, world, port, out_path, blocks=None):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    import paper_0904_3151_b200 as eg
    from paper_0904_3151_b200 import distributed, workloads
    x = workloads.planted_clusters(400, 8, 8, 20, 0.03, 5)
    params = eg.MsmParams(epsilon=0.05, gamma=1e-3, length=24, mismatch=2, blocks=4,
                          replicates=3, seed=7)
    res = distributed.build_step(torch.from_numpy(x), params, "cosine", world, rank,
                                 ops=OracleOps(orc, x, blocks))
    if rank == 0:
        np.savez(out_path, keys=res["keys"].numpy(), dist=res["dist"].numpy())
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.mark.parametrize("blocks", [None, 3, 6, 10703])
def test_two_rank_build_equals_single_process(oracle, tmp_path, blocks):
    """Sharded build == single-process reference, for the reference block
    count and for planned counts k' != k (the pair set is independent of k)."""
    out = str(tmp_path / "merged.npz")
    mp.spawn(_worker, args=(2, _free_port(), out, blocks), nprocs=2, join=True)
    got = np.load(out)
    from paper_0904_3151_b200 import workloads
    x = workloads.planted_clusters(400, 8, 8, 20, 0.03, 5)
    ref = oracle.build_graph(x, 0.05, 24, 2, 4, 3, 7)
    k = got["keys"].view(np.uint64)
    pairs = np.stack([(k >> np.uint64(32)).astype(np.int64),
                      (k & np.uint64(0xffffffff)).astype(np.int64)], axis=1)
    np.testing.assert_array_equal(pairs, ref.pairs)
    np.testing.assert_allclose(got["dist"], ref.distances, rtol=0, atol=1e-12)


def _bad_worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    import paper_0904_3151_b200 as eg
    from paper_0904_3151_b200 import distributed, workloads
    x = workloads.planted_clusters(400, 8, 8, 20, 0.03, 5)
    x[301] = 0.0                       # in rank 1's shard
    x[350] = 0.0
    params = eg.MsmParams(epsilon=0.05, gamma=1e-3, length=24, mismatch=2, blocks=4,
                          replicates=1, seed=7)
    try:
        distributed.build_step(torch.from_numpy(x), params, "cosine", world, rank,
                               ops=OracleOps(orc, x))
        msg = "no error"
    except eg.DataError as e:
        msg = str(e)
    with open(f"{out_path}.{rank}", "w") as f:
        f.write(msg)
    tdist.destroy_process_group()


def test_bad_rows_raise_on_every_rank(oracle, tmp_path):
    """A zero row in one rank's shard: every rank raises the reference's
    DataError for the first offending global row (no rank is left waiting
    in a collective)."""
    out = str(tmp_path / "msg")
    mp.spawn(_bad_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        assert open(f"{out}.{r}").read() == "row 301 has zero norm and cannot be projected"


def test_unit_and_row_sharding_cover_exactly_once():
    from paper_0904_3151_b200 import distributed
    for total, world in [(660, 8), (28, 3), (5, 8)]:
        seen = sorted(u for r in range(world) for u in distributed.my_units(total, world, r))
        assert seen == list(range(total))
    for n, world in [(1_600_000, 8), (10, 3), (7, 8)]:
        rows = []
        for r in range(world):
            lo, hi, per = distributed.row_shard(n, world, r)
            assert hi - lo <= per
            rows.extend(range(lo, hi))
        assert rows == list(range(n))
