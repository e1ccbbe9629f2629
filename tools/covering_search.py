"""Search for small covering designs C(v, m, t): families of m-subsets of
{0..v-1} ("masked block sets") such that every t-subset lies inside at least
one of them.  The MSM units of a design keep the v - m other blocks; every
pair differing in at most t blocks then shares a masked key in some unit.

Simulated annealing on a fixed family size (cost = uncovered t-subsets, move =
exchange one element of one member), shrinking the family while a cover is
found.  Writes the tables used by paper_0904_3151_b200/designs.py.

    python tools/covering_search.py --t 3 --vmax 14 --seconds 20 --out /tmp/designs.json
"""
import argparse
import itertools
import json
import math
import random
import time


def popcount(x):
    return bin(x).count("1")


def tsubsets_of(mask, t):
    bits = [i for i in range(mask.bit_length()) if mask >> i & 1]
    return [sum(1 << b for b in c) for c in itertools.combinations(bits, t)]


def greedy(v, m, t, rng):
    tsubs = [sum(1 << b for b in c) for c in itertools.combinations(range(v), t)]
    uncovered = set(tsubs)
    fam = []
    cands = [sum(1 << b for b in c) for c in itertools.combinations(range(v), m)]
    while uncovered:
        best, bestc = None, -1
        sample = cands if len(cands) <= 4000 else rng.sample(cands, 4000)
        for c in sample:
            cnt = sum(1 for s in tsubsets_of(c, t) if s in uncovered)
            if cnt > bestc or (cnt == bestc and rng.random() < 0.3):
                best, bestc = c, cnt
        fam.append(best)
        uncovered.difference_update(tsubsets_of(best, t))
    return fam


def anneal(v, m, t, size, rng, seconds):
    """Try to find a cover with `size` members; returns the family or None."""
    tsubs = [sum(1 << b for b in c) for c in itertools.combinations(range(v), t)]
    idx = {s: i for i, s in enumerate(tsubs)}
    cover_cache = {}

    def covers(mask):
        r = cover_cache.get(mask)
        if r is None:
            r = [idx[s] for s in tsubsets_of(mask, t)]
            cover_cache[mask] = r
        return r

    allm = [sum(1 << b for b in c) for c in itertools.combinations(range(v), m)]
    fam = [rng.choice(allm) for _ in range(size)]
    cnt = [0] * len(tsubs)
    for f in fam:
        for i in covers(f):
            cnt[i] += 1
    cost = sum(1 for c in cnt if c == 0)
    T = 0.6
    end = time.time() + seconds
    it = 0
    full = (1 << v) - 1
    while cost and time.time() < end:
        it += 1
        j = rng.randrange(size)
        old = fam[j]
        ins = [b for b in range(v) if old >> b & 1]
        outs = [b for b in range(v) if not old >> b & 1]
        new = old ^ (1 << rng.choice(ins)) ^ (1 << rng.choice(outs))
        delta = 0
        co, cn = covers(old), covers(new)
        for i in co:
            cnt[i] -= 1
            if cnt[i] == 0:
                delta += 1
        for i in cn:
            if cnt[i] == 0:
                delta -= 1
            cnt[i] += 1
        if delta <= 0 or rng.random() < math.exp(-delta / T):
            fam[j] = new
            cost += delta
        else:
            for i in cn:
                cnt[i] -= 1
            for i in co:
                cnt[i] += 1
        if it % 20000 == 0:
            T = max(0.15, T * 0.97)
    return fam if cost == 0 else None


def schoenheim(v, m, t):
    b = 1
    for i in range(t):
        b = -(-b * (v - t + 1 + i) // (m - t + 1 + i))
    return b


def search(v, m, t, seconds, seed=0):
    rng = random.Random(seed)
    best = greedy(v, m, t, rng)
    lb = schoenheim(v, m, t)
    end = time.time() + seconds
    while len(best) > lb and time.time() < end:
        got = anneal(v, m, t, len(best) - 1, rng, min(seconds / 4, end - time.time()))
        if got is None:
            continue
        best = got
    return sorted(best), lb


def check(v, m, t, fam):
    assert all(popcount(f) == m and f < (1 << v) for f in fam)
    for c in itertools.combinations(range(v), t):
        s = sum(1 << b for b in c)
        assert any(f & s == s for f in fam), (v, m, t, c)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t", type=int, nargs="+", default=[2, 3])
    ap.add_argument("--vmax", type=int, default=14)
    ap.add_argument("--seconds", type=float, default=10.0)
    ap.add_argument("--out", default="/tmp/designs.json")
    ap.add_argument("--only", type=str, default="")
    a = ap.parse_args()
    out = {}
    todo = []
    if a.only:
        for s in a.only.split(";"):
            todo.append(tuple(int(x) for x in s.split(",")))
    else:
        for t in a.t:
            for v in range(t + 2, a.vmax + 1):
                for m in range(t + 1, v - 1):
                    todo.append((v, m, t))
    for v, m, t in todo:
        fam, lb = search(v, m, t, a.seconds)
        check(v, m, t, fam)
        complete = math.comb(v, t)
        print(f"C({v},{m},{t}) = {len(fam)} (bound {lb}; complete C({v},{t}) = {complete})", flush=True)
        out[f"{v},{m},{t}"] = fam
    with open(a.out, "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
