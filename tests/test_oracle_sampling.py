"""Pins for oracle/sampling.py (Sec 4.1.1 :448-462).

Pinned by a hand-worked example, by set identities (the shards partition the
distinct keys: numpy's unique, not the oracle's own sorted(set())), by the
splitter semantics (every key of shard r lies in [spl_r, spl_{r+1})), and by
the regular-sampling balance bound: rank i contributes to partition r at most
(c_ir + 1) ceil(|D_i| / S) keys, c_ir = rank i's samples inside the partition
(consecutive samples of D_i are at most ceil(|D_i| / S) indices apart)."""
import math

import numpy as np
import pytest

from oracle import sampling as S


def test_hand_worked_example():
    # P = 2, S = 2: D0 = [1, 3, 5, 7] samples idx 0, 2 -> 1, 5; D1 = [2, 4, 6, 8] -> 2, 6.
    # Sorted samples [1, 2, 5, 6], M = 4, splitter r = 1 at floor(1 * 4 / 2) = 2 -> 5.
    shards, spl = S.dedup_sorted([[7, 3, 5, 1, 3], [8, 2, 6, 4, 8]], 2)
    assert spl == [5]
    assert shards == [[1, 2, 3, 4], [5, 6, 7, 8]]


def test_samples_positions():
    D = list(range(100, 110))              # |D| = 10
    assert S.regular_samples(D, 4) == [100, 102, 105, 107]   # floor(k 10 / 4) = 0, 2, 5, 7
    assert S.regular_samples(D, 10) == D
    assert S.regular_samples(D, 16) == D                     # |D| < S: all of D
    assert S.regular_samples([], 8) == []


def test_splitters_positions():
    smp = [9, 1, 8, 2, 7, 3, 6, 4, 5, 0]   # sorted 0..9, M = 10
    assert S.select_splitters(smp, 4) == [2, 5, 7]           # floor(r 10 / 4) = 2, 5, 7
    assert S.select_splitters(smp, 1) == []
    assert S.select_splitters([], 3) == [0, 0]


def test_bounds_lower_bound():
    D = [2, 4, 4, 6, 9]
    assert S.split_bounds(D, [4, 7]) == [0, 1, 4, 5]
    assert S.split_bounds(D, [0, 100]) == [0, 0, 5, 5]


def test_w2_integer_order_roundtrip():
    rng = np.random.Generator(np.random.PCG64(3))
    k = rng.integers(0, 2**64, size=(500, 2), dtype=np.uint64)
    k[:50, 1] = 0
    xs = S.to_ints(k, 2)
    assert np.array_equal(S.from_ints(xs, 2), k)
    order = np.lexsort((k[:, 0], k[:, 1]))        # word 1 major, independent of the oracle
    assert np.array_equal(S.from_ints(sorted(xs), 2), k[order])


def _check_protocol(local, Ssz):
    P = len(local)
    shards, spl = S.dedup_sorted(local, Ssz)
    allk = [int(v) for x in local for v in x]
    ref = [int(v) for v in np.unique(np.array(allk, dtype=np.uint64))]
    assert [x for sh in shards for x in sh] == ref                     # partition of the distinct keys
    lo = [-math.inf] + spl
    hi = spl + [math.inf]
    for r, sh in enumerate(shards):
        assert all(lo[r] <= x < hi[r] for x in sh)
        assert sh == sorted(sh) and len(set(sh)) == len(sh)
    # balance bound
    D = [sorted(set(x)) for x in local]
    smp = [S.regular_samples(d, Ssz) for d in D]
    for r, sh in enumerate(shards):
        bound = 0
        for i in range(P):
            c = sum(1 for x in smp[i] if lo[r] <= x < hi[r])
            bound += (c + 1) * math.ceil(len(D[i]) / Ssz) if D[i] else 0
        assert len(sh) <= bound, (r, len(sh), bound)
    return shards


@pytest.mark.parametrize("P,Ssz,seed", [(1, 8, 1), (2, 4, 2), (4, 16, 3), (8, 64, 4), (3, 5, 5)])
def test_protocol_random(P, Ssz, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    local = [rng.integers(0, 5000, size=int(rng.integers(0, 3000))).tolist() for _ in range(P)]
    _check_protocol(local, Ssz)


def test_protocol_skewed_and_empty_ranks():
    rng = np.random.Generator(np.random.PCG64(9))
    heavy = [7] * 2000 + rng.integers(0, 100, size=500).tolist()
    _check_protocol([heavy, [], [7, 7, 7], rng.integers(0, 1 << 40, size=800).tolist()], 32)


def test_balance_uniform_keys():
    # regular sampling on uniform distinct keys: shards within 10% of each other (P = 8, S = 256)
    rng = np.random.Generator(np.random.PCG64(11))
    local = [rng.integers(0, 1 << 62, size=20000).tolist() for _ in range(8)]
    shards = _check_protocol(local, 256)
    sizes = [len(s) for s in shards]
    assert max(sizes) / min(sizes) < 1.1
