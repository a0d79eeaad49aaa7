"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's sort-based regular-sampling de-duplication (
PAPER.md Sec 4.1.1 :448-462), written step by step in the paper's order with
Python integers (a key = the integer whose bit t is orbital t; at W = 2 word 1
is the high word), sorted() and bisect:

  Step 1 (:454)  each rank sorts its buffer D_i (and drops duplicates, DESIGN.md
                 reading r15) and takes S pivots at indices floor(k |D_i| / S),
                 k = 0..S-1 (all of D_i when |D_i| < S);
  Step 2 (:457)  the root sorts the P x S gathered samples and takes the P-1
                 splitters at equidistant positions floor(r M / P), r = 1..P-1;
                 every rank finds its partition bounds by binary search
                 (bisect_left: partition r = [spl_r, spl_{r+1}));
  Step 3 (:460)  all-to-all-v, then merge + stream compaction at the receiver
                 (sorted(set(...))).

Shares no code with the CUDA path.
"""
from __future__ import annotations

import bisect

import numpy as np


def to_ints(keys, W: int) -> list[int]:
    k = np.asarray(keys, dtype=np.uint64).reshape(-1, W)
    if W == 1:
        return [int(x) for x in k[:, 0]]
    return [int(a) | (int(b) << 64) for a, b in zip(k[:, 0], k[:, 1])]


def from_ints(xs, W: int) -> np.ndarray:
    out = np.zeros((len(xs), W), dtype=np.uint64)
    for i, x in enumerate(xs):
        out[i, 0] = x & ((1 << 64) - 1)
        if W == 2:
            out[i, 1] = x >> 64
    return out


def sort_unique(xs) -> list[int]:
    """Step 1, first half: the rank's sorted buffer without duplicates."""
    return sorted(set(xs))


def regular_samples(D: list[int], S: int) -> list[int]:
    """Step 1, second half: S pivots at indices floor(k |D| / S)."""
    if len(D) < S:
        return list(D)
    return [D[(k * len(D)) // S] for k in range(S)]


def select_splitters(samples: list[int], P: int) -> list[int]:
    """Step 2: sort the gathered samples, P-1 splitters at floor(r M / P)."""
    srt = sorted(samples)
    M = len(srt)
    return [srt[(r * M) // P] if M else 0 for r in range(1, P)]


def split_bounds(D: list[int], spl: list[int]) -> list[int]:
    """Step 2, last sentence: binary search of each splitter in the sorted array."""
    return [0] + [bisect.bisect_left(D, x) for x in spl] + [len(D)]


def dedup_sorted(local: list[list[int]], S: int):
    """The whole protocol over P logical ranks: (shards, splitters)."""
    P = len(local)
    D = [sort_unique(x) for x in local]
    samples = [s for d in D for s in regular_samples(d, S)]
    spl = select_splitters(samples, P)
    bounds = [split_bounds(d, spl) for d in D]
    shards = []
    for r in range(P):
        recv = [x for i in range(P) for x in D[i][bounds[i][r]:bounds[i][r + 1]]]
        shards.append(sorted(set(recv)))
    return shards, spl
