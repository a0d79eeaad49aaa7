"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Stage-3 contraction: the plain definition of

    e[s] = sum over records r with src[r] = s of  H[r] * psi[idx(key[r])]

(Eq. 5 :267-270, the inner sum sum_{j in C_i} H_ij psi_j; Stage 3
:398-403 maps psi back to the non-unique records through a reverse index,
:634).  idx(key) = position of the key in the unique set; psi is aligned with
that set.  Reduction (reading r14): each product p = fl64(H * psi)
is rounded half-to-even to the grid 2^-80 and the integers are summed exactly
(Python ints), e[s] = that exact sum rounded once to fp64.  A record whose key
is not in the set contributes nothing and is counted as missing.

Written from the definition with Python integers and a dict; shares no code
with the CUDA path.
"""
from __future__ import annotations

import math

import numpy as np


def round80(p: float) -> int:
    """round_half_even(p * 2^80) as an exact integer."""
    if p == 0.0:
        return 0
    f, E = math.frexp(p)            # p = f * 2^E, 0.5 <= |f| < 1
    m = int(f * (1 << 53))          # exact: f has 53 significant bits
    sh = E - 53 + 80
    if sh >= 0:
        return m << sh if m >= 0 else -((-m) << sh)
    r = -sh
    am = abs(m)
    whole, rem, half = am >> r, am & ((1 << r) - 1), 1 << (r - 1)
    if rem > half or (rem == half and (whole & 1)):
        whole += 1
    return whole if m >= 0 else -whole


def contract(keys, hij, src, n_parents: int, space_keys, psi, W: int):
    """Returns (e float64 [n_parents], n_missing)."""
    keys = np.asarray(keys, dtype=np.uint64).reshape(-1, W)
    space_keys = np.asarray(space_keys, dtype=np.uint64).reshape(-1, W)
    index = {tuple(int(x) for x in k): i for i, k in enumerate(space_keys)}
    acc = [0] * n_parents
    missing = 0
    for k, h, s in zip(keys, np.asarray(hij, dtype=np.float64), np.asarray(src)):
        i = index.get(tuple(int(x) for x in k))
        if i is None:
            missing += 1
            continue
        p = float(h) * float(psi[i])    # one IEEE fp64 multiply
        if not abs(p) < 2.0 ** 20:
            raise ValueError("|H psi| >= 2^20")
        acc[int(s)] += round80(p)
    e = np.array([math.ldexp(float(a), -80) for a in acc], dtype=np.float64)
    return e, missing
