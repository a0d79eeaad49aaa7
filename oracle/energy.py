"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Stage-3 contraction: the plain definition of

    e[s] = sum over records r with src[r] = s of  H[r] * psi[idx(key[r])]

(Eq. 5 :267-270, the inner sum sum_{j in C_i} H_ij psi_j; Stage 3
:398-403 maps psi back to the non-unique records through a reverse index,
:634).  idx(key) = position of the key in the unique set; psi is aligned with
that set.  Each term is the IEEE fp64 product fl(H * psi) and e[s] is the
EXACT sum of its terms rounded once to fp64 (math.fsum, which is correctly
rounded).  The paper fixes no summation order (:398-403 "reduction
operations"), so the order-free exact sum is the definition; any GPU
summation order is compared against it within a tolerance (DESIGN.md r14).
A record whose key is not in the set contributes nothing and is counted as
missing.

Written from the definition with a dict and math.fsum; shares no code with
the CUDA path.
"""
from __future__ import annotations

import math

import numpy as np


def contract(keys, hij, src, n_parents: int, space_keys, psi, W: int):
    """Returns (e float64 [n_parents], n_missing, absterm float64 [n_parents]);
    absterm[s] = fsum of |terms| (the condition scale of e[s])."""
    keys = np.asarray(keys, dtype=np.uint64).reshape(-1, W)
    space_keys = np.asarray(space_keys, dtype=np.uint64).reshape(-1, W)
    index = {tuple(int(x) for x in k): i for i, k in enumerate(space_keys)}
    terms = [[] for _ in range(n_parents)]
    missing = 0
    for k, h, s in zip(keys, np.asarray(hij, dtype=np.float64), np.asarray(src)):
        i = index.get(tuple(int(x) for x in k))
        if i is None:
            missing += 1
            continue
        terms[int(s)].append(float(h) * float(psi[i]))    # one IEEE fp64 multiply
    e = np.array([math.fsum(t) for t in terms], dtype=np.float64)
    absterm = np.array([math.fsum(abs(x) for x in t) for t in terms], dtype=np.float64)
    return e, missing, absterm
