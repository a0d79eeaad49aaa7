"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

One step of the selected-CI growth loop with the heat-bath surrogate
selector (Sec 2.2 :308-312: generate the coupled
sets of S, de-duplicate, select the top-K new configurations, merge them into
S; the NNQS amplitude is replaced by the heat-bath score, DESIGN.md reading
r16), written from the definition with Python dicts and sorted():

    records (i -> j, H_ij)      = the oracle's gen_coupled over S
    p(i, j)                     = fl(H_ij * psi_i)             (one fp64 multiply)
    v(i, j)                     = bits(|p|) << 1 | [p < 0]     (|p| first, then the sign)
    score_j                     = max over records of v(i, j),  j not in S, v > 0
    selected                    = the K largest scores, ties by the pool hash order pi
    S'                          = S u selected
    psi'_i = psi_i (i in S),    psi'_j = -p_j (j selected, p_j the product behind score_j)

Shares no code with the CUDA path.
"""
from __future__ import annotations

import struct

import numpy as np

MASK = (1 << 64) - 1


def _fmix64(x: int) -> int:
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & MASK
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & MASK
    x ^= x >> 31
    return x


def pi_order(key: tuple) -> tuple:
    """The pool hash order pi(j) = (hi, lo) (reading r13)."""
    if len(key) == 1:
        return (_fmix64(key[0]), 0)
    lo = _fmix64(key[1] ^ 0x9E3779B97F4A7C15)
    return (_fmix64(key[0] ^ lo), lo)


def _bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def _from_bits(b: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def score_value(p: float) -> int:
    return (_bits(abs(p)) << 1) | (1 if p < 0.0 else 0)


def grow_step(S_keys, psi, rec, K: int, W: int):
    """S_keys [|S|, W] and psi [|S|] aligned (any order); rec = the oracle's
    gen_coupled(S_keys) dict.  Returns (new space as {key tuple: psi},
    selected keys in selection order, number of candidates)."""
    S_keys = np.asarray(S_keys, dtype=np.uint64).reshape(-1, W)
    space = {tuple(int(x) for x in k): float(p) for k, p in zip(S_keys, psi)}
    best: dict = {}
    for k, h, s in zip(np.asarray(rec["keys"]).reshape(-1, W), rec["hij"], rec["src"]):
        p = float(h) * float(psi[int(s)])
        v = score_value(p)
        key = tuple(int(x) for x in k)
        if v > best.get(key, 0):
            best[key] = v
    cand = [(key, v) for key, v in best.items() if key not in space and v > 0]
    cand.sort(key=lambda kv: (-kv[1], pi_order(kv[0])))
    selected = cand[:K]
    out = dict(space)
    for key, v in selected:
        a = _from_bits(v >> 1)
        out[key] = a if (v & 1) else -a          # psi_j = -p
    return out, [key for key, _ in selected], len(cand)
