"""Brute-force second-quantised Hamiltonian (test pin for the oracle).

H = sum_pq h_pq a+_p a_q + 1/2 sum_pqrs <pq|rs> a+_p a+_q a_s a_r
with <pq|rs> = (PR|QS) d(s_p,s_r) d(s_q,s_s) (chemist (PR|QS) from the
integral FACTORS B^L, not from the packed array), applied to occupation-number
kets with explicit Jordan-Wigner signs: a+_t / a_t on |n> carry
(-1)^(number of occupied orbitals with index < t).  No Slater-Condon rule, no
excitation enumeration, no packed-ERI indexing is shared with oracle/.

Only spatial orbitals listed in `active` are given nonzero integrals, so the
operator sums run over active spin orbitals only while the kets may carry
frozen electrons anywhere in m <= 128 bits (their signs still count).
"""
from __future__ import annotations

import numpy as np


def full_eri_from_factors(B: np.ndarray, K: int) -> np.ndarray:
    """(PQ|RS) = sum_L B^L_PQ B^L_RS as a dense [K,K,K,K] array (einsum order)."""
    Bf = np.zeros((B.shape[0], K, K))
    for P in range(K):
        for Q in range(P + 1):
            Bf[:, P, Q] = B[:, P * (P + 1) // 2 + Q]
            Bf[:, Q, P] = B[:, P * (P + 1) // 2 + Q]
    return np.einsum("lpq,lrs->pqrs", Bf, Bf)


def _ann(state: int, t: int):
    if not (state >> t) & 1:
        return None, 0
    sign = -1 if bin(state & ((1 << t) - 1)).count("1") % 2 else 1
    return state ^ (1 << t), sign


def _cre(state: int, t: int):
    if (state >> t) & 1:
        return None, 0
    sign = -1 if bin(state & ((1 << t) - 1)).count("1") % 2 else 1
    return state | (1 << t), sign


def apply_H(ket: int, h: np.ndarray, eri4: np.ndarray, active_spatial, spatial_of=None) -> dict:
    """H|ket> as {bra_state: amplitude}.  h, eri4 are indexed by *spatial*
    index via spatial_of[P_active] (identity by default)."""
    act = []
    for P in active_spatial:
        act += [2 * P, 2 * P + 1]
    sp = (lambda t: t // 2)
    out: dict[int, float] = {}

    def add(s, v):
        out[s] = out.get(s, 0.0) + v

    occ = [t for t in act if (ket >> t) & 1]
    # one-body
    for q in occ:
        s1, g1 = _ann(ket, q)
        for p in act:
            if p % 2 != q % 2:
                continue
            s2, g2 = _cre(s1, p)
            if s2 is None:
                continue
            v = h[sp(p), sp(q)]
            if v != 0.0:
                add(s2, g1 * g2 * v)
    # two-body: 1/2 <pq|rs> a+p a+q a_s a_r
    for r in occ:
        s1, g1 = _ann(ket, r)
        for s in occ:
            s2, g2 = _ann(s1, s)
            if s2 is None:
                continue
            for q in act:
                if q % 2 != s % 2:
                    continue
                s3, g3 = _cre(s2, q)
                if s3 is None:
                    continue
                for p in act:
                    if p % 2 != r % 2:
                        continue
                    s4, g4 = _cre(s3, p)
                    if s4 is None:
                        continue
                    v = eri4[sp(p), sp(r), sp(q), sp(s)]  # <pq|rs> = (PR|QS)
                    if v != 0.0:
                        add(s4, 0.5 * g1 * g2 * g3 * g4 * v)
    return out


def key_to_int(row) -> int:
    row = np.atleast_1d(row)
    return sum(int(w) << (64 * i) for i, w in enumerate(row))


def int_to_key(x: int, W: int) -> np.ndarray:
    return np.array([(x >> (64 * i)) & ((1 << 64) - 1) for i in range(W)], dtype=np.uint64)
