"""Pins of the f4 growth-step oracle (oracle/heatbath.py; SURVEY 8(f) f4,
PAPER.md Sec 2.2 :308-312, reading r16) against what is fixed
independently of it:

* the heat-bath scores against the BRUTE-FORCE second-quantised Hamiltonian
  (tests/fock.py): score_j = max_i |<j|H|i> psi_i| over i in S, j not in S;
* a hand example (S = {HF}, psi = 1: the selection is the K largest |H_HF,j|);
* set algebra: the selection is a subset of C \\ S, |S'| = |S| + min(K, #cand),
  smaller K gives a prefix of the larger K's selection, K >= #cand takes all."""
import numpy as np
import pytest

import oracle
import synth
from oracle import heatbath as HB
from tests import fock


def _lih(g=1):
    K, na, nb = 6, 2, 2
    ints = synth.make_integrals(K, g, 0x5EED0000 + 40 + g)
    return K, na, nb, ints, synth.full_space(K, na, nb)


@pytest.mark.parametrize("g", [1, 4])
def test_scores_against_bruteforce(g):
    K, na, nb, ints, full = _lih(g)
    rng = np.random.default_rng(g)
    S = full[np.sort(rng.choice(len(full), 30, replace=False))]
    psi = rng.uniform(-1, 1, size=len(S))
    rec = oracle.gen_coupled(2 * K, na, nb, S, ints, 0.0)
    new, sel, ncand = HB.grow_step(S, psi, rec, 10 ** 6, 1)
    e4 = fock.full_eri_from_factors(ints.factors, K)
    Sset = {int(k[0]) for k in S}
    best = {}
    for i, k in enumerate(S):
        col = fock.apply_H(int(k[0]), ints.h, e4, list(range(K)))   # <j|H|i>
        for j, v in col.items():
            if j in Sset or v == 0.0:
                continue
            t = abs(v * psi[i])
            if t > best.get(j, (0.0, 0.0))[0]:
                best[j] = (t, -v * psi[i])
    assert ncand == len(best) == len(sel)
    for j, (t, amp) in best.items():
        assert abs(abs(new[(j,)]) - t) <= 1e-12 * max(t, 1e-300)
        assert abs(new[(j,)] - amp) <= 1e-12 * max(t, 1e-300)


def test_hand_example_hf_reference():
    K, na, nb, ints, full = _lih()
    hf = synth.occ_to_keys(np.array([[1, 1, 1, 1] + [0] * 8], dtype=bool), 12)
    rec = oracle.gen_coupled(12, na, nb, hf, ints, 0.0)
    order = sorted(zip(rec["hij"], (int(k[0]) for k in rec["keys"])), key=lambda t: -abs(t[0]))
    new, sel, ncand = HB.grow_step(hf, np.array([1.0]), rec, 5, 1)
    assert ncand == len(rec["src"])
    got = [k[0] for k in sel]
    assert sorted(abs(new[(j,)]) for j in got) == sorted(abs(h) for h, _ in order[:5])
    for h, j in order:
        if (j,) in new:
            assert new[(j,)] == -h                  # psi_j = -H_j,HF * 1


def test_selection_set_algebra():
    wl, ints, par = synth.workload_inputs("h2o", n_parents=40)
    psi = np.random.default_rng(3).uniform(-1, 1, size=len(par))
    rec = oracle.gen_coupled(wl.m, 5, 5, par, ints, 0.0)
    big, sel_big, ncand = HB.grow_step(par, psi, rec, 500, 1)
    small, sel_small, _ = HB.grow_step(par, psi, rec, 120, 1)
    every, sel_all, _ = HB.grow_step(par, psi, rec, 10 ** 9, 1)
    Sset = {(int(k[0]),) for k in par}
    C = {(int(k[0]),) for k in rec["keys"]}
    assert set(sel_big) <= C - Sset
    assert sel_small == sel_big[:120]
    assert len(big) == len(par) + min(500, ncand) and len(sel_all) == ncand
    assert all(every[k] == big[k] for k in big)
