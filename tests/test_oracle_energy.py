"""Pins of the Stage-3 contraction oracle (oracle/energy.py, SURVEY 8(f) f1,
PAPER.md Eq. 5 :267-270; reduction = DESIGN.md reading r14) against what the
mathematics fixes: the rounding rule on hand-computed values, exact dyadic
sums, order independence, and delta amplitudes reproducing single matrix
elements (Hermiticity of the coupled records)."""
import math
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from oracle import energy


def test_round80_closed_forms():
    t = 2.0 ** -80
    assert energy.round80(0.0) == 0
    assert energy.round80(t) == 1
    assert energy.round80(0.5 * t) == 0           # tie -> even (0)
    assert energy.round80(1.5 * t) == 2           # tie -> even (2)
    assert energy.round80(2.5 * t) == 2           # tie -> even (2)
    assert energy.round80(-2.5 * t) == -2
    assert energy.round80(1.25 * t) == 1 and energy.round80(1.75 * t) == 2
    assert energy.round80(1.0) == 1 << 80
    assert energy.round80(-3.0) == -(3 << 80)
    assert energy.round80(2.0 ** -200) == 0
    # dyadic values above the grid are exact
    rng = random.Random(1)
    for _ in range(1000):
        x = rng.randint(-(1 << 40), 1 << 40) * 2.0 ** -30
        assert energy.round80(x) == int(Fraction(x) * (1 << 80))


def test_dyadic_sums_exact_and_order_independent():
    rng = np.random.default_rng(3)
    n, npar = 5000, 17
    keys = np.arange(1, n + 1, dtype=np.uint64).reshape(-1, 1)
    hij = rng.integers(-(1 << 32), 1 << 32, size=n) * 2.0 ** -30
    src = rng.integers(0, npar, size=n)
    space = keys.copy()
    psi = np.ones(n)
    e, miss = energy.contract(keys, hij, src, npar, space, psi, 1)
    assert miss == 0
    for s in range(npar):
        assert e[s] == math.fsum(hij[src == s])   # exact sum of dyadic terms
    perm = rng.permutation(n)
    e2, _ = energy.contract(keys[perm], hij[perm], src[perm], npar, space, psi, 1)
    assert np.array_equal(e, e2)


def test_missing_keys_counted():
    keys = np.array([[5], [6], [7], [8]], dtype=np.uint64)
    e, miss = energy.contract(keys, [1.0, 2.0, 4.0, 8.0], [0, 0, 1, 1], 2, keys[::2], np.array([1.0, 1.0]), 1)
    assert miss == 2 and e[0] == 1.0 and e[1] == 4.0


@pytest.mark.parametrize("j0", [0, 37, 224])
def test_delta_psi_gives_matrix_elements(j0):
    """psi = delta_{j0} over the LiH full space: e[s] = H_{s, j0} (0 if j0 is
    not coupled to s), which also equals H_{j0, s} (bit-exact Hermiticity)."""
    wl, ints, par = synth.workload_inputs("lih")
    rec = oracle.gen_coupled(wl.m, wl.n_alpha, wl.n_beta, par, ints, 0.0)
    psi = np.zeros(len(par))
    psi[j0] = 1.0
    e, miss = energy.contract(rec["keys"], rec["hij"], rec["src"], len(par), par, psi, 1)
    assert miss == 0
    row = {int(k[0]): h for k, h, s in zip(rec["keys"], rec["hij"], rec["src"]) if s == j0}
    for s in range(len(par)):
        sel = (rec["src"] == s) & (rec["keys"][:, 0] == par[j0, 0])
        h_s_j0 = float(rec["hij"][sel][0]) if sel.any() else 0.0
        assert e[s] == h_s_j0
        assert e[s] == row.get(int(par[s, 0]), 0.0)
