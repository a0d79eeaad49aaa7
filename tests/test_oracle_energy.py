"""Pins of the Stage-3 contraction oracle (oracle/energy.py, SURVEY 8(f) f1,
PAPER.md Eq. 5 :267-270: e_i = sum_{j in C_i} H_ij psi_j) against what the
mathematics fixes:

* a hand-computed example;
* exact rational arithmetic (fractions.Fraction) of the same products,
  rounded once -- fsum must agree bit for bit (the definition is the exact
  sum, not a summation order);
* delta amplitudes reproduce single matrix elements (e[s] = H_{s, j0}) and
  bit-exact Hermiticity;
* against the BRUTE-FORCE second-quantised Hamiltonian (tests/fock.py,
  explicit creation/annihilation operators over the full Sz sector): with
  a random psi over the whole LiH space, e[s] = sum_{j != s} <s|H|j> psi_j
  within 1e-12 of the absolute term sum -- an independent construction of
  the same off-diagonal matrix-vector product;
* missing keys counted and contribute nothing; order independence."""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from oracle import energy
from tests import fock


def test_hand_example():
    keys = np.array([[3], [5], [9], [5]], dtype=np.uint64)
    hij = [0.5, -0.25, 2.0, 1.0]
    src = [0, 0, 1, 1]
    space = np.array([[5], [9], [3]], dtype=np.uint64)   # idx(3) = 2, idx(5) = 0, idx(9) = 1
    psi = np.array([4.0, -1.0, 8.0])
    e, miss, ab = energy.contract(keys, hij, src, 2, space, psi, 1)
    # e0 = 0.5*psi[2] + (-0.25)*psi[0] = 4 - 1 = 3;  e1 = 2*psi[1] + 1*psi[0] = -2 + 4 = 2
    assert miss == 0 and e.tolist() == [3.0, 2.0] and ab.tolist() == [5.0, 6.0]


def test_exact_rational_sum():
    rng = np.random.default_rng(3)
    n, npar = 4000, 13
    keys = rng.choice(1 << 40, size=n, replace=False).astype(np.uint64).reshape(-1, 1)
    hij = rng.standard_normal(n) * 10.0 ** rng.integers(-12, 2, size=n)
    src = rng.integers(0, npar, size=n)
    space = keys[rng.permutation(n)]
    psi = rng.uniform(-1, 1, size=n)
    e, miss, _ = energy.contract(keys, hij, src, npar, space, psi, 1)
    pos = {int(k[0]): i for i, k in enumerate(space)}
    for s in range(npar):
        exact = sum((Fraction(float(hij[r]) * float(psi[pos[int(keys[r, 0])]])) for r in range(n) if src[r] == s),
                    Fraction(0))
        assert e[s] == float(exact)          # float(Fraction) is correctly rounded
    perm = rng.permutation(n)
    e2, _, _ = energy.contract(keys[perm], hij[perm], src[perm], npar, space, psi, 1)
    assert np.array_equal(e, e2)


def test_missing_keys_counted():
    keys = np.array([[5], [6], [7], [8]], dtype=np.uint64)
    e, miss, _ = energy.contract(keys, [1.0, 2.0, 4.0, 8.0], [0, 0, 1, 1], 2, keys[::2], np.array([1.0, 1.0]), 1)
    assert miss == 2 and e[0] == 1.0 and e[1] == 4.0


@pytest.mark.parametrize("j0", [0, 37, 224])
def test_delta_psi_gives_matrix_elements(j0):
    """psi = delta_{j0} over the LiH full space: e[s] = H_{s, j0} (0 if j0 is
    not coupled to s), which also equals H_{j0, s} (bit-exact Hermiticity)."""
    wl, ints, par = synth.workload_inputs("lih")
    rec = oracle.gen_coupled(wl.m, wl.n_alpha, wl.n_beta, par, ints, 0.0)
    psi = np.zeros(len(par))
    psi[j0] = 1.0
    e, miss, _ = energy.contract(rec["keys"], rec["hij"], rec["src"], len(par), par, psi, 1)
    assert miss == 0
    row = {int(k[0]): h for k, h, s in zip(rec["keys"], rec["hij"], rec["src"]) if s == j0}
    for s in range(len(par)):
        sel = (rec["src"] == s) & (rec["keys"][:, 0] == par[j0, 0])
        h_s_j0 = float(rec["hij"][sel][0]) if sel.any() else 0.0
        assert e[s] == h_s_j0
        assert e[s] == row.get(int(par[s, 0]), 0.0)


@pytest.mark.parametrize("g", [1, 4])
def test_against_bruteforce_hamiltonian(g):
    """e = (H - diag H) psi over the full LiH Sz = 0 space, H from explicit
    second-quantised operators (tests/fock.py), psi random."""
    K, na, nb = 6, 2, 2
    ints = synth.make_integrals(K, g, 0x5EED0000 + g)
    e4 = fock.full_eri_from_factors(ints.factors, K)
    par = synth.full_space(K, na, nb)
    rng = np.random.default_rng(g)
    psi = rng.uniform(-1, 1, size=len(par))
    rec = oracle.gen_coupled(2 * K, na, nb, par, ints, 0.0)
    e, miss, ab = energy.contract(rec["keys"], rec["hij"], rec["src"], len(par), par, psi, 1)
    assert miss == 0
    idx = {int(k[0]): i for i, k in enumerate(par)}
    for s, p in enumerate(par):
        ket = fock.key_to_int(p)
        col = fock.apply_H(ket, ints.h, e4, list(range(K)))   # H|s> = sum_j <j|H|s> |j>, H real symmetric
        ref = math.fsum(v * psi[idx[j]] for j, v in col.items() if j != ket)
        scale = math.fsum(abs(v * psi[idx[j]]) for j, v in col.items() if j != ket)
        assert abs(e[s] - ref) <= 1e-12 * max(scale, 1e-300), (s, e[s], ref)
        assert ab[s] == pytest.approx(scale, rel=1e-12, abs=1e-14)
