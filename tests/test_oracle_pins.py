"""Pins for the oracle (oracle/oracle.cpp) against things other than itself:
the paper's / SPEC's printed examples, closed-form counts, a brute-force
second-quantised Hamiltonian, bit-exact Hermiticity, the LiH closure, and
std::set-free set algebra.  CPU only (-m "not gpu")."""
import json
import os
from itertools import combinations
from math import comb

import numpy as np
import pytest

import oracle
import synth
from tests import fock

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------- SPEC examples
def test_render_paper_example():
    for e in GOLD["render"]:
        occ = np.zeros((1, e["m"]), dtype=bool)
        occ[0, e["occupied"]] = True
        assert synth.render(synth.occ_to_keys(occ, e["m"])[0], e["m"]) == e["text"]
        assert synth.render(synth.parse(e["text"]), e["m"]) == e["text"]


@pytest.mark.parametrize("e", GOLD["apply_single"], ids=lambda e: e["cite"])
def test_apply_single_spec(e):
    out, par = oracle.apply_single(synth.parse(e["c"]), e["p"], e["a"])
    assert synth.render(out, len(e["c"])) == e["result"]
    assert par == e["parity"]


@pytest.mark.parametrize("e", GOLD["apply_double"], ids=lambda e: e["cite"])
def test_apply_double_spec(e):
    out, par = oracle.apply_double(synth.parse(e["c"]), e["p"], e["q"], e["a"], e["b"])
    assert synth.render(out, len(e["c"])) == e["result"]
    assert par == e["parity"]


def test_apply_invalid():
    with pytest.raises(ValueError):
        oracle.apply_single(synth.parse("1100"), 2, 3)   # p unoccupied
    with pytest.raises(ValueError):
        oracle.apply_double(synth.parse("1100"), 0, 1, 1, 3)  # a occupied


def test_apply_single_twice_restores():
    # p->a then a->p restores c with parity product +1 (m up to 128)
    rng = np.random.default_rng(1)
    for m in (8, 64, 100, 128):
        W = synth.words_for(m)
        for _ in range(200):
            occ = np.zeros((1, m), dtype=bool)
            occ[0, rng.choice(m, m // 3, replace=False)] = True
            c = synth.occ_to_keys(occ, m)[0]
            p = int(rng.choice(np.nonzero(occ[0])[0]))
            a = int(rng.choice(np.nonzero(~occ[0])[0]))
            c1, s1 = oracle.apply_single(c, p, a)
            c2, s2 = oracle.apply_single(c1, a, p)
            assert np.array_equal(c2, c) and s1 * s2 == 1
            assert len(c1) == W


# ---------------------------------------------------------------- closed forms
def closed_form(K, na, nb):
    va, vb = K - na, K - nb
    singles = na * va + nb * vb
    same = comb(na, 2) * comb(va, 2) + comb(nb, 2) * comb(vb, 2)
    opp = na * va * nb * vb
    return singles + same + opp


@pytest.mark.parametrize("K,na,nb,npar,expect", [
    (6, 2, 2, 225, 92),          # LiH-like, full space (16 + 12 + 64)
    (13, 5, 5, 20, 2240),        # H2O-like dense
    (6, 3, 1, 20, None),         # open shell
    (28, 7, 7, 2, 30723),        # N2-like dense
    (48, 8, 8, 1, 146720),       # C2H4-like dense, W = 2
])
def test_closed_form_counts(K, na, nb, npar, expect):
    ints = synth.make_integrals(K, 1, 11 + K)          # dense: no accidental zeros
    if K == 6 and npar == 225:
        par = synth.full_space(K, na, nb)
    else:
        par = synth.hf_ball_parents(K, na, nb, npar, 1, 99 + K)
    r = oracle.gen_coupled(2 * K, na, nb, par, ints, 0.0)
    cf = closed_form(K, na, nb)
    if expect is not None:
        assert cf == expect
    counts = np.bincount(r["src"], minlength=len(par))
    assert np.all(counts == cf)


@pytest.mark.slow
def test_closed_form_m120():
    K, n = 60, 12
    ints = synth.make_integrals(K, 1, 5)
    par = synth.hf_ball_parents(K, n, n, 1, 1, 5)
    r = oracle.gen_coupled(2 * K, n, n, par, ints, 0.0)
    assert len(r["src"]) == closed_form(K, n, n) == 481824


# ---------------------------------------------------------------- brute force
def _embedded_integrals(K_full, active, g, seed):
    """Integrals on K_full spatial orbitals, nonzero only on `active`."""
    small = synth.make_integrals(len(active), g, seed)
    h = np.zeros((K_full, K_full))
    for i, P in enumerate(active):
        for j, Q in enumerate(active):
            h[P, Q] = small.h[i, j]
    npair = K_full * (K_full + 1) // 2
    eri = np.zeros(npair * (npair + 1) // 2)
    e4s = fock.full_eri_from_factors(small.factors, len(active))
    e4 = np.zeros((K_full,) * 4)
    ia = np.array(active)
    e4[np.ix_(ia, ia, ia, ia)] = e4s
    # packed copy of the SAME small ERI values (read from small.eri, the packed generator output)
    for i, P in enumerate(active):
        for j, Q in enumerate(active):
            for k, R in enumerate(active):
                for l, S in enumerate(active):
                    eri[synth.eri_index(P, Q, R, S)] = small.eri[synth.eri_index(i, j, k, l)]
    ints = synth.Integrals(K_full, g, h, eri, None, seed)
    return ints, e4


def _check_against_bruteforce(m, na, nb, parents, ints, e4, active, eps=0.0):
    W = parents.shape[1]
    r = oracle.gen_coupled(m, na, nb, parents, ints, eps)
    n_checked = 0
    for s, par in enumerate(parents):
        ket = fock.key_to_int(par)
        col = fock.apply_H(ket, ints.h, e4, active)
        brute = {j: v for j, v in col.items() if j != ket and abs(v) > 1e-12}
        sel = np.nonzero(r["src"] == s)[0]
        got = {fock.key_to_int(r["keys"][x]): (r["hij"][x], r["phase"][x]) for x in sel}
        assert set(got) == set(brute), f"coupled set differs for parent {s}"
        for j, (H, ph) in got.items():
            assert abs(H - brute[j]) <= 1e-12 * max(1.0, abs(brute[j])), (s, j, H, brute[j])
            assert ph in (-1, 1)
            n_checked += 1
        assert len(r["keys"][sel]) == len(got)
        assert all(len(k) == W for k in r["keys"][sel])
    return n_checked


@pytest.mark.parametrize("K,na,nb,g", [(4, 2, 2, 1), (4, 2, 1, 1), (5, 3, 2, 2), (6, 2, 2, 1), (6, 2, 2, 4)])
def test_bruteforce_fock_full_space(K, na, nb, g):
    """Every record of the full Sz sector equals <j|H|i> from explicit operators."""
    ints = synth.make_integrals(K, g, 1000 + K + g)
    e4 = fock.full_eri_from_factors(ints.factors, K)
    par = synth.full_space(K, na, nb)
    if len(par) > 120:
        par = par[:: max(1, len(par) // 120)]
    n = _check_against_bruteforce(2 * K, na, nb, par, ints, e4, list(range(K)))
    assert n > 0


def test_bruteforce_across_word_boundary():
    """m = 128 (W = 2): active spatial orbitals straddle spin-orbital 64, with
    frozen electrons in between (their Jordan-Wigner signs still count)."""
    K_full = 64
    active = [3, 21, 31, 32, 33, 50, 63]
    ints, e4 = _embedded_integrals(K_full, active, 1, 4242)
    rng = np.random.default_rng(5)
    m = 2 * K_full
    parents = []
    for _ in range(12):
        occ = np.zeros(m, dtype=bool)
        # frozen electrons on inactive orbitals
        inactive = [t for t in range(m) if t // 2 not in active]
        occ[rng.choice(inactive, 20, replace=False)] = True
        # 3 alpha + 3 beta active electrons
        occ[[2 * P for P in rng.choice(active, 3, replace=False)]] = True
        occ[[2 * P + 1 for P in rng.choice(active, 3, replace=False)]] = True
        parents.append(occ)
    par = synth.occ_to_keys(np.array(parents), m)
    na = int(synth.keys_to_occ(par, m)[0, 0::2].sum())
    nb = int(synth.keys_to_occ(par, m)[0, 1::2].sum())
    n = _check_against_bruteforce(m, na, nb, par, ints, e4, active)
    assert n > 50


# ---------------------------------------------------------------- Hermiticity / closure
@pytest.mark.parametrize("g", [1, 4])
def test_lih_hermiticity_bit_exact_and_closure(g):
    K, na, nb = 6, 2, 2
    ints = synth.make_integrals(K, g, 0x5EED0000)
    par = synth.full_space(K, na, nb)
    r = oracle.gen_coupled(12, na, nb, par, ints, 0.0)
    idx = {int(k[0]): s for s, k in enumerate(par)}
    table = {(int(r["src"][x]), idx[int(r["keys"][x, 0])]): r["hij"][x] for x in range(len(r["src"]))}
    for (i, j), H in table.items():
        assert table[(j, i)] == H            # bit-exact H_ij = H_ji (reading r5)
    if g == 1:
        assert len(r["src"]) == 20700         # 225 x 92 (SURVEY 8(c) pins)
        u, mult = np.unique(r["keys"][:, 0], return_counts=True)
        assert len(u) == 225 and np.all(mult == 92)
        assert np.array_equal(oracle.dedup(r["keys"], 1), par)


def test_h2o_hermiticity_sampled():
    """Records whose target is also a parent: H(i->j) == H(j->i) bit-exactly."""
    wl, ints, par = synth.workload_inputs("h2o", n_parents=400)
    r = oracle.gen_coupled(wl.m, wl.n_alpha, wl.n_beta, par, ints, 0.0)
    idx = {int(k[0]): s for s, k in enumerate(par)}
    table = {}
    for x in range(len(r["src"])):
        j = idx.get(int(r["keys"][x, 0]))
        if j is not None:
            table[(int(r["src"][x]), j)] = r["hij"][x]
    assert len(table) > 100
    for (i, j), H in table.items():
        assert table[(j, i)] == H


# ---------------------------------------------------------------- screening
def test_threshold_monotone_and_limits():
    wl, ints, par = synth.workload_inputs("h2o", n_parents=50)
    r0 = oracle.gen_coupled(wl.m, 5, 5, par, ints, 0.0)
    assert np.all(np.abs(r0["hij"]) > 0)
    prev = None
    for eps in (0.0, 1e-6, 1e-4, 1e-3, 1e-2):
        r = oracle.gen_coupled(wl.m, 5, 5, par, ints, eps)
        assert np.all(np.abs(r["hij"]) > eps)
        s = set(zip(r["src"].tolist(), r["keys"][:, 0].tolist()))
        if prev is not None:
            assert s <= prev
        # records above eps are exactly the eps=0 records with |H| > eps
        ref = set((int(a), int(b)) for a, b, h in zip(r0["src"], r0["keys"][:, 0], r0["hij"]) if abs(h) > eps)
        assert s == ref
        prev = s
    r_inf = oracle.gen_coupled(wl.m, 5, 5, par, ints, float("inf"))
    assert len(r_inf["src"]) == 0


def test_point_group_zeros_drop_out():
    """g = 4: every record of a totally symmetric parent is totally symmetric,
    and fewer records than the dense closed form survive."""
    wl, ints, par = synth.workload_inputs("h2o", n_parents=30)
    r = oracle.gen_coupled(wl.m, 5, 5, par, ints, 0.0)
    occ = synth.keys_to_occ(r["keys"], wl.m)
    irr = (np.arange(wl.m) // 2) % 4
    sym = np.bitwise_xor.reduce(np.where(occ, irr[None, :], 0), axis=1)
    assert np.all(sym == 0)
    assert len(r["src"]) < 30 * closed_form(13, 5, 5)


# ---------------------------------------------------------------- validation
def test_validate_parents():
    wl, ints, par = synth.workload_inputs("h2o", n_parents=10)
    assert oracle.validate(26, 5, 5, par) == -1
    bad = par.copy()
    bad[3, 0] |= np.uint64(1 << 30)           # bit >= m
    assert oracle.validate(26, 5, 5, bad) == 3
    bad = par.copy()
    bad[7, 0] ^= np.uint64(1)                # wrong alpha count
    assert oracle.validate(26, 5, 5, bad) == 7


# ---------------------------------------------------------------- dedup / owner / merge
def _np_owner(keys, W, P):
    """owner(j) = floor(mix(j) P / 2^64), mix per DESIGN.md reading r9 (Python ints)."""
    M = (1 << 64) - 1

    def fm(x):
        x ^= x >> 30
        x = (x * 0xBF58476D1CE4E5B9) & M
        x ^= x >> 27
        x = (x * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)
    out = []
    for k in keys:
        mix = fm(int(k[0])) if W == 1 else fm(int(k[0]) ^ fm(int(k[1]) ^ 0x9E3779B97F4A7C15))
        out.append((mix * P) >> 64)
    return np.array(out)


@pytest.mark.parametrize("W", [1, 2])
def test_dedup_against_sort_unique_and_owners(W):
    keys = synth.zipf_keys(200_000, W, 1.1, 1 << 15, seed=3 + W)
    u_all = oracle.dedup(keys, W, 1, 0)
    ref = synth.unique_keys(keys)
    assert np.array_equal(u_all, ref)
    for P in (2, 4, 8):
        shards = [oracle.dedup(keys, W, P, r) for r in range(P)]
        cat = np.concatenate(shards)
        assert len(cat) == len(ref)                       # disjoint + complete
        assert np.array_equal(synth.unique_keys(cat), ref)
        for r, sh in enumerate(shards):
            assert np.array_equal(sh, synth.sort_keys(sh))    # each shard sorted
            if len(sh):
                assert np.all(_np_owner(sh[:2000], W, P) == r)
        assert np.array_equal(oracle.owner(ref[:3000], W, P), _np_owner(ref[:3000], W, P))


def test_dedup_empty():
    assert len(oracle.dedup(np.zeros((0, 1), dtype=np.uint64), 1)) == 0


@pytest.mark.parametrize("W", [1, 2])
def test_merge_set_algebra(W):
    rng = np.random.default_rng(9)
    A = synth.unique_keys(rng.integers(1, 5000, size=(3000, W), dtype=np.uint64))
    B = synth.unique_keys(rng.integers(1, 5000, size=(2000, W), dtype=np.uint64))
    S2, ins = oracle.merge(A, B, W)
    sa = set(map(tuple, A.tolist()))
    sb = set(map(tuple, B.tolist()))
    assert set(map(tuple, S2.tolist())) == sa | sb
    assert set(map(tuple, ins.tolist())) == sb - sa
    assert len(S2) == len(A) + len(ins)
    assert np.array_equal(S2, synth.sort_keys(S2)) and np.array_equal(ins, synth.sort_keys(ins))
    S3, ins2 = oracle.merge(S2, B, W)                      # idempotence
    assert np.array_equal(S3, S2) and len(ins2) == 0
    S4, ins4 = oracle.merge(np.zeros((0, W), np.uint64), B, W)
    assert np.array_equal(S4, B) and np.array_equal(ins4, B)


def test_lih_merge_inserts_nothing():
    K = 6
    ints = synth.make_integrals(K, 1, 0x5EED0000)
    par = synth.full_space(K, 2, 2)
    r = oracle.gen_coupled(12, 2, 2, par, ints, 0.0)
    U = oracle.dedup(r["keys"], 1)
    S2, ins = oracle.merge(par, U, 1)
    assert len(ins) == 0 and np.array_equal(S2, par)
