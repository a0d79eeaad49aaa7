"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no excitation enumeration,
no Slater-Condon rule, no phase, no dedup): it only draws input data --
integrals and parent determinants -- with the shapes and structure of the
paper's workloads.  Recipe: SURVEY.md section 8(d), restated in DESIGN.md
"Input recipe".

Conventions shared by every consumer (DESIGN.md "Readings" r1-r3):
  * spin orbital t = 2*P + sigma (interleaved; sigma 0 = alpha, 1 = beta);
    P = t // 2 is the spatial index.
  * a determinant is W = 1 (m <= 64) or W = 2 (m <= 128) uint64 words;
    orbital t lives in word t // 64, bit t % 64.
  * keys are compared as one big unsigned integer, word W-1 most significant.
  * integrals: h is a dense symmetric K*K float64 array; the two-electron
    integrals (PQ|RS) (chemist notation) are stored 8-fold packed:
        ij  = max(P,Q)*(max(P,Q)+1)/2 + min(P,Q)
        idx = max(ij,kl)*(max(ij,kl)+1)/2 + min(ij,kl)
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15


# ----------------------------------------------------------------------------
# counter-based splitmix64 stream (vectorised): value i = mix(seed + (i+1)*gamma)
# ----------------------------------------------------------------------------
def splitmix64_stream(seed: int, count: int, start: int = 0) -> np.ndarray:
    i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & MASK64) + i * np.uint64(GOLDEN_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_pm1(seed: int, count: int, start: int = 0) -> np.ndarray:
    """u ~ U(-1, 1) from the top 53 bits of the splitmix64 stream."""
    z = splitmix64_stream(seed, count, start)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0


# ----------------------------------------------------------------------------
# integrals
# ----------------------------------------------------------------------------
def pair_index(p: int, q: int) -> int:
    hi, lo = (p, q) if p >= q else (q, p)
    return hi * (hi + 1) // 2 + lo


def eri_index(p: int, q: int, r: int, s: int) -> int:
    return pair_index(pair_index(p, q), pair_index(r, s))


@dataclass
class Integrals:
    n_spatial: int          # K
    g: int                  # number of irreps of the synthetic point group (1 = dense)
    h: np.ndarray           # float64 [K, K], symmetric
    eri: np.ndarray         # float64 [npair*(npair+1)/2], 8-fold packed (PQ|RS)
    factors: np.ndarray     # float64 [2K, npair]: B^L_{PQ} (packed pair index); eri = sum_L B B
    seed: int

    @property
    def irreps(self) -> np.ndarray:
        return np.arange(self.n_spatial) % self.g


def make_integrals(K: int, g: int = 1, seed: int = 0x5EED0000) -> Integrals:
    """Synthetic 8-fold-symmetric real integrals G(K, g, seed).

    e_P = -2 + 2.5 P/(K-1);  h_PQ = e_P d_PQ + 0.05 u exp(-|P-Q|/3), zero unless
    irrep(P) xor irrep(Q) = 0;  (PQ|RS) = sum_{L<2K} B^L_PQ B^L_RS with
    B^L_PQ = u exp(-|P-Q|/4)/sqrt(2K), zero unless irrep(P) xor irrep(Q) = L mod g.
    Irreps are P mod g (g a power of two, XOR product).  u values are drawn in
    the fixed order: h for P >= Q (row-major), then B for P >= Q, L ascending.
    The ERI is accumulated over L ascending in float64 (exact products, adds
    in a fixed order), so both sides of every parity test read identical bits.
    """
    assert g in (1, 2, 4, 8), "g must be a power of two <= 8"
    assert K >= 2
    gam = np.arange(K) % g
    npair = K * (K + 1) // 2
    P_idx = np.array([p for p in range(K) for q in range(p + 1)])
    Q_idx = np.array([q for p in range(K) for q in range(p + 1)])
    # one-electron
    u_h = uniform_pm1(seed, npair, 0)
    e = -2.0 + 2.5 * np.arange(K) / (K - 1)
    h = np.zeros((K, K))
    dist = np.abs(P_idx - Q_idx).astype(np.float64)
    hv = 0.05 * u_h * np.exp(-dist / 3.0)
    hv = np.where(P_idx == Q_idx, e[P_idx] + hv, hv)
    hv = np.where((gam[P_idx] ^ gam[Q_idx]) == 0, hv, 0.0)
    h[P_idx, Q_idx] = hv
    h[Q_idx, P_idx] = hv
    # two-electron factors
    nL = 2 * K
    u_b = uniform_pm1(seed, npair * nL, npair).reshape(npair, nL)  # P>=Q major, L minor
    scale = np.exp(-dist / 4.0) / math.sqrt(2 * K)
    B = (u_b * scale[:, None]).T.copy()  # [L, pair]
    sym_ok = ((gam[P_idx] ^ gam[Q_idx])[None, :] == (np.arange(nL) % g)[:, None])
    B = np.where(sym_ok, B, 0.0)
    M = np.zeros((npair, npair))
    for L in range(nL):          # L ascending: fixed accumulation order
        b = B[L]
        M += np.multiply.outer(b, b)
    rows, cols = np.tril_indices(npair)
    eri = np.zeros(npair * (npair + 1) // 2)
    eri[rows * (rows + 1) // 2 + cols] = M[rows, cols]
    return Integrals(K, g, h, eri, B, seed)


# ----------------------------------------------------------------------------
# determinants
# ----------------------------------------------------------------------------
def words_for(m: int) -> int:
    assert 2 <= m <= 128
    return 1 if m <= 64 else 2


def occ_to_keys(occ: np.ndarray, m: int) -> np.ndarray:
    """occ: bool [N, m] (spin-orbital occupancy) -> uint64 [N, W]."""
    W = words_for(m)
    N = occ.shape[0]
    out = np.zeros((N, W), dtype=np.uint64)
    for t in range(m):
        out[:, t // 64] |= occ[:, t].astype(np.uint64) << np.uint64(t % 64)
    return out


def keys_to_occ(keys: np.ndarray, m: int) -> np.ndarray:
    keys = np.asarray(keys, dtype=np.uint64).reshape(len(keys), -1)
    occ = np.zeros((keys.shape[0], m), dtype=bool)
    for t in range(m):
        occ[:, t] = ((keys[:, t // 64] >> np.uint64(t % 64)) & np.uint64(1)).astype(bool)
    return occ


def sort_keys(keys: np.ndarray) -> np.ndarray:
    """Sort uint64 [N, W] rows by the big-integer order (word W-1 most significant)."""
    keys = np.asarray(keys, dtype=np.uint64)
    order = np.lexsort(tuple(keys[:, w] for w in range(keys.shape[1])))
    return keys[order]


def unique_keys(keys: np.ndarray) -> np.ndarray:
    """Sorted unique rows (big-integer order)."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    if len(keys) == 0:
        return keys.reshape(0, keys.shape[1] if keys.ndim == 2 else 1)
    s = sort_keys(keys)
    keep = np.ones(len(s), dtype=bool)
    keep[1:] = np.any(s[1:] != s[:-1], axis=1)
    return s[keep]


def render(key, m: int) -> str:
    """Text form: orbital 0 is the leftmost character."""
    words = [int(x) for x in np.atleast_1d(np.asarray(key, dtype=np.uint64))]
    return "".join("1" if (words[t // 64] >> (t % 64)) & 1 else "0" for t in range(m))


def parse(text: str) -> np.ndarray:
    m = len(text)
    W = words_for(m)
    w = [0] * W
    for t, c in enumerate(text):
        if c == "1":
            w[t // 64] |= 1 << (t % 64)
        elif c != "0":
            raise ValueError("bitstring must contain only 0/1")
    return np.array(w, dtype=np.uint64)


def full_space(K: int, n_alpha: int, n_beta: int) -> np.ndarray:
    """All determinants with n_alpha / n_beta electrons, sorted (e.g. LiH: 225;
    H2O-like K = 13, 5/5: 1,656,369)."""
    from itertools import combinations
    m = 2 * K
    if m <= 64:   # vectorised: every alpha string OR every beta string
        a = np.array([sum(1 << (2 * P) for P in c) for c in combinations(range(K), n_alpha)], dtype=np.uint64)
        b = np.array([sum(1 << (2 * P + 1) for P in c) for c in combinations(range(K), n_beta)], dtype=np.uint64)
        return np.sort((a[:, None] | b[None, :]).reshape(-1)).reshape(-1, 1)
    rows = []
    for ca in combinations(range(K), n_alpha):
        for cb in combinations(range(K), n_beta):
            occ = np.zeros(m, dtype=bool)
            occ[[2 * P for P in ca]] = True
            occ[[2 * P + 1 for P in cb]] = True
            rows.append(occ)
    return sort_keys(occ_to_keys(np.array(rows), m))


LEVEL_WEIGHTS = (0.001, 0.05, 0.45, 0.20, 0.30)
_HERE = os.path.dirname(os.path.abspath(__file__))
_SAMPLER_SO = os.path.join(_HERE, "_sampler.so")
_sampler = None


def build_sampler(force: bool = False) -> str:
    src = os.path.join(_HERE, "sampler.c")
    if force or not os.path.exists(_SAMPLER_SO) or os.path.getmtime(_SAMPLER_SO) < os.path.getmtime(src):
        tmp = _SAMPLER_SO + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, src, "-lm"])
        os.replace(tmp, _SAMPLER_SO)
    return _SAMPLER_SO


def _lib():
    global _sampler
    if _sampler is None:
        lib = ctypes.CDLL(build_sampler())
        lib.synth_hf_ball.restype = ctypes.c_longlong
        lib.synth_hf_ball.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_longlong, ctypes.c_uint64, ctypes.c_double,
                                      ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p]
        _sampler = lib
    return _sampler


def hf_ball_parents(K: int, n_alpha: int, n_beta: int, n_parents: int, g: int = 1,
                    seed: int = 0xFA7E0000, tau: float | None = None,
                    level_weights=LEVEL_WEIGHTS, max_draws: int = 1 << 34) -> np.ndarray:
    """HF-ball sampler; the draw loop is in synth/sampler.c (see
    its header for the recipe).  tau = K/8 by default.  Returns the first
    n_parents distinct determinants in draw order, sorted: uint64 [n_parents, W]."""
    tau = K / 8.0 if tau is None else float(tau)
    W = words_for(2 * K)
    out = np.zeros((n_parents, W), dtype=np.uint64)
    lw = np.ascontiguousarray(level_weights, dtype=np.float64)
    got = _lib().synth_hf_ball(K, n_alpha, n_beta, g, n_parents, seed & MASK64, tau,
                               lw.ctypes.data, len(lw), max_draws, out.ctypes.data)
    if got < n_parents:
        raise RuntimeError(f"hf_ball_parents: only {got} distinct determinants found")
    return sort_keys(out)


# ----------------------------------------------------------------------------
# the five BASELINE.json workloads
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Workload:
    name: str
    K: int
    n_alpha: int
    n_beta: int
    g: int
    n_parents: int     # 0 = full space
    config_no: int

    @property
    def m(self) -> int:
        return 2 * self.K

    @property
    def words(self) -> int:
        return words_for(self.m)


WORKLOADS = {
    "lih": Workload("LiH-like", 6, 2, 2, 1, 0, 0),
    "lih_g4": Workload("LiH-like (g=4)", 6, 2, 2, 4, 0, 0),
    "h2o": Workload("H2O-like", 13, 5, 5, 4, 10_000, 1),
    "h2o_dense": Workload("H2O-like (dense)", 13, 5, 5, 1, 10_000, 1),
    "n2": Workload("N2 cc-pVDZ-like", 28, 7, 7, 8, 1_000_000, 2),
    "c2h4": Workload("C2H4-like", 48, 8, 8, 8, 10_000_000, 3),
    "m120": Workload("large-active-space m=120", 60, 12, 12, 8, 1_700, 4),
}


def workload_inputs(key: str, n_parents: int | None = None):
    """(Workload, Integrals, parents uint64 [N, W]) for a named workload."""
    wl = WORKLOADS[key]
    ints = make_integrals(wl.K, wl.g, 0x5EED0000 + wl.config_no)
    if wl.n_parents == 0:
        par = full_space(wl.K, wl.n_alpha, wl.n_beta)
    else:
        n = wl.n_parents if n_parents is None else n_parents
        par = hf_ball_parents(wl.K, wl.n_alpha, wl.n_beta, n, wl.g, 0xFA7E0000 + wl.config_no)
    return wl, ints, par


def zipf_keys(n: int, W: int, theta: float = 1.1, universe: int = 1 << 20, seed: int = 7) -> np.ndarray:
    """Zipf(theta)-distributed random keys (SPEC S:332 dedup stress): a universe of
    random 64W-bit keys, drawn with Zipf weights.  Keys are never 0."""
    rng = np.random.Generator(np.random.PCG64(seed))
    base = rng.integers(1, 2**63, size=(universe, W), dtype=np.uint64, endpoint=False)
    base |= np.uint64(1)
    ranks = np.arange(1, universe + 1, dtype=np.float64)
    p = ranks ** (-theta)
    p /= p.sum()
    idx = rng.choice(universe, size=n, p=p)
    return base[idx]
