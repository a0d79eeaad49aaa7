"""GPU parity: the CUDA path (through the C ABI, paper_2604_15768_b200) against
the oracle, element by element on the same seeded inputs.

Bar (BASELINE.json north_star): configuration sets, counts and phases
bit-exact; H_ij within 1e-12 relative (we also assert the expected exact
equality, reading r5)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2604_15768_b200 as P
    return P


@pytest.fixture(scope="module")
def ctx(P):
    c = P.Context(0)
    yield c
    c.close()


def fmix64(x):
    x = np.asarray(x, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


def hash_hi_lo(keys, W):
    """Hash order pi(j) = (hi, lo) (reading r13), written from its definition."""
    keys = np.asarray(keys, dtype=np.uint64).reshape(-1, W)
    if W == 1:
        return fmix64(keys[:, 0]), np.zeros(len(keys), dtype=np.uint64)
    lo = fmix64(keys[:, 1] ^ np.uint64(0x9E3779B97F4A7C15))
    return fmix64(keys[:, 0] ^ lo), lo


def hash_sort(keys, W):
    keys = np.asarray(keys, dtype=np.uint64).reshape(-1, W)
    hi, lo = hash_hi_lo(keys, W)
    return keys[np.lexsort((lo, hi))]


def assert_hash_sorted_unique(keys, W):
    hi, lo = hash_hi_lo(keys, W)
    if len(hi) > 1:
        assert np.all((hi[1:] > hi[:-1]) | ((hi[1:] == hi[:-1]) & (lo[1:] > lo[:-1]))), "not strictly in hash order"


def canon(keys, src, *cols):
    """sort records by (src, key big-integer)"""
    keys = np.asarray(keys).reshape(len(keys), -1)
    order = np.lexsort(tuple(keys[:, w] for w in range(keys.shape[1])) + (np.asarray(src),))
    return (keys[order], np.asarray(src)[order]) + tuple(np.asarray(c)[order] for c in cols)


def run_gen(P, ctx, wl_m, na, nb, par, ints, eps):
    sp = P.Space(wl_m, na, nb)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    tpar = torch.from_numpy(par.astype(np.uint64)).cuda()
    rec = ctx.gen_coupled(sp, tpar, di, eps, with_src=True, with_phase=True)
    torch.cuda.synchronize()
    return (rec.keys.cpu().numpy(), rec.src.cpu().numpy().astype(np.uint32), rec.hij.cpu().numpy(),
            rec.phase.cpu().numpy())


def assert_gen_parity(P, ctx, m, na, nb, par, ints, eps=0.0):
    g_keys, g_src, g_h, g_ph = run_gen(P, ctx, m, na, nb, par, ints, eps)
    ref = oracle.gen_coupled(m, na, nb, par, ints, eps)
    assert len(g_src) == len(ref["src"]), "record counts differ"
    gk, gs, gh, gp = canon(g_keys, g_src, g_h, g_ph)
    rk, rs, rh, rp = canon(ref["keys"], ref["src"], ref["hij"], ref["phase"])
    assert np.array_equal(gs, rs) and np.array_equal(gk, rk), "coupled sets differ"
    assert np.array_equal(gp, rp), "phases differ"
    rel = np.abs(gh - rh) / np.maximum(np.abs(rh), 1e-300)
    assert np.all(rel <= 1e-12), f"max rel err {rel.max()}"
    assert np.array_equal(gh, rh), "H not bit-identical (expected under reading r5)"
    # per-parent counts
    assert np.array_equal(np.bincount(gs, minlength=len(par)), np.bincount(rs, minlength=len(par)))
    return len(gs)


@pytest.mark.parametrize("key", ["lih", "lih_g4"])
def test_gen_lih_full_space(P, ctx, key):
    wl, ints, par = synth.workload_inputs(key)
    n = assert_gen_parity(P, ctx, wl.m, wl.n_alpha, wl.n_beta, par, ints)
    if key == "lih":
        assert n == 20700


def test_gen_h2o_10k(P, ctx):
    wl, ints, par = synth.workload_inputs("h2o")
    assert len(par) == 10_000
    assert_gen_parity(P, ctx, wl.m, wl.n_alpha, wl.n_beta, par, ints)


def test_gen_h2o_dense_and_threshold(P, ctx):
    wl, ints, par = synth.workload_inputs("h2o_dense", n_parents=2000)
    n0 = assert_gen_parity(P, ctx, wl.m, 5, 5, par, ints, 0.0)
    assert n0 == 2000 * 2240
    assert_gen_parity(P, ctx, wl.m, 5, 5, par, ints, 1e-4)
    assert_gen_parity(P, ctx, wl.m, 5, 5, par, ints, 3e-3)


def test_gen_open_shell(P, ctx):
    ints = synth.make_integrals(9, 2, 77)
    par = synth.hf_ball_parents(9, 4, 2, 500, 1, 78)
    assert_gen_parity(P, ctx, 18, 4, 2, par, ints)


def test_gen_n2_prefix_and_sample(P, ctx):
    wl, ints, par = synth.workload_inputs("n2", n_parents=20_000)
    rng = np.random.default_rng(0)
    sel = np.sort(rng.choice(len(par), 300, replace=False))
    assert_gen_parity(P, ctx, wl.m, 7, 7, par[:200], ints)
    assert_gen_parity(P, ctx, wl.m, 7, 7, par[sel], ints)


def test_gen_c2h4_w2(P, ctx):
    wl, ints, par = synth.workload_inputs("c2h4", n_parents=2000)
    rng = np.random.default_rng(1)
    sel = np.sort(rng.choice(len(par), 60, replace=False))
    assert_gen_parity(P, ctx, wl.m, 8, 8, par[sel], ints)


def test_gen_m120_w2(P, ctx):
    wl, ints, par = synth.workload_inputs("m120", n_parents=40)
    assert_gen_parity(P, ctx, wl.m, 12, 12, par[:12], ints)


@pytest.mark.parametrize("eps", [1e-6, 1e-4])
def test_gen_w2_threshold(P, ctx, eps):
    """W = 2 screening (a6) at eps > 0: C2H4-like and m = 120 samples."""
    wl, ints, par = synth.workload_inputs("c2h4", n_parents=2000)
    rng = np.random.default_rng(7)
    sel = np.sort(rng.choice(len(par), 40, replace=False))
    n_eps = assert_gen_parity(P, ctx, wl.m, 8, 8, par[sel], ints, eps)
    assert n_eps < oracle_count(wl, par[sel], ints, 0.0)
    wl, ints, par = synth.workload_inputs("m120", n_parents=40)
    assert_gen_parity(P, ctx, wl.m, 12, 12, par[:10], ints, eps)


def oracle_count(wl, par, ints, eps):
    return len(oracle.gen_coupled(wl.m, wl.n_alpha, wl.n_beta, par, ints, eps)["src"])


def test_gen_w2_invalid_parents(P, ctx):
    wl, ints, par = synth.workload_inputs("c2h4", n_parents=50)
    sp = P.Space(wl.m, 8, 8)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    for word, bit in ((1, 40), (0, 3)):          # a bit >= m = 96 (word 1, bit 40); a flipped spin
        bad = par.copy()
        bad[31, word] ^= np.uint64(1 << bit)
        with pytest.raises(P.CusciError) as e:
            ctx.gen_coupled_count(sp, torch.from_numpy(bad).cuda(), di, 1e-6)
        assert e.value.code == 2 and "parent 31" in str(e.value)


def test_h2o_full_space_closure(P, ctx):
    """SURVEY 8(c) at-scale pin with no oracle: the dense H2O-like full Sz = 0
    space (C(13,5)^2 = 1,656,369 parents) generates 2,240 x 1,656,369 =
    3.71e9 records whose union is exactly the space, every key reached by
    exactly 2,240 parents (the coupling relation is symmetric), in the
    bench's batched gen -> dedup_global -> merge_space launch configuration."""
    wl, ints, _ = synth.workload_inputs("h2o_dense", n_parents=1)
    par = synth.full_space(13, 5, 5)
    assert len(par) == 1_656_369
    sp = P.Space(26, 5, 5)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    tpar = torch.from_numpy(par).cuda()
    pv = tpar.view(torch.int64).reshape(-1)                 # keys < 2^26: int64 order = key order
    mult = torch.zeros(len(par), dtype=torch.int64, device="cuda")
    pool = ctx.pool(sp, 1 << 21)
    batch = 250_000
    total = 0
    for a in range(0, len(par), batch):
        rec = ctx.gen_coupled(sp, tpar[a:a + batch], di, 0.0, with_src=False)
        total += rec.count
        u = ctx.dedup_global(sp, rec.keys)
        ctx.merge_space(pool, u)
        k = rec.keys.view(torch.int64).reshape(-1)
        idx = torch.searchsorted(pv, k)
        assert bool((pv[idx.clamp(max=len(par) - 1)] == k).all()), "a record outside the Sz = 0 space"
        mult += torch.bincount(idx, minlength=len(par))
        del rec, u, k, idx
    assert total == 2240 * len(par) == 3_710_266_560
    assert bool((mult == 2240).all()), f"multiplicities in [{int(mult.min())}, {int(mult.max())}]"
    got = pool.keys().cpu().numpy()
    assert len(got) == len(par)
    assert_hash_sorted_unique(got, 1)
    assert np.array_equal(synth.sort_keys(got), par)
    pool.close()


def test_gen_m128_dense_word_boundary(P, ctx):
    ints = synth.make_integrals(64, 1, 5)
    par = synth.hf_ball_parents(64, 3, 3, 8, 1, 6)
    assert_gen_parity(P, ctx, 128, 3, 3, par, ints)


# ------------------------------------------------------------------ edge cases / errors
def test_gen_edges_and_errors(P, ctx):
    wl, ints, par = synth.workload_inputs("h2o", n_parents=100)
    sp = P.Space(wl.m, 5, 5)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    tpar = torch.from_numpy(par).cuda()
    # empty
    r = ctx.gen_coupled(sp, tpar[:0], di, 0.0, capacity=10)
    assert r.count == 0
    # eps = inf -> nothing
    assert ctx.gen_coupled_count(sp, tpar, di, float("inf")) == 0
    # capacity overflow then retry
    total = ctx.gen_coupled_count(sp, tpar, di, 0.0)
    with pytest.raises(P.CusciError) as e:
        ctx.gen_coupled(sp, tpar, di, 0.0, capacity=total - 1)
    assert e.value.code == 3
    r = ctx.gen_coupled(sp, tpar, di, 0.0, capacity=total)
    assert r.count == total
    # invalid parent: a bit >= m, wrong spin count
    bad = par.copy()
    bad[17, 0] |= np.uint64(1 << 40)
    with pytest.raises(P.CusciError) as e:
        ctx.gen_coupled(sp, torch.from_numpy(bad).cuda(), di, 0.0, capacity=total)
    assert e.value.code == 2 and "parent 17" in str(e.value)
    bad = par.copy()
    bad[5, 0] ^= np.uint64(1)
    with pytest.raises(P.CusciError) as e:
        ctx.gen_coupled_count(sp, torch.from_numpy(bad).cuda(), di, 0.0)
    assert e.value.code == 2
    # bad arguments
    with pytest.raises(P.CusciError) as e:
        ctx.gen_coupled_count(sp, tpar, di, float("nan"))
    assert e.value.code == 1
    with pytest.raises(P.CusciError) as e:
        ctx.gen_coupled_count(sp, tpar, di, -1.0)
    assert e.value.code == 1
    with pytest.raises(P.CusciError) as e:
        ctx.gen_coupled_count(P.Space(130, 5, 5), tpar, di, 0.0)
    assert e.value.code == 1


def test_gen_full_size_sampled(P, ctx):
    """N2 at the bench's launch configuration (one batch of 125k parents):
    sampled parents compared record by record; properties checked for all."""
    wl, ints, par = synth.workload_inputs("n2", n_parents=125_000)
    sp = P.Space(wl.m, 7, 7)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    tpar = torch.from_numpy(par).cuda()
    rec = ctx.gen_coupled(sp, tpar, di, 0.0, with_src=True)
    src = rec.src.cpu().numpy().astype(np.int64)
    hij = rec.hij.cpu().numpy()
    assert np.all(np.abs(hij) > 0)
    rng = np.random.default_rng(3)
    sel = np.sort(rng.choice(len(par), 40, replace=False))
    ref = oracle.gen_coupled(wl.m, 7, 7, par[sel], ints, 0.0)
    keys = rec.keys.cpu().numpy()
    mask = np.isin(src, sel)
    remap = {int(s): i for i, s in enumerate(sel)}
    g_src = np.array([remap[int(s)] for s in src[mask]], dtype=np.uint32)
    gk, gs, gh = canon(keys[mask], g_src, hij[mask])
    rk, rs, rh = canon(ref["keys"], ref["src"], ref["hij"])
    assert np.array_equal(gk, rk) and np.array_equal(gs, rs) and np.array_equal(gh, rh)


# ------------------------------------------------------------------ dedup
def _dedup_gpu(P, ctx, sp, keys):
    out = ctx.dedup_global(sp, torch.from_numpy(keys).cuda())
    return out.cpu().numpy()


def test_dedup_lih_closure(P, ctx):
    wl, ints, par = synth.workload_inputs("lih")
    sp = P.Space(12, 2, 2)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    rec = ctx.gen_coupled(sp, torch.from_numpy(par).cuda(), di, 0.0)
    u = ctx.dedup_global(sp, rec.keys).cpu().numpy()
    assert_hash_sorted_unique(u, 1)
    assert np.array_equal(synth.sort_keys(u), par)          # 20,700 records -> the 225 parents


@pytest.mark.parametrize("W,n", [(1, 0), (1, 1), (1, 5000), (1, 1_000_003), (2, 700_001)])
def test_dedup_zipf(P, ctx, W, n):
    sp = P.Space(64 * W, 1, 1)
    keys = synth.zipf_keys(max(n, 1), W, 1.1, 1 << 18, seed=11 + W)[:n]
    got = _dedup_gpu(P, ctx, sp, keys).reshape(-1, W)
    ref = oracle.dedup(keys, W)
    assert_hash_sorted_unique(got, W)
    assert np.array_equal(synth.sort_keys(got), ref.reshape(-1, W))


def test_dedup_generated_stream(P, ctx):
    wl, ints, par = synth.workload_inputs("h2o")
    sp = P.Space(wl.m, 5, 5)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    rec = ctx.gen_coupled(sp, torch.from_numpy(par).cuda(), di, 0.0)
    got = ctx.dedup_global(sp, rec.keys).cpu().numpy()
    ref = oracle.dedup(rec.keys.cpu().numpy(), 1)
    assert_hash_sorted_unique(got, 1)
    assert np.array_equal(synth.sort_keys(got), ref)


@pytest.mark.parametrize("W,Pn", [(1, 2), (1, 4), (1, 8), (2, 4)])
def test_dedup_logical_ranks(P, ctx, W, Pn):
    """P logical ranks on one GPU: partition on each rank, exchange by device
    copies in the harness, finalize per owner; compare with the oracle's
    per-owner shards (multi-GPU host logic)."""
    sp = P.Space(64 * W, 1, 1)
    allk = synth.zipf_keys(400_000, W, 1.1, 1 << 16, seed=5)
    parts = np.array_split(allk, Pn)
    bins = []
    for r in range(Pn):
        b, counts = ctx.dedup_partition(sp, torch.from_numpy(parts[r]).cuda(), Pn)
        offs = np.concatenate([[0], np.cumsum(counts)])
        bins.append([b[offs[o]:offs[o + 1]] for o in range(Pn)])
        # each bin holds only its owner's keys, locally unique
        for o in range(Pn):
            kb = bins[r][o].cpu().numpy()
            assert len(np.unique(kb, axis=0)) == len(kb)
            if len(kb):
                assert np.all(oracle.owner(kb, W, Pn) == o)
    total = 0
    for o in range(Pn):
        recv = torch.cat([bins[r][o] for r in range(Pn)])
        ref = oracle.dedup(allk, W, Pn, o)
        got = ctx.dedup_finalize(sp, recv).cpu().numpy().reshape(-1, W)
        assert_hash_sorted_unique(got, W)
        assert np.array_equal(synth.sort_keys(got), ref.reshape(-1, W))
        # the owner-side finalize dedup_global uses: the runs read in place, no partition pass
        got2 = ctx.dedup_finalize_runs(sp, recv, [bins[r][o].shape[0] for r in range(Pn)]).cpu().numpy()
        assert np.array_equal(got2.reshape(-1, W), got)
        total += len(got)
    assert total == len(oracle.dedup(allk, W))


@pytest.mark.parametrize("W,Pn,n", [(1, 3, 3_000_000), (2, 5, 900_001), (1, 8, 20)])
def test_dedup_finalize_runs(P, ctx, W, Pn, n):
    """runs_dedup on runs with heavy overlap (every key on several ranks) and
    empty runs, at sizes spanning many buckets."""
    sp = P.Space(64 * W, 1, 1)
    allk = synth.zipf_keys(n, W, 0.9, 1 << 21, seed=17 + Pn)
    runs = [ctx.dedup_global(sp, torch.from_numpy(allk[r::Pn]).cuda()) for r in range(Pn)]
    runs[1] = runs[1][:0]
    recv = torch.cat(runs)
    got = ctx.dedup_finalize_runs(sp, recv, [x.shape[0] for x in runs]).cpu().numpy().reshape(-1, W)
    keep = np.concatenate([allk[r::Pn] for r in range(Pn) if r != 1]) if Pn > 1 else allk
    assert_hash_sorted_unique(got, W)
    assert np.array_equal(synth.sort_keys(got), oracle.dedup(keep, W).reshape(-1, W))


@pytest.mark.parametrize("W,Pn,n", [(1, 8, 4_000_000), (2, 3, 1_500_000), (1, 6, 2_000_000)])
def test_dedup_finalize_runs_owner_range(P, ctx, W, Pn, n):
    """What dedup_global's owner r receives at P ranks: every rank's bin for
    owner r, i.e. keys from 1/P of the hash space (owner(j) = floor(hi P / 2^64)).
    The finalize must bucket over that range -- the exact slow path (a full
    LSD sort) is not taken -- and give the oracle's set for the owner."""
    sp = P.Space(64 * W, 1, 1)
    allk = synth.zipf_keys(n, W, 0.9, 1 << 22, seed=29 + Pn)
    r_own = Pn // 2
    runs = []
    for r in range(Pn):
        bins, counts = ctx.dedup_partition(sp, torch.from_numpy(allk[r::Pn]).cuda(), Pn)
        off = sum(counts[:r_own])
        runs.append(bins[off:off + counts[r_own]].clone())
    recv = torch.cat(runs)
    ctx.dedup_stats(reset=True)
    got = ctx.dedup_finalize_runs(sp, recv, [x.shape[0] for x in runs]).cpu().numpy().reshape(-1, W)
    st = ctx.dedup_stats(reset=True)
    assert st["slow_path_calls"] == 0
    assert_hash_sorted_unique(got, W)
    assert np.array_equal(synth.sort_keys(got), oracle.dedup(allk, W, Pn, r_own).reshape(-1, W))


# ------------------------------------------------------------------ merge
@pytest.mark.parametrize("W", [1, 2])
def test_merge_parity(P, ctx, W):
    rng = np.random.default_rng(2 + W)
    sp = P.Space(64 * W, 1, 1)
    S0 = synth.unique_keys(rng.integers(1, 1 << 40, size=(300_000, W), dtype=np.uint64))
    pool = ctx.pool(sp, capacity=1000)           # forces growth
    ins0 = ctx.merge_space(pool, torch.from_numpy(hash_sort(S0, W)).cuda(), want_inserted=True).cpu().numpy()
    assert np.array_equal(synth.sort_keys(ins0), S0) and len(pool) == len(S0)
    for it in range(3):
        U = synth.unique_keys(np.concatenate([S0[rng.choice(len(S0), 50_000)],
                                              rng.integers(1, 1 << 40, size=(80_000, W), dtype=np.uint64)]))
        before = pool.keys().cpu().numpy()
        ins = ctx.merge_space(pool, torch.from_numpy(hash_sort(U, W)).cuda(), want_inserted=True).cpu().numpy()
        ref_s, ref_ins = oracle.merge(before, U, W)
        after = pool.keys().cpu().numpy()
        assert_hash_sorted_unique(after, W)
        assert_hash_sorted_unique(ins, W)
        assert np.array_equal(synth.sort_keys(after), ref_s)
        assert np.array_equal(synth.sort_keys(ins), ref_ins)
        assert len(pool) == len(before) + len(ins)
    # idempotence
    again = ctx.merge_space(pool, torch.from_numpy(hash_sort(U, W)).cuda(), want_inserted=True)
    assert again.shape[0] == 0
    # input not in the hash order is rejected
    with pytest.raises(P.CusciError) as e:
        ctx.merge_space(pool, torch.from_numpy(hash_sort(U, W)[::-1].copy()).cuda())
    assert e.value.code == 1
    pool.close()


@pytest.mark.parametrize("W", [1, 2])
def test_merge_into_empty_pool(P, ctx, W):
    """Empty pool: S' = U (copy path) -- still validated, inserted = U."""
    rng = np.random.default_rng(40 + W)
    sp = P.Space(64 * W, 1, 1)
    U = synth.unique_keys(rng.integers(1, 1 << 40, size=(50_001, W), dtype=np.uint64))
    pool = ctx.pool(sp, capacity=16)
    ins = ctx.merge_space(pool, torch.from_numpy(hash_sort(U, W)).cuda(), want_inserted=True).cpu().numpy()
    assert_hash_sorted_unique(pool.keys().cpu().numpy(), W)
    assert np.array_equal(synth.sort_keys(pool.keys().cpu().numpy()), U) and np.array_equal(synth.sort_keys(ins), U)
    pool.clear()
    with pytest.raises(P.CusciError) as e:
        ctx.merge_space(pool, torch.from_numpy(hash_sort(U, W)[::-1].copy()).cuda())
    assert e.value.code == 1
    pool.close()


@pytest.mark.parametrize("W", [1, 2])
def test_merge_sparse_paths(P, ctx, W):
    """|U| << |S| (with inserted) and |S| << |U| (without): the sparse merge
    (locate + shifted copy) must equal the set algebra."""
    rng = np.random.default_rng(60 + W)
    sp = P.Space(64 * W, 1, 1)
    big = synth.unique_keys(rng.integers(1, 1 << 40, size=(400_000, W), dtype=np.uint64))
    small = synth.unique_keys(np.concatenate([big[rng.choice(len(big), 2000, replace=False)],
                                              rng.integers(1, 1 << 40, size=(3000, W), dtype=np.uint64)]))
    # U small into a big pool, inserted requested
    pool = ctx.pool(sp, 16)
    ctx.merge_space(pool, torch.from_numpy(hash_sort(big, W)).cuda())
    ins = ctx.merge_space(pool, torch.from_numpy(hash_sort(small, W)).cuda(), want_inserted=True).cpu().numpy()
    ref_s, ref_ins = oracle.merge(big, small, W)
    after = pool.keys().cpu().numpy()
    assert_hash_sorted_unique(after, W)
    assert np.array_equal(synth.sort_keys(after), ref_s) and np.array_equal(synth.sort_keys(ins), ref_ins)
    assert_hash_sorted_unique(ins, W)
    # S small, U big, no inserted
    pool.clear()
    ctx.merge_space(pool, torch.from_numpy(hash_sort(small, W)).cuda())
    ctx.merge_space(pool, torch.from_numpy(hash_sort(big, W)).cuda())
    after = pool.keys().cpu().numpy()
    assert_hash_sorted_unique(after, W)
    assert np.array_equal(synth.sort_keys(after), oracle.merge(small, big, W)[0])
    # unsorted small U is rejected
    with pytest.raises(P.CusciError) as e:
        ctx.merge_space(pool, torch.from_numpy(hash_sort(small, W)[::-1].copy()).cuda())
    assert e.value.code == 1
    pool.close()


@pytest.mark.parametrize("W", [1, 2])
def test_merge_sparse_clustered_inserts(P, ctx, W):
    """Inserts clustered in the hash order: > 31 inserts land in one warp span of
    the big run (the copy kernel's search fallback) next to spans with none."""
    rng = np.random.default_rng(70 + W)
    sp = P.Space(64 * W, 1, 1)
    big = hash_sort(synth.unique_keys(rng.integers(1, 1 << 40, size=(300_007, W), dtype=np.uint64)), W)
    extra = hash_sort(synth.unique_keys(rng.integers(1 << 41, 1 << 42, size=(200_000, W), dtype=np.uint64)), W)
    hb, _ = hash_hi_lo(big, W)
    he, _ = hash_hi_lo(extra, W)
    lo, hi = hb[100_000], hb[100_400]                 # a 400-key window of the big run (< 2 warp spans)
    clustered = extra[(he > lo) & (he < hi)][:3000]
    small = np.concatenate([clustered, big[rng.choice(len(big), 1000, replace=False)]])
    small = hash_sort(synth.unique_keys(small), W)
    assert len(clustered) > 64
    pool = ctx.pool(sp, 16)
    ctx.merge_space(pool, torch.from_numpy(big).cuda())
    ins = ctx.merge_space(pool, torch.from_numpy(small).cuda(), want_inserted=True).cpu().numpy()
    ref_s, ref_ins = oracle.merge(big, small, W)
    after = pool.keys().cpu().numpy()
    assert_hash_sorted_unique(after, W)
    assert np.array_equal(synth.sort_keys(after), ref_s) and np.array_equal(synth.sort_keys(ins), ref_ins)
    # and the other direction (big U into a small pool, no inserted)
    pool.clear()
    ctx.merge_space(pool, torch.from_numpy(small).cuda())
    ctx.merge_space(pool, torch.from_numpy(big).cuda())
    after = pool.keys().cpu().numpy()
    assert_hash_sorted_unique(after, W)
    assert np.array_equal(synth.sort_keys(after), oracle.merge(small, big, W)[0])
    pool.close()


@pytest.mark.parametrize("W", [1, 2])
@pytest.mark.parametrize("where", ["span_start", "lane0", "mid", "last"])
def test_merge_copy_paths_reject_one_swap(P, ctx, W, where):
    """One adjacent swap anywhere in a large U must be caught by the copy kernels'
    order check (empty pool, and |S| << |U| sparse), wherever it falls relative
    to the warp spans (R x 32 keys) and lanes."""
    rng = np.random.default_rng(80 + W)
    sp = P.Space(64 * W, 1, 1)
    U = hash_sort(synth.unique_keys(rng.integers(1, 1 << 40, size=(100_003, W), dtype=np.uint64)), W)
    span = 32 * (16 if W == 1 else 8)
    i = {"span_start": 7 * span, "lane0": 7 * span + 32 * 3, "mid": 7 * span + 32 * 3 + 17, "last": len(U) - 1}[where]
    bad = U.copy()
    bad[[i - 1, i]] = bad[[i, i - 1]]
    pool = ctx.pool(sp, 16)
    with pytest.raises(P.CusciError) as e:
        ctx.merge_space(pool, torch.from_numpy(bad).cuda())
    assert e.value.code == 1
    pool.clear()
    ctx.merge_space(pool, torch.from_numpy(U[::997].copy()).cuda())   # a small S: the sparse path copies U
    with pytest.raises(P.CusciError) as e:
        ctx.merge_space(pool, torch.from_numpy(bad).cuda())
    assert e.value.code == 1
    pool.close()


@pytest.mark.parametrize("W", [1, 2])
def test_pool_merge_equals_merge_space(P, ctx, W):
    """cusci_pool_merge (src = another pool, not re-validated) gives the same pool
    and inserted set as merge_space with src's keys, on all three paths
    (empty destination, sparse, general), and merging a pool into itself is a no-op."""
    rng = np.random.default_rng(90 + W)
    sp = P.Space(64 * W, 1, 1)
    A = hash_sort(synth.unique_keys(rng.integers(1, 1 << 40, size=(200_003, W), dtype=np.uint64)), W)
    B = hash_sort(synth.unique_keys(rng.integers(1, 1 << 40, size=(150_001, W), dtype=np.uint64)), W)
    for dst_keys in (A[:0], A[::500].copy(), A):           # empty, sparse (|S| << |U|), general
        src = ctx.pool(sp, 16)
        ctx.merge_space(src, torch.from_numpy(B).cuda())
        d1, d2 = ctx.pool(sp, 16), ctx.pool(sp, 16)
        if len(dst_keys):
            ctx.merge_space(d1, torch.from_numpy(dst_keys).cuda())
            ctx.merge_space(d2, torch.from_numpy(dst_keys).cuda())
        ins1 = ctx.merge_pool(d1, src, want_inserted=True).cpu().numpy()
        ins2 = ctx.merge_space(d2, src.keys(), want_inserted=True).cpu().numpy()
        k1 = d1.keys().cpu().numpy()
        assert np.array_equal(k1, d2.keys().cpu().numpy()) and np.array_equal(ins1, ins2)
        ref_s, ref_ins = oracle.merge(dst_keys, B, W)
        assert np.array_equal(synth.sort_keys(k1), ref_s) and np.array_equal(synth.sort_keys(ins1), ref_ins)
        n = len(d1)
        assert ctx.merge_pool(d1, d1, want_inserted=True).shape[0] == 0 and len(d1) == n
        for x in (src, d1, d2):
            x.close()


def test_pipeline_lih_merge_inserts_nothing(P, ctx):
    wl, ints, par = synth.workload_inputs("lih")
    sp = P.Space(12, 2, 2)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    tp = torch.from_numpy(par).cuda()
    pool = ctx.pool(sp, 256)
    ctx.merge_space(pool, torch.from_numpy(hash_sort(par, 1)).cuda())
    rec = ctx.gen_coupled(sp, tp, di, 0.0)
    u = ctx.dedup_global(sp, rec.keys)
    ins = ctx.merge_space(pool, u, want_inserted=True)
    assert ins.shape[0] == 0 and len(pool) == 225


def test_radix_multi_portion_subprocess():
    """The onesweep passes chain <= 2^28-key portions on the device; shrink the
    portion to 2^16 keys (CUSCI_PORTION_LOG2) to exercise that path at small n."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2604_15768_b200 as P, oracle, synth
ctx = P.Context(0)
for W, m, n in [(1, 56, 300_000), (1, 26, 200_001), (2, 96, 150_000), (2, 120, 70_001)]:
    rng = np.random.default_rng(n)
    base = rng.integers(1, 1 << min(m, 62), size=(max(1, n // 4), W), dtype=np.uint64)
    if W == 2:
        base[:, 1] &= np.uint64((1 << (m - 64)) - 1)
    keys = base[rng.integers(0, len(base), size=n)]
    sp = P.Space(m, 1, 1)
    got = ctx.dedup_global(sp, torch.from_numpy(keys).cuda()).cpu().numpy().reshape(-1, W)
    assert np.array_equal(synth.sort_keys(got), oracle.dedup(keys, W).reshape(-1, W)), (W, m, n)
print("OK")
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUSCI_PORTION_LOG2="16")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


def test_dedup_bucket_split_knob_subprocess():
    """The half-bucket work split (CUSCI_BUCKET_SPLIT=1) gives the same sets."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2604_15768_b200 as P, oracle, synth
ctx = P.Context(0)
for W, n in [(1, 2_000_000), (2, 600_000)]:
    keys = synth.zipf_keys(n, W, 1.05, 1 << 20, seed=3 + W)
    got = ctx.dedup_global(P.Space(64 * W, 1, 1), torch.from_numpy(keys).cuda()).cpu().numpy().reshape(-1, W)
    assert np.array_equal(synth.sort_keys(got), oracle.dedup(keys, W).reshape(-1, W)), W
print("OK")
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUSCI_BUCKET_SPLIT="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


def _fmix64_inv(h):
    """inverse of the splitmix64 finalizer (to build keys with chosen hash)."""
    M = (1 << 64) - 1
    i2 = pow(0x94D049BB133111EB, -1, 1 << 64)
    i1 = pow(0xBF58476D1CE4E5B9, -1, 1 << 64)
    out = []
    for x in h:
        x = int(x)
        x ^= (x >> 31) ^ (x >> 62)
        x = (x * i2) & M
        x ^= (x >> 27) ^ (x >> 54)
        x = (x * i1) & M
        x ^= (x >> 30) ^ (x >> 60)
        out.append(x)
    return np.array(out, dtype=np.uint64)


def test_dedup_bucket_overflow_slow_path(P, ctx):
    """Keys whose hash lands in ONE bucket (more distinct keys than its
    shared-memory table): the bucket is flagged and the host finishes with the
    full hash-order sort + unique -- the result must still be exact."""
    rng = np.random.default_rng(17)
    hi = rng.integers(1, 1 << 40, size=9000, dtype=np.uint64)        # top 24 bits zero
    keys = _fmix64_inv(hi).reshape(-1, 1)
    assert np.array_equal(fmix64(keys[:, 0]), hi)
    other = rng.integers(1, 1 << 62, size=(12000, 1), dtype=np.uint64)
    allk = np.concatenate([keys, keys[:3000], other])
    sp = P.Space(64, 1, 1)
    got = ctx.dedup_global(sp, torch.from_numpy(allk).cuda()).cpu().numpy()
    assert_hash_sorted_unique(got, 1)
    assert np.array_equal(synth.sort_keys(got), oracle.dedup(allk, 1))


def _t_fmix64(x):
    """splitmix64 finalizer on int64 torch tensors (logical shifts, wrapping multiplies)."""
    def srl(v, s):
        return (v >> s) & ((1 << (64 - s)) - 1)
    c1 = 0xBF58476D1CE4E5B9 - (1 << 64)
    c2 = 0x94D049BB133111EB - (1 << 64)
    x = x ^ srl(x, 30)
    x = x * c1
    x = x ^ srl(x, 27)
    x = x * c2
    return x ^ srl(x, 31)


def _t_fmix64_inv(x):
    """inverse of the splitmix64 finalizer on int64 torch tensors."""
    def srl(v, s):
        return (v >> s) & ((1 << (64 - s)) - 1)
    i2 = pow(0x94D049BB133111EB, -1, 1 << 64)
    i1 = pow(0xBF58476D1CE4E5B9, -1, 1 << 64)
    i2 = i2 - (1 << 64) if i2 >= 1 << 63 else i2
    i1 = i1 - (1 << 64) if i1 >= 1 << 63 else i1
    x = x ^ srl(x, 31) ^ srl(x, 62)
    x = x * i2
    x = x ^ srl(x, 27) ^ srl(x, 54)
    x = x * i1
    return x ^ srl(x, 30) ^ srl(x, 60)


def test_dedup_hist_free_pass_overflow_falls_back(P, ctx):
    """70M keys whose hash shares its top byte (one group): the hist-free first
    pass overflows its region and the call redoes the pass with histograms --
    the result must still be exact."""
    g = torch.Generator(device="cuda").manual_seed(5)
    D = 40_000_000
    hi = torch.randint(0, 1 << 56, (D,), device="cuda", generator=g, dtype=torch.int64) | (0x5A << 56)
    hi = torch.unique(hi)
    base = _t_fmix64_inv(hi)
    assert torch.equal(_t_fmix64(base), hi)
    keys = torch.cat([base, base[: 30_000_000]])
    keys = keys[torch.randperm(keys.numel(), device="cuda", generator=g)]
    u = ctx.dedup_global(P.Space(64, 1, 1), keys.view(torch.uint64).reshape(-1, 1))
    ui = u.view(torch.int64).reshape(-1)
    flip = -(1 << 63)
    assert u.shape[0] == base.numel()
    h = _t_fmix64(ui) ^ flip
    assert bool((h[1:] > h[:-1]).all())
    assert torch.equal(torch.sort(ui ^ flip).values, torch.sort(base ^ flip).values)


@pytest.mark.parametrize("W", [1, 2])
def test_dedup_histogram_free_passes(P, ctx, W):
    """1e8 keys (4e7 distinct): both partition passes run without histograms
    (region cursors), checked by the stats, the exact count, strict hash order
    and set equality."""
    g = torch.Generator(device="cuda").manual_seed(9 + W)
    D, n = 40_000_000, 100_000_000
    C = 0x9E3779B97F4A7C15 - (1 << 64)
    base = torch.arange(1, D + 1, dtype=torch.int64, device="cuda") * C
    if W == 2:
        base = torch.stack([base, torch.arange(D, dtype=torch.int64, device="cuda") % 977], dim=1)
    keys = torch.cat([base, base[torch.randint(0, D, (n - D,), device="cuda", generator=g)]])
    keys = keys[torch.randperm(n, device="cuda", generator=g)].contiguous()
    ctx.dedup_stats(reset=True)
    u = ctx.dedup_global(P.Space(64 * W, 1, 1), keys.view(torch.uint64).reshape(-1, W))
    st = ctx.dedup_stats(reset=True)
    assert st["hist_keys"] == 0 and st["hist_free_keys"] == n and st["key_passes"] == 2 * n, st
    assert u.shape[0] == D
    flip = -(1 << 63)
    if W == 1:
        ui = u.view(torch.int64).reshape(-1)
        h = _t_fmix64(ui) ^ flip
        assert bool((h[1:] > h[:-1]).all())
        assert torch.equal(torch.sort(ui ^ flip).values, torch.sort(base ^ flip).values)
    else:
        got = synth.sort_keys(u.cpu().numpy().reshape(-1, 2))
        ref = synth.sort_keys(base.cpu().numpy().view(np.uint64).reshape(-1, 2))
        assert np.array_equal(got, ref)
        assert_hash_sorted_unique(u.cpu().numpy().reshape(-1, 2), 2)


_AT_SCALE = r"""
import sys, torch
sys.path.insert(0, %r)
import paper_2604_15768_b200 as P
from tests.test_gpu_parity import _t_fmix64
ctx = P.Context(0)
D, R = 660_000_000, 100_000_000
C = 0x9E3779B97F4A7C15 - (1 << 64)          # odd: i -> i * C is a bijection of Z/2^64
base = torch.arange(1, D + 1, dtype=torch.int64, device="cuda") * C
g = torch.Generator(device="cuda").manual_seed(7)
rep = base[torch.randint(0, D, (R,), device="cuda", generator=g)]
keys = torch.cat([base, rep])
del rep
keys = keys[torch.randperm(keys.numel(), device="cuda", generator=g)]
ctx.dedup_stats(reset=True)
u = ctx.dedup_global(P.Space(64, 1, 1), keys.view(torch.uint64).reshape(-1, 1))
st = ctx.dedup_stats(reset=True)
del keys
assert u.shape[0] == D
assert st["key_passes"] == %d * (D + R) and st["slow_path_calls"] == 0, st
ui = u.view(torch.int64).reshape(-1)
flip = -(1 << 63)
hi = _t_fmix64(ui) ^ flip                      # signed order of hi ^ 2^63 = unsigned order of hi
assert bool((hi[1:] > hi[:-1]).all()), "not strictly in hash order"
del hi
assert torch.equal(torch.sort(ui ^ flip).values, torch.sort(base ^ flip).values)
print("OK")
"""


@pytest.mark.parametrize("distinct_target,passes", [(None, 2), ("1536", 3)])
def test_dedup_at_scale(distinct_target, passes):
    """0.76e9 keys (0.66e9 distinct, 1e8 repeated), shuffled: exercises the
    HyperLogLog plan with one further partition pass (default bucket target)
    and with two (a smaller distinct-per-bucket target via the tuning knob).
    Too large for the oracle: checked by the exact distinct count, strict hash
    order and set equality with the generating set (torch sort on the GPU)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    if distinct_target:
        env["CUSCI_BUCKET_DISTINCT"] = distinct_target
    r = subprocess.run([sys.executable, "-c", _AT_SCALE % (root, passes)], env=env, capture_output=True, text=True,
                       timeout=900, cwd=root)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


_N2_BATCH = r"""
import sys, torch
sys.path.insert(0, %r)
import paper_2604_15768_b200 as P, synth
wl, ints, par = synth.workload_inputs("n2", n_parents=1_000_000)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7)
di = P.DeviceIntegrals(ints.h, ints.eri)
shard = ctx.dedup_global(sp, torch.from_numpy(par).cuda())
rec = ctx.gen_coupled(sp, shard[:500_000], di, 0.0, with_src=False)
assert rec.count == 1_938_044_316, rec.count
ctx.dedup_stats(reset=True)
u = ctx.dedup_global(sp, rec.keys)
st = ctx.dedup_stats(reset=True)
assert st["hist_free_keys"] == rec.count and st["slow_path_calls"] == 0, st   # the bench's hist-free plan ran
# strict hash order on the device (hi = fmix64(key), W = 1)
def srl(x, k):  # logical shift right of int64 bit patterns
    return (x >> k) & ((1 << (64 - k)) - 1)
def fmix(x):  # splitmix64 finalizer on int64 bit patterns (multiplications wrap mod 2^64)
    x = x ^ srl(x, 30); x = x * -4658895280553007687; x = x ^ srl(x, 27); x = x * -7723592293110705685
    return x ^ srl(x, 31)
hi = fmix(u.view(torch.int64).reshape(-1)) ^ (-(2 ** 63))   # unsigned order as signed order
assert bool((hi[1:] > hi[:-1]).all()), "not strictly increasing in the hash order"
del hi
# the set: torch's sort-based unique of the same 1.94e9 keys (library code, independent of libcusci)
ref = torch.unique(rec.keys.view(torch.int64).reshape(-1))
del rec
got = torch.sort(u.view(torch.int64).reshape(-1)).values
assert got.shape == ref.shape and bool(torch.equal(got, ref)), (got.shape, ref.shape)
del got, ref
# the bench's merges at full size: the unique pool over both batches (the general
# merge), then S <- S u C from the parents (the sparse path), against torch.unique
ctx.release_cached()
torch.cuda.empty_cache()
pool = ctx.pool(sp, 1 << 20)
ctx.merge_space(pool, u)
rec2 = ctx.gen_coupled(sp, shard[500_000:], di, 0.0, with_src=False)
u2 = ctx.dedup_global(sp, rec2.keys)
del rec2
ctx.release_cached()
torch.cuda.empty_cache()
ctx.merge_space(pool, u2)
ref = torch.unique(torch.cat([u.view(torch.int64).reshape(-1), u2.view(torch.int64).reshape(-1)]))
got = torch.sort(pool.keys().view(torch.int64).reshape(-1)).values
assert got.shape == ref.shape and bool(torch.equal(got, ref)), (got.shape, ref.shape)
spool = ctx.pool(sp, 1 << 20)
ctx.merge_space(spool, shard)
ctx.merge_pool(spool, pool)
ref = torch.unique(torch.cat([ref, shard.view(torch.int64).reshape(-1)]))
got = torch.sort(spool.keys().view(torch.int64).reshape(-1)).values
assert got.shape == ref.shape and bool(torch.equal(got, ref)), (got.shape, ref.shape)
print("OK", int(ref.shape[0]))
"""


def test_dedup_n2_bench_batch(P, ctx):
    """The bench's own dedup call at full size: the first N2 batch (5e5 parents ->
    1,938,044,316 generated keys, 86% redundant) through the histogram-free
    plan, against torch.unique of the same keys (set equality) with strict
    hash order checked on the device; then the bench's merges at full size
    (the unique pool over both batches, S <- S u C from the parents)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ctx.release_cached()          # this process's cached device memory: the subprocess needs ~100 GB
    torch.cuda.empty_cache()
    r = subprocess.run([sys.executable, "-c", _N2_BATCH % root], capture_output=True, text=True, timeout=1200, cwd=root)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


# ------------------------------------------------------------------ Stage-3 contraction
def _contract_case(P, ctx, wl_key, n_par, W, seed, keep_every=1):
    from oracle import energy
    wl, ints, par = synth.workload_inputs(wl_key, n_parents=n_par)
    sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    rec = ctx.gen_coupled(sp, torch.from_numpy(par).cuda(), di, 0.0, with_src=True)
    uniq = ctx.dedup_global(sp, rec.keys)[::keep_every].contiguous()
    rng = np.random.default_rng(seed)
    psi = rng.uniform(-1.0, 1.0, size=uniq.shape[0])
    e, miss = ctx.energy_contract(sp, rec, len(par), uniq, torch.from_numpy(psi).cuda())
    keys = rec.keys[:rec.count].cpu().numpy().reshape(-1, W)
    src = rec.src[:rec.count].cpu().numpy()
    ref, rmiss, absterm = energy.contract(keys, rec.hij[:rec.count].cpu().numpy(), src,
                                          len(par), uniq.cpu().numpy().reshape(-1, W), psi, W)
    assert miss == rmiss
    assert_contract_close(e.cpu().numpy(), ref, np.bincount(src, minlength=len(par)))
    return miss


def assert_contract_close(got, ref, nterms):
    """e vs the exact (fsum) definition: |e - e_exact| <= 1e-12 |e_exact|.  The
    kernel's own bound (DESIGN.md r14) is half an ulp of e plus 2^-81 per term
    (products rounded to the 2^-80 grid), far inside 1e-12 |e| unless the sum
    cancels to < 1e-9; an exactly zero reference must be reproduced up to
    that grid term."""
    err = np.abs(got - ref)
    tol = 1e-12 * np.abs(ref) + (ref == 0) * nterms * 2.0 ** -80
    assert np.all(err <= tol), f"max rel err {np.max(err / np.maximum(np.abs(ref), 1e-300))}"


def test_contract_lih(P, ctx):
    assert _contract_case(P, ctx, "lih", None, 1, 1) == 0


def test_contract_h2o_with_missing(P, ctx):
    assert _contract_case(P, ctx, "h2o", 300, 1, 2) == 0
    assert _contract_case(P, ctx, "h2o", 300, 1, 3, keep_every=2) > 0


def test_contract_c2h4_w2(P, ctx):
    assert _contract_case(P, ctx, "c2h4", 4, 2, 4, keep_every=3) > 0


@pytest.mark.parametrize("wl_key,n_par,W,keep_every", [("lih", None, 1, 1), ("h2o", 2000, 1, 1), ("h2o", 2000, 1, 3),
                                                        ("c2h4", 6, 2, 3)])
def test_contract_partitioned(P, ctx, wl_key, n_par, W, keep_every):
    """the pi-partitioned contraction (records scattered into 256 regions first,
    CUSCI_OPT_CONTRACT_PARTITION = 1) against the exact-sum definition, incl.
    absent amplitudes; and bit-identical to the unpartitioned kernel"""
    try:
        ctx.contract_partition(1)
        miss = _contract_case(P, ctx, wl_key, n_par, W, 11, keep_every=keep_every)
        assert (miss > 0) == (keep_every > 1)
        wl, ints, par = synth.workload_inputs(wl_key, n_parents=n_par)
        sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
        rec = ctx.gen_coupled(sp, torch.from_numpy(par).cuda(), P.DeviceIntegrals(ints.h, ints.eri), 0.0, with_src=True)
        uniq = ctx.dedup_global(sp, rec.keys)
        psi = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, uniq.shape[0])).cuda()
        e1, m1 = ctx.energy_contract(sp, rec, len(par), uniq, psi)
        ctx.contract_partition(-1)
        e0, m0 = ctx.energy_contract(sp, rec, len(par), uniq, psi)
        assert m0 == m1 and torch.equal(e0, e1)
    finally:
        ctx.contract_partition(0)


def test_contract_rejects_bad_src(P, ctx):
    wl, ints, par = synth.workload_inputs("lih")
    sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
    rec = ctx.gen_coupled(sp, torch.from_numpy(par).cuda(), P.DeviceIntegrals(ints.h, ints.eri), 0.0, with_src=True)
    uniq = ctx.dedup_global(sp, rec.keys)
    psi = torch.ones(uniq.shape[0], dtype=torch.float64, device="cuda")
    with pytest.raises(P.CusciError) as e:   # records of parents 0..224, n_parents = 100
        ctx.energy_contract(sp, rec, 100, uniq, psi)
    assert e.value.code == 1 and "src" in str(e.value)
    with pytest.raises(ValueError):
        ctx.energy_contract(sp, rec, len(par), uniq, psi, e=torch.empty(10, dtype=torch.float64, device="cuda"))


def test_contract_rejects_large_products(P, ctx):
    wl, ints, par = synth.workload_inputs("lih")
    sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
    rec = ctx.gen_coupled(sp, torch.from_numpy(par).cuda(), P.DeviceIntegrals(ints.h, ints.eri), 0.0, with_src=True)
    uniq = ctx.dedup_global(sp, rec.keys)
    psi = torch.full((uniq.shape[0],), 2.0 ** 30, dtype=torch.float64, device="cuda")
    with pytest.raises(P.CusciError) as e:
        ctx.energy_contract(sp, rec, len(par), uniq, psi)
    assert e.value.code == 1


# ---- the paper's regular-sampling sorted dedup (oracle/sampling.py)
def _f2_keys(W, n, seed):
    return synth.zipf_keys(max(n, 1), W, 1.1, 1 << 16, seed=seed)[:n]


@pytest.mark.parametrize("W,n", [(1, 0), (1, 1), (1, 4097), (1, 300_001), (2, 150_001)])
def test_f2_sort_unique(P, ctx, W, n):
    from oracle import sampling as S
    sp = P.Space(64 * W, 1, 1)
    keys = _f2_keys(W, n, 31 + W)
    got = ctx.sort_unique(sp, torch.from_numpy(keys).cuda()).cpu().numpy().reshape(-1, W)
    ref = S.from_ints(S.sort_unique(S.to_ints(keys, W)), W)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("W", [1, 2])
def test_f2_blocks_virtual_ranks(P, ctx, W):
    """Steps 1-3 composed from the exported blocks over 5 virtual ranks on one GPU
    (the NCCL transport is dedup_global's) against the oracle protocol."""
    from oracle import sampling as S
    sp = P.Space(64 * W, 1, 1)
    keys = _f2_keys(W, 90_000, 41 + W)
    Pn, Ssz = 5, 37
    parts = [keys[i::Pn] for i in range(Pn)]
    parts[3] = parts[3][:0]                                   # an empty rank
    local = [S.to_ints(x, W) for x in parts]
    D_ref = [S.sort_unique(x) for x in local]
    D = [ctx.sort_unique(sp, torch.from_numpy(x).cuda()) if len(x) else torch.empty((0, W), dtype=torch.uint64, device="cuda")
         for x in parts]
    smp = []
    for d, dr in zip(D, D_ref):
        assert np.array_equal(d.cpu().numpy().reshape(-1, W), S.from_ints(dr, W))
        s = ctx.regular_samples(sp, d, Ssz)
        assert np.array_equal(s.cpu().numpy().reshape(-1, W), S.from_ints(S.regular_samples(dr, Ssz), W))
        smp.append(s)
    gathered = torch.cat(smp[::-1])                           # any order
    spl = ctx.select_splitters(sp, gathered, Pn)
    spl_ref = S.select_splitters([x for dr in D_ref for x in S.regular_samples(dr, Ssz)], Pn)
    assert np.array_equal(spl.cpu().numpy().reshape(-1, W), S.from_ints(spl_ref, W))
    recv = [[] for _ in range(Pn)]
    for d, dr in zip(D, D_ref):
        b = ctx.split_bounds(sp, d, spl, Pn)
        assert b == S.split_bounds(dr, spl_ref)
        for r in range(Pn):
            recv[r].append(d[b[r]:b[r + 1]])
    shards_ref, _ = S.dedup_sorted(local, Ssz)
    for r in range(Pn):
        got = ctx.sort_unique(sp, torch.cat(recv[r])).cpu().numpy().reshape(-1, W) if sum(len(x) for x in recv[r]) else np.zeros((0, W), np.uint64)
        assert np.array_equal(got, S.from_ints(shards_ref[r], W)), r


@pytest.mark.parametrize("W", [1, 2])
def test_f2_dedup_sorted_world1(P, ctx, W):
    from oracle import sampling as S
    sp = P.Space(64 * W, 1, 1)
    keys = _f2_keys(W, 200_003, 51 + W)
    got = ctx.dedup_sorted(sp, torch.from_numpy(keys).cuda(), 64).cpu().numpy().reshape(-1, W)
    assert np.array_equal(got, S.from_ints(S.sort_unique(S.to_ints(keys, W)), W))


def test_f2_n2_records_sorted_dedup(P, ctx):
    """Sorted dedup of a generated N2 stream equals the hash-order dedup's set, re-sorted."""
    wl, ints, par = synth.workload_inputs("n2", n_parents=300)
    sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    rec = ctx.gen_coupled(sp, torch.from_numpy(par).cuda(), di, 0.0, with_src=False)
    got = ctx.dedup_sorted(sp, rec.keys, 256).cpu().numpy().reshape(-1)
    ref = np.unique(oracle.dedup(rec.keys.cpu().numpy(), 1).reshape(-1))
    assert np.array_equal(got, ref)
