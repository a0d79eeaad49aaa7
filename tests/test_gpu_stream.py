"""GPU parity of the memory-centric streaming stages (
PAPER.md Sec 4.3 :583-634): mini-batched Stage 1 (gen -> dedup -> merge with
H2D prefetch and D2H offload of the original set) and Stage 3 (reload, or
regenerate) must give exactly what the unbatched calls give -- and the
oracle's sets / exact sums."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import energy
from tests.test_gpu_parity import assert_contract_close, assert_hash_sorted_unique, canon

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


@pytest.mark.parametrize("key,n_par,batch", [("h2o", 10_000, 3_001), ("c2h4", 90, 25), ("lih", None, 1000)])
def test_stream_stages(P, ctx, key, n_par, batch):
    wl, ints, par = synth.workload_inputs(key, n_parents=n_par)
    W = wl.words
    sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    ph = torch.from_numpy(par).pin_memory()
    total = ctx.gen_coupled_count(sp, ph.cuda(), di, 0.0)
    host = P.HostRecords(total, W)
    pool = ctx.pool(sp, 1024)
    st = ctx.stream_generate(sp, ph, di, 0.0, batch, pool, host)
    assert st["records"] == total == host.count
    assert st["batches"] == -(-len(par) // batch)
    assert st["peak_device_bytes"] > 0 and st["ms_wall"] > 0
    # the host original set = the oracle's records (src = global parent index)
    ref = oracle.gen_coupled(wl.m, wl.n_alpha, wl.n_beta, par, ints, 0.0)
    hk, hs, hh = canon(host.keys.numpy(), host.src.numpy().astype(np.uint32), host.hij.numpy())
    rk, rs, rh = canon(ref["keys"], ref["src"], ref["hij"])
    assert np.array_equal(hk, rk) and np.array_equal(hs, rs) and np.array_equal(hh, rh)
    # the pool = the distinct coupled configurations
    u = pool.keys().cpu().numpy().reshape(-1, W)
    assert st["unique"] == len(u)
    assert_hash_sorted_unique(u, W)
    assert np.array_equal(synth.sort_keys(u), oracle.dedup(ref["keys"], W).reshape(-1, W))
    # Stage 3: reload (odd record batches) == regenerate == one energy_contract (bit for bit), ~ oracle
    uk = pool.keys()
    psi = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, size=uk.shape[0])).cuda()
    e1, m1, s1 = ctx.stream_energy(sp, host, len(par), uk, psi, batch_records=max(1, total // 3 + 7))
    e2, m2, s2 = ctx.stream_energy_regen(sp, ph, di, 0.0, batch, uk, psi)
    rec = ctx.gen_coupled(sp, ph.cuda(), di, 0.0, with_src=True)
    e3, m3 = ctx.energy_contract(sp, rec, len(par), uk, psi)
    assert m1 == m2 == m3 == 0
    assert torch.equal(e1, e2) and torch.equal(e1, e3)
    assert s1["records"] == s2["records"] == total
    eref, _, _ = energy.contract(ref["keys"], ref["hij"], ref["src"], len(par), uk.cpu().numpy(), psi.cpu().numpy(), W)
    assert_contract_close(e1.cpu().numpy(), eref, np.bincount(ref["src"], minlength=len(par)))
    pool.close()


def test_stream_without_offload_and_capacity(P, ctx):
    wl, ints, par = synth.workload_inputs("h2o", n_parents=2000)
    sp = P.Space(wl.m, 5, 5)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    ph = torch.from_numpy(par).pin_memory()
    pool = ctx.pool(sp, 1024)
    st = ctx.stream_generate(sp, ph, di, 0.0, 777, pool)            # records consumed on the device
    assert st["d2h_bytes"] == 0 and st["unique"] == len(pool)
    ref = ctx.dedup_global(sp, ctx.gen_coupled(sp, ph.cuda(), di, 0.0).keys).cpu().numpy()
    assert np.array_equal(synth.sort_keys(pool.keys().cpu().numpy()), synth.sort_keys(ref))
    small = P.HostRecords(1000, 1)
    pool.clear()
    with pytest.raises(P.CusciError) as e:
        ctx.stream_generate(sp, ph, di, 0.0, 777, pool, small)
    assert e.value.code == 3 and small.count == 1000
    assert len(pool) == len(ref)                                     # the pool is complete regardless
    pool.close()


def test_stream_collective(P):
    """stream_generate's collective path (batch-count agreement + dedup_global's
    protocol) on a forced 1-rank communicator."""
    c = P.Context(0, 0, 1, nccl_id=P.Context.nccl_unique_id())
    c.force_collective(True)
    wl, ints, par = synth.workload_inputs("h2o", n_parents=1500)
    sp = P.Space(wl.m, 5, 5)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    pool = c.pool(sp, 1024)
    st = c.stream_generate(sp, torch.from_numpy(par).pin_memory(), di, 0.0, 400, pool)
    ref = oracle.dedup(oracle.gen_coupled(wl.m, 5, 5, par, ints, 0.0)["keys"], 1)
    assert st["batches"] == 4 and np.array_equal(synth.sort_keys(pool.keys().cpu().numpy()), ref)
    pool.close()
    c.close()


# ------------------------------------------------------------------ f4: SCI growth (heat-bath surrogate)
@pytest.mark.parametrize("key,n_par,K,iters", [("lih", None, 40, 3), ("h2o", 50, 2000, 3), ("n2", 20, 800, 2),
                                               ("c2h4", 3, 300, 2)])
def test_sci_grow_steps(P, ctx, key, n_par, K, iters):
    """sci_grow_step from a small start space vs the oracle step by step: the
    space, the selection and every amplitude bit for bit."""
    from oracle import heatbath as HB
    wl, ints, par = synth.workload_inputs(key, n_parents=n_par)
    W = wl.words
    if key == "lih":
        par = par[:5]
    sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    pool = ctx.pool(sp, 1024)
    ctx.merge_space(pool, ctx.dedup_global(sp, torch.from_numpy(par).cuda()))
    keys = pool.keys().cpu().numpy().reshape(-1, W)
    psi = np.random.default_rng(5).uniform(-1, 1, size=len(keys))
    ref = {tuple(int(x) for x in k): p for k, p in zip(keys, psi)}
    psi_d = torch.from_numpy(psi).cuda()
    for it in range(iters):
        S = np.array(list(ref.keys()), dtype=np.uint64).reshape(-1, W)
        rec = oracle.gen_coupled(wl.m, wl.n_alpha, wl.n_beta, S, ints, 0.0)
        ref, sel, ncand = HB.grow_step(S, np.array(list(ref.values())), rec, K, W)
        psi_d, st = ctx.sci_grow_step(sp, pool, psi_d, di, 0.0, K)
        assert st["records"] == len(rec["src"]) and st["candidates"] == ncand
        assert st["selected"] == len(sel) == min(K, ncand) and st["space_after"] == len(ref)
        got = pool.keys().cpu().numpy().reshape(-1, W)
        assert_hash_sorted_unique(got, W)
        gp = psi_d.cpu().numpy()
        assert {tuple(int(x) for x in k): p for k, p in zip(got, gp)} == ref, f"iteration {it}"
    pool.close()
