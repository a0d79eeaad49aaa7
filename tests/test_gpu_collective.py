"""GPU parity of the collective protocol (SURVEY 8(a) a10 exchange, 8(e)) on
real NCCL: a 1-rank communicator with CUSCI_OPT_FORCE_COLLECTIVE runs the
whole multi-rank code path of dedup_global / dedup_sorted -- the status-
carrying count exchange (ncclSend/ncclRecv), the status all-reduce, the
payload all-to-all-v (the own bin through NCCL to self), the owner-side
finalize -- and of dedup_sorted's sample all-gather.  Results are compared
with the oracle exactly as the 1-rank shortcut is (PAPER.md :453-460)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import sampling as OS
from tests.test_gpu_parity import assert_hash_sorted_unique

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2604_15768_b200 as P
    return P


@pytest.fixture(scope="module")
def cctx(P):
    c = P.Context(0, 0, 1, nccl_id=P.Context.nccl_unique_id())
    c.force_collective(True)
    yield c
    c.close()


def test_force_needs_communicator(P):
    c = P.Context(0)
    with pytest.raises(P.CusciError) as e:
        c.force_collective(True)
    assert e.value.code == 1
    c.close()


@pytest.mark.parametrize("W,n", [(1, 0), (1, 1), (1, 70_001), (1, 1_000_003), (2, 300_001)])
def test_collective_dedup_zipf(P, cctx, W, n):
    sp = P.Space(64 * W, 1, 1)
    keys = synth.zipf_keys(max(n, 1), W, 1.1, 1 << 17, seed=21 + W)[:n]
    l0 = cctx.kernel_launches
    got = cctx.dedup_global(sp, torch.from_numpy(keys).cuda()).cpu().numpy().reshape(-1, W)
    assert cctx.kernel_launches > l0 or n == 0
    assert_hash_sorted_unique(got, W)
    assert np.array_equal(synth.sort_keys(got), oracle.dedup(keys, W).reshape(-1, W))


def test_collective_dedup_generated_stream(P, cctx):
    wl, ints, par = synth.workload_inputs("n2", n_parents=400)
    sp = P.Space(wl.m, 7, 7)
    rec = cctx.gen_coupled(sp, torch.from_numpy(par).cuda(), P.DeviceIntegrals(ints.h, ints.eri), 0.0)
    got = cctx.dedup_global(sp, rec.keys).cpu().numpy()
    assert_hash_sorted_unique(got, 1)
    assert np.array_equal(synth.sort_keys(got), oracle.dedup(rec.keys.cpu().numpy(), 1))


def test_collective_error_agreement_and_recovery(P, cctx):
    """A rank whose arguments fail still takes part in the count exchange (its
    failure marker), every rank returns the error, and the communicator stays
    usable for the next call."""
    keys = torch.from_numpy(synth.zipf_keys(5000, 1, 1.1, 1 << 12, seed=3)).cuda()
    with pytest.raises(P.CusciError) as e:
        cctx.dedup_global(P.Space(130, 1, 1), keys)            # m > 128 -> E_INVALID_ARG
    assert e.value.code == 1
    with pytest.raises(P.CusciError) as e:
        cctx.dedup_sorted(P.Space(64, 1, 1), keys, 0)            # n_samples < 1
    assert e.value.code == 1
    got = cctx.dedup_global(P.Space(64, 1, 1), keys).cpu().numpy()
    assert np.array_equal(synth.sort_keys(got), oracle.dedup(keys.cpu().numpy(), 1))


@pytest.mark.parametrize("W,n", [(1, 0), (1, 4097), (1, 250_001), (2, 120_001)])
def test_collective_dedup_sorted(P, cctx, W, n):
    sp = P.Space(64 * W, 1, 1)
    keys = synth.zipf_keys(max(n, 1), W, 1.05, 1 << 16, seed=31 + W)[:n]
    got = cctx.dedup_sorted(sp, torch.from_numpy(keys).cuda(), 512).cpu().numpy().reshape(-1, W)
    ref = OS.from_ints(OS.sort_unique(OS.to_ints(keys, W)), W).reshape(-1, W)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("wl_key,n_par,W,keep_every", [("h2o", 300, 1, 1), ("h2o", 300, 1, 3), ("c2h4", 4, 2, 2)])
def test_collective_energy_contract(P, cctx, wl_key, n_par, W, keep_every):
    """f1 through the owner protocol (requests -> owner lookup -> answers back)
    vs the exact-sum oracle, with keys missing from the space."""
    from oracle import energy
    from tests.test_gpu_parity import assert_contract_close
    wl, ints, par = synth.workload_inputs(wl_key, n_parents=n_par)
    sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
    rec = cctx.gen_coupled(sp, torch.from_numpy(par).cuda(), P.DeviceIntegrals(ints.h, ints.eri), 0.0, with_src=True)
    uniq = cctx.dedup_global(sp, rec.keys)[::keep_every].contiguous()
    psi = np.random.default_rng(9).uniform(-1.0, 1.0, size=uniq.shape[0])
    e, miss = cctx.energy_contract(sp, rec, len(par), uniq, torch.from_numpy(psi).cuda())
    src = rec.src[:rec.count].cpu().numpy()
    ref, rmiss, _ = energy.contract(rec.keys.cpu().numpy().reshape(-1, W), rec.hij.cpu().numpy(), src, len(par),
                                    uniq.cpu().numpy().reshape(-1, W), psi, W)
    assert miss == rmiss and (miss > 0) == (keep_every > 1)
    assert_contract_close(e.cpu().numpy(), ref, np.bincount(src, minlength=len(par)))
