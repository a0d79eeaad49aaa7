"""Drive every libcusci kernel path on small inputs (for compute-sanitizer):
    compute-sanitizer --tool memcheck python tools/sanitize_run.py [small|large]
small: LiH / H2O / C2H4-like gen, dedup (bucket + slow path), merge (general,
sparse, empty pool, pool merge), f1 contraction, f2 sorted dedup, f3 streaming,
f4 growth, the collective protocol on a 1-rank communicator.  large: adds one
dedup of 2^26 keys (the histogram-free partition passes).  Results are checked
for self-consistency only (parity is the tests' job)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_15768_b200 as P  # noqa: E402
import synth  # noqa: E402


def check_sorted_unique(t):
    n = t.shape[0]
    assert n == 0 or len(np.unique(t.cpu().numpy(), axis=0)) == n


def run_workload(ctx, key, n_par, batch, collective=False):
    wl, ints, par = synth.workload_inputs(key, n_parents=n_par)
    sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    tp = torch.from_numpy(par).cuda()
    rec = ctx.gen_coupled(sp, tp, di, 0.0, with_src=True, with_phase=True)
    rec2 = ctx.gen_coupled(sp, tp, di, 1e-3, with_src=True)
    assert rec2.count <= rec.count
    u = ctx.dedup_global(sp, rec.keys)
    check_sorted_unique(u)
    pool = ctx.pool(sp, 64)
    ctx.merge_space(pool, ctx.dedup_global(sp, tp))           # empty pool: validated copy
    ins = ctx.merge_space(pool, u, want_inserted=True)       # general or sparse merge
    half = ctx.dedup_global(sp, rec.keys[: rec.count // 2])
    ctx.merge_space(pool, half)                              # everything already present
    other = ctx.pool(sp, 64)
    ctx.merge_space(other, half)
    ctx.merge_pool(other, pool, want_inserted=True)
    assert len(other) == len(pool) and ins.shape[0] <= u.shape[0]
    psi = torch.rand(len(pool), dtype=torch.float64, device="cuda") - 0.5
    e, miss = ctx.energy_contract(sp, rec, len(par), pool.keys(), psi)
    srt = ctx.dedup_sorted(sp, rec.keys, 64)
    assert srt.shape[0] == u.shape[0]
    if collective:  # the streaming stages and the growth step are one-rank calls
        print(f"{key} (collective): {rec.count} records, {u.shape[0]} unique, missing {miss}")
        return
    ph = torch.from_numpy(par).pin_memory()
    host = P.HostRecords(rec.count, wl.words)
    spool = ctx.pool(sp, 64)
    st = ctx.stream_generate(sp, ph, di, 0.0, batch, spool, host)
    assert st["records"] == rec.count and len(spool) == u.shape[0]
    uk = spool.keys()
    psi2 = torch.rand(uk.shape[0], dtype=torch.float64, device="cuda") - 0.5
    e1, _, _ = ctx.stream_energy(sp, host, len(par), uk, psi2, batch_records=max(1, rec.count // 3 + 7))
    e2, _, _ = ctx.stream_energy_regen(sp, ph, di, 0.0, batch, uk, psi2)
    assert torch.equal(e1, e2)
    gpool = ctx.pool(sp, 64)
    ctx.merge_space(gpool, ctx.dedup_global(sp, tp[:20]))
    gpsi = torch.ones(len(gpool), dtype=torch.float64, device="cuda")
    for _ in range(2):
        gpsi, _ = ctx.sci_grow_step(sp, gpool, gpsi, di, 0.0, 4 * len(gpool))
    for p_ in (pool, other, spool, gpool):
        p_.close()
    print(f"{key}: {rec.count} records, {u.shape[0]} unique, missing {miss}")


def main():
    size = sys.argv[1] if len(sys.argv) > 1 else "small"
    nid = P.Context.nccl_unique_id()
    ctx = P.Context(0, 0, 1, nccl_id=nid)
    run_workload(ctx, "lih", None, 100)
    run_workload(ctx, "h2o", 1500, 700)
    run_workload(ctx, "c2h4", 40, 15)
    # the collective protocol on a 1-rank communicator (NCCL self exchange)
    ctx.force_collective(True)
    run_workload(ctx, "h2o", 800, 300, collective=True)
    ctx.force_collective(False)
    # bucket overflow -> slow path: one bucket with more distinct keys than its table
    sp = P.Space(64, 32, 32)
    g = torch.Generator(device="cuda").manual_seed(3)
    keys = torch.randint(0, 2**62, (300_000, 1), device="cuda", generator=g, dtype=torch.int64).view(torch.uint64)
    check_sorted_unique(ctx.dedup_global(sp, keys))
    if size == "large":  # histogram-free partition passes (>= 2^26 keys), 90% duplicates
        n = 1 << 26
        base = torch.randint(0, 2**62, (n // 10, 1), device="cuda", generator=g, dtype=torch.int64)
        big = base[torch.randint(0, n // 10, (n,), device="cuda", generator=g)].contiguous().view(torch.uint64)
        u = ctx.dedup_global(sp, big)
        assert u.shape[0] == torch.unique(big).shape[0]
        print(f"large dedup: {n} keys -> {u.shape[0]}")
    torch.cuda.synchronize()
    print(f"sanitize_run {size}: OK ({ctx.kernel_launches} kernel launches)")
    ctx.close()


if __name__ == "__main__":
    main()
