"""Measured model of one rank's work in the P-GPU N2 step, on one GPU:
the 10^6 parents are split by hash owner into P shards; for every shard r we time
gen_coupled and the local unique filter + owner partition (dedup_partition) and keep
the bin destined to owner 0; then owner 0's finalize over the P received runs
(dedup_finalize_runs) and its merge into the pool are timed.  Prints one JSON line:
per-rank ms (max over shards) and bytes each rank sends.
    python tools/shard_model.py [P] [parents]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_15768_b200 as PK  # noqa: E402
import synth  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
npar = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
wl, ints, par = synth.workload_inputs("n2", n_parents=npar)
ctx = PK.Context(0)
sp = PK.Space(wl.m, wl.n_alpha, wl.n_beta)
di = PK.DeviceIntegrals(ints.h, ints.eri)
bins, counts = ctx.dedup_partition(sp, torch.from_numpy(par).cuda(), P)   # parents by hash owner
offs = [0]
for c in counts:
    offs.append(offs[-1] + c)


def timed(fn, reps=2):
    """the last of `reps` runs (the first grows the scratch arena)"""
    for _ in range(reps - 1):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    return r, e0.elapsed_time(e1)


rows, runs, run_counts = [], [], []
for r in range(P):
    shard = bins[offs[r]:offs[r + 1]]
    rec, t_gen = timed(lambda: ctx.gen_coupled(sp, shard, di, 0.0, with_src=True))
    (lb, lc), t_ded = timed(lambda: ctx.dedup_partition(sp, rec.keys, P))
    rows.append({"parents": int(shard.shape[0]), "records": int(rec.count), "gen_ms": t_gen, "local_dedup_ms": t_ded,
                 "local_unique": int(sum(lc)), "sent_keys": int(sum(lc) - lc[r])})
    runs.append(lb[:lc[0]].clone())
    run_counts.append(lc[0])
    del rec, lb
recv = torch.cat(runs)
u, t_fin = timed(lambda: ctx.dedup_finalize_runs(sp, recv, run_counts), reps=3)
# owner 0's pool already holds the other half of its shard (S u U_new, |S| ~ |U|)
half = u.shape[0] // 2
pool = ctx.pool(sp, 1 << 20)


def merge_once():
    pool.clear()
    ctx.merge_space(pool, u[::2].contiguous())   # (every other key: still pi-sorted)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.merge_space(pool, u[1::2].contiguous())
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


merge_once()
t_merge = merge_once()
W = wl.words
out = {"P": P, "parents": npar, "ranks": rows, "owner0_received_keys": int(recv.shape[0]), "owner0_unique": int(u.shape[0]),
       "owner0_finalize_ms": t_fin, "owner0_merge_ms": t_merge,
       "max_gen_ms": max(x["gen_ms"] for x in rows), "max_local_dedup_ms": max(x["local_dedup_ms"] for x in rows),
       "max_sent_bytes": max(x["sent_keys"] for x in rows) * 8 * W}
out["exchange_ms_at_600GBs"] = out["max_sent_bytes"] / 600e9 * 1e3
out["model_rank_ms"] = out["max_gen_ms"] + out["max_local_dedup_ms"] + out["exchange_ms_at_600GBs"] + t_fin + t_merge
print(json.dumps(out))
