"""Owner-side finalize (dedup_finalize_runs) on what owner 0 receives from P ranks
(each rank's keys with owner 0: a 1/P slice of the hash range), timed against
dedup_finalize on the concatenation; dedup stats show the slow-path count."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as PK  # noqa: E402

ctx = PK.Context(0)
sp = PK.Space(56, 7, 7)
g = torch.Generator(device="cuda").manual_seed(1)
for P, n_per in ((8, 200_000_000), (2, 100_000_000), (3, 100_000_000), (8, 2_000_000), (5, 20_000_000)):
    base = torch.randint(0, 2**55, (n_per * P // 3, 1), device="cuda", generator=g, dtype=torch.int64)
    runs, cnts = [], []
    for r in range(P):
        pick = base[torch.randint(0, base.shape[0], (n_per,), device="cuda", generator=g)].view(torch.uint64)
        bins, c = ctx.dedup_partition(sp, pick, P)
        runs.append(bins[: c[0]].clone())
        cnts.append(c[0])
        del bins, pick
    recv = torch.cat(runs)
    del runs
    for rep in range(2):
        ctx.profile(True)
        ctx.profile_read()
        ctx.dedup_stats(reset=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = ctx.dedup_finalize_runs(sp, recv, cnts)
        e1.record()
        torch.cuda.synchronize()
        pr = ctx.profile_read()
        st = ctx.dedup_stats(reset=True)
    ref = torch.unique(recv.view(torch.int64)).shape[0]
    print(P, recv.shape[0], out.shape[0], ref, "runs %.2f ms" % e0.elapsed_time(e1),
          {k: round(v[0], 2) for k, v in pr.items()}, "slow_path", st["slow_path_calls"], "buckets", st["buckets"])
    assert out.shape[0] == ref
