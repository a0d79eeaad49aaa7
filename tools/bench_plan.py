"""Dedup plan of each bench batch (N2, 1e6 parents, 2 batches)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth
wl, ints, par = synth.workload_inputs("n2", n_parents=1_000_000)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7); di = P.DeviceIntegrals(ints.h, ints.eri)
shard = ctx.dedup_global(sp, torch.from_numpy(par).cuda())
for a, b in [(0, 500_000), (500_000, 1_000_000)]:
    rec = ctx.gen_coupled(sp, shard[a:b], di, 0.0, with_src=False)
    ctx.dedup_stats(reset=True)
    u = ctx.dedup_global(sp, rec.keys)
    print(a, b, rec.count, u.shape[0], ctx.dedup_stats(reset=True))
    del rec, u
