"""Print the dedup plan statistics for the bench's N2 batch (5e5 parents)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth
npar = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
wl, ints, par = synth.workload_inputs("n2", n_parents=npar)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7); di = P.DeviceIntegrals(ints.h, ints.eri)
shard = ctx.dedup_global(sp, torch.from_numpy(par).cuda())
rec = ctx.gen_coupled(sp, shard, di, 0.0, with_src=False)
ctx.dedup_stats(reset=True)
ctx.profile(True); ctx.profile_read()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
u = ctx.dedup_global(sp, rec.keys); torch.cuda.synchronize()
e0.record(); u = ctx.dedup_global(sp, rec.keys); e1.record(); torch.cuda.synchronize()
p = ctx.profile_read()
print(rec.count, u.shape[0], ctx.dedup_stats(reset=True), f"{e0.elapsed_time(e1):.2f} ms", {k: round(v[0] / 2, 2) for k, v in p.items()})
