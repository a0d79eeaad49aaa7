import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth
npar = int(sys.argv[1]) if len(sys.argv) > 1 else 250_000
wl, ints, par = synth.workload_inputs("n2", n_parents=npar)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7); di = P.DeviceIntegrals(ints.h, ints.eri)
rec = ctx.gen_coupled(sp, torch.from_numpy(par).cuda(), di, 0.0, with_src=False)
for _ in range(2):
    u = ctx.dedup_global(sp, rec.keys)
torch.cuda.synchronize()
print(rec.count, u.shape)
