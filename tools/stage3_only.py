"""Time energy_contract alone on the bench's N2 data (first batch)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth
wl, ints, par = synth.workload_inputs("n2", n_parents=1_000_000)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7); di = P.DeviceIntegrals(ints.h, ints.eri)
shard = ctx.dedup_global(sp, torch.from_numpy(par).cuda())
rec = ctx.gen_coupled(sp, shard[:500_000], di, 0.0, with_src=True)
u = ctx.dedup_global(sp, rec.keys)
psi = torch.rand(u.shape[0], dtype=torch.float64, device="cuda") * 2 - 1
for _ in range(2):
    e, miss = ctx.energy_contract(sp, rec, 500_000, u, psi)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); e, miss = ctx.energy_contract(sp, rec, 500_000, u, psi); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"contract {rec.count} records, space {u.shape[0]}: {ms:.2f} ms, {rec.count/ms/1e6:.3e} rec/s, missing {miss}")
