"""Time the f2 building blocks (sort_unique = hash dedup + LSD radix sort) on one N2 batch."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth
npar = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
wl, ints, par = synth.workload_inputs("n2", n_parents=npar)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7); di = P.DeviceIntegrals(ints.h, ints.eri)
r = ctx.gen_coupled(sp, torch.from_numpy(par).cuda(), di, 0.0, with_src=False)
u = ctx.dedup_global(sp, r.keys)
for name, fn in [("dedup_global", lambda: ctx.dedup_global(sp, r.keys)),
                 ("sort_unique(raw)", lambda: ctx.sort_unique(sp, r.keys)),
                 ("sort_unique(distinct)", lambda: ctx.sort_unique(sp, u))]:
    fn(); torch.cuda.synchronize(); ctx.profile(True); ctx.profile_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); x = fn(); e1.record(); torch.cuda.synchronize(); del x
    p = ctx.profile_read()
    print(f"{name}: n={r.count if 'raw' in name or name == 'dedup_global' else u.shape[0]} {e0.elapsed_time(e1):.2f} ms  " +
          " ".join(f"{k}={v[0]:.2f}/{v[1]}" for k, v in sorted(p.items(), key=lambda kv: -kv[1][0])))
