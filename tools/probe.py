"""Exploratory probe: host wall time per library call (synchronised) for the
bench workload, to separate kernel time from host/allocation overhead."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_15768_b200 as P, synth

wlname = sys.argv[1] if len(sys.argv) > 1 else "n2"
npar = int(sys.argv[2]) if len(sys.argv) > 2 else None
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 250_000
wl, ints, par = synth.workload_inputs(wlname, n_parents=npar)
ctx = P.Context(0)
sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
di = P.DeviceIntegrals(ints.h, ints.eri)
tp = torch.from_numpy(par).cuda()
tph = ctx.dedup_global(sp, tp)  # parents in the pool (hash) order
batches = [(i, min(i + batch, len(par))) for i in range(0, len(par), batch)]
cnts = [ctx.gen_coupled_count(sp, tp[a:b], di) for a, b in batches]
cap = max(cnts)
out = P.Records(torch.empty((cap, wl.words), dtype=torch.uint64, device="cuda"),
                torch.empty(cap, dtype=torch.float64, device="cuda"),
                torch.empty(cap, dtype=torch.int32, device="cuda"), None, cap)
def T(): torch.cuda.synchronize(); return time.perf_counter()
upool = ctx.pool(sp, 1 << 20); spool = ctx.pool(sp, 1 << 20)
for it in range(5):
    ctx.profile(True); ctx.profile_read()
    t0 = T(); tim = {}
    upool.clear(); spool.clear()
    for a, b in batches:
        t = T(); rec = ctx.gen_coupled(sp, tp[a:b], di, 0.0, out=out); tim["gen"] = tim.get("gen", 0) + T() - t
        t = T(); u = ctx.dedup_global(sp, rec.keys); tim["dedup"] = tim.get("dedup", 0) + T() - t
        t = T(); ctx.merge_space(upool, u); tim["merge"] = tim.get("merge", 0) + T() - t
        del u
    t = T(); ctx.merge_space(spool, tph); ctx.merge_pool(spool, upool)
    tim["final"] = T() - t
    tot = T() - t0
    prof = ctx.profile_read()
    ksum = sum(v[0] for v in prof.values())
    print(f"iter {it}: total {tot*1e3:.1f} ms, kernels {ksum:.1f} ms, " + ", ".join(f"{k} {v*1e3:.1f}" for k, v in tim.items()))
    print("   ", {k: round(v[0], 2) for k, v in prof.items()})
print("torch reserved GB", torch.cuda.memory_reserved() / 1e9)
