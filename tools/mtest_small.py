import sys, os, torch, time
sys.path.insert(0, '/root/repo')
import paper_2604_15768_b200 as P, synth
wl, ints, par = synth.workload_inputs("n2", n_parents=1_000_000)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7)
shard = ctx.dedup_global(sp, torch.from_numpy(par).cuda())
for cap in (1 << 20, 1 << 22):
    pool = ctx.pool(sp, cap)
    for rep in range(3):
        pool.clear(); torch.cuda.synchronize()
        ctx.profile(True); ctx.profile_read()
        t0 = time.perf_counter(); ctx.merge_space(pool, shard); torch.cuda.synchronize(); t1 = time.perf_counter()
        print(cap, rep, f"{(t1-t0)*1e3:.2f} ms wall", ctx.profile_read(), len(pool))
