"""Compare device-resident vs host-input step timings (bench's e2e gap)."""
import sys, os, time, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth
wl, ints, par = synth.workload_inputs("n2", n_parents=1_000_000)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7); di = P.DeviceIntegrals(ints.h, ints.eri)
shard = ctx.dedup_global(sp, torch.from_numpy(par).cuda())
pinned = torch.from_numpy(shard.cpu().numpy()).pin_memory()
batches = [(0, 500_000), (500_000, 1_000_000)]
counts = [ctx.gen_coupled_count(sp, shard[a:b], di, 0.0) for a, b in batches]
cap = max(counts)
out = P.Records(torch.empty((cap, 1), dtype=torch.uint64, device="cuda"), torch.empty(cap, dtype=torch.float64, device="cuda"),
                torch.empty(cap, dtype=torch.int32, device="cuda"), None, cap)
up, spool = ctx.pool(sp, 1 << 20), ctx.pool(sp, 1 << 20)
def step(pd):
    up.clear(); spool.clear(); n = 0
    for a, b in batches:
        r = ctx.gen_coupled(sp, pd[a:b], di, 0.0, out=out); n += r.count
        u = ctx.dedup_global(sp, r.keys); ctx.merge_space(up, u); del u
    ctx.merge_space(spool, pd); ctx.merge_pool(spool, up)
    return n
for _ in range(2): step(shard)
def timeit(name, f, k=3):
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(k): f()
    e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"{name}: {e0.elapsed_time(e1)/k:.1f} ms/step (wall {(t1-t0)*1e3/k:.1f})")
timeit("device", lambda: step(shard))
def e2e():
    pd = torch.empty_like(shard); pd.copy_(pinned, non_blocking=True); step(pd)
timeit("e2e", e2e)
timeit("device again", lambda: step(shard))
pd0 = torch.empty_like(shard); pd0.copy_(pinned)
timeit("fresh tensor reused", lambda: step(pd0))
