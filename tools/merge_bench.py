"""Time merge_space alone on N2-like unique shards (per kernel class)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth
npar = int(sys.argv[1]) if len(sys.argv) > 1 else 250_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl, ints, par = synth.workload_inputs("n2", n_parents=npar)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7); di = P.DeviceIntegrals(ints.h, ints.eri)
half = npar // 2
r1 = ctx.gen_coupled(sp, torch.from_numpy(par[:half]).cuda(), di, 0.0, with_src=False)
u1 = ctx.dedup_global(sp, r1.keys); del r1
r2 = ctx.gen_coupled(sp, torch.from_numpy(par[half:]).cuda(), di, 0.0, with_src=False)
u2 = ctx.dedup_global(sp, r2.keys); del r2
pool = ctx.pool(sp, 1 << 20)
def once():
    pool.clear()
    ctx.merge_space(pool, u1)
    ctx.merge_space(pool, u2)
once(); once()
torch.cuda.synchronize()
ctx.profile(True); ctx.profile_read()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    once()
e1.record(); torch.cuda.synchronize()
p = ctx.profile_read()
n_in = u1.shape[0] * 2 + u2.shape[0]; n_out = u1.shape[0] + len(pool)
gb = (n_in + n_out) * 8 / 1e9
ms = e0.elapsed_time(e1) / reps
print(f"merge |U1|={u1.shape[0]} |U2|={u2.shape[0]} -> {len(pool)}: {ms:.2f} ms/pair ({gb/ms*1e3:.0f} GB/s algorithmic)  " + " ".join(f"{k}={v[0]/reps:.2f}" for k, v in sorted(p.items(), key=lambda kv: -kv[1][0])))
if len(sys.argv) > 3 and sys.argv[3] == "nosparse":
    sys.exit(0)
# sparse: a pool of the parents (1 / |U| ~ 1/400) merged with the union (S <- S u C)
spool = ctx.pool(sp, 1 << 20)
pd = ctx.dedup_global(sp, torch.from_numpy(par).cuda())
def once_sparse():
    spool.clear()
    ctx.merge_space(spool, pd)
    ctx.merge_pool(spool, pool)
once_sparse(); torch.cuda.synchronize(); ctx.profile_read()
e0.record()
for _ in range(reps):
    once_sparse()
e1.record(); torch.cuda.synchronize()
p = ctx.profile_read()
ms = e0.elapsed_time(e1) / reps
gb = 2 * len(pool) * 8 / 1e9
print(f"sparse |S|={npar} |U|={len(pool)} -> {len(spool)}: {ms:.2f} ms ({gb/ms*1e3:.0f} GB/s copy-equivalent)  " + " ".join(f"{k}={v[0]/reps:.3f}" for k, v in sorted(p.items(), key=lambda kv: -kv[1][0])))
