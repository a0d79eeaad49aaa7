"""Time dedup_global alone on an N2-like generated key stream (per kernel class)."""
import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth
npar = int(sys.argv[1]) if len(sys.argv) > 1 else 250_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl, ints, par = synth.workload_inputs("n2", n_parents=npar)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7); di = P.DeviceIntegrals(ints.h, ints.eri)
rec = ctx.gen_coupled(sp, torch.from_numpy(par).cuda(), di, 0.0, with_src=False)
u = ctx.dedup_global(sp, rec.keys)
u2 = ctx.dedup_global(sp, u)          # all-distinct input (finalize-like)
torch.cuda.synchronize()
ctx.profile(True); ctx.profile_read()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    u = ctx.dedup_global(sp, rec.keys)
e1.record(); torch.cuda.synchronize()
p = ctx.profile_read()
ms = e0.elapsed_time(e1) / reps
print(f"dedup n={rec.count} -> {u.shape[0]}: {ms:.2f} ms/call  " + " ".join(f"{k}={v[0]/reps:.2f}" for k, v in sorted(p.items(), key=lambda kv: -kv[1][0])))
e0.record()
for _ in range(reps):
    u2 = ctx.dedup_global(sp, u)
e1.record(); torch.cuda.synchronize()
p = ctx.profile_read()
print(f"dedup distinct n={u.shape[0]}: {e0.elapsed_time(e1)/reps:.2f} ms/call  " + " ".join(f"{k}={v[0]/reps:.2f}" for k, v in sorted(p.items(), key=lambda kv: -kv[1][0])))
