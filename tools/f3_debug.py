import sys, os, json, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth
wl, ints, par = synth.workload_inputs("n2", n_parents=100_000)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7); di = P.DeviceIntegrals(ints.h, ints.eri)
ph = torch.from_numpy(par).pin_memory()
tot = ctx.gen_coupled_count(sp, ph.cuda(), di, 0.0)
host = P.HostRecords(tot, 1)
print("pinned", host.keys.is_pinned(), ph.is_pinned())
pool = ctx.pool(sp, 1 << 20)
ctx.profile(True); ctx.profile_read()
for mode in ["offload", "offload", "none", "none"]:
    pool.clear()
    t0 = time.time()
    st = ctx.stream_generate(sp, ph, di, 0.0, 25_000, pool, host if mode == "offload" else None)
    pr = ctx.profile_read()
    print(mode, f"{time.time()-t0:.3f}s", json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in st.items()}))
    print("   ", {k: (round(v[0], 2), v[1]) for k, v in pr.items()})
