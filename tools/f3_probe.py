"""C2H4 streamed Stage 1 (no offload): unique-pool growth and time vs parents."""
import sys, os, json, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth
wl, ints, par = synth.workload_inputs("c2h4", n_parents=int(sys.argv[1]) if len(sys.argv) > 1 else 400_000)
ctx = P.Context(0)
sp = P.Space(wl.m, wl.n_alpha, wl.n_beta); di = P.DeviceIntegrals(ints.h, ints.eri)
ph = torch.from_numpy(par).pin_memory()
for n in [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [50_000, 100_000, 200_000, 400_000]:
    pool = ctx.pool(sp, 1 << 24)
    t0 = time.time()
    st = ctx.stream_generate(sp, ph[:n], di, 0.0, 20_000, pool)
    print(json.dumps({"parents": n, "wall_s": time.time() - t0, **st, "redundancy": 1 - st["unique"] / st["records"]}), flush=True)
    pool.close()
    torch.cuda.empty_cache()
