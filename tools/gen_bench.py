"""Time gen_coupled alone (device-resident parents, preallocated outputs)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth, json
wl_name = sys.argv[1] if len(sys.argv) > 1 else "n2"
npar = int(sys.argv[2]) if len(sys.argv) > 2 else 250_000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
with_src = (sys.argv[4] != "nosrc") if len(sys.argv) > 4 else True
wl, ints, par = synth.workload_inputs(wl_name, n_parents=npar)
ctx = P.Context(0)
sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
di = P.DeviceIntegrals(ints.h, ints.eri)
tp = torch.from_numpy(par).cuda()
cnt = ctx.gen_coupled_count(sp, tp, di)
out = P.Records(torch.empty((cnt, wl.words), dtype=torch.uint64, device="cuda"), torch.empty(cnt, dtype=torch.float64, device="cuda"),
                torch.empty(cnt, dtype=torch.int32, device="cuda") if with_src else None, None, cnt)
for _ in range(2): ctx.gen_coupled(sp, tp, di, 0.0, out=out)
torch.cuda.synchronize()
ctx.profile(True); ctx.profile_read()
for _ in range(reps): ctx.gen_coupled(sp, tp, di, 0.0, out=out)
prof = ctx.profile_read()
ms = prof["gen"][0] / prof["gen"][1]
B = cnt * (8 * wl.words + 8 + (4 if with_src else 0)) + len(par) * 8 * wl.words
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6545.3
print(f"gen {wl_name} parents={len(par)} records={cnt} ({cnt/len(par):.0f}/parent): {ms:.3f} ms/launch, "
      f"{cnt/ms/1e6:.3e} rec/s, {B/ms/1e6:.0f} GB/s = {B/ms/1e6/peak*100:.1f}% of {peak} GB/s")
