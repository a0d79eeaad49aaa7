"""Time our local sort (dedup_finalize = onesweep LSD passes + unique) and the
dedup partition on distinct random keys; compare with tools/cub_bench."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 56
ctx = P.Context(0)
g = torch.Generator(device="cuda"); g.manual_seed(1)
keys = torch.randint(0, 1 << 62, (n, 1), device="cuda", dtype=torch.int64, generator=g)
keys &= (1 << bits) - 1
keys = keys.view(torch.uint64)
sp = P.Space(bits if bits % 2 == 0 else bits + 1, 1, 1)
for name, fn in [("finalize(sort+unique)", lambda: ctx.dedup_finalize(sp, keys)),
                 ("dedup_global(all distinct)", lambda: ctx.dedup_global(sp, keys))]:
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ctx.profile(True); ctx.profile_read()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); reps = 3
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    prof = {k: round(v[0] / reps, 3) for k, v in ctx.profile_read().items()}
    ctx.profile(False)
    print(f"{name}: n={n} bits={bits}: {ms:.3f} ms; per kernel class {prof}", flush=True)
