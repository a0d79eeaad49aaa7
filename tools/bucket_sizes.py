"""Bucket-size spread of an N2 batch's key stream in the hash order (top bits of hi)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth
npar = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
wl, ints, par = synth.workload_inputs("n2", n_parents=npar)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7); di = P.DeviceIntegrals(ints.h, ints.eri)
rec = ctx.gen_coupled(sp, torch.from_numpy(par).cuda(), di, 0.0, with_src=False)
k = rec.keys.view(torch.int64).reshape(-1)
def fmix(x):
    M = (1 << 64) - 1
    x = x ^ (x >> 30 & ((1 << 34) - 1)); x = x * (0xBF58476D1CE4E5B9 - (1 << 64))
    x = x ^ (x >> 27 & ((1 << 37) - 1)); x = x * (0x94D049BB133111EB - (1 << 64))
    x = x ^ (x >> 31 & ((1 << 33) - 1)); return x
for ch in range(0, 1):
    h = torch.empty_like(k)
    step = 1 << 28
    for a in range(0, k.numel(), step):
        h[a:a + step] = fmix(k[a:a + step])
u = torch.unique(h)
for bits in (14, 15, 16, 17, 18):
    top = (h >> (64 - bits)) & ((1 << bits) - 1)
    c = torch.bincount(top, minlength=1 << bits).double()
    cu = torch.bincount((u >> (64 - bits)) & ((1 << bits) - 1), minlength=1 << bits).double()
    print(f"bits {bits}: keys/bucket mean {c.mean():.0f} max {c.max():.0f} ({c.max()/c.mean():.3f}x) p99.99 {torch.quantile(c[:1<<16], 0.9999):.0f}; distinct mean {cu.mean():.0f} max {cu.max():.0f} ({cu.max()/cu.mean():.3f}x)")
# heaviest keys
vals, cnts = torch.unique(k, return_counts=True)
top = torch.topk(cnts, 5)
print("n", k.numel(), "distinct", vals.numel(), "top multiplicities", top.values.tolist())
