import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, synth
ctx = P.Context(0)
for W, m, n in [(1, 56, int(sys.argv[1])), (2, 96, int(sys.argv[1]) // 2)]:
    rng = np.random.default_rng(n)
    base = rng.integers(1, 1 << min(m, 62), size=(max(1, n // 4), W), dtype=np.uint64)
    keys = base[rng.integers(0, len(base), size=n)]
    sp = P.Space(m, 1, 1)
    got = ctx.dedup_global(sp, torch.from_numpy(keys).cuda()).cpu().numpy()
    ref = synth.unique_keys(keys)
    print(W, n, len(got), len(ref), np.array_equal(got, ref), flush=True)
