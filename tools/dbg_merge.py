import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2604_15768_b200 as P, oracle, synth
from test_gpu_parity import hash_sort, hash_hi_lo
ctx = P.Context(0)
W = int(sys.argv[1]) if len(sys.argv) > 1 else 1
trials = int(sys.argv[2]) if len(sys.argv) > 2 else 5
N0 = int(sys.argv[3]) if len(sys.argv) > 3 else 300_000
bad = 0
for trial in range(trials):
    rng = np.random.default_rng(2 + W + trial)
    sp = P.Space(64 * W, 1, 1)
    S0 = synth.unique_keys(rng.integers(1, 1 << 40, size=(N0, W), dtype=np.uint64))
    pool = ctx.pool(sp, capacity=1000)
    ctx.merge_space(pool, torch.from_numpy(hash_sort(S0, W)).cuda())
    for it in range(3):
        U = synth.unique_keys(np.concatenate([S0[rng.choice(len(S0), N0 // 6)], rng.integers(1, 1 << 40, size=(N0 // 4, W), dtype=np.uint64)]))
        before = pool.keys().cpu().numpy()
        ins = ctx.merge_space(pool, torch.from_numpy(hash_sort(U, W)).cuda(), want_inserted=True).cpu().numpy()
        after = pool.keys().cpu().numpy()
        hi, lo = hash_hi_lo(after, W)
        okord = bool(np.all((hi[1:] > hi[:-1]) | ((hi[1:] == hi[:-1]) & (lo[1:] > lo[:-1]))))
        ref_s, ref_ins = oracle.merge(before, U, W)
        okset = np.array_equal(synth.sort_keys(after), ref_s)
        if not (okord and okset):
            bad += 1
            badpos = np.nonzero(~((hi[1:] > hi[:-1]) | ((hi[1:] == hi[:-1]) & (lo[1:] > lo[:-1]))))[0]
            print("trial", trial, "it", it, "order", okord, "set", okset, len(after), len(ref_s), "bad positions", badpos[:10], "tile", badpos[:10] // 2048, flush=True)
    pool.close()
print("bad", bad)
