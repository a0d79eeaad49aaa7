import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, oracle, synth
ctx = P.Context(0)
W, Pn = 1, 4
sp = P.Space(64 * W, 1, 1)
allk = synth.zipf_keys(400_000, W, 1.1, 1 << 16, seed=5)
parts = np.array_split(allk, Pn)
refp = [oracle.dedup(allk, W, Pn, o) for o in range(Pn)]
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    bins = []
    for r in range(Pn):
        b, counts = ctx.dedup_partition(sp, torch.from_numpy(parts[r]).cuda(), Pn)
        offs = np.concatenate([[0], np.cumsum(counts)])
        bins.append([b[offs[o]:offs[o + 1]] for o in range(Pn)])
        ref_r = oracle.dedup(parts[r], W)
        allb = b.cpu().numpy()
        ok_part = np.array_equal(synth.unique_keys(allb), ref_r) and len(allb) == len(ref_r)
        if not ok_part:
            print("trial", trial, "rank", r, "partition wrong", len(allb), len(ref_r), len(synth.unique_keys(allb)))
    for o in range(Pn):
        recv = torch.cat([bins[r][o] for r in range(Pn)])
        got = ctx.dedup_finalize(sp, recv).cpu().numpy()
        if not np.array_equal(got.reshape(-1, W), refp[o].reshape(-1, W)):
            rk = recv.cpu().numpy()
            s = np.sort(got[:, 0])
            print("trial", trial, "owner", o, "finalize wrong: got", len(got), "ref", len(refp[o]),
                  "sorted?", np.all(got[1:, 0] > got[:-1, 0]), "set-equal?", np.array_equal(np.unique(got[:, 0]), refp[o][:, 0]),
                  "recv unique", len(np.unique(rk[:, 0])))
print("done")
