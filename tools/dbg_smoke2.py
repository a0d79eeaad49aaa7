import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_15768_b200 as P, oracle, synth
ctx = P.Context(0)
for trial in range(4):
  for key, n in (("lih", None), ("h2o", 2000)):
    wl, ints, par = synth.workload_inputs(key, n_parents=n)
    sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
    di = P.DeviceIntegrals(ints.h, ints.eri)
    tp = torch.from_numpy(par).cuda()
    rec = ctx.gen_coupled(sp, tp, di, 0.0, with_src=True)
    uniq = ctx.dedup_global(sp, rec.keys)
    pool = ctx.pool(sp, 1024)
    pd = ctx.dedup_global(sp, tp)
    pdn = pd.cpu().numpy()
    ok1 = np.array_equal(synth.sort_keys(pdn), par)
    ctx.merge_space(pool, pd)
    pk = pool.keys().cpu().numpy()
    ok2 = np.array_equal(pk, pdn)
    un = uniq.cpu().numpy()
    ins = ctx.merge_space(pool, uniq, want_inserted=True)
    pk2 = pool.keys().cpu().numpy()
    ref_s, ref_ins = oracle.merge(par, synth.unique_keys(un), 1)
    ok3 = np.array_equal(synth.sort_keys(pk2), ref_s)
    print(trial, key, "parents-dedup", ok1, "pool1", ok2, "merge", ok3, len(pk2), len(ref_s),
          "extra", len(np.setdiff1d(pk2[:, 0], ref_s[:, 0])), "missing", len(np.setdiff1d(ref_s[:, 0], pk2[:, 0])), flush=True)
    pool.close()
