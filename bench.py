"""bench.py -- one step of the selected-CI hot path (QiankunNet-cuSCI,
arXiv 2604.15768) on N B200s:

    for each parent batch of this rank's shard:
        gen_coupled(batch, integrals, eps)      # coupled configs + H_ij (a1-a7)
        dedup_global(records.keys)              # global de-dup (a8-a11), NCCL when N > 1
        merge_space(unique_pool, U_batch)       # GPU-resident union of the unique set
    merge_space(space_pool, unique_pool)        # S <- S u C (a12)

Workload (default, --workload n2): the N2 cc-pVDZ-like configuration of
BASELINE.json (56 spin orbitals, 14 electrons, 10^6 parents, synthetic
D2h-like integrals, eps = 0); parents are sharded across ranks by hash owner
(strong scaling: fixed total work).  Prints ONE JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "coupled configs/sec (with H_ij) and unique configs/sec after global dedup, 1/2/4/8 B200"
HBM_NOMINAL_GBS = 7700.0  # B200 HBM3e spec (B200_PROFILING.md); the roofline peak is the measured copy


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="n2")
    ap.add_argument("--parents", type=int, default=None, help="override the workload's parent count")
    ap.add_argument("--batch", type=int, default=None, help="parents per gen_coupled call")
    ap.add_argument("--eps", type=float, default=0.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-stage3", action="store_true", help="skip the Stage-3 contraction measurement (SURVEY 8(f) f1)")
    ap.add_argument("--no-f2", action="store_true", help="skip the regular-sampling dedup measurement (SURVEY 8(f) f2)")
    ap.add_argument("--no-f3", action="store_true", help="skip the streaming-stage measurement (SURVEY 8(f) f3)")
    ap.add_argument("--f3-parents", type=int, default=100_000, help="parents of the f3 offload measurement")
    ap.add_argument("--no-f4", action="store_true", help="skip the SCI growth measurement (SURVEY 8(f) f4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=None, help="parents in the oracle's bounded sample")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- distributed
def dist_setup(gpus: int):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != gpus:
        raise SystemExit(f"--gpus {gpus} but WORLD_SIZE={world}")
    pg = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    return rank, world, local, pg


def bcast_bytes(pg, payload: bytes | None, rank: int) -> bytes:
    if pg is None:
        return payload
    obj = [payload if rank == 0 else None]
    pg.broadcast_object_list(obj, src=0)
    return obj[0]


def _reduce_device(pg):
    import torch
    return "cuda" if pg.get_backend() == "nccl" else "cpu"


def allreduce_max(pg, x: float) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=_reduce_device(pg))
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(pg, x: float) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=_reduce_device(pg))
    pg.all_reduce(t, op=pg.ReduceOp.SUM)
    return float(t.item())


def plan_batches(pg, n_par: int, batch: int):
    """Parent batches of this rank's shard.  dedup_global is collective, so every
    rank must make the same number of calls: the batch count is agreed (max
    over ranks) and each shard is split evenly into that many batches."""
    n_batches = int(allreduce_max(pg, float(max(1, -(-n_par // max(1, batch))))))
    edges = [round(i * n_par / n_batches) for i in range(n_batches + 1)]
    return [(edges[i], edges[i + 1]) for i in range(n_batches)]


def barrier(pg):
    if pg is not None:
        pg.barrier()


# ----------------------------------------------------------------------------- oracle (cpu baseline)
def oracle_sample(wl, ints, par, n_sample: int):
    """The oracle as it stands, single host thread, on a bounded sample of the
    workload: the first n_sample parents through gen -> dedup -> merge."""
    import oracle
    sample = par[:n_sample]
    t0 = time.perf_counter()
    rec = oracle.gen_coupled(wl.m, wl.n_alpha, wl.n_beta, sample, ints, 0.0)
    u = oracle.dedup(rec["keys"], wl.words)
    s2, ins = oracle.merge(sample, u, wl.words)
    dt = time.perf_counter() - t0
    return len(rec["src"]), len(u), dt


def oracle_sample_mt(wl, ints, par, n_sample: int, threads: int):
    """oracle-MT: the same unmodified oracle calls with the parents
    sharded over host threads (ctypes releases the GIL inside the C++ oracle):
    per-shard gen + std::set dedup in parallel, then one std::set dedup of the
    shards' unique keys and the set_union merge."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    sample = par[:n_sample]
    shards = [x for x in np.array_split(sample, threads) if len(x)]
    t0 = time.perf_counter()

    def work(sh):
        rec = oracle.gen_coupled(wl.m, wl.n_alpha, wl.n_beta, sh, ints, 0.0)
        return len(rec["src"]), oracle.dedup(rec["keys"], wl.words)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        parts = list(ex.map(work, shards))
    nrec = sum(p[0] for p in parts)
    u = oracle.dedup(np.concatenate([p[1] for p in parts]), wl.words)
    oracle.merge(sample, u, wl.words)
    return nrec, len(u), time.perf_counter() - t0


def default_cpu_sample(wl) -> int:
    return {"lih": 225, "h2o": 4000, "h2o_dense": 1000, "n2": 1000, "c2h4": 40, "m120": 4}.get(wl, 100)


def run_reference(args):
    """--impl reference: the oracle (the one reference this tier has), timed as
    it stands on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    # bounded: ~15 s of oracle work per step at --steps 5, shrunk for longer runs
    n_sample = args.cpu_sample or max(1, int(default_cpu_sample(args.workload) * min(1.0, 5.0 / max(1, args.steps))))
    wl, ints, par = synth.workload_inputs(args.workload, n_parents=max(n_sample, 1) if args.parents is None else args.parents)
    for _ in range(args.warmup):
        oracle_sample(wl, ints, par, max(1, n_sample // 10))
    recs, uniq, times = 0, 0, []
    for _ in range(args.steps):
        r, u, dt = oracle_sample(wl, ints, par, n_sample)
        recs, uniq = r, u
        times.append(dt)
    t = sum(times) / len(times)
    value = recs / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "coupled configs/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{wl.name} ({args.workload})", "m": wl.m, "n_alpha": wl.n_alpha,
                   "n_beta": wl.n_beta, "point_group_irreps": wl.g, "parents": n_sample, "eps": 0.0},
        "unique_configs_per_s": uniq / t,
        "cpu_baseline": {"value": value, "unit": "coupled configs/s", "cores": 1, "kind": "oracle",
                         "sample": f"{n_sample} parents (first distinct sampler draws) of the {args.workload} workload through "
                                   f"oracle gen -> std::set dedup -> set_union merge ({recs} records, {uniq} unique)"},
        "e2e": {"value": value, "unit": "coupled configs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- ours
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    import paper_2604_15768_b200 as P
    import synth

    rank, world, local, pg = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nid = bcast_bytes(pg, P.Context.nccl_unique_id() if (world > 1 and rank == 0) else None, rank)
    ctx = P.Context(local, rank, world, nccl_id=nid)
    stream = ctx.stream

    wl, ints, par_all = synth.workload_inputs(args.workload, n_parents=args.parents)
    sp = P.Space(wl.m, wl.n_alpha, wl.n_beta)
    W = wl.words
    di = P.DeviceIntegrals(ints.h, ints.eri, dev)
    # shard the parent set by hash owner (the same owner function as the pool)
    mine = np.array_split(par_all, world)[rank]
    shard = ctx.dedup_global(sp, torch.from_numpy(mine).to(dev))   # parents owned by this rank (sorted)
    n_par = int(shard.shape[0])
    batch = args.batch or {"n2": 500_000, "c2h4": 20_000}.get(args.workload, max(1, n_par))
    batches = plan_batches(pg, n_par, batch)
    batch = max(b - a for a, b in batches) if batches else 0
    # plan: exact record counts per batch (buffer sizing; outside the timed region)
    counts = [ctx.gen_coupled_count(sp, shard[a:b], di, args.eps) for a, b in batches]
    cap = max(counts) if counts else 1
    keys_buf = torch.empty((cap, W), dtype=torch.uint64, device=dev)
    hij_buf = torch.empty(cap, dtype=torch.float64, device=dev)
    src_buf = torch.empty(cap, dtype=torch.int32, device=dev)
    out = P.Records(keys_buf, hij_buf, src_buf, None, cap)
    shard_host = shard.cpu().numpy()
    shard_pinned = torch.from_numpy(shard_host).pin_memory()

    upool = ctx.pool(sp, 1 << 20)   # union of the unique coupled configurations C
    spool = ctx.pool(sp, 1 << 20)   # the space S (starts as the parent shard)

    mstat = [0]  # merge algorithmic bytes (read |S| + |U|, write |S'|) accumulated by step()

    def merge_acc(pool, n_new, fn):
        before = len(pool)
        fn()
        mstat[0] += (before + n_new + len(pool)) * 8 * W

    def step(parents_dev, e2e=False):
        """one pass of the hot path; returns (records, unique, space_size)."""
        nrec = 0
        upool.clear()
        spool.clear()
        for (a, b) in batches:
            rec = ctx.gen_coupled(sp, parents_dev[a:b], di, args.eps, out=out)
            nrec += rec.count
            u = ctx.dedup_global(sp, rec.keys)
            merge_acc(upool, u.shape[0], lambda: ctx.merge_space(upool, u))
            del u
        merge_acc(spool, parents_dev.shape[0], lambda: ctx.merge_space(spool, parents_dev))
        merge_acc(spool, len(upool), lambda: ctx.merge_pool(spool, upool))
        return nrec, len(upool), len(spool)

    # warm-up
    for _ in range(args.warmup):
        step(shard)
    torch.cuda.synchronize()

    # ---------------- timed region (device-resident inputs)
    clocks = ClockSampler(local)
    clocks.start()
    ctx.profile(True)
    ctx.profile_read()
    ctx.dedup_stats(reset=True)
    mstat[0] = 0
    launches0 = ctx.kernel_launches
    barrier(pg)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    tot_rec = tot_uni = 0
    for _ in range(args.steps):
        r, u, s = step(shard)
        tot_rec += r
        tot_uni += u
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(pg)
    ms_local = ev0.elapsed_time(ev1)
    prof = ctx.profile_read()
    dstats = ctx.dedup_stats(reset=True)
    merge_bytes = mstat[0] // args.steps
    ctx.profile(False)
    launches = ctx.kernel_launches - launches0
    clk = clocks.stop()
    ms = allreduce_max(pg, ms_local)
    recs_all = allreduce_sum(pg, tot_rec)
    uni_all = allreduce_sum(pg, tot_uni)
    value = recs_all / (ms / 1e3)
    unique_rate = uni_all / (ms / 1e3)

    # ---------------- Stage-3 contraction (not part of the headline step):
    # e[s] = sum_j H_sj psi_j over every batch's records, psi synthetic and
    # aligned with the unique set C (the upool), reverse index just in time
    stage3 = None
    if not args.no_stage3 and world == 1:
        ukeys = upool.keys()
        g = torch.Generator(device=dev).manual_seed(11)
        psi = torch.rand(ukeys.shape[0], dtype=torch.float64, device=dev, generator=g) * 2.0 - 1.0
        e_all = torch.empty(n_par, dtype=torch.float64, device=dev)
        s_ms, s_rec, s_miss = 0.0, 0, 0
        for rep in range(2):  # first pass = warm-up
            s_ms, s_rec, s_miss = 0.0, 0, 0
            for (a, b) in batches:
                rec = ctx.gen_coupled(sp, shard[a:b], di, args.eps, out=out)
                c0 = torch.cuda.Event(enable_timing=True)
                c1 = torch.cuda.Event(enable_timing=True)
                c0.record(stream)
                _, miss = ctx.energy_contract(sp, rec, b - a, ukeys, psi, e=e_all[a:b])
                c1.record(stream)
                torch.cuda.synchronize()
                s_ms += c0.elapsed_time(c1)
                s_rec += rec.count
                s_miss += miss
        s_bytes = s_rec * (8 * W + 8 + 4 + 8)   # record read + one psi gather per record
        stage3 = {"records_per_s": s_rec / (s_ms / 1e3), "ms_per_step": s_ms, "records": s_rec, "missing": s_miss,
                  "space": int(ukeys.shape[0]), "achieved_GBs": s_bytes / (s_ms / 1e3) / 1e9,
                  "e_checksum": float(e_all.abs().sum().item())}
        del ukeys, psi, e_all

    # ---------------- the paper's regular-sampling sorted dedup (not in the headline step):
    # dedup_sorted on one batch's records against dedup_global on the same keys, and
    # Table-1 balance (max/min, CV of the owned unique shard sizes) for P = 8 virtual
    # ranks (the batch split by parent, as ranks would own it): regular-sampling
    # splitters (S = 1024, PAPER.md :454) vs the hash owner (DESIGN.md r9)
    f2 = None
    if not args.no_f2 and world == 1 and batches:
        a, b = batches[0]
        rec = ctx.gen_coupled(sp, shard[a:b], di, args.eps, out=out)
        kk = rec.keys
        def timed(fn, reps=2):
            for _ in range(2):   # the 2nd call settles the library's scratch arena (one-time consolidation)
                fn()
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            for _ in range(reps):
                r = fn()
                del r
            t1.record(stream)
            torch.cuda.synchronize()
            return t0.elapsed_time(t1) / reps
        ms_sorted = timed(lambda: ctx.dedup_sorted(sp, kk, 1024))
        ms_hash = timed(lambda: ctx.dedup_global(sp, kk))
        Pv, Sv = 8, 1024
        ends = [a + (b - a) * i // Pv for i in range(Pv + 1)]
        smp, spl_in = [], None
        for i in range(Pv):   # Step 1 per virtual rank: sort + unique, regular samples
            ri = ctx.gen_coupled(sp, shard[ends[i]:ends[i + 1]], di, args.eps, out=out, with_src=False)
            d = ctx.sort_unique(sp, ri.keys)
            smp.append(ctx.regular_samples(sp, d, Sv).clone())
            del d
        spl = ctx.select_splitters(sp, torch.cat(smp), Pv)
        rec = ctx.gen_coupled(sp, shard[a:b], di, args.eps, out=out)
        glob_sorted = ctx.sort_unique(sp, rec.keys)
        bnd = ctx.split_bounds(sp, glob_sorted, spl, Pv)
        n_uni = int(glob_sorted.shape[0])
        del glob_sorted
        _, hcounts = ctx.dedup_partition(sp, rec.keys, Pv)
        def bal(c):
            c = np.asarray(c, dtype=np.float64)
            return {"sizes": [int(x) for x in c], "max_over_min": float(c.max() / max(c.min(), 1)),
                    "cv": float(c.std() / c.mean())}
        f2 = {"records": int(rec.count), "unique": n_uni,
              "dedup_sorted_ms": ms_sorted, "dedup_sorted_keys_per_s": rec.count / (ms_sorted / 1e3),
              "dedup_global_ms": ms_hash, "dedup_global_keys_per_s": rec.count / (ms_hash / 1e3),
              "table1_P8": {"samples_per_rank": Sv,
                            "regular_sampling": bal([bnd[r + 1] - bnd[r] for r in range(Pv)]),
                            "hash_owner": bal(hcounts)}}

    # ---------------- f3: memory-centric streaming (Sec 4.3; not in the headline step)
    # Stage 1 with the original set offloaded to pinned host memory (3 streams), then
    # Stage 3 both ways: reload the original set H2D, or regenerate it on the device
    f3 = None
    if not args.no_f3 and world == 1:
        ctx.release_cached()   # the step's scratch peak: the stage runs in a fresh device budget
        nf = min(args.f3_parents, n_par)
        sh_h = torch.from_numpy(shard_host[:nf].copy()).pin_memory()
        tot_f = ctx.gen_coupled_count(sp, shard[:nf], di, args.eps)
        host = P.HostRecords(tot_f, W)
        fpool = ctx.pool(sp, 1 << 20)
        fb = max(1, nf // 4)
        ctx.stream_generate(sp, sh_h, di, args.eps, fb, fpool, host)      # warm-up (allocator, pinned pages)
        fpool.clear()
        st1 = ctx.stream_generate(sp, sh_h, di, args.eps, fb, fpool, host)
        fk = fpool.keys()
        g = torch.Generator(device=dev).manual_seed(13)
        fpsi = torch.rand(fk.shape[0], dtype=torch.float64, device=dev, generator=g) * 2.0 - 1.0
        ctx.stream_energy(sp, host, nf, fk, fpsi, batch_records=max(1, tot_f // 4))
        e_r, _, st3 = ctx.stream_energy(sp, host, nf, fk, fpsi, batch_records=max(1, tot_f // 4))
        e_g, _, st3g = ctx.stream_energy_regen(sp, sh_h, di, args.eps, fb, fk, fpsi)
        rb = 8 * W + 12
        f3 = {"parents": nf, "batches": st1["batches"], "records": st1["records"], "unique": st1["unique"],
              "stage1_offload": {**st1, "overlap_ms": st1["ms_h2d"] + st1["ms_compute"] + st1["ms_d2h"] - st1["ms_wall"],
                                 "d2h_GBs": st1["d2h_bytes"] / max(st1["ms_d2h"], 1e-9) / 1e6},
              "stage3_reload": {**st3, "h2d_GBs": st3["h2d_bytes"] / max(st3["ms_h2d"], 1e-9) / 1e6,
                                "records_per_s": st3["records"] / (st3["ms_wall"] / 1e3)},
              "stage3_regenerate": {**st3g, "records_per_s": st3g["records"] / (st3g["ms_wall"] / 1e3)},
              "stage3_identical": bool(torch.equal(e_r, e_g)), "record_bytes": rb}
        del host, fk, fpsi, e_r, e_g, sh_h
        fpool.close()

    # ---------------- f4: SCI growth with the heat-bath surrogate (SURVEY 8(f) f4; Sec 2.2, :822-833)
    f4 = None
    if not args.no_f4 and world == 1:
        gpool = ctx.pool(sp, 1 << 20)
        s0 = shard[: min(2000, n_par)]
        ctx.merge_space(gpool, ctx.dedup_global(sp, s0))
        g = torch.Generator(device=dev).manual_seed(17)
        gpsi = torch.rand(len(gpool), dtype=torch.float64, device=dev, generator=g) * 2.0 - 1.0
        curve = []
        for it in range(4):
            gpsi, gst = ctx.sci_grow_step(sp, gpool, gpsi, di, args.eps, 4 * len(gpool))
            curve.append({**gst, "redundancy": 1.0 - gst["unique"] / max(gst["records"], 1),
                          "records_per_s": gst["records"] / (gst["ms"] / 1e3)})
        f4 = {"start_space": int(s0.shape[0]), "K": "4 x |S| per iteration", "iterations": curve}
        gpool.close()

    # ---------------- e2e through the public streaming API (f3's stream_generate): the
    # parents come from pinned HOST memory every step (H2D prefetch on the copy stream,
    # gen -> dedup_global -> merge_space per mini-batch), then S <- S u C with the
    # parents copied in again, and the step's counts read back to the host
    e2e = None
    if not args.no_e2e:
        del out, keys_buf, hij_buf, src_buf      # stream_generate keeps its own record slot
        torch.cuda.empty_cache()
        ctx.release_cached()                     # the earlier sections' scratch peaks

        def e2e_step():
            upool.clear()
            spool.clear()
            st = ctx.stream_generate(sp, shard_pinned, di, args.eps, batch, upool, None, batch_records=cap)
            pd = shard_pinned.to(dev, non_blocking=True)
            ctx.merge_space(spool, pd)
            ctx.merge_pool(spool, upool)
            res = torch.tensor([st["records"], len(upool), len(spool)], dtype=torch.int64).to(dev).cpu()  # D2H
            return int(res[0])

        for _ in range(max(1, min(args.warmup, 2))):  # warm the host-input path (allocator, pinned copies)
            e2e_step()
        barrier(pg)
        torch.cuda.synchronize()
        eclocks = ClockSampler(local)
        eclocks.start()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        er = 0
        for _ in range(args.steps):
            er += e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        eclk = eclocks.stop()
        barrier(pg)
        ems = allreduce_max(pg, e0.elapsed_time(e1))
        e2e = {"value": allreduce_sum(pg, er) / (ems / 1e3), "unit": "coupled configs/s",
               "h2d_bytes_per_step": int(2 * shard_pinned.numel() * 8), "d2h_bytes_per_step": 24,
               "ms_per_step": ems / args.steps, "clocks": eclk,
               "path": "stream_generate (pinned host parents, H2D prefetch stream) + merge_space + merge_pool; "
                       "the unique set stays GPU-resident (the pool), counts read back"}

    # ---------------- roofline of the dominant kernel class
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    rec_bytes = 8 * W + 8 + 4

    # algorithmic bytes per step for each kernel class,
    # from the library's own dedup plan (keys x partition passes)
    ds = dstats
    alg = {
        "gen": sum(counts) * rec_bytes + n_par * 8 * W,                  # records written + parents read
        "part_scatter": ds["key_passes"] * 16 * W // args.steps,         # partition: read + write a key per pass
        "part_hist": ds["hist_keys"] * 8 * W // args.steps,              # histogram passes: read a key
        "bucket_unique": (ds["keys_in"] + ds["keys_out"]) * 8 * W // args.steps,  # read every key, write survivors
        "merge": merge_bytes,                                            # read S and U, write S'
    }
    # merge_space runs as merge_split + merge_tile (general / sparse) or a validated
    # copy (sorted_check, empty pool): its bytes are timed against all of them
    mparts = [prof[c] for c in ("merge_split", "merge_tile", "sorted_check") if c in prof]
    timing = dict(prof)
    if mparts:
        timing["merge"] = (sum(x[0] for x in mparts), sum(x[1] for x in mparts))
    kernels = {}
    for name, (kms, kl) in timing.items():
        if name in alg and kl:
            ach = alg[name] * args.steps / (kms / 1e3) / 1e9
            # frac: vs the measured copy bandwidth (a read-only stream can exceed it);
            # frac_nominal: vs the 7.7 TB/s HBM3e spec (B200_PROFILING.md)
            kernels[name] = {"ms_per_step": kms / args.steps, "achieved_GBs": ach, "frac": ach / hbm_peak,
                             "frac_nominal": ach / HBM_NOMINAL_GBS}
    dname = max(prof.items(), key=lambda kv: kv[1][0])[0] if prof else None
    # the headline roofline: the dominant kernel among those with algorithmic bytes in
    # SURVEY 8(d) (gen, bucket_unique = the dedup's N*8W read + U*8W write, merge); the
    # partition passes move bytes no dedup has to move (implementation overhead): they
    # are in kernel_roofline with their own read + write and in dedup_roofline's
    # traffic amplification, not in the headline
    cand = {k: v for k, v in kernels.items() if k in ("gen", "bucket_unique", "merge")}
    rname = max(cand, key=lambda k: cand[k]["ms_per_step"]) if cand else None
    # measured DRAM traffic per launch of each class: the committed ncu launch list
    # of this command for THIS workload (profiles/<round>_<workload>_traffic.json,
    # newest round) -- null if absent
    traffic, traffic_src = {}, None
    try:
        import glob
        tj = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_{args.workload}_traffic.json")))
        if tj:
            d = json.load(open(tj[-1]))
            if d.get("parents") in (None, len(par_all)) and d.get("eps", 0.0) == args.eps:
                traffic = d.get("classes", {})
                traffic_src = os.path.relpath(tj[-1], ROOT)
    except (OSError, ValueError):
        pass
    roof = None
    if rname:
        launches_r = timing[rname][1] / args.steps
        tr = traffic.get(rname, {}).get("dram_bytes_per_launch")
        roof = {"bound": "hbm", "kernel": rname, "achieved": kernels[rname]["achieved_GBs"], "peak": hbm_peak,
                "unit": "GB/s", "frac": kernels[rname]["frac"],
                "frac_nominal": kernels[rname]["frac_nominal"], "peak_nominal": HBM_NOMINAL_GBS,
                "traffic": tr, "traffic_source": traffic_src,
                "alg_bytes_per_launch": alg[rname] / launches_r if launches_r else None,
                "peak_source": peak_src, "dominant_class": dname,
                "note": "partition passes (part_scatter) are implementation overhead (SURVEY 8(d)); see dedup_roofline"}
        for k in kernels:
            kernels[k]["dram_bytes_per_launch_ncu"] = traffic.get(k, {}).get("dram_bytes_per_launch")
            kernels[k]["alg_bytes_per_launch"] = alg[k] / (timing[k][1] / args.steps)
    # the dedup as a whole against what ANY dedup must move: read the N
    # input keys, write the U distinct ones; the partition passes and the pack are
    # implementation overhead, reported as traffic amplification (measured DRAM bytes
    # of every dedup kernel / these algorithmic bytes)
    dedup_roof = None
    dcls = [c for c in ("part_scatter", "part_hist", "bucket_unique", "pack") if c in prof]
    if dcls:
        d_ms = sum(prof[c][0] for c in dcls) / args.steps
        d_alg = (ds["keys_in"] + ds["keys_out"]) * 8 * W / args.steps
        d_dram = None
        if traffic and all(c in traffic for c in dcls):
            d_dram = sum(traffic[c]["dram_bytes_per_launch"] * prof[c][1] / args.steps for c in dcls)
        dedup_roof = {"bound": "hbm", "alg_bytes_per_step": d_alg, "ms_per_step": d_ms,
                      "achieved": d_alg / (d_ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                      "frac": d_alg / (d_ms / 1e3) / 1e9 / hbm_peak, "kernels": dcls,
                      "dram_bytes_per_step_ncu": d_dram,
                      "traffic_amplification": (d_dram / d_alg) if d_dram else None,
                      "keys_per_s": ds["keys_in"] / args.steps / (d_ms / 1e3)}
    if "part_scatter" in kernels:
        kernels["part_scatter"]["bytes"] = "the pass's own read + write of every key (implementation overhead of the dedup, see dedup_roofline)"
    gen_roof = None
    if "gen" in kernels:
        gen_roof = {"achieved": kernels["gen"]["achieved_GBs"], "frac": kernels["gen"]["frac"],
                    "records_per_s_kernel": tot_rec / (prof["gen"][0] / 1e3)}

    # ---------------- cpu baseline (oracle, rank 0, N=1 only)
    cpu = cpu_mt = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_sample = args.cpu_sample or default_cpu_sample(args.workload)
        _, _, par_s = synth.workload_inputs(args.workload, n_parents=n_sample)
        r, u, dt = oracle_sample(wl, ints, par_s, n_sample)
        cpu = {"value": r / dt, "unit": "coupled configs/s", "cores": 1, "kind": "oracle",
               "sample": f"{n_sample} parents (first distinct sampler draws) of the workload through oracle gen -> std::set dedup -> "
                         f"set_union merge ({r} records, {u} unique, {dt:.1f} s)"}
        # oracle-MT: the same oracle sharded over every host core
        nth = max(1, len(os.sched_getaffinity(0)))
        n_mt = n_sample * nth
        _, _, par_m = synth.workload_inputs(args.workload, n_parents=n_mt)
        rm, um, dtm = oracle_sample_mt(wl, ints, par_m, n_mt, nth)
        cpu_mt = {"value": rm / dtm, "unit": "coupled configs/s", "cores": nth, "kind": "oracle-MT",
                  "sample": f"{n_mt} parents sharded over {nth} threads ({rm} records, {um} unique, {dtm:.1f} s)"}

    if stage3:
        stage3["frac"] = stage3["achieved_GBs"] / hbm_peak
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "coupled configs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{wl.name} ({args.workload})", "m": wl.m, "n_alpha": wl.n_alpha,
                       "n_beta": wl.n_beta, "point_group_irreps": wl.g, "parents": int(len(par_all)),
                       "parents_per_batch": batch, "eps": args.eps, "records_per_step": int(recs_all / args.steps),
                       "unique_per_step": int(uni_all / args.steps),
                       "parallelism": f"dp{world} (hash-owner shards, NCCL all-to-all-v)",
                       "l2": "inputs larger than L2 (records per batch >> 126 MB)"},
            "unique_configs_per_s": unique_rate,
            "redundancy": 1.0 - uni_all / max(recs_all, 1),
            "roofline": roof,
            "dedup_roofline": dedup_roof,
            "gen_kernel": gen_roof,
            "kernel_roofline": kernels,
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])},
            "stage3_contract": stage3,
            "f2_regular_sampling": f2,
            "f3_streaming": f3,
            "f4_sci_growth": f4,
            "cpu_baseline": cpu,
            "cpu_baseline_mt": cpu_mt,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
