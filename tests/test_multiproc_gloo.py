"""World-size-2 gloo tests of the multi-rank host logic (CPU, no GPU):
the NCCL unique-id broadcast, max/sum-over-ranks timing reductions used by
bench.py, and the owner-sharded protocol (each rank partitions its local
keys by owner, the bins are exchanged with all_to_all, each owner dedups what
it received) checked against the oracle's per-owner shards."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import oracle
        import synth
        # 1) unique-id broadcast (payload from rank 0 reaches every rank)
        payload = bytes(range(128)) if rank == 0 else None
        got = bench.bcast_bytes(dist, payload, rank)
        assert got == bytes(range(128))
        # 2) timing reductions
        assert bench.allreduce_max(dist, float(rank + 1)) == float(world)
        assert bench.allreduce_sum(dist, 1.5) == 1.5 * world
        # 2b) collective batch plan: unequal shards still give equal call counts
        n_par = 500_300 if rank == 0 else 499_700
        plan = bench.plan_batches(dist, n_par, 500_000)
        assert len(plan) == 2 and plan[0][0] == 0 and plan[-1][1] == n_par
        assert all(b > a for a, b in plan) and all(plan[i][1] == plan[i + 1][0] for i in range(len(plan) - 1))
        # 3) owner-sharded dedup protocol (logical; oracle arithmetic)
        for W in (1, 2):
            allk = synth.zipf_keys(60_000, W, 1.1, 1 << 12, seed=21)
            mine = np.array_split(allk, world)[rank]
            own = oracle.owner(mine, W, world)
            sends = [torch.from_numpy(np.ascontiguousarray(mine[own == r]).view(np.int64).reshape(-1))
                     for r in range(world)]
            counts = torch.tensor([len(x) for x in sends], dtype=torch.int64)
            rcounts = torch.empty(world, dtype=torch.int64)
            dist.all_to_all_single(rcounts, counts)
            recv = torch.empty(int(rcounts.sum()), dtype=torch.int64)
            dist.all_to_all_single(recv, torch.cat(sends), [int(c) for c in rcounts], [int(c) for c in counts])
            shard = oracle.dedup(recv.numpy().view(np.uint64).reshape(-1, W), W)
            ref = oracle.dedup(allk, W, world, rank)
            assert np.array_equal(shard, ref), (rank, W)
            tot = bench.allreduce_sum(dist, float(len(shard)))
            assert tot == len(oracle.dedup(allk, W))
        # 4) the paper's regular-sampling protocol (oracle arithmetic)
        from oracle import sampling as S
        for W in (1, 2):
            allk = synth.zipf_keys(40_000, W, 1.1, 1 << 12, seed=23)
            local = [S.to_ints(x, W) for x in np.array_split(allk, world)]
            D = S.sort_unique(local[rank])
            gathered = [None] * world
            dist.all_gather_object(gathered, S.regular_samples(D, 64))
            spl = S.select_splitters([x for g in gathered for x in g], world)
            b = S.split_bounds(D, spl)
            outgoing = [D[b[r]:b[r + 1]] for r in range(world)]
            # all-to-all-v of the runs (object transport)
            got = [None] * world
            dist.all_gather_object(got, outgoing)
            shard = sorted(set(x for i in range(world) for x in got[i][rank]))
            ref_shards, ref_spl = S.dedup_sorted(local, 64)
            assert spl == ref_spl and shard == ref_shards[rank], (rank, W)
        q.put((rank, "ok"))
    except Exception as e:  # surface failures to the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_gloo_world2_protocol():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: "ok", 1: "ok"}, res
