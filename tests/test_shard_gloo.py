"""N>1 host path on CPU (gloo, world_size 2): shard planning, global RNG indexing, max-over-ranks timing
and the gather reproduce the unsharded result bit for bit.  The per-rank compute is the oracle (CPU
stand-in for the CUDA kernel, which has the same global-index contract; the GPU side of the contract is
tests/test_gpu_parity.py::test_shard_invariance)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1810_11359_b200.shard import gather_rows, lpt_plan, max_over_ranks, plan_imbalance, receiver_shard


def test_receiver_shard_partition():
    for M in (0, 1, 7, 16, 16384, 100003):
        for world in (1, 2, 3, 8):
            got = [receiver_shard(M, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == M
            for (a, b), (c, d) in zip(got, got[1:]):
                assert b == c
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1


def test_lpt_plan_balanced_and_complete():
    import workloads as W
    from paper_1810_11359_b200.shard import room_cost
    rb = W.cfg5(2000)
    costs = [room_cost(rb.room[i], rb.Tdiff[i], rb.Tmax[i], rb.fs) for i in range(rb.n)]
    plan = lpt_plan(costs, 8)
    allidx = np.sort(np.concatenate(plan))
    assert np.array_equal(allidx, np.arange(rb.n))
    assert plan_imbalance(costs, plan) < 1.01
    assert all(np.array_equal(a, b) for a, b in zip(plan, lpt_plan(costs, 8)))  # deterministic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle
    import workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = W.cfg3(6, "diffuse")
    sc.Tdiff, sc.Tmax = 0.02, 0.05
    beta, _ = oracle.beta_sabine(sc.room, sc.T60)
    nb = oracle.t2n(sc.Tdiff, sc.room)
    a, b = receiver_shard(6, world, rank)
    h = oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv[a:b], nb, sc.Tdiff, sc.Tmax, pattern=sc.pattern,
                            orV_rcv=sc.orV_rcv[a:b], seed=sc.seed, rir_index_base=a)[0]
    full = gather_rows(torch.from_numpy(h), 6, world, rank)
    t = max_over_ranks(1.0 + rank)
    if rank == 0:
        ref = oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv, nb, sc.Tdiff, sc.Tmax, pattern=sc.pattern,
                                  orV_rcv=sc.orV_rcv, seed=sc.seed)[0]
        q.put((bool(np.array_equal(full.numpy(), ref)), t))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shard_gather_bitwise():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    same, t = q.get(timeout=10)
    assert same
    assert t == 2.0


def _batch_worker(rank, world, port, q):
    """config 5 host path: batch_shard + gather_ragged over gloo, with synthetic per-room rows standing in for
    the batch call's output (each room's row encodes its global index and sample, so any misplacement shows)."""
    import torch.distributed as dist

    import workloads as W
    from paper_1810_11359_b200.shard import batch_shard, gather_ragged, room_cost
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rb = W.cfg5(300)
    ns = [int(np.ceil(rb.Tmax[i] * rb.fs - 1e-6)) for i in range(rb.n)]
    rooms = [dict(rir_index=i, n=ns[i], Tmax=rb.Tmax[i]) for i in range(rb.n)]
    costs = [room_cost(rb.room[i], rb.Tdiff[i], rb.Tmax[i], rb.fs) for i in range(rb.n)]
    idx, mine, tot = batch_shard(rooms, costs, world, rank)
    local = torch.empty((tot,), dtype=torch.float64)
    for r in mine:  # the "RIR" of room i: 1e6 i + k at sample k
        n = int(np.ceil(r["Tmax"] * rb.fs - 1e-6))
        local[r["out_offset"]:r["out_offset"] + n] = torch.arange(n, dtype=torch.float64) + 1e6 * r["rir_index"]
    full = gather_ragged(local, idx, ns, world, rank)
    if rank == 0:
        ref = np.concatenate([np.arange(ns[i], dtype=np.float64) + 1e6 * i for i in range(rb.n)])
        q.put(bool(np.array_equal(full.numpy(), ref)) and sorted(int(i) for i in idx) != list(range(rb.n)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_batch_shard_gather():
    """LPT shards of rooms (non-contiguous global indices) gathered back to rank 0 in
    global room order, world_size 2 over gloo."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert q.get(timeout=10)
