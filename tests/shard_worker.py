"""One rank of the config-5 multi-GPU path for tests/test_gpu_parity.py::test_cfg5_two_ranks_...:
LPT-shard a batch of rooms over WORLD_SIZE ranks, one gpurir_simulate_rir_batch call per rank on this rank's
GPU (cuda:LOCAL_RANK modulo the devices present — the test runs both ranks on cuda:0), then gather the ragged
outputs to rank 0 over gloo, which saves them.  Launched with torch.distributed.run (127.0.0.1)."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rooms_of(P, W, n):
    rb = W.cfg5(n)
    rooms, costs, ns = [], [], []
    from paper_1810_11359_b200 import shard
    for i in range(rb.n):
        beta, _ = P.beta_sabine(rb.room[i], rb.T60[i])
        nb = P.t2n(rb.Tdiff[i], rb.room[i])
        n_i = P.nsamples(rb.Tmax[i], rb.fs)
        rooms.append(dict(room_sz=rb.room[i], beta=beta, pos_src=rb.pos_src[i], pos_rcv=rb.pos_rcv[i], nb_img=nb,
                          Tdiff=rb.Tdiff[i], Tmax=rb.Tmax[i], rir_index=i, n=n_i))
        costs.append(shard.room_cost(rb.room[i], rb.Tdiff[i], rb.Tmax[i], rb.fs))
        ns.append(n_i)
    return rb, rooms, costs, ns


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rooms", type=int, default=600)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    import paper_1810_11359_b200 as P
    import workloads as W
    from paper_1810_11359_b200 import shard
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    rb, rooms, costs, ns = rooms_of(P, W, args.rooms)
    idx, mine, tot = shard.batch_shard(rooms, costs, world, rank)
    out = torch.empty((tot,), dtype=torch.float32, device="cuda")
    P.simulate_rir_batch(mine, rb.fs, out, seed=rb.seed, mode="poly", sync=True)
    full = shard.gather_ragged(out.cpu(), idx, ns, world, rank)
    if rank == 0:
        np.save(args.out, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
