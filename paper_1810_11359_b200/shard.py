"""Multi-GPU sharding of independent RIRs: host-side planning and gather.

RIRs (receivers of one room, or whole rooms) are independent, so the
path shards with no data-path collective: one process per GPU computes its
shard through the C ABI with `rir_index_base` = the global index of its first
RIR, which keeps every tail RNG stream (reading C16) and therefore every output
sample identical to a 1-GPU run.  Results stay on the devices (dataset
generation) or are gathered to rank 0 (`gather_rows`).  No NCCL call sits on
the hot path; torch.distributed is used for the barrier, the max-over-ranks
timing and the optional gather.
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np


def receiver_shard(M_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [start, stop) of the M_total RIRs owned by `rank` (sizes differ by at most 1)."""
    if not (0 <= rank < world) or M_total < 0:
        raise ValueError("bad shard arguments")
    q, r = divmod(M_total, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


def room_cost(room_sz: Sequence[float], Tdiff: float, Tmax: float, fs: float, c: float = 343.0,
              Tw: float = 4e-3) -> float:
    """Estimated work of one room's RIR: in-window taps of the images inside the Tdiff sphere
    (image density 4 pi c^3 t^2 / V, SURVEY §7 hard part 2) plus the samples written."""
    V = float(np.prod(np.asarray(room_sz, dtype=np.float64)))
    n_img = 4.0 / 3.0 * math.pi * (c * Tdiff) ** 3 / V
    taps = n_img * Tw * fs
    return taps * 13.0 + Tmax * fs * 4.0


def lpt_plan(costs: Sequence[float], world: int) -> list[np.ndarray]:
    """Longest-processing-time-first assignment of jobs to `world` ranks (deterministic: ties by index)."""
    costs = np.asarray(costs, dtype=np.float64)
    order = np.lexsort((np.arange(costs.size), -costs))
    load = np.zeros(world)
    owner = np.empty(costs.size, dtype=np.int64)
    for j in order:
        r = int(np.argmin(load))  # lowest loaded rank, lowest index on ties
        owner[j] = r
        load[r] += costs[j]
    return [np.nonzero(owner == r)[0] for r in range(world)]


def plan_imbalance(costs: Sequence[float], plan: list[np.ndarray]) -> float:
    """max / mean rank load of a plan."""
    costs = np.asarray(costs, dtype=np.float64)
    loads = np.array([costs[p].sum() for p in plan])
    return float(loads.max() / loads.mean()) if loads.mean() > 0 else 1.0


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timings: the job ends when the slowest rank ends)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local, M_total: int, world: int, rank: int):
    """Gather contiguous receiver shards [M_local, nS] to rank 0 as [M_total, nS] (None on other ranks).

    Shards are padded to the largest shard for the collective; works with gloo (CPU) and nccl (CUDA)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or world == 1:
        return local
    sizes = [receiver_shard(M_total, world, r) for r in range(world)]
    mx = max(b - a for a, b in sizes)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad, gather_list=bufs, dst=0)
    if rank != 0:
        return None
    return torch.cat([bufs[r][: sizes[r][1] - sizes[r][0]] for r in range(world)], dim=0)


def batch_shard(rooms: Sequence[dict], costs: Sequence[float], world: int, rank: int):
    """The rooms of `rank` under the LPT plan (config 5 over `world` GPUs): (global indices, rooms with their
    global `rir_index` kept — so each tail RNG stream, reading C16, is the unsharded one — and compact ragged
    `out_offset`s, total samples).  `rooms` are gpurir_room dicts whose `out_offset` is ignored here; the
    samples of room i are `n_samples[i]` = ceil(Tmax_i fs), passed in as the dicts' 'n' key."""
    plan = lpt_plan(costs, world)
    idx = plan[rank]
    mine, off = [], 0
    for i in idx:
        r = dict(rooms[i])
        r["rir_index"] = int(rooms[i].get("rir_index", i))
        r["out_offset"] = off
        off += int(r.pop("n"))
        mine.append(r)
    return idx, mine, off


def gather_ragged(local, idx, n_samples: Sequence[int], world: int, rank: int):
    """Gather every rank's compact batch output (1-D, rooms in `idx` order) to rank 0 as one ragged buffer in
    global room order (None on other ranks).  Host-side (gloo or nccl), outside any timed region."""
    import torch
    import torch.distributed as dist
    n_samples = np.asarray(n_samples, dtype=np.int64)
    starts = np.concatenate([[0], np.cumsum(n_samples)])
    if not dist.is_initialized() or world == 1:
        out = torch.empty(int(starts[-1]), dtype=local.dtype, device=local.device)
        pos = 0
        for i in idx:
            out[starts[i]:starts[i + 1]] = local[pos:pos + n_samples[i]]
            pos += int(n_samples[i])
        return out
    sizes = torch.tensor([local.numel()], dtype=torch.int64, device=local.device)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes)
    mx = int(max(s.item() for s in all_sizes))
    pad = torch.zeros((mx,), dtype=local.dtype, device=local.device)
    pad[: local.numel()] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad, gather_list=bufs, dst=0)
    idxs = [None] * world
    dist.all_gather_object(idxs, [int(i) for i in idx])
    if rank != 0:
        return None
    out = torch.empty(int(starts[-1]), dtype=local.dtype, device=local.device)
    for r in range(world):
        pos = 0
        for i in idxs[r]:
            out[starts[i]:starts[i + 1]] = bufs[r][pos:pos + n_samples[i]]
            pos += int(n_samples[i])
    return out
