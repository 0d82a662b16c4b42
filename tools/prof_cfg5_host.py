"""Host-side cost of one config-5 batch call (100 000 rooms): the Python size check, the C planner alone
(gpurir_workspace_bytes) and the whole call's host time against its device time.  Run on a GPU box."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_11359_b200 as P  # noqa: E402
from paper_1810_11359_b200 import api, shard, _lib  # noqa: E402
import workloads as W  # noqa: E402

rb = W.cfg5(100_000)
rooms, costs = [], []
for i in range(rb.n):
    beta, _ = P.beta_sabine(rb.room[i], rb.T60[i])
    nb = P.t2n(rb.Tdiff[i], rb.room[i])
    rooms.append(dict(room_sz=rb.room[i], beta=beta, pos_src=rb.pos_src[i], pos_rcv=rb.pos_rcv[i], nb_img=nb,
                      Tdiff=rb.Tdiff[i], Tmax=rb.Tmax[i], rir_index=i, n=P.nsamples(rb.Tmax[i], rb.fs)))
    costs.append(shard.room_cost(rb.room[i], rb.Tdiff[i], rb.Tmax[i], rb.fs))
idx, mine, tot = shard.batch_shard(rooms, costs, 1, 0)
arr = P.room_array(mine)
out = torch.empty((tot,), dtype=torch.float32, device="cuda")
lib = _lib.lib()
o = api.make_opts("poly")
for r in range(3):
    t = time.perf_counter(); n = api._batch_need(arr, rb.fs); a = time.perf_counter() - t
    t = time.perf_counter(); b = lib.gpurir_workspace_bytes(len(arr), arr, C.c_double(rb.fs), C.c_double(343.0), C.byref(o))
    w = time.perf_counter() - t
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter(); e0.record(); P.simulate_rir_batch(arr, rb.fs, out, seed=rb.seed, mode="poly"); e1.record()
    h = time.perf_counter() - t
    torch.cuda.synchronize()
    print(f"_batch_need {a*1e3:6.1f} ms  planner (workspace_bytes) {w*1e3:6.1f} ms  whole call host {h*1e3:6.1f} ms"
          f"  events around the call {e0.elapsed_time(e1):6.1f} ms  ({b / 1e6:.1f} MB workspace)", flush=True)

# the bench's loop: flush, event, call, event, no synchronisation between steps
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
stream = torch.cuda.current_stream()
for variant in ("bench loop", "no flush"):
    torch.cuda.synchronize()
    K = 8
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    hs = []
    t0 = time.perf_counter()
    for i in range(K):
        if variant == "bench loop":
            flush.zero_()
        ev[i][0].record(stream)
        t = time.perf_counter()
        P.simulate_rir_batch(arr, rb.fs, out, seed=rb.seed, mode="poly", stream=stream)
        hs.append((time.perf_counter() - t) * 1e3)
        ev[i][1].record(stream)
    t_enq = time.perf_counter() - t0
    torch.cuda.synchronize()
    t_all = time.perf_counter() - t0
    st = [a.elapsed_time(b) for a, b in ev]
    print(f"{variant}: host per call {' '.join(f'{x:.1f}' for x in hs)} ms; enqueue {t_enq*1e3:.0f} ms, wall {t_all*1e3:.0f} ms;"
          f" event step ms {' '.join(f'{x:.1f}' for x in st)}", flush=True)
