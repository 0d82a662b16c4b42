"""Is graph-replay time per call quantised?  Replays a spin kernel of 1..20 us (every CTA spins) from a CUDA graph,
with and without a cluster attribute, and prints us per replay (diagnostic; build: nvcc -shared tools/probe/spin.cu)."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = C.CDLL(os.path.join(ROOT, "build", "spin.so"))
lib.spin_launch.argtypes = [C.c_longlong, C.c_int, C.c_int, C.c_int, C.c_void_p]
MHZ = 1965.0


def per_replay(us, blocks, threads, cluster, n=50):
    s = torch.cuda.Stream()
    cyc = int(us * MHZ)
    with torch.cuda.stream(s):
        assert lib.spin_launch(cyc, blocks, threads, cluster, C.c_void_p(s.cuda_stream)) == 0
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        assert lib.spin_launch(cyc, blocks, threads, cluster, C.c_void_p(s.cuda_stream)) == 0
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000.0 / n


for blocks, threads, cluster in ((1, 32, 0), (128, 1024, 0), (128, 1024, 8)):
    row = []
    for k in range(0, 81):
        us = 0.25 * k
        row.append(f"{us:5.2f}:{per_replay(us, blocks, threads, cluster):6.2f}")
    print(f"blocks={blocks} threads={threads} cluster={cluster}")
    for i in range(0, len(row), 9):
        print("  " + "  ".join(row[i:i + 9]))
    sys.stdout.flush()
