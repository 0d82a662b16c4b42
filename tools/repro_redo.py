"""Reproducer: the polyphase count-guard redo (split = -3) on config 3 (i) with 64 receivers (GPU box)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_1810_11359_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from helpers import derive, run_gpu  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 64
split = int(sys.argv[2]) if len(sys.argv) > 2 else -3
sc = W.cfg3(M, "diffuse")
beta, nb = derive(oracle, sc)
g = run_gpu(P, sc, beta, nb, mode="poly", split=split)
print("ok", M, split, float(np.abs(g).max()), flush=True)
