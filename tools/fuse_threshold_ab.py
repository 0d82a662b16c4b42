"""A/B of the fused-tail threshold (run under gpurun with GPURIR_LIB=build/<variant>.so): device time of one
polyphase cfg3 (i) call per M, L2 flushed, median of 9."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sweep import scene_call, time_call  # noqa: E402
import workloads as W  # noqa: E402

for M in [int(x) for x in os.environ.get("AB_MS", "148,296,444,592,888,1184,2048").split(",")]:
    fn, _ = scene_call(W.cfg3(M, "diffuse"), "poly")
    ms = time_call(fn, reps=9, warm=3)
    print(json.dumps({"lib": os.environ.get("GPURIR_LIB", "default"), "M": M, "ms": round(ms, 4),
                      "rirs_per_s": round(M / ms * 1e3)}), flush=True)
