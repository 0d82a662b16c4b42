"""paper_1810_11359_b200 — B200-native (sm_100a) Image Source Method RIR engine.

The hot path of gpuRIR (Diaz-Guerra et al., arXiv 1810.11359) as hand-written
CUDA kernels behind the C ABI in include/gpurir.h (libgpurir.so); this package is
the thin Python binding (same names) plus the multi-GPU shard planner.
There is no CPU fallback: without the built extension every call raises.
"""
from .api import (att2t_sabine, beta_sabine, beta_sabine_weighted, device_status, image_params, lut_table, poly_table, poly_fir_table, make_opts, nsamples,
                  room_array, sabine_t60, simulate_rir, simulate_rir_batch, simulate_rir_host, simulate_trajectory, t2n, version,
                  workspace_bytes)
from ._lib import EXPORTS, LIB_PATH, MODES, PATTERNS, GpurirError

__all__ = ["simulate_rir", "simulate_rir_batch", "simulate_rir_host", "simulate_trajectory", "sabine_t60", "beta_sabine", "beta_sabine_weighted", "att2t_sabine", "t2n", "nsamples",
           "lut_table", "poly_table", "poly_fir_table", "image_params", "device_status", "make_opts", "room_array", "version", "GpurirError",
           "workspace_bytes",
           "MODES", "PATTERNS", "EXPORTS", "LIB_PATH"]
