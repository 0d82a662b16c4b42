"""ctypes loader for libgpurir.so (the C ABI declared in include/gpurir.h).

Argument marshalling only.  There is no fallback: if the CUDA extension is not
built, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GPURIR_LIB", os.path.join(_HERE, "libgpurir.so"))  # override: A/B builds only

OK, EINVAL, EDEGENERATE, EINFEASIBLE, ENOMEM, ECUDA, ECAPACITY = range(7)
FLAG_SYNC = 1
MODES = {"fp32": 0, "lut": 1, "fp16": 2, "lut_tex": 3, "poly": 4}
PATTERNS = {"omni": 0, "subcardioid": 1, "cardioid": 2, "hypercardioid": 3, "bidirectional": 4}

# Every symbol include/gpurir.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "gpurir_opts_default", "gpurir_simulate_rir", "gpurir_simulate_rir_batch", "gpurir_nsamples",
    "gpurir_sabine_t60", "gpurir_beta_sabine", "gpurir_att2t_sabine", "gpurir_t2n", "gpurir_image_params",
    "gpurir_lut_table", "gpurir_device_status", "gpurir_strerror", "gpurir_last_cuda_error", "gpurir_version",
    "gpurir_simulate_trajectory", "gpurir_simulate_rir_dir", "gpurir_beta_sabine_weighted", "gpurir_poly_table",
    "gpurir_simulate_rir_host", "gpurir_workspace_bytes", "gpurir_batch_extent", "gpurir_poly_fir_table",
]


class Opts(C.Structure):
    _fields_ = [("mode", C.c_int), ("Tw", C.c_double), ("lut_Q", C.c_int), ("seed", C.c_uint64),
                ("rir_index_base", C.c_uint64), ("stream", C.c_void_p), ("split", C.c_int), ("flags", C.c_uint),
                ("ev_ism", C.c_void_p * 2), ("ev_tail", C.c_void_p * 2), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("status", C.c_void_p)]


class Room(C.Structure):
    _fields_ = [("room_sz", C.c_float * 3), ("beta", C.c_float * 6), ("pos_src", C.c_float * 3),
                ("pos_rcv", C.c_float * 3), ("orV_rcv", C.c_float * 3), ("mic_pattern", C.c_int),
                ("nb_img", C.c_int * 3), ("Tdiff", C.c_double), ("Tmax", C.c_double), ("out_offset", C.c_longlong),
                ("orV_src", C.c_float * 3), ("spkr_pattern", C.c_int), ("rir_index", C.c_ulonglong)]


class GpurirError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        msg = f"{where}: {strerror(status)} (status {status})"
        if detail:
            msg += f": {detail}"
        super().__init__(msg)
        self.status = status


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built (run `python -c 'import __graft_entry__ as g; g.build()'`); "
                           "there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    fp, ip, dp, vp = C.POINTER(C.c_float), C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_void_p
    L.gpurir_opts_default.restype = None
    L.gpurir_opts_default.argtypes = [C.POINTER(Opts)]
    L.gpurir_simulate_rir.restype = C.c_int
    L.gpurir_simulate_rir.argtypes = [fp, fp, vp, C.c_int, vp, C.c_int, vp, C.c_int, ip, C.c_double, C.c_double,
                                      C.c_double, C.c_double, vp, C.POINTER(Opts)]
    L.gpurir_simulate_rir_dir.restype = C.c_int
    L.gpurir_simulate_rir_dir.argtypes = [fp, fp, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, C.c_int, ip, C.c_double,
                                          C.c_double, C.c_double, C.c_double, vp, C.POINTER(Opts)]
    L.gpurir_simulate_rir_host.restype = C.c_int
    L.gpurir_simulate_rir_host.argtypes = [fp, fp, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, C.c_int, ip, C.c_double,
                                           C.c_double, C.c_double, C.c_double, vp, C.POINTER(Opts)]
    L.gpurir_beta_sabine_weighted.restype = C.c_int
    L.gpurir_beta_sabine_weighted.argtypes = [fp, C.c_double, fp, C.c_int, C.c_int, fp, ip]
    L.gpurir_simulate_rir_batch.restype = C.c_int
    L.gpurir_simulate_rir_batch.argtypes = [C.c_int, C.POINTER(Room), C.c_double, C.c_double, vp, C.POINTER(Opts)]
    L.gpurir_workspace_bytes.restype = C.c_size_t
    L.gpurir_batch_extent.restype = C.c_longlong
    L.gpurir_batch_extent.argtypes = [C.c_int, C.POINTER(Room), C.c_double]
    L.gpurir_workspace_bytes.argtypes = [C.c_int, C.POINTER(Room), C.c_double, C.c_double, C.POINTER(Opts)]
    L.gpurir_simulate_trajectory.restype = C.c_int
    L.gpurir_simulate_trajectory.argtypes = [vp, C.c_longlong, vp, C.c_int, C.c_int, C.c_longlong, vp, C.POINTER(Opts)]
    L.gpurir_nsamples.restype = C.c_longlong
    L.gpurir_nsamples.argtypes = [C.c_double, C.c_double]
    L.gpurir_sabine_t60.restype = C.c_double
    L.gpurir_sabine_t60.argtypes = [fp, fp]
    L.gpurir_beta_sabine.restype = C.c_int
    L.gpurir_beta_sabine.argtypes = [fp, C.c_double, C.c_int, C.c_int, fp, ip]
    L.gpurir_att2t_sabine.restype = C.c_double
    L.gpurir_att2t_sabine.argtypes = [C.c_double, C.c_double]
    L.gpurir_t2n.restype = C.c_int
    L.gpurir_t2n.argtypes = [C.c_double, fp, C.c_double, ip]
    L.gpurir_image_params.restype = C.c_int
    L.gpurir_image_params.argtypes = [fp, fp, fp, fp, fp, C.c_int, fp, C.c_int, ip, C.c_double, C.c_double, vp, vp,
                                      vp]
    L.gpurir_poly_table.restype = C.c_int
    L.gpurir_poly_table.argtypes = [C.c_double, C.c_double, ip, fp, C.c_longlong]
    L.gpurir_poly_fir_table.restype = C.c_int
    L.gpurir_poly_fir_table.argtypes = [C.c_double, C.c_double, ip, ip, ip, fp, C.c_longlong]
    L.gpurir_lut_table.restype = C.c_longlong
    L.gpurir_lut_table.argtypes = [C.c_double, C.c_double, C.c_int, fp, C.c_longlong]
    L.gpurir_device_status.restype = C.c_int
    L.gpurir_device_status.argtypes = [C.c_int]
    L.gpurir_strerror.restype = C.c_char_p
    L.gpurir_strerror.argtypes = [C.c_int]
    L.gpurir_last_cuda_error.restype = C.c_char_p
    L.gpurir_last_cuda_error.argtypes = []
    L.gpurir_version.restype = C.c_char_p
    L.gpurir_version.argtypes = []
    _lib = L
    return L


def strerror(status: int) -> str:
    try:
        return lib().gpurir_strerror(int(status)).decode()
    except RuntimeError:
        return "?"


def check(status: int, where: str) -> None:
    if status != OK:
        detail = lib().gpurir_last_cuda_error().decode() if status == ECUDA else ""
        raise GpurirError(status, where, detail)
