"""CPU double-precision oracle for the ISM RIR path (gpuRIR, arXiv 1810.11359).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package
`paper_1810_11359_b200`.  It shares no code with the CUDA path.

This module is argument marshalling (ctypes + numpy) over oracle/oracle.c; all
arithmetic lives in that C file, each function citing the PAPER.md passage it
follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
SRC_PATH = os.path.join(_HERE, "oracle.c")

STATUS = {0: "OK", 1: "EINVAL", 2: "EDEGENERATE", 3: "EINFEASIBLE"}
PATTERNS = {"omni": 0, "subcardioid": 1, "cardioid": 2, "hypercardioid": 3, "bidirectional": 4}


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, OpenMP)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", LIB_PATH, SRC_PATH, "-lm"]
        subprocess.run(cmd, check=True)
    return LIB_PATH


_native_path = None


def use_native() -> str:
    """Switch this process to an -O3 -march=native build of oracle.c (bench.py's timed oracle arms only; the
    arithmetic is the same source).  Built where it runs, in the temp directory, because -march=native code
    from another host may not execute on this one.  Call before the first oracle function."""
    global _native_path, _lib
    import tempfile
    tag = f"{int(os.path.getmtime(SRC_PATH))}_{os.uname().nodename}"
    path = os.path.join(tempfile.gettempdir(), f"liboracle_native_{tag}.so")
    if not os.path.exists(path):
        tmp = path + f".{os.getpid()}"
        subprocess.run(["gcc", "-O3", "-march=native", "-fopenmp", "-fPIC", "-shared", "-o", tmp, SRC_PATH, "-lm"],
                       check=True)
        os.replace(tmp, path)
    _native_path = path
    _lib = None
    return path


def build_flags() -> str:
    return "-O3 -march=native" if _native_path else "-O2"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class OracleError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: oracle status {status} ({STATUS.get(status, '?')})")
        self.status = status


_lib = None


def lib():
    global _lib
    if _lib is None:
        if _native_path is None:
            build()
        L = C.CDLL(_native_path or LIB_PATH)
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        L.oracle_nsamples.restype = C.c_long
        L.oracle_nsamples.argtypes = [C.c_double, C.c_double]
        L.oracle_image_coord.restype = C.c_double
        L.oracle_image_coord.argtypes = [C.c_int, C.c_double, C.c_double]
        L.oracle_wall_crossings.restype = None
        L.oracle_wall_crossings.argtypes = [C.c_int, ip, ip]
        L.oracle_windowed_sinc.restype = C.c_double
        L.oracle_windowed_sinc.argtypes = [C.c_double, C.c_double, C.c_double]
        L.oracle_sabine_t60.restype = C.c_double
        L.oracle_sabine_t60.argtypes = [dp, dp]
        L.oracle_beta_sabine.restype = C.c_int
        L.oracle_beta_sabine.argtypes = [dp, C.c_double, C.c_int, C.c_int, dp, ip]
        L.oracle_att2t.restype = C.c_double
        L.oracle_att2t.argtypes = [C.c_double, C.c_double]
        L.oracle_t2n.restype = C.c_int
        L.oracle_t2n.argtypes = [C.c_double, dp, C.c_double, ip]
        L.oracle_philox4x32_10.restype = None
        L.oracle_philox4x32_10.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.oracle_uniform.restype = C.c_double
        L.oracle_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.oracle_logistic.restype = C.c_double
        L.oracle_logistic.argtypes = [C.c_double]
        L.oracle_image_set.restype = C.c_long
        L.oracle_image_set.argtypes = [dp, dp, dp, dp, dp, C.c_int, dp, C.c_int, ip, C.c_double, C.c_double, ip,
                                       dp, dp, dp]
        L.oracle_beta_sabine_weighted.restype = C.c_int
        L.oracle_beta_sabine_weighted.argtypes = [dp, C.c_double, dp, C.c_int, C.c_int, dp, ip]
        L.oracle_simulate_rir.restype = C.c_int
        L.oracle_simulate_rir.argtypes = [dp, dp, dp, C.c_int, dp, C.c_int, dp, C.c_int, dp, C.c_int, ip, C.c_double,
                                          C.c_double, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                          C.c_uint64, C.c_int, C.c_int, dp]
        L.oracle_max_threads.restype = C.c_int
        L.oracle_max_threads.argtypes = []
        L.oracle_lut_build.restype = C.c_long
        L.oracle_lut_build.argtypes = [C.c_double, C.c_double, C.c_int, dp, C.c_long]
        L.oracle_lut_lookup.restype = C.c_double
        L.oracle_lut_lookup.argtypes = [dp, C.c_long, C.c_int, C.c_double, C.c_double]
        L.oracle_logistic_stream.restype = None
        L.oracle_logistic_stream.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_long, dp]
        L.oracle_simulate_trajectory.restype = C.c_int
        L.oracle_simulate_trajectory.argtypes = [dp, C.c_long, dp, C.c_int, C.c_int, C.c_long, dp]
        L.oracle_sin_pi_poly.restype = C.c_double
        L.oracle_sin_pi_poly.argtypes = [C.c_double]
        L.oracle_cos_pi_poly.restype = C.c_double
        L.oracle_cos_pi_poly.argtypes = [C.c_double]
        _lib = L
    return _lib


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def nsamples(T: float, fs: float) -> int:
    return int(lib().oracle_nsamples(float(T), float(fs)))


def image_coord(n: int, L: float, s: float) -> float:
    return lib().oracle_image_coord(int(n), float(L), float(s))


def wall_crossings(n: int) -> tuple[int, int]:
    a, b = C.c_int(), C.c_int()
    lib().oracle_wall_crossings(int(n), C.byref(a), C.byref(b))
    return a.value, b.value


def windowed_sinc(t: float, Tw: float = 4e-3, fc: float = 8000.0) -> float:
    return lib().oracle_windowed_sinc(float(t), float(Tw), float(fc))


def sabine_t60(room, beta) -> float:
    r, b = _d(room), _d(beta)
    return lib().oracle_sabine_t60(_dp(r), _dp(b))


def beta_sabine(room, T60: float, sign: int = -1, clamp: bool = False) -> tuple[np.ndarray, bool]:
    r = _d(room)
    out = np.zeros(6)
    cl = C.c_int(0)
    st = lib().oracle_beta_sabine(_dp(r), float(T60), int(sign), int(bool(clamp)), _dp(out), C.byref(cl))
    if st != 0:
        raise OracleError(st, "beta_sabine")
    return out, bool(cl.value)


def beta_sabine_weighted(room, T60: float, weights, sign: int = -1, clamp: bool = False) -> tuple[np.ndarray, bool]:
    """NEXT row f3 (reading R9): alpha_i = w_i alpha0 with Sabine's T60 (Eq. 7) met exactly."""
    r, w = _d(room), _d(weights)
    out = np.zeros(6)
    cl = C.c_int(0)
    st = lib().oracle_beta_sabine_weighted(_dp(r), float(T60), _dp(w), int(sign), int(bool(clamp)), _dp(out),
                                           C.byref(cl))
    if st != 0:
        raise OracleError(st, "beta_sabine_weighted")
    return out, bool(cl.value)


def att2t(att_dB: float, T60: float) -> float:
    return lib().oracle_att2t(float(att_dB), float(T60))


def t2n(T: float, room, c: float = 343.0) -> np.ndarray:
    r = _d(room)
    nb = np.zeros(3, dtype=np.int32)
    st = lib().oracle_t2n(float(T), _dp(r), float(c), _ip(nb))
    if st != 0:
        raise OracleError(st, "t2n")
    return nb


def philox4x32_10(ctr, key) -> np.ndarray:
    c = (C.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (C.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (C.c_uint32 * 4)()
    lib().oracle_philox4x32_10(c, k, o)
    return np.array(list(o), dtype=np.uint32)


def uniform(seed: int, r: int, k: int) -> float:
    return lib().oracle_uniform(int(seed), int(r), int(k))


def logistic(u: float) -> float:
    return lib().oracle_logistic(float(u))


def logistic_stream(seed: int, r: int, k0: int, n: int) -> np.ndarray:
    out = np.zeros(int(n))
    lib().oracle_logistic_stream(int(seed), int(r), int(k0), int(n), _dp(out))
    return out


def image_set(room, beta, src, rcv, nb, fs=16000.0, c=343.0, pattern=0, orv=None, spkr_pattern=0, ors=None):
    """All lattice images of one (src, rcv): dict with n [N,3], x (delay in samples), A, beta."""
    nb = np.ascontiguousarray(np.asarray(nb, dtype=np.int32))
    N = int(np.prod(nb.astype(np.int64)))
    n_out = np.zeros((N, 3), dtype=np.int32)
    x_out = np.zeros(N)
    A_out = np.zeros(N)
    b_out = np.zeros(N)
    r, b, s, q = _d(room), _d(beta), _d(src), _d(rcv)
    o = _d(orv if orv is not None else [0.0, 0.0, 1.0])
    os_ = _d(ors if ors is not None else [0.0, 0.0, 1.0])
    cnt = lib().oracle_image_set(_dp(r), _dp(b), _dp(s), _dp(q), _dp(o), int(pattern), _dp(os_), int(spkr_pattern),
                                 _ip(nb), float(fs), float(c), _ip(n_out), _dp(x_out), _dp(A_out), _dp(b_out))
    if cnt < 0:
        raise OracleError(-cnt, "image_set")
    return {"n": n_out, "x": x_out, "A": A_out, "beta": b_out}


def simulate_rir(room, beta, pos_src, pos_rcv, nb_img, Tdiff, Tmax, fs=16000.0, c=343.0, pattern=0,
                 orV_rcv=None, Tw=4e-3, seed=0, rir_index_base=0, dense=False, nthreads=0, spkr_pattern=0,
                 orV_src=None) -> np.ndarray:
    """Oracle RIRs [M_src][M_rcv][nSamples] in float64 (P:274 layout)."""
    src = _d(pos_src).reshape(-1, 3)
    rcv = _d(pos_rcv).reshape(-1, 3)
    Ms, Mr = src.shape[0], rcv.shape[0]
    nS = nsamples(Tmax, fs)
    out = np.zeros((Ms, Mr, nS))
    orv = None if orV_rcv is None else _d(orV_rcv).reshape(-1, 3)
    ors = None if orV_src is None else _d(orV_src).reshape(-1, 3)
    nb = np.ascontiguousarray(np.asarray(nb_img, dtype=np.int32))
    r, b = _d(room), _d(beta)
    st = lib().oracle_simulate_rir(_dp(r), _dp(b), _dp(src), Ms, _dp(rcv), Mr,
                                   _dp(orv) if orv is not None else None, int(pattern),
                                   _dp(ors) if ors is not None else None, int(spkr_pattern), _ip(nb), float(Tdiff),
                                   float(Tmax), float(fs), float(c), float(Tw), int(seed), int(rir_index_base),
                                   int(bool(dense)), int(nthreads), _dp(out))
    if st != 0:
        raise OracleError(st, "simulate_rir")
    return out


def simulate_trajectory(signal, rirs) -> np.ndarray:
    """NEXT row f1: moving source through per-point RIR banks rirs [n_points][n_mics][L]."""
    sig = _d(signal).reshape(-1)
    R = _d(rirs)
    if R.ndim != 3:
        raise ValueError("rirs must be [n_points][n_mics][L]")
    P_, M, L = R.shape
    out = np.zeros((M, sig.size + L - 1))
    st = lib().oracle_simulate_trajectory(_dp(sig), sig.size, _dp(R), P_, M, L, _dp(out))
    if st != 0:
        raise OracleError(st, "simulate_trajectory")
    return out


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def lut_build(Tw: float = 4e-3, fs: float = 16000.0, Q: int = 16) -> tuple[np.ndarray, int]:
    half = lib().oracle_lut_build(float(Tw), float(fs), int(Q), None, 0)
    out = np.zeros(2 * half + 1)
    lib().oracle_lut_build(float(Tw), float(fs), int(Q), _dp(out), out.size)
    return out, int(half)


def lut_lookup(lut: np.ndarray, half: int, Q: int, fs: float, t: float) -> float:
    lut = _d(lut)
    return lib().oracle_lut_lookup(_dp(lut), int(half), int(Q), float(fs), float(t))


def sin_pi_poly(x: float) -> float:
    return lib().oracle_sin_pi_poly(float(x))


def cos_pi_poly(x: float) -> float:
    return lib().oracle_cos_pi_poly(float(x))
