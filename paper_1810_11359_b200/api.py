"""Thin Python binding of libgpurir (include/gpurir.h), same names as the C ABI.

Argument marshalling only: torch supplies device memory and streams; every step
of the RIR path runs in the library's CUDA kernels.  Citations as in the header.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import FLAG_SYNC, MODES, PATTERNS, GpurirError, Opts, Room, check, lib


def _f3(v, n=3):
    a = (C.c_float * n)(*[float(x) for x in np.asarray(v, dtype=np.float64).reshape(-1)[:n]])
    if len(np.asarray(v).reshape(-1)) != n:
        raise ValueError(f"expected {n} values")
    return a


def _i3(v):
    vv = [int(x) for x in np.asarray(v).reshape(-1)]
    if len(vv) != 3:
        raise ValueError("expected 3 values")
    return (C.c_int * 3)(*vv)


def _pattern(p) -> int:
    return PATTERNS[p] if isinstance(p, str) else int(p)


def _mode(m) -> int:
    return MODES[m] if isinstance(m, str) else int(m)


def _stream_handle(stream) -> int | None:
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def make_opts(mode="fp32", Tw=4e-3, lut_Q=16, seed=0, rir_index_base=0, stream=None, split=0, sync=False,
              ev_ism=None, ev_tail=None, workspace=None, status=None) -> Opts:
    o = Opts()
    lib().gpurir_opts_default(C.byref(o))
    o.mode = _mode(mode)
    o.Tw = float(Tw)
    o.lut_Q = int(lut_Q)
    o.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    o.rir_index_base = int(rir_index_base)
    o.stream = _stream_handle(stream)
    o.split = int(split)
    o.flags = FLAG_SYNC if sync else 0
    if ev_ism is not None:  # torch.cuda.Event pair recorded around the ISM kernel
        o.ev_ism[0], o.ev_ism[1] = ev_ism[0].cuda_event, ev_ism[1].cuda_event
    if ev_tail is not None:
        o.ev_tail[0], o.ev_tail[1] = ev_tail[0].cuda_event, ev_tail[1].cuda_event
    if workspace is not None:  # caller-owned device scratch (uint8 CUDA tensor) of the batch call
        o.workspace = workspace.data_ptr()
        o.workspace_bytes = workspace.numel() * workspace.element_size()
    if status is not None:  # caller-owned device int32 status word of this call
        o.status = status.data_ptr()
    return o


def _on_device(t):
    """The calling thread's current device is the library's device (gpurir.h conventions): switch to t's."""
    import torch
    return torch.cuda.device(t.device)


def nsamples(T: float, fs: float) -> int:
    """ceil(T fs) under reading C9."""
    return int(lib().gpurir_nsamples(float(T), float(fs)))


def _dev_f32(t, name, rows=None):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch tensor")
    if t.dtype != torch.float32 or not t.is_contiguous():
        raise TypeError(f"{name} must be contiguous float32")
    if rows is not None and (t.dim() != 2 or t.shape[1] != 3):
        raise ValueError(f"{name} must have shape [M, 3]")
    return t


def simulate_rir(room_sz, beta, pos_src, pos_rcv, nb_img, Tdiff, Tmax, fs, c=343.0, orV_rcv=None,
                 mic_pattern="omni", mode="fp32", Tw=4e-3, lut_Q=16, seed=0, rir_index_base=0, out=None,
                 stream=None, split=0, sync=False, ev_ism=None, ev_tail=None, orV_src=None, spkr_pattern="omni"):
    """gpurir_simulate_rir: RIRs [M_src][M_rcv][ceil(Tmax fs)] (float32, on pos_src's device).

    room_sz (3) and beta (6, wall order x0,x1,y0,y1,z0,z1) are host values; pos_src [M_src,3],
    pos_rcv [M_rcv,3] and orV_rcv [M_rcv,3] are CUDA float32 tensors.  Stream-ordered; returns `out`.
    A directional source (orV_src [M_src,3], spkr_pattern; NEXT row f3) goes through gpurir_simulate_rir_dir.
    """
    import torch
    pos_src = _dev_f32(pos_src, "pos_src", rows=True)
    pos_rcv = _dev_f32(pos_rcv, "pos_rcv", rows=True)
    pat = _pattern(mic_pattern)
    spat = _pattern(spkr_pattern)
    if orV_rcv is not None:
        orV_rcv = _dev_f32(orV_rcv, "orV_rcv", rows=True)
    if orV_src is not None:
        orV_src = _dev_f32(orV_src, "orV_src", rows=True)
    Ms, Mr = pos_src.shape[0], pos_rcv.shape[0]
    nS = nsamples(Tmax, fs)
    if out is None:
        out = torch.empty((Ms, Mr, nS), dtype=torch.float32, device=pos_src.device)
    elif out.dtype != torch.float32 or not out.is_contiguous() or out.numel() < Ms * Mr * nS:
        raise ValueError("out must be contiguous float32 with M_src*M_rcv*nSamples elements")
    for t, nm in ((pos_rcv, "pos_rcv"), (orV_rcv, "orV_rcv"), (orV_src, "orV_src"), (out, "out")):
        if t is not None and t.device != pos_src.device:
            raise ValueError(f"{nm} must be on {pos_src.device}")
    with _on_device(pos_src):
        return _simulate_rir(room_sz, beta, pos_src, pos_rcv, nb_img, Tdiff, Tmax, fs, c, orV_rcv, pat, mode, Tw,
                             lut_Q, seed, rir_index_base, out, stream, split, sync, ev_ism, ev_tail, orV_src, spat,
                             Ms, Mr)


def _simulate_rir(room_sz, beta, pos_src, pos_rcv, nb_img, Tdiff, Tmax, fs, c, orV_rcv, pat, mode, Tw, lut_Q, seed,
                  rir_index_base, out, stream, split, sync, ev_ism, ev_tail, orV_src, spat, Ms, Mr):
    o = make_opts(mode, Tw, lut_Q, seed, rir_index_base, stream, split, sync, ev_ism, ev_tail)
    ov = orV_rcv.data_ptr() if orV_rcv is not None else None
    if spat == 0 and orV_src is None:
        st = lib().gpurir_simulate_rir(_f3(room_sz), _f3(beta, 6), pos_src.data_ptr(), Ms, pos_rcv.data_ptr(), Mr,
                                       ov, pat, _i3(nb_img), float(Tdiff), float(Tmax), float(fs), float(c),
                                       out.data_ptr(), C.byref(o))
        check(st, "gpurir_simulate_rir")
    else:
        st = lib().gpurir_simulate_rir_dir(_f3(room_sz), _f3(beta, 6), pos_src.data_ptr(), Ms,
                                           orV_src.data_ptr() if orV_src is not None else None, spat,
                                           pos_rcv.data_ptr(), Mr, ov, pat, _i3(nb_img), float(Tdiff), float(Tmax),
                                           float(fs), float(c), out.data_ptr(), C.byref(o))
        check(st, "gpurir_simulate_rir_dir")
    return out


def _host_f32(x, name, rows=False):
    """A host float32 C-contiguous buffer (numpy array or CPU torch tensor, pinned or not) and its pointer."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous():
                raise ValueError(f"{name} must be a contiguous float32 CPU tensor")
            if rows and (x.dim() != 2 or x.shape[1] != 3):
                raise ValueError(f"{name} must have shape [M, 3]")
            return x, x.data_ptr()
    except ImportError:
        pass
    a = np.ascontiguousarray(x, dtype=np.float32)
    if rows and (a.ndim != 2 or a.shape[1] != 3):
        raise ValueError(f"{name} must have shape [M, 3]")
    return a, a.ctypes.data


def simulate_rir_host(room_sz, beta, pos_src, pos_rcv, nb_img, Tdiff, Tmax, fs, c=343.0, orV_rcv=None,
                      mic_pattern="omni", mode="fp32", Tw=4e-3, lut_Q=16, seed=0, rir_index_base=0, out=None,
                      stream=None, split=0, orV_src=None, spkr_pattern="omni"):
    """gpurir_simulate_rir_host: simulate_rir from host memory, host<->device copies inside the call.

    pos_src / pos_rcv / orV_* are host [M,3] float32 arrays (numpy or CPU tensors; pinned tensors let the
    copies overlap the kernels); `out` (optional) a host float32 buffer of M_src*M_rcv*nSamples elements —
    a numpy array is allocated if omitted.  Synchronous: returns `out` filled, shape [M_src, M_rcv, nS].
    """
    src, p_src = _host_f32(pos_src, "pos_src", rows=True)
    rcv, p_rcv = _host_f32(pos_rcv, "pos_rcv", rows=True)
    orv, p_orv = _host_f32(orV_rcv, "orV_rcv", rows=True) if orV_rcv is not None else (None, None)
    ors, p_ors = _host_f32(orV_src, "orV_src", rows=True) if orV_src is not None else (None, None)
    Ms, Mr = src.shape[0], rcv.shape[0]
    nS = nsamples(Tmax, fs)
    if out is None:
        out = np.empty((Ms, Mr, nS), dtype=np.float32)
    hold, p_out = _host_f32(out, "out")
    if (hold.numel() if hasattr(hold, "numel") else hold.size) < Ms * Mr * nS:
        raise ValueError("out must hold M_src*M_rcv*nSamples float32 elements")
    if hold is not out:
        raise ValueError("out must be a contiguous float32 host buffer")
    o = make_opts(mode, Tw, lut_Q, seed, rir_index_base, stream, split, False)
    st = lib().gpurir_simulate_rir_host(_f3(room_sz), _f3(beta, 6), p_src, Ms, p_ors, _pattern(spkr_pattern), p_rcv,
                                        Mr, p_orv, _pattern(mic_pattern), _i3(nb_img), float(Tdiff), float(Tmax),
                                        float(fs), float(c), p_out, C.byref(o))
    check(st, "gpurir_simulate_rir_host")
    return out


def room_array(rooms) -> C.Array:
    """Build a gpurir_room[n] array from a sequence of dicts with the struct's field names."""
    arr = (Room * len(rooms))()
    for i, r in enumerate(rooms):
        R = arr[i]
        R.room_sz[:] = [float(x) for x in r["room_sz"]]
        R.beta[:] = [float(x) for x in r["beta"]]
        R.pos_src[:] = [float(x) for x in r["pos_src"]]
        R.pos_rcv[:] = [float(x) for x in r["pos_rcv"]]
        R.orV_rcv[:] = [float(x) for x in r.get("orV_rcv", (0.0, 0.0, 1.0))]
        R.mic_pattern = _pattern(r.get("mic_pattern", 0))
        R.orV_src[:] = [float(x) for x in r.get("orV_src", (0.0, 0.0, 1.0))]
        R.spkr_pattern = _pattern(r.get("spkr_pattern", 0))
        R.nb_img[:] = [int(x) for x in r["nb_img"]]
        R.Tdiff = float(r["Tdiff"])
        R.Tmax = float(r["Tmax"])
        R.out_offset = int(r["out_offset"])
        R.rir_index = int(r.get("rir_index", i))  # tail RNG stream: rir_index_base + rir_index (reading C16)
    return arr


def _batch_need(arr, fs) -> int:
    """Elements of `out` the rooms write: max(out_offset + ceil(Tmax fs)) (gpurir_batch_extent, one C call)."""
    n = int(lib().gpurir_batch_extent(len(arr), arr, float(fs)))
    if n < 0:
        raise ValueError("invalid rooms / fs")
    return n


def workspace_bytes(rooms, fs, c=343.0, mode="fp32", Tw=4e-3, lut_Q=16, split=0) -> int:
    """gpurir_workspace_bytes: device scratch the batch call needs for these rooms (opts.workspace)."""
    arr = rooms if isinstance(rooms, C.Array) else room_array(rooms)
    o = make_opts(mode, Tw, lut_Q, split=split, stream=0)
    return int(lib().gpurir_workspace_bytes(len(arr), arr, float(fs), float(c), C.byref(o)))


def simulate_rir_batch(rooms, fs, out, c=343.0, mode="fp32", Tw=4e-3, lut_Q=16, seed=0, rir_index_base=0,
                       stream=None, split=0, sync=False, workspace=None, status=None, ev_ism=None, ev_tail=None):
    """gpurir_simulate_rir_batch: one RIR per independent room into ragged rows of `out` (CUDA float32).

    `rooms` is a ctypes gpurir_room array (see room_array) or a sequence of dicts; room i's tail stream is
    rir_index_base + its rir_index (default i).  Stream-ordered (no host synchronisation unless sync).
    """
    import torch
    arr = rooms if isinstance(rooms, C.Array) else room_array(rooms)
    if not (isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == torch.float32 and out.is_contiguous()):
        raise TypeError("out must be a contiguous CUDA float32 tensor")
    if out.numel() < _batch_need(arr, fs):
        raise ValueError(f"out holds {out.numel()} elements; the rooms write up to {_batch_need(arr, fs)}")
    with _on_device(out):
        o = make_opts(mode, Tw, lut_Q, seed, rir_index_base, stream, split, sync, ev_ism, ev_tail, workspace, status)
        st = lib().gpurir_simulate_rir_batch(len(arr), arr, float(fs), float(c), out.data_ptr(), C.byref(o))
    check(st, "gpurir_simulate_rir_batch")
    return out


def simulate_trajectory(signal, rirs, out=None, stream=None, sync=False, split=0):
    """gpurir_simulate_trajectory: filter a mono `signal` [n_sig] (CUDA float32) through the per-point RIR
    banks `rirs` [n_points][n_mics][L] of a source trajectory; returns [n_mics][n_sig + L - 1].
    split: 0 automatic (tensor-core kernel when L % 4 == 0), -1 the CUDA-core kernel, > 0 the tensor-core
    kernel with that K split (test hooks)."""
    import torch
    signal = signal.reshape(-1)
    if not (isinstance(signal, torch.Tensor) and signal.is_cuda and signal.dtype == torch.float32):
        raise TypeError("signal must be a CUDA float32 tensor")
    if not (isinstance(rirs, torch.Tensor) and rirs.is_cuda and rirs.dtype == torch.float32 and rirs.dim() == 3):
        raise TypeError("rirs must be a CUDA float32 tensor [n_points, n_mics, L]")
    signal = signal.contiguous()
    rirs = rirs.contiguous()
    n_points, n_mics, L = rirs.shape
    n_out = signal.numel() + L - 1
    if out is None:
        out = torch.empty((n_mics, n_out), dtype=torch.float32, device=signal.device)
    elif not (out.is_cuda and out.dtype == torch.float32 and out.is_contiguous() and tuple(out.shape) == (n_mics, n_out)):
        raise TypeError(f"out must be a contiguous CUDA float32 tensor of shape {(n_mics, n_out)}")
    if rirs.device != signal.device or out.device != signal.device:
        raise ValueError("signal, rirs and out must be on one device")
    with _on_device(signal):
        o = make_opts(stream=stream, sync=sync, split=split)
        st = lib().gpurir_simulate_trajectory(signal.data_ptr(), signal.numel(), rirs.data_ptr(), n_points, n_mics,
                                              L, out.data_ptr(), C.byref(o))
    check(st, "gpurir_simulate_trajectory")
    return out


# ---- host helpers ------------------------------------------------------------------

def sabine_t60(room_sz, beta) -> float:
    """Eq. 7."""
    return float(lib().gpurir_sabine_t60(_f3(room_sz), _f3(beta, 6)))


def beta_sabine(room_sz, T60: float, sign: int = -1, clamp: bool = False) -> tuple[np.ndarray, bool]:
    """A17 / reading C17: uniform-absorption beta for a target T60 (negative by default)."""
    out = (C.c_float * 6)()
    cl = C.c_int(0)
    st = lib().gpurir_beta_sabine(_f3(room_sz), float(T60), int(sign), int(bool(clamp)), out, C.byref(cl))
    check(st, "gpurir_beta_sabine")
    return np.array(list(out), dtype=np.float32), bool(cl.value)


def beta_sabine_weighted(room_sz, T60: float, weights, sign: int = -1, clamp: bool = False) -> tuple[np.ndarray, bool]:
    """Non-uniform absorption (NEXT row f3, reading R9): alpha_i = w_i alpha0, Sabine's T60 met exactly."""
    out = (C.c_float * 6)()
    cl = C.c_int(0)
    st = lib().gpurir_beta_sabine_weighted(_f3(room_sz), float(T60), _f3(weights, 6), int(sign), int(bool(clamp)),
                                           out, C.byref(cl))
    check(st, "gpurir_beta_sabine_weighted")
    return np.array(list(out), dtype=np.float32), bool(cl.value)


def att2t_sabine(att_dB: float, T60: float) -> float:
    return float(lib().gpurir_att2t_sabine(float(att_dB), float(T60)))


def t2n(T: float, room_sz, c: float = 343.0) -> np.ndarray:
    out = (C.c_int * 3)()
    st = lib().gpurir_t2n(float(T), _f3(room_sz), float(c), out)
    check(st, "gpurir_t2n")
    return np.array(list(out), dtype=np.int32)


def lut_table(Tw: float = 4e-3, fs: float = 16000.0, Q: int = 16) -> tuple[np.ndarray, int]:
    half = int(lib().gpurir_lut_table(float(Tw), float(fs), int(Q), None, 0))
    if half < 0:
        raise GpurirError(-half, "gpurir_lut_table")
    buf = (C.c_float * (2 * half + 1))()
    lib().gpurir_lut_table(float(Tw), float(fs), int(Q), buf, 2 * half + 1)
    return np.array(list(buf), dtype=np.float32), half


def poly_table(Tw: float = 4e-3, fs: float = 16000.0) -> tuple[np.ndarray, int]:
    """gpurir_poly_table: the polyphase coefficients P [ntaps, 8] of GPURIR_POLY and the first tap m_lo (R11)."""
    mlo = C.c_int(0)
    n = int(lib().gpurir_poly_table(float(Tw), float(fs), C.byref(mlo), None, 0))
    if n < 0:
        raise GpurirError(-n, "gpurir_poly_table")
    buf = (C.c_float * (8 * n))()
    lib().gpurir_poly_table(float(Tw), float(fs), C.byref(mlo), buf, 8 * n)
    return np.array(list(buf), dtype=np.float32).reshape(n, 8), int(mlo.value)


def poly_fir_table(Tw: float = 4e-3, fs: float = 16000.0) -> dict:
    """gpurir_poly_fir_table: the rotated low-rank FIR form of GPURIR_POLY (reading R13) — far [2, ntaps, 2],
    near [2, nn, 2], Q [2, 4, 4], m_lo, nmi0, nn."""
    mlo, nmi0, nn = C.c_int(0), C.c_int(0), C.c_int(0)
    n = int(lib().gpurir_poly_fir_table(float(Tw), float(fs), C.byref(mlo), C.byref(nmi0), C.byref(nn), None, 0))
    if n < 0:
        raise GpurirError(-n, "gpurir_poly_fir_table")
    k = nn.value
    cap = 4 * n + 4 * k + 32
    buf = (C.c_float * cap)()
    lib().gpurir_poly_fir_table(float(Tw), float(fs), C.byref(mlo), C.byref(nmi0), C.byref(nn), buf, cap)
    a = np.array(list(buf), dtype=np.float32)
    return {"far": a[:4 * n].reshape(2, n, 2), "near": a[4 * n:4 * n + 4 * k].reshape(2, k, 2),
            "Q": a[4 * n + 4 * k:].reshape(2, 4, 4), "mlo": int(mlo.value), "nmi0": int(nmi0.value), "nn": k}


def image_params(room_sz, beta, src, rcv, nb_img, fs, c=343.0, mic_pattern="omni", orv=None, device=None,
                 spkr_pattern="omni", ors=None):
    """gpurir_image_params: (delay in samples float64 [N], amplitude float32 [N]) in lattice order."""
    import torch
    N = int(np.prod(np.asarray(nb_img, dtype=np.int64)))
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    x = torch.empty(N, dtype=torch.float64, device=dev)
    A = torch.empty(N, dtype=torch.float32, device=dev)
    o = _f3(orv) if orv is not None else None
    os_ = _f3(ors) if ors is not None else None
    st = lib().gpurir_image_params(_f3(room_sz), _f3(beta, 6), _f3(src), _f3(rcv), o, _pattern(mic_pattern), os_,
                                   _pattern(spkr_pattern), _i3(nb_img), float(fs), float(c), x.data_ptr(), A.data_ptr(),
                                   _stream_handle(None))
    check(st, "gpurir_image_params")
    return x, A


def device_status(reset: bool = True) -> int:
    return int(lib().gpurir_device_status(int(bool(reset))))


def version() -> str:
    return lib().gpurir_version().decode()
