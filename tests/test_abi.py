"""The C-ABI library loads and exports every symbol include/gpurir.h declares; host helpers agree with
the oracle's (-m "not gpu": no device compute is called)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    from paper_1810_11359_b200 import build as B
    B.build()
    import paper_1810_11359_b200 as P
    return P


def _declared():
    src = open(os.path.join(ROOT, "include", "gpurir.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gpurir_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(P):
    names = _declared()
    assert len(names) >= 14
    lib = ctypes.CDLL(P.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(P.EXPORTS) == names


def test_version(P):
    assert "sm_100a" in P.version()


def test_lib_is_sm100a_fatbin(P):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_helpers_match_oracle(P, oracle):
    rng = np.random.default_rng(4)
    for _ in range(200):
        room = rng.uniform(2, 10, 3).astype(np.float32)
        T60 = float(rng.uniform(0.2, 2.0))
        try:
            bo, clo = oracle.beta_sabine(room, T60)
        except oracle.OracleError as e:
            with pytest.raises(P.GpurirError) as ei:
                P.beta_sabine(room, T60)
            assert ei.value.status == e.status == 3
            continue
        bg, clg = P.beta_sabine(room, T60)
        assert clg == clo and np.allclose(bg, bo, rtol=1e-6)
        beta = rng.uniform(-1, 1, 6).astype(np.float32)
        assert P.sabine_t60(room, beta) == pytest.approx(oracle.sabine_t60(room, beta), rel=1e-12)
        T = float(rng.uniform(0.01, 2.0))
        assert list(P.t2n(T, room)) == list(oracle.t2n(T, room))
        assert P.att2t_sabine(15.0, T60) == pytest.approx(oracle.att2t(15.0, T60), rel=1e-15)
        assert P.nsamples(T, 16000.0) == oracle.nsamples(T, 16000.0)


def test_lut_table_matches_eq9_oracle(P, oracle):
    for fs in (16000.0, 44100.0, 48000.0):
        g, hg = P.lut_table(4e-3, fs, 16)
        r, hr = oracle.lut_build(4e-3, fs, 16)
        assert hg == hr
        assert np.max(np.abs(g - r)) < 1e-7


def test_invalid_arguments_rejected_on_host(P):
    # host validation happens before any device work: EINVAL without touching CUDA
    assert P._lib.lib().gpurir_simulate_rir(None, None, None, 0, None, 0, None, 0, None, 0.1, 0.1, 16000.0, 343.0,
                                            None, None) == 1


def test_weighted_beta_matches_oracle(P, oracle):
    """f3 helper (reading R9): library and oracle agree, including infeasible and clamped cases."""
    rng = np.random.default_rng(11)
    for _ in range(200):
        room = rng.uniform(2, 10, 3).astype(np.float32)
        w = rng.uniform(0.0, 1.0, 6).astype(np.float32)
        T60 = float(rng.uniform(0.2, 2.0))
        try:
            bo, _ = oracle.beta_sabine_weighted(room, T60, w)
        except oracle.OracleError as e:
            with pytest.raises(P.GpurirError) as ei:
                P.beta_sabine_weighted(room, T60, w)
            assert ei.value.status == e.status == 3
            bg, cl = P.beta_sabine_weighted(room, T60, w, clamp=True)
            assert cl and np.all(bg == 0)
            continue
        bg, cl = P.beta_sabine_weighted(room, T60, w)
        assert not cl and np.allclose(bg, bo, rtol=1e-6, atol=1e-7)
    with pytest.raises(P.GpurirError):
        P.beta_sabine_weighted([3, 4, 2.5], 0.5, [0.0] * 6)


def _dir_call(P, spkr, ors, mode=0, Q=16, buf=None, Tdiff=0.01, Tmax=0.01, fs=16000.0):
    """gpurir_simulate_rir_dir with dummy (never dereferenced on a rejected call) device pointers."""
    L = P._lib.lib()
    f3 = (ctypes.c_float * 3)(3.0, 4.0, 2.5)
    b6 = (ctypes.c_float * 6)(*([0.5] * 6))
    nb = (ctypes.c_int * 3)(3, 3, 3)
    o = P._lib.Opts()
    L.gpurir_opts_default(ctypes.byref(o))
    o.mode, o.lut_Q = mode, Q
    dummy = ctypes.c_void_p(16)
    return L.gpurir_simulate_rir_dir(f3, b6, dummy, 1, ors, spkr, dummy, 1, None, 0, nb, Tdiff, Tmax, fs,
                                     343.0, dummy, ctypes.byref(o))


def test_directional_source_validated_on_host(P):
    """f3: a directional source needs orientations; patterns outside 0..4 are rejected (EINVAL = 1)."""
    assert _dir_call(P, 2, None) == 1
    assert _dir_call(P, 5, ctypes.c_void_p(16)) == 1
    assert _dir_call(P, -1, None) == 1


def test_mode_validation_on_host(P):
    """LUT needs a power-of-two Q (R4); the texture LUT (f2) does not; unknown modes are EINVAL.  A call
    that passes host validation goes on to the device, which this container lacks (ECUDA = 5)."""
    import torch
    assert _dir_call(P, 0, None, mode=1, Q=10) == 1
    assert _dir_call(P, 0, None, mode=5) == 1
    if not torch.cuda.is_available():
        assert _dir_call(P, 0, None, mode=3, Q=10) == 5
        assert _dir_call(P, 0, None, mode=1, Q=16) == 5


def test_host_call_validated_on_host(P):
    """gpurir_simulate_rir_host rejects bad arguments before touching the device (EINVAL = 1)."""
    L = P._lib.lib()
    f3 = (ctypes.c_float * 3)(3.0, 4.0, 2.5)
    b6 = (ctypes.c_float * 6)(*([0.5] * 6))
    nb = (ctypes.c_int * 3)(3, 3, 3)
    buf = (ctypes.c_float * 64)()
    o = P._lib.Opts()
    L.gpurir_opts_default(ctypes.byref(o))
    args = lambda **k: dict(dict(src=buf, ms=1, ors=None, sp=0, rcv=buf, mr=1, orv=None, mp=0, Tmax=0.01, out=buf), **k)
    def call(a):
        return L.gpurir_simulate_rir_host(f3, b6, ctypes.cast(a["src"], ctypes.c_void_p) if a["src"] else None, a["ms"],
                                          a["ors"], a["sp"], ctypes.cast(a["rcv"], ctypes.c_void_p), a["mr"], a["orv"],
                                          a["mp"], nb, 0.005, a["Tmax"], 16000.0, 343.0,
                                          ctypes.cast(a["out"], ctypes.c_void_p) if a["out"] else None, ctypes.byref(o))
    assert call(args(src=None)) == 1
    assert call(args(out=None)) == 1
    assert call(args(ms=0)) == 1
    assert call(args(mp=2)) == 1            # cardioid receivers need orientations
    assert call(args(sp=6)) == 1            # no such pattern
    assert call(args(Tmax=-1.0)) == 1


def test_ism_length_cap(P):
    """The kernels floor delays in fp32 with the 1.5 2^23 magic, exact below 2^22 samples: an ISM part
    longer than 2^22 - 8192 samples (87 s at 48 kHz) is EINVAL on the host, for every mode; the diffuse
    tail has no such limit."""
    import torch
    for mode in (0, 4):
        assert _dir_call(P, 0, None, mode=mode, Tdiff=90.0, Tmax=90.0, fs=48000.0) == 1
        if not torch.cuda.is_available():  # passes host validation, then needs the device
            assert _dir_call(P, 0, None, mode=mode, Tdiff=80.0, Tmax=200.0, fs=48000.0) == 5


@pytest.mark.parametrize("fs", [8000.0, 16000.0, 22050.0, 44100.0, 48000.0, 96000.0])
def test_poly_table_reproduces_eq6(P, oracle, fs):
    """Reading R11: the host's Chebyshev expansion (exactly the table GPURIR_POLY uploads) reproduces the
    oracle's Eq. 6 windowed sinc at every integer tap and fractional delay to < 1e-6 of its peak; taps past
    the open support are zero."""
    Tw = 4e-3
    tab, mlo = P.poly_table(Tw, fs)
    rng = np.random.default_rng(int(fs))
    phi = np.concatenate([rng.random(200), [0.0, 1e-7, 0.5, 1 - 6e-8]])
    T = np.cos(np.arange(8)[:, None] * np.arccos(2 * phi - 1)[None, :])  # T_d(2 phi - 1)
    approx = tab.astype(np.float64) @ T                                     # [tap, phi]
    worst = 0.0
    for mi in range(tab.shape[0]):
        m = mlo + mi
        exact = np.array([oracle.windowed_sinc((m - f) / fs, Tw, fs / 2) for f in phi])
        worst = max(worst, float(np.max(np.abs(approx[mi] - exact))))
    assert worst < 1e-6, worst
    H = Tw * fs / 2
    assert mlo == int(np.floor(-H)) + 1 and tab.shape[0] % 8 == 0
    with pytest.raises(P.GpurirError):
        P.poly_table(Tw, 300000.0)  # Tw fs > 1022 taps


@pytest.mark.parametrize("fs", [3000.0, 8000.0, 16000.0, 22050.0, 44100.0, 48000.0, 96000.0])
def test_poly_fir_table_reproduces_eq6(P, oracle, fs):
    """Reading R13: the rotated, low-rank FIR form the kernel runs (channels G' = Q G; rotated channels 4..7 only
    on their window: 8 taps m = -3 .. 4 for tables of <= 64 taps, else 16-24 aligned taps) reproduces the oracle's Eq. 6 windowed sinc at every integer tap and fractional delay
    to < 1e-6 of its peak, as the unrotated table does; Q is orthogonal and block diagonal over the parities."""
    Tw = 4e-3
    F = P.poly_fir_table(Tw, fs)
    far, near, Qc, mlo, nmi0, nn = F["far"], F["near"], F["Q"], F["mlo"], F["nmi0"], F["nn"]
    n = far.shape[1]
    Q = np.zeros((8, 8))
    for par in range(2):
        for k in range(4):
            for i in range(4):
                Q[2 * k + par, 2 * i + par] = Qc[par, k, i]
    assert np.abs(Q @ Q.T - np.eye(8)).max() < 1e-6
    assert 0 <= nmi0 and nmi0 + nn <= n
    if n <= 64:  # the window m = -3 .. 4 (clamped to the table)
        assert nn == 8 and (nmi0 == min(-3 - mlo, n - 8) or nmi0 == 0)
    else:        # longer tables: an aligned 16- or 24-tap window covering m = -6 .. 7
        assert nn in (16, 24) and nmi0 % 8 == 0 and nmi0 <= -6 - mlo and nmi0 + nn >= 8 - mlo
    Pr = np.zeros((n, 8))  # rotated coefficients per tap
    Pr[:, 0:4] = far.transpose(1, 0, 2).reshape(n, 4)
    Pr[nmi0:nmi0 + nn, 4:8] = near.transpose(1, 0, 2).reshape(nn, 4)
    rng = np.random.default_rng(int(fs) + 1)
    phi = np.concatenate([rng.random(200), [0.0, 1e-7, 0.5, 1 - 6e-8]])
    T = np.cos(np.arange(8)[:, None] * np.arccos(2 * phi - 1)[None, :])  # T_d(2 phi - 1)
    approx = Pr @ (Q @ T)                                                  # [tap, phi]
    worst = 0.0
    for mi in range(n):
        m = mlo + mi
        exact = np.array([oracle.windowed_sinc((m - f) / fs, Tw, fs / 2) for f in phi])
        worst = max(worst, float(np.max(np.abs(approx[mi] - exact))))
    assert worst < 1e-6, worst
    tab, mlo0 = P.poly_table(Tw, fs)  # the same expansion: unrotated channels = Q^T rotated
    assert mlo0 == mlo and tab.shape[0] == n


@pytest.mark.parametrize("Tw,fs", [(2e-3, 16000.0), (2e-3, 48000.0), (8e-3, 16000.0), (8e-3, 48000.0), (16e-3, 16000.0)])
def test_poly_fir_table_other_windows(P, oracle, Tw, fs):
    """Reading R13 at other window lengths T_w (2-16 ms: 32-384 taps): the rotated low-rank FIR equals the
    unrotated expansion to < 1e-7 and the oracle's Eq. 6 to < 1e-6 of its peak at every tap."""
    F = P.poly_fir_table(Tw, fs)
    far, near, Qc, mlo, nmi0, nn = F["far"], F["near"], F["Q"], F["mlo"], F["nmi0"], F["nn"]
    n = far.shape[1]
    Q = np.zeros((8, 8))
    for par in range(2):
        for k in range(4):
            for i in range(4):
                Q[2 * k + par, 2 * i + par] = Qc[par, k, i]
    Pr = np.zeros((n, 8))
    Pr[:, 0:4] = far.transpose(1, 0, 2).reshape(n, 4)
    Pr[nmi0:nmi0 + nn, 4:8] = near.transpose(1, 0, 2).reshape(nn, 4)
    phi = np.linspace(0.0, 1.0, 61)[:-1]
    T = np.cos(np.arange(8)[:, None] * np.arccos(2 * phi - 1)[None, :])
    approx = Pr @ (Q @ T)
    tab, _ = P.poly_table(Tw, fs)
    assert np.abs(approx - tab.astype(np.float64) @ T).max() < 1e-7
    worst = max(float(np.max(np.abs(approx[mi] - [oracle.windowed_sinc((mlo + mi - f) / fs, Tw, fs / 2) for f in phi])))
                for mi in range(n))
    assert worst < 1e-6, worst


def test_batch_extent_on_host(P):
    """gpurir_batch_extent (the binding's output-size check of a batch call): max(out_offset + ceil(Tmax fs)),
    reading C9 / R1, computed on the host without a device; -1 for invalid arguments."""
    rooms = [dict(room_sz=[3, 4, 2.5], beta=[-0.9] * 6, pos_src=[1, 1, 1], pos_rcv=[2, 2, 1], nb_img=[5, 5, 5],
                  Tdiff=0.05, Tmax=T, out_offset=off) for T, off in ((0.3, 0), (0.1, 4800), (0.2, 6400), (0.05, 100))]
    arr = P.room_array(rooms)
    want = max(r["out_offset"] + P.nsamples(r["Tmax"], 16000.0) for r in rooms)
    assert want == 9600
    assert P._lib.lib().gpurir_batch_extent(len(arr), arr, 16000.0) == want
    assert P._lib.lib().gpurir_batch_extent(0, arr, 16000.0) == 0
    assert P._lib.lib().gpurir_batch_extent(1, arr, 0.0) == -1
