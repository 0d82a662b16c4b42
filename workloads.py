"""Seeded synthetic input generators for the five BASELINE.json configs.

Shared by tests/, bench.py and __graft_entry__.smoke(): it draws geometry and
positions only and holds NONE of the method's arithmetic (no Sabine inversion,
no image lattice sizing, no RIR maths).  Each consumer derives beta / nb_img
with its own side's helpers (the oracle's in tests and the cpu_baseline, the
CUDA library's in the product path).

Recipes follow SURVEY.md §8(d) "Concrete synthetic input" (restated in
DESIGN.md §"Input recipe"):

  cfg1  3x4x2.5 m, T60 0.3, src (1.2,1.5,1.1), rcv (2.1,2.9,1.4), omni, ISM to 0.3 s, 16 kHz
  cfg2  6x4x3 m, T60 in {0.1..2.0}, src (2.0,1.5,1.2), rcv (4.1,2.9,1.6), ISM to T60/4, tail to T60
  cfg3  3x4x2.5 m, T60 0.7, src (1.5,1.0,1.2), M rcv uniform in [0.3, L-0.3]^3 (seed 3),
        orientations uniform on S^2 (seed 3), cardioid; (i) Tdiff 0.175 / Tmax 0.7, (ii) ISM to 0.7
  cfg4  3x4x2.5 m, T60 1.0, src (1.0,1.0,1.5), 32-mic UCA r=0.10 m at (2.0,2.5,1.3), omni, 48 kHz;
        (a) Tdiff 0.25 / Tmax 1.0, (b) ISM to 0.5 s
  cfg5  n rooms (seed 5): L ~ U(3,10) x U(3,8) x U(2.5,4.5), T60 ~ U(0.2,1.5), src/rcv uniform with
        0.5 m wall margin, omni, 16 kHz, Tdiff = T60/4, Tmax = T60
  traj1 (NEXT row f1) cfg3's room and T60, a source moving on a straight line (0.5,1.0,1.2) ->
        (2.5,3.0,1.2) sampled at 100 trajectory points, 32-mic UCA r=0.10 m at (1.5,2.5,1.3), omni,
        16 kHz, Tdiff 0.175 / Tmax 0.7 (L = 11200), 1 s of unit-variance white noise (seed 11)

Positions, room sizes and orientations are float32 (the C ABI's type); the
oracle receives the same float32 values widened to double.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

C_SOUND = 343.0  # reading C5
PATTERN = {"omni": 0, "subcardioid": 1, "cardioid": 2, "hypercardioid": 3, "bidirectional": 4}
SEED_BASE = 0x5EED0000


@dataclass
class Scene:
    """One gpurir_simulate_rir call's raw inputs (beta and nb_img are derived by the consumer)."""
    name: str
    room: np.ndarray            # float32 [3]
    T60: float                  # target reverberation time (beta derived via Sabine inversion, sign -1)
    pos_src: np.ndarray         # float32 [M_src, 3]
    pos_rcv: np.ndarray         # float32 [M_rcv, 3]
    orV_rcv: np.ndarray | None  # float32 [M_rcv, 3] or None
    pattern: int
    Tdiff: float
    Tmax: float
    fs: float
    c: float = C_SOUND
    seed: int = 0
    nb_time: float | None = None  # time nb_img must reach (default Tdiff); C6
    clamp: bool = False           # clamp infeasible T60 to beta = 0 (C18)
    meta: dict = field(default_factory=dict)

    @property
    def M(self) -> int:
        return int(self.pos_src.shape[0] * self.pos_rcv.shape[0])


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def cfg1() -> Scene:
    return Scene("cfg1", _f32([3, 4, 2.5]), 0.3, _f32([[1.2, 1.5, 1.1]]), _f32([[2.1, 2.9, 1.4]]), None,
                 PATTERN["omni"], 0.3, 0.3, 16000.0, seed=SEED_BASE + 1)


CFG2_T60 = [round(0.1 * i, 1) for i in range(1, 21)]


def cfg2(T60: float) -> Scene:
    return Scene(f"cfg2_T60_{T60:.1f}", _f32([6, 4, 3]), float(T60), _f32([[2.0, 1.5, 1.2]]),
                 _f32([[4.1, 2.9, 1.6]]), None, PATTERN["omni"], T60 / 4.0, float(T60), 16000.0,
                 seed=SEED_BASE + 2, clamp=True)


def _receivers_cfg3(M: int, room: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(3)
    lo = 0.3
    pos = lo + rng.random((M, 3)) * (room.astype(np.float64) - 2 * lo)
    v = rng.standard_normal((M, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return _f32(pos), _f32(v)


def cfg3(M: int, variant: str = "diffuse") -> Scene:
    room = _f32([3, 4, 2.5])
    rcv, orv = _receivers_cfg3(M, room)
    if variant == "diffuse":
        Tdiff, Tmax = 0.175, 0.7
    elif variant == "full":
        Tdiff, Tmax = 0.7, 0.7
    else:
        raise ValueError(variant)
    return Scene(f"cfg3_{variant}_M{M}", room, 0.7, _f32([[1.5, 1.0, 1.2]]), rcv, orv, PATTERN["cardioid"],
                 Tdiff, Tmax, 16000.0, seed=SEED_BASE + 3)


def cfg4(variant: str = "a", n_mics: int = 32) -> Scene:
    ang = 2.0 * np.pi * np.arange(n_mics) / n_mics
    rcv = np.stack([2.0 + 0.10 * np.cos(ang), 2.5 + 0.10 * np.sin(ang), np.full(n_mics, 1.3)], axis=1)
    if variant == "a":
        Tdiff, Tmax = 0.25, 1.0
    elif variant == "b":
        Tdiff, Tmax = 0.5, 0.5
    else:
        raise ValueError(variant)
    return Scene(f"cfg4{variant}", _f32([3, 4, 2.5]), 1.0, _f32([[1.0, 1.0, 1.5]]), _f32(rcv), None,
                 PATTERN["omni"], Tdiff, Tmax, 48000.0, seed=SEED_BASE + 4)


def traj1(n_points: int = 100, n_mics: int = 32, n_sig: int = 16000) -> Scene:
    t = np.linspace(0.0, 1.0, n_points)
    src = np.stack([0.5 + 2.0 * t, 1.0 + 2.0 * t, np.full(n_points, 1.2)], axis=1)
    ang = 2.0 * np.pi * np.arange(n_mics) / n_mics
    rcv = np.stack([1.5 + 0.10 * np.cos(ang), 2.5 + 0.10 * np.sin(ang), np.full(n_mics, 1.3)], axis=1)
    return Scene(f"traj1_P{n_points}_M{n_mics}", _f32([3, 4, 2.5]), 0.7, _f32(src), _f32(rcv), None,
                 PATTERN["omni"], 0.175, 0.7, 16000.0, seed=SEED_BASE + 11, meta={"n_sig": n_sig})


def traj_signal(n_sig: int, seed: int = SEED_BASE + 11) -> np.ndarray:
    """The source signal of a trajectory workload: unit-variance white noise, float32."""
    return _f32(np.random.default_rng(seed).standard_normal(n_sig))


@dataclass
class RoomBatch:
    """cfg5: independent rooms, one src / one omni rcv each."""
    room: np.ndarray     # float32 [n, 3]
    T60: np.ndarray      # float64 [n]
    pos_src: np.ndarray  # float32 [n, 3]
    pos_rcv: np.ndarray  # float32 [n, 3]
    Tdiff: np.ndarray    # float64 [n]
    Tmax: np.ndarray     # float64 [n]
    fs: float = 16000.0
    c: float = C_SOUND
    seed: int = SEED_BASE + 5

    @property
    def n(self) -> int:
        return int(self.room.shape[0])


def cfg5(n_rooms: int = 100_000) -> RoomBatch:
    rng = np.random.default_rng(5)
    L = np.stack([rng.uniform(3, 10, n_rooms), rng.uniform(3, 8, n_rooms), rng.uniform(2.5, 4.5, n_rooms)], axis=1)
    L = L.astype(np.float32)
    T60 = rng.uniform(0.2, 1.5, n_rooms)
    m = 0.5
    src = m + rng.random((n_rooms, 3)) * (L.astype(np.float64) - 2 * m)
    rcv = m + rng.random((n_rooms, 3)) * (L.astype(np.float64) - 2 * m)
    return RoomBatch(_f32(L), T60, _f32(src), _f32(rcv), T60 / 4.0, T60.copy())


def random_small_scene(rng: np.random.Generator, fs: float = 16000.0, max_src: int = 2, max_rcv: int = 3,
                       T: float | None = None) -> Scene:
    """Small random scene (SPEC S:525 style): rooms 2-8 m, T60 0.3-1.0 s, ISM only to a short time."""
    room = _f32(rng.uniform(2.0, 8.0, 3))
    T60 = float(rng.uniform(0.3, 1.0))
    Ms, Mr = int(rng.integers(1, max_src + 1)), int(rng.integers(1, max_rcv + 1))
    r64 = room.astype(np.float64)
    src = _f32(0.2 + rng.random((Ms, 3)) * (r64 - 0.4))
    rcv = _f32(0.2 + rng.random((Mr, 3)) * (r64 - 0.4))
    pat = int(rng.integers(0, 5))
    orv = None
    if pat != 0:
        v = rng.standard_normal((Mr, 3))
        orv = _f32(v / np.linalg.norm(v, axis=1, keepdims=True))
    Tm = float(T if T is not None else rng.uniform(0.02, 0.06))
    return Scene("random", room, T60, src, rcv, orv, pat, Tm, Tm, fs, seed=int(rng.integers(0, 2**31)))
