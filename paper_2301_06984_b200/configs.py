"""Seeded synthetic inputs for the five BASELINE.json configs.

Every draw is ``rng_word(seed, uid, j)`` (random.hpp:13-28, restated in numpy
uint64 arithmetic), so the arrays are a pure function of (config, n, seed)
and identical bits feed the GPU engine and both CPU oracles. Transcendental
draws (lognormal diameters) happen only here, on the host.

No public benchmark dataset is involved: the paper's models live in a
companion artifact that is not present; these generators stand in for them
with the shapes, sizes and distributions BASELINE.json names.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

# mean of 12 neighbours within R = 12
DENSITY = 12.0 / (4.0 / 3.0 * math.pi * 12.0 ** 3)

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)
_C1 = np.uint64(0x632BE59BD9B4E019)


def rng_word(seed, stream, counter) -> np.ndarray:
    """Vectorised random.hpp:13-28 (uint64 wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        s = np.asarray(stream, dtype=np.uint64)
        c = np.asarray(counter, dtype=np.uint64)
        x = np.uint64(seed) + _M1 * (s + _C1)
        x = x + _M2 * (c + np.uint64(1))
        for _ in range(2):
            x = x ^ (x >> np.uint64(30))
            x = x * _M2
            x = x ^ (x >> np.uint64(27))
            x = x * _M3
            x = x ^ (x >> np.uint64(31))
    return x


def u01(w: np.ndarray) -> np.ndarray:
    """random.hpp:38-40 next_double."""
    return (w >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


@dataclass
class Workload:
    name: str
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    d: np.ndarray
    mask: np.ndarray | None
    params: dict = field(default_factory=dict)  # SimulationParams fields
    steps: int = 1
    bytes_per_agent_iteration: int = 128
    tags: np.ndarray | None = None          # Agent::tag (reference models)
    rng_counters: np.ndarray | None = None  # Agent::rng_counter after population build

    @property
    def n(self) -> int:
        return len(self.x)


def c1_relaxation(n: int = 131_072, seed: int = 0) -> Workload:
    """configs[0]: uniform cube at 12 mean neighbours, d ~ U[8, 12], dt 0.01."""
    L = (n / DENSITY) ** (1.0 / 3.0)
    uid = np.arange(n, dtype=np.uint64)
    x, y, z = (u01(rng_word(seed, uid, j)) * L for j in range(3))
    d = 8.0 + 4.0 * u01(rng_word(seed, uid, 3))
    return Workload("c1_mechanical_relaxation", x, y, z, d, None,
                    dict(seed=seed, simulation_time_step=0.01), steps=100)


def c2_proliferation(side: int = 16, seed: int = 0, rate: float = 34.0) -> Workload:
    """configs[1]: side^3 lattice (spacing 20, d 10); volume grows by `rate`
    per step, division above the volume of d = 14 (absim_models.h)."""
    g = np.arange(side, dtype=np.float64) * 20.0
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    n = side ** 3
    d = np.full(n, 10.0)
    vdiv = math.pi / 6.0 * (14.0 * 14.0 * 14.0)
    return Workload("c2_proliferation", X.ravel().copy(), Y.ravel().copy(), Z.ravel().copy(), d,
                    None, dict(seed=seed, simulation_time_step=0.01,
                               model=N.MODEL_PROLIFERATION, model_params=[rate, vdiv]),
                    steps=200, bytes_per_agent_iteration=144)


def c3_spheroid(n: int = 1 << 23, seed: int = 0, speed: float = 1.0) -> Workload:
    """configs[2]: n sites of an FCC lattice (nearest-neighbour spacing
    10 + sqrt(3), contact-free under +-0.5 jitter) closest to the centre;
    the outer 10% (by radius rank) are driven outward each step."""
    a = 10.0 + math.sqrt(3.0)          # nearest-neighbour distance
    cube = a * math.sqrt(2.0)          # FCC cubic cell edge
    r_est = (n * cube ** 3 / 4.0 / (4.0 / 3.0 * math.pi)) ** (1.0 / 3.0)
    m = int(math.ceil(r_est / cube)) + 2
    ax = np.arange(-m, m + 1, dtype=np.float64) * cube
    X, Y, Z = np.meshgrid(ax, ax, ax, indexing="ij")
    base = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
    h = cube / 2.0
    pts = np.concatenate([base, base + [h, h, 0], base + [h, 0, h], base + [0, h, h]])
    r2 = (pts * pts).sum(1)
    order = np.argsort(r2, kind="stable")[:n]
    pts = pts[order]
    uid = np.arange(n, dtype=np.uint64)
    jit = [(u01(rng_word(seed, uid, 10 + j)) - 0.5) for j in range(3)]
    x, y, z = pts[:, 0] + jit[0], pts[:, 1] + jit[1], pts[:, 2] + jit[2]
    mask = np.zeros(n, np.uint8)
    mask[int(0.9 * n):] = 1
    return Workload("c3_static_spheroid", x, y, z, np.full(n, 10.0), mask,
                    dict(seed=seed, simulation_time_step=0.01, detect_static_agents=True,
                         model=N.MODEL_DRIVE, model_params=[0.0, 0.0, 0.0, speed]),
                    steps=100, bytes_per_agent_iteration=134)


def c4_large_uniform(n: int = 1 << 26, seed: int = 0) -> Workload:
    """configs[3]: uniform cube at 12 mean neighbours, d ~ lognormal(ln 10, 0.1)
    (Box-Muller on the host), Morton re-sort every 10 steps, 50 steps."""
    L = (n / DENSITY) ** (1.0 / 3.0)
    uid = np.arange(n, dtype=np.uint64)
    x, y, z = (u01(rng_word(seed, uid, j)) * L for j in range(3))
    u1 = 1.0 - u01(rng_word(seed, uid, 4))  # (0, 1]
    u2 = u01(rng_word(seed, uid, 5))
    zn = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
    d = np.exp(math.log(10.0) + 0.1 * zn)
    return Workload("c4_large_uniform", x, y, z, d, None,
                    dict(seed=seed, simulation_time_step=0.01, sorting_frequency=10),
                    steps=50)


def c5_sir(n: int = 10_000_000, seed: int = 0) -> Workload:
    """configs[4]: n point agents uniform in a periodic cube at ~5 agents
    within the infection radius 2 (rho = 0.1492 => L = (n / rho)^(1/3),
    406.2 at 10^7), unit random-walk steps, p = 0.1 per infected neighbour,
    recovery after 20 iterations, 1 % initially infected (absim_models.h)."""
    rho = 5.0 / (4.0 / 3.0 * math.pi * 8.0)
    L = (n / rho) ** (1.0 / 3.0)
    uid = np.arange(n, dtype=np.uint64)
    x, y, z = (u01(rng_word(seed, uid, j)) * L for j in range(3))
    return Workload("c5_sir", x, y, z, np.ones(n), None,
                    dict(seed=seed, model=N.MODEL_SIR, model_params=[L, 2.0, 1.0, 20.0, 0.1]),
                    steps=300, bytes_per_agent_iteration=120)


def _cube_side(n: int) -> int:
    s = 1
    while s * s * s < n:
        s += 1
    return s


def ref_proliferation(n: int = 4096) -> Workload:
    """The reference's own build_proliferation (models.cpp:21-38): a cubic
    lattice of ceil(n^(1/3))^3 cells (x-major), spacing 20, d 10, each with
    models::GrowDivide(rate 2, threshold 14, initial 10) (models.hpp:15-37)."""
    s = _cube_side(n)
    g = np.arange(s, dtype=np.float64) * 20.0
    x, y, z = (a.ravel() for a in np.meshgrid(g, g, g, indexing="ij"))
    m = len(x)
    return Workload("ref_proliferation", x.copy(), y.copy(), z.copy(), np.full(m, 10.0), None,
                    dict(seed=42, model=N.MODEL_GROW_DIVIDE, model_params=[2.0, 14.0, 10.0]),
                    steps=40, bytes_per_agent_iteration=128, tags=np.zeros(m, np.uint32),
                    rng_counters=np.zeros(m, np.uint64))


def ref_proliferation_die(n: int = 4096, p_remove: float = 0.02, sorting_frequency: int = 0) -> Workload:
    """ref_proliferation with every cell also removing itself with probability
    p_remove per iteration (ABS_MODEL_GROW_DIVIDE_DIE: models::GrowDivide +
    AgentContext::remove_self): additions and removals in the same commits,
    optionally with the Morton re-sort, so daughter uids and removal slots
    follow the reference's reordered storage."""
    wl = ref_proliferation(n)
    wl.name = "ref_proliferation_die"
    wl.params = dict(seed=42, model=N.MODEL_GROW_DIVIDE_DIE, model_params=[2.0, 14.0, 10.0, p_remove],
                     sorting_frequency=sorting_frequency)
    return wl


def ref_clustering(n: int = 10_000, seed: int = 42) -> Workload:
    """The reference's own build_clustering (models.cpp:40-61): n cells of
    two interleaved types (tag = uid % 2) uniformly in a cube of side
    cbrt(n) * 20, positions from each agent's own stream (counters 0..2, so
    its rng_counter is 3 afterwards), d 10, models::Cohere(30, 1)
    (models.hpp:42-64); tune_clustering_params pins the box length to 30."""
    side = math.cbrt(float(n)) * 20.0
    uid = np.arange(n, dtype=np.uint64)
    x, y, z = (0.0 + (side - 0.0) * u01(rng_word(seed, uid, j)) for j in range(3))
    return Workload("ref_clustering", x, y, z, np.full(n, 10.0), None,
                    dict(seed=seed, model=N.MODEL_COHERE, model_params=[30.0, 1.0], fixed_box_length=30.0),
                    steps=40, bytes_per_agent_iteration=128, tags=(uid % np.uint64(2)).astype(np.uint32),
                    rng_counters=np.full(n, 3, np.uint64))


CONFIGS = {
    "c1": c1_relaxation,
    "c2": c2_proliferation,
    "c3": c3_spheroid,
    "c4": c4_large_uniform,
    "c5": c5_sir,
}
