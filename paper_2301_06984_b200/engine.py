"""Reference-shaped host API over the B200 engine (include/absim_gpu.h).

Mirrors the reference's public surface for the hot path so call sites read
like the reference's own tests:

* ``SimulationParams``  — params.hpp:17-52 (hot-path fields + device knobs)
* ``Simulation``        — simulation.hpp:89-123: ``add_agents`` (batched
  ``add_agent``), ``simulate(iterations)``, ``report()``, ``environment()``,
  ``iteration``; failures raise like the reference (ValueError for
  std::invalid_argument, AbsimError(RuntimeError) for runtime/logic errors).
* ``UniformGrid``       — the Environment contract (environment.hpp:36-51):
  ``update()``, ``largest_agent_diameter()``, ``max_query_radius()``,
  ``name()``, plus UniformGrid's ``box_length/origin/dims/box_index_of``
  (uniform_grid.hpp:40-57), batched: ``cell_ids()`` and ``neighbors()``.
* ``SimulationReport``  — report.hpp:18-41 counters.

All compute runs in the sm_100a kernels of libabsim_gpu.so; there is no CPU
path.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


def peak_rss_bytes() -> int:
    """High-water-mark RSS of this process (report.cpp: VmHWM), 0 if unavailable."""
    try:
        with open("/proc/self/status") as f:
            for line in f:
                if line.startswith("VmHWM:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


ENVIRONMENTS = {"uniform_grid": N.ENV_UNIFORM_GRID, "brute_force": N.ENV_BRUTE_FORCE, "kdtree": N.ENV_KD_TREE, "kd_tree": N.ENV_KD_TREE}


@dataclass
class SimulationParams:
    seed: int = 42
    simulation_time_step: float = 0.1
    repulsion_coefficient: float = 2.0
    max_displacement: float = 3.0
    force_threshold: float = 0.0
    fixed_box_length: float = 0.0
    sorting_frequency: int = 0
    detect_static_agents: bool = False
    # device-side behaviour model (ABS_MODEL_*) and its parameters
    model: int = N.MODEL_NONE
    model_params: list = field(default_factory=lambda: [0.0] * 8)
    capacity: int = 0
    record_forces: bool = True
    bins_per_box: int = 0      # sub-bins per box edge along y, z (0 = auto)
    bins_per_box_x: int = 0    # sub-bins per box edge along x (0 = auto)
    # EnvironmentKind (params.hpp:9): "uniform_grid", "brute_force" or "kdtree" (params.cpp:7-30 names)
    environment: str = "uniform_grid"
    # per-agent candidate lists between environment rebuilds:
    # True = auto (used when the path allows it and a build pays off), False =
    # re-bin every step, "always" = build whenever the lists do not cover a step;
    # neighbor_skin 0 = 0.2 x the largest diameter
    neighbor_list: bool | str = True
    neighbor_skin: float = 0.0

    def validate(self):
        """SimulationParams::validate (params.cpp:44-72), hot-path subset."""
        if self.fixed_box_length < 0.0:
            raise ValueError("fixed_box_length must be >= 0")
        if not self.simulation_time_step > 0.0:
            raise ValueError("simulation_time_step must be > 0")
        if self.repulsion_coefficient < 0.0:
            raise ValueError("repulsion_coefficient must be >= 0")
        if not self.max_displacement > 0.0:
            raise ValueError("max_displacement must be > 0")
        if self.force_threshold < 0.0:
            raise ValueError("force_threshold must be >= 0")
        if self.environment not in ENVIRONMENTS:
            raise ValueError(f"unknown environment kind {self.environment!r}")
        if self.sorting_frequency > 0 and self.environment != "uniform_grid":
            raise ValueError("sorting requires the uniform_grid environment")  # params.cpp:52-55

    def to_c(self) -> N.Config:
        c = N.Config()
        N.load().abs_gpu_default_config(C.byref(c))
        c.seed = self.seed
        c.simulation_time_step = self.simulation_time_step
        c.repulsion_coefficient = self.repulsion_coefficient
        c.max_displacement = self.max_displacement
        c.force_threshold = self.force_threshold
        c.fixed_box_length = self.fixed_box_length
        c.sorting_frequency = self.sorting_frequency
        c.detect_static_agents = 1 if self.detect_static_agents else 0
        c.model = self.model
        mp = list(self.model_params) + [0.0] * (8 - len(self.model_params))
        for i in range(8):
            c.model_params[i] = float(mp[i])
        c.capacity = self.capacity
        c.record_forces = 1 if self.record_forces else 0
        c.bins_per_box = self.bins_per_box
        c.bins_per_box_x = self.bins_per_box_x
        c.environment = ENVIRONMENTS[self.environment]
        c.neighbor_list = 1 if self.neighbor_list == "always" else (0 if self.neighbor_list else -1)
        c.neighbor_skin = float(self.neighbor_skin)
        return c


@dataclass
class SimulationReport:
    """SimulationReport (report.hpp:18-41). Counters are cumulative. The wall
    buckets are device time of the iterations run while timing is enabled
    (Simulation.reset_timers(True)); total_wall_ms is the host wall time of
    simulate() calls, as in the reference."""
    iterations: int = 0
    final_agent_count: int = 0
    uid_count: int = 0
    force_evaluations: int = 0
    force_skips: int = 0
    agents_added: int = 0
    agents_removed: int = 0
    kernel_launches: int = 0
    agent_iterations: int = 0        # sum of the agents at the start of every iteration since the upload
    total_wall_ms: float = 0.0
    agent_ops_ms: float = 0.0
    env_update_ms: float = 0.0
    sorting_ms: float = 0.0
    setup_teardown_ms: float = 0.0
    per_iteration_ms: list = field(default_factory=list)
    per_operation_ms: dict = field(default_factory=dict)
    agents_sorted: int = 0           # cross-domain migrations during sorting: one domain per device
    same_domain_steals: int = 0      # no work stealing on the device (grid scheduler)
    cross_domain_steals: int = 0
    allocator_batch_migrations: int = 0
    peak_rss_bytes: int = 0


def _p(a, ct):
    return None if a is None else a.ctypes.data_as(C.POINTER(ct))


class UniformGrid:
    """Environment contract over the device grid (uniform_grid.hpp:26-94).
    With SimulationParams(environment="brute_force") it is the
    BruteForceEnvironment (environment.hpp:53-80): every agent is a
    candidate, max_query_radius is unbounded and there are no cell ids."""

    def __init__(self, sim: "Simulation"):
        self._sim = sim

    def name(self) -> str:
        return self._sim.params.environment

    def update(self) -> None:
        N.check(N.load().abs_gpu_env_update(self._sim._ctx), self._sim._ctx)

    def _info(self):
        g = np.zeros(5)
        dims = np.zeros(3, np.uint32)
        N.check(N.load().abs_gpu_grid_info(self._sim._ctx, _p(g, C.c_double), _p(dims, C.c_uint32)),
                self._sim._ctx)
        return g, dims

    def largest_agent_diameter(self) -> float:
        return float(self._info()[0][4])

    def box_length(self) -> float:
        return float(self._info()[0][3])

    def max_query_radius(self) -> float:
        if self._sim.params.environment != "uniform_grid":
            return math.inf
        return self.box_length()

    def origin(self) -> np.ndarray:
        return self._info()[0][:3].copy()

    def dims(self) -> np.ndarray:
        return self._info()[1].copy()

    def cell_ids(self) -> np.ndarray:
        """box_index_of for every agent, in device storage order."""
        n = self._sim.agent_count()
        out = np.zeros(n, np.uint64)
        N.check(N.load().abs_gpu_cell_ids(self._sim._ctx, _p(out, C.c_uint64)), self._sim._ctx)
        return out

    def neighbors(self):
        """CSR (offsets[n+1], uids) of sorted neighbour uids within the force
        query radius 0.5 (d + dmax) (simulation.cpp:469), storage order."""
        lib, ctx = N.load(), self._sim._ctx
        n = self._sim.agent_count()
        offsets = np.zeros(n + 1, np.uint64)
        total = C.c_uint64(0)
        N.check(lib.abs_gpu_neighbors(ctx, _p(offsets, C.c_uint64), None, 0, C.byref(total)), ctx)
        uids = np.zeros(max(1, total.value), np.uint64)
        N.check(lib.abs_gpu_neighbors(ctx, _p(offsets, C.c_uint64), _p(uids, C.c_uint64),
                                      total.value, C.byref(total)), ctx)
        return offsets, uids[: total.value]


class Simulation:
    """Simulation-shaped front end (simulation.hpp:89-123) on one B200."""

    def __init__(self, params: SimulationParams | None = None, device: int = 0):
        self.params = params or SimulationParams()
        self.params.validate()
        lib = N.load()
        self._wall_ms = 0.0  # host wall time of simulate() (report.total_wall_ms)
        self._cfg = self.params.to_c()
        ctx = C.c_void_p()
        N.check(lib.abs_gpu_create(C.byref(self._cfg), device, C.byref(ctx)), None)
        self._ctx = ctx
        self._env = UniformGrid(self)

    def close(self):
        if getattr(self, "_ctx", None):
            N.load().abs_gpu_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- population ------------------------------------------------------
    def add_agents(self, x, y, z, d, behaviour_mask=None, uid=None, volume=None, flags=None,
                   partners=None, uid_count: int = 0):
        """Batched Simulation::add_agent: replaces the population (uids
        0..n-1 in array order unless given)."""
        x, y, z, d = (np.ascontiguousarray(a, np.float64) for a in (x, y, z, d))
        m = None if behaviour_mask is None else np.ascontiguousarray(behaviour_mask, np.uint8)
        u = None if uid is None else np.ascontiguousarray(uid, np.uint64)
        v = None if volume is None else np.ascontiguousarray(volume, np.float64)
        f = None if flags is None else np.ascontiguousarray(flags, np.uint8)
        pa = None if partners is None else np.ascontiguousarray(partners, np.uint32)
        N.check(N.load().abs_gpu_upload(self._ctx, len(x), _p(u, C.c_uint64), _p(x, C.c_double),
                                        _p(y, C.c_double), _p(z, C.c_double), _p(d, C.c_double),
                                        _p(m, C.c_uint8), _p(v, C.c_double), _p(f, C.c_uint8),
                                        _p(pa, C.c_uint32), uid_count), self._ctx)

    def add_agents_device(self, x_ptr, y_ptr, z_ptr, d_ptr, n, uid_ptr=None, mask_ptr=None, uid_count: int = 0):
        """Population from device-resident arrays (e.g. torch CUDA tensors).
        With explicit uids, uid_count (> every uid) is required."""
        N.check(N.load().abs_gpu_upload_device(self._ctx, n, uid_ptr, x_ptr, y_ptr, z_ptr, d_ptr,
                                               mask_ptr, uid_count if uid_ptr else n), self._ctx)

    def remove_agents(self, uids):
        u = np.ascontiguousarray(uids, np.uint64)
        N.check(N.load().abs_gpu_remove(self._ctx, _p(u, C.c_uint64), len(u)), self._ctx)

    # -- schedule --------------------------------------------------------
    def simulate(self, iterations: int) -> None:
        t0 = time.perf_counter()
        N.check(N.load().abs_gpu_simulate(self._ctx, iterations), self._ctx)
        self._wall_ms += (time.perf_counter() - t0) * 1e3

    def set_grid_override(self, grid=None, dims=None) -> None:
        """Multi-domain: force the grid of all ranks (origin[3], box, dmax; dims)."""
        if grid is None:
            N.check(N.load().abs_gpu_set_grid_override(self._ctx, None, None), self._ctx)
            return
        g = np.ascontiguousarray(grid, np.float64)
        dm = np.ascontiguousarray(dims, np.uint32)
        N.check(N.load().abs_gpu_set_grid_override(self._ctx, _p(g, C.c_double), _p(dm, C.c_uint32)),
                self._ctx)

    def local_bounds(self) -> np.ndarray:
        """[min x, min y, min z, max x, max y, max z, max d] of the population."""
        out = np.zeros(7)
        N.check(N.load().abs_gpu_local_bounds(self._ctx, _p(out, C.c_double)), self._ctx)
        return out

    def sir_counts(self):
        """Config 5: [S, I, R] after the last iteration."""
        out = np.zeros(3, np.uint64)
        N.check(N.load().abs_gpu_sir_counts(self._ctx, _p(out, C.c_uint64)), self._ctx)
        return [int(v) for v in out]

    def sir_state(self):
        """Config 5: (state per agent, infection iteration), storage order."""
        n = self.agent_count()
        st = np.zeros(n, np.uint8)
        ti = np.zeros(n, np.uint32)
        N.check(N.load().abs_gpu_sir_state(self._ctx, _p(st, C.c_uint8), _p(ti, C.c_uint32)), self._ctx)
        return st, ti

    # -- Agent::tag / rng_counter (reference models) -------------------------
    def set_agent_ext(self, tags=None, rng_counters=None) -> None:
        """Per-agent tags / RandomStream counters in the current storage order."""
        t = None if tags is None else np.ascontiguousarray(tags, np.uint32)
        r = None if rng_counters is None else np.ascontiguousarray(rng_counters, np.uint64)
        N.check(N.load().abs_gpu_set_agent_ext(self._ctx, _p(t, C.c_uint32), _p(r, C.c_uint64)), self._ctx)

    def agent_ext(self):
        """(tags, rng_counters) in the device storage order."""
        n = self.report().final_agent_count
        t = np.zeros(n, np.uint32)
        r = np.zeros(n, np.uint64)
        N.check(N.load().abs_gpu_download_ext(self._ctx, _p(t, C.c_uint32), _p(r, C.c_uint64)), self._ctx)
        return t, r

    # -- multi-domain additions (deferred commit) ---------------------------
    def set_defer_commit(self, defer: bool) -> None:
        N.check(N.load().abs_gpu_set_defer_commit(self._ctx, 1 if defer else 0), self._ctx)

    def division_marks(self, out_ptr=None, cap: int = 0) -> int:
        """Copy this context's uid-indexed division marks of the pending
        iteration into a device buffer (uint32, >= uid_count entries);
        returns uid_count (call with out_ptr=None to size the buffer)."""
        n = C.c_uint64(0)
        rc = N.load().abs_gpu_division_marks(self._ctx, out_ptr, cap, C.byref(n))
        if out_ptr is not None:
            N.check(rc, self._ctx)
        return int(n.value)

    def commit(self, global_marks_ptr=None, length: int = 0) -> None:
        """Finish the pending iteration's additions with the rank-summed marks."""
        N.check(N.load().abs_gpu_commit(self._ctx, global_marks_ptr, length), self._ctx)

    def set_iteration(self, iteration: int) -> None:
        N.check(N.load().abs_gpu_set_iteration(self._ctx, iteration), self._ctx)

    def synchronize(self):
        N.check(N.load().abs_gpu_synchronize(self._ctx), self._ctx)

    def sort(self):
        """sort_and_balance (sort_balance.cpp:22-148) on the current storage."""
        N.check(N.load().abs_gpu_sort(self._ctx), self._ctx)

    def environment(self) -> UniformGrid:
        return self._env

    def _stats(self) -> N.Stats:
        s = N.Stats()
        N.check(N.load().abs_gpu_stats(self._ctx, C.byref(s)), self._ctx)
        return s

    @property
    def iteration(self) -> int:
        return int(self._stats().iterations)

    def agent_count(self) -> int:
        return int(self._stats().agents)

    def report(self) -> SimulationReport:
        s = self._stats()
        return SimulationReport(iterations=s.iterations, final_agent_count=s.agents,
                                uid_count=s.uid_count, force_evaluations=s.force_evaluations,
                                force_skips=s.force_skips, agents_added=s.agents_added,
                                agents_removed=s.agents_removed, kernel_launches=s.kernel_launches,
                                agent_iterations=s.agent_iterations, total_wall_ms=self._wall_ms, peak_rss_bytes=peak_rss_bytes())

    def phase_report(self) -> SimulationReport:
        """report() plus the device-time categories of the timed iterations."""
        r = self.report()
        out4 = np.zeros(4)
        n = C.c_uint64(0)
        N.check(N.load().abs_gpu_phase_times(self._ctx, _p(out4, C.c_double), None, 0, C.byref(n)), self._ctx)
        per = np.zeros(max(int(n.value), 1))
        N.check(N.load().abs_gpu_phase_times(self._ctx, _p(out4, C.c_double), _p(per, C.c_double), len(per),
                                             C.byref(n)), self._ctx)
        r.env_update_ms, r.sorting_ms, r.agent_ops_ms, r.setup_teardown_ms = (float(v) for v in out4)
        r.per_iteration_ms = per[:int(n.value)].tolist()
        r.per_operation_ms = {"environment_update": r.env_update_ms, "sorting": r.sorting_ms,
                              "agent_operations": r.agent_ops_ms, "commit": r.setup_teardown_ms}
        return r

    def agents(self) -> dict:
        """Download the population (device storage order)."""
        n = self.agent_count()
        out = {"uid": np.zeros(n, np.uint64), "x": np.zeros(n), "y": np.zeros(n), "z": np.zeros(n),
               "d": np.zeros(n), "fx": np.zeros(n), "fy": np.zeros(n), "fz": np.zeros(n),
               "partners": np.zeros(n, np.uint32), "flags": np.zeros(n, np.uint8),
               "volume": np.zeros(n)}
        nn = C.c_uint64(0)
        N.check(N.load().abs_gpu_download(
            self._ctx, C.byref(nn), _p(out["uid"], C.c_uint64),
            *(_p(out[k], C.c_double) for k in ("x", "y", "z", "d", "fx", "fy", "fz")),
            _p(out["partners"], C.c_uint32), _p(out["flags"], C.c_uint8),
            _p(out["volume"], C.c_double)), self._ctx)
        return out

    def fields(self, *names) -> dict:
        """Download a subset of agents() (uid, x, y, z, d, partners, flags), device storage order."""
        n = self.agent_count()
        dt = {"uid": np.uint64, "partners": np.uint32, "flags": np.uint8}
        out = {k: np.zeros(n, dt.get(k, np.float64)) for k in names}
        nn = C.c_uint64(0)
        g = lambda k, ct: _p(out[k], ct) if k in out else None  # noqa: E731
        N.check(N.load().abs_gpu_download(
            self._ctx, C.byref(nn), g("uid", C.c_uint64), g("x", C.c_double), g("y", C.c_double),
            g("z", C.c_double), g("d", C.c_double), None, None, None, g("partners", C.c_uint32),
            g("flags", C.c_uint8), None), self._ctx)
        return out

    def positions(self, x, y, z) -> int:
        """Download positions into caller-owned float64 arrays (e.g. pinned);
        returns the agent count (device storage order)."""
        nn = C.c_uint64(0)
        N.check(N.load().abs_gpu_download(self._ctx, C.byref(nn), None, _p(x, C.c_double),
                                          _p(y, C.c_double), _p(z, C.c_double), None, None, None,
                                          None, None, None, None), self._ctx)
        return int(nn.value)

    def run_frames(self, inputs, outputs, iterations: int = 1, first_iteration: int = 0, uids=None) -> list:
        """Host-boundary pipeline (abs_gpu_run_frames): for each frame f,
        upload inputs[f] = (x, y, z, d), run `iterations` iterations from
        iteration first_iteration + f * iterations, and write the positions
        into outputs[f] = (x, y, z) (float64 arrays, ideally page-locked);
        uids[f] (uint64, optional) receives the uid of each output row.
        The next frame's upload and the previous frame's download overlap
        the current frame's iterations. Returns the agent count per frame."""
        if len(inputs) != len(outputs):
            raise ValueError("one output triple per input frame")
        frames = (N.Frame * len(inputs))()
        keep, counts = [], (C.c_uint64 * max(1, len(inputs)))()
        for f, (inp, out) in enumerate(zip(inputs, outputs)):
            a = [np.ascontiguousarray(v, np.float64) for v in inp]
            o = list(out)
            for v in o:
                if v.dtype != np.float64 or not v.flags.c_contiguous:
                    raise ValueError("outputs must be contiguous float64 arrays")
            keep += a
            n = len(a[0])
            if any(len(v) != n for v in a):
                raise ValueError("frame arrays differ in length")
            u = None if uids is None else uids[f]
            if u is not None and (u.dtype != np.uint64 or not u.flags.c_contiguous):
                raise ValueError("uids must be contiguous uint64 arrays")
            cap = min(len(v) for v in o + ([u] if u is not None else []))
            frames[f] = N.Frame(n, *(_p(v, C.c_double) for v in a), *(_p(v, C.c_double) for v in o), cap,
                                C.cast(C.byref(counts, 8 * f), C.POINTER(C.c_uint64)), _p(u, C.c_uint64))
        t0 = time.perf_counter()
        N.check(N.load().abs_gpu_run_frames(self._ctx, frames, len(inputs), iterations, first_iteration),
                self._ctx)
        self._wall_ms += (time.perf_counter() - t0) * 1e3
        del keep
        return [int(counts[f]) for f in range(len(inputs))]

    # -- timing of the dominant kernel --------------------------------------
    def reset_timers(self, enable: bool = True):
        N.check(N.load().abs_gpu_reset_timers(self._ctx, 1 if enable else 0), self._ctx)

    def list_stats(self) -> dict:
        """Neighbour-list counters (abs_gpu_list_stats): builds, list steps,
        timed build launches + their CUDA-event ms, largest candidate count."""
        out = np.zeros(4, np.uint64)
        ms = C.c_double(0)
        N.check(N.load().abs_gpu_list_stats(self._ctx, _p(out, C.c_uint64), C.byref(ms)), self._ctx)
        return {"builds": int(out[0]), "list_steps": int(out[1]), "build_launches": int(out[2]),
                "max_candidates": int(out[3]), "build_ms": ms.value}

    def record_evaluations(self, enable: bool = True):
        """Record every agent's force evaluations per iteration (parity hook)."""
        N.check(N.load().abs_gpu_record_evaluations(self._ctx, 1 if enable else 0), self._ctx)

    def evaluations(self) -> np.ndarray:
        """Per-agent force evaluations of the last iteration, download order."""
        out = np.zeros(max(1, self.agent_count()), np.uint32)
        N.check(N.load().abs_gpu_download_evaluations(self._ctx, _p(out, C.c_uint32), len(out)), self._ctx)
        return out[:self.agent_count()]

    def storage_keys(self) -> np.ndarray:
        """Each agent's slot in the reference's storage order (download order);
        agents()[k][np.argsort(storage_keys())] is the reference's for_each_agent order."""
        out = np.zeros(max(1, self.agent_count()), np.uint32)
        N.check(N.load().abs_gpu_download_storage_keys(self._ctx, _p(out, C.c_uint32), len(out)), self._ctx)
        return out[:self.agent_count()]

    def force_kernel_time(self):
        ms = C.c_double(0)
        launches = C.c_uint64(0)
        N.check(N.load().abs_gpu_force_kernel_time(self._ctx, C.byref(ms), C.byref(launches)),
                self._ctx)
        return ms.value, launches.value

    @property
    def stream(self) -> int:
        return N.load().abs_gpu_stream(self._ctx) or 0
