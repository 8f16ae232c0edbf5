"""TEST INFRASTRUCTURE ONLY — ctypes front-ends for the two CPU oracles.

* ``RefSim``  drives the UNMODIFIED reference engine (oracle/_ref/libabsim_ref.so,
  built by oracle/Makefile from /root/reference/proj/src + ref_harness.cpp).
* ``PortSim`` drives the C restatement (oracle/_build/liboracle.so, built from
  oracle/absim_oracle.c).

Both expose the same methods so tests can run them side by side. Only tests/,
``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference arm may
import this module; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libabsim_ref.so")
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REFERENCE_SRC = "/root/reference/proj/src"

MODEL_NONE, MODEL_PROLIFERATION, MODEL_DRIVE, MODEL_GROW, MODEL_SIR = 0, 1, 2, 3, 4

F_STATIC, F_MOVED, F_GREW, F_NEWLY_ADDED, F_NVIOL, F_NNEW = 1, 2, 4, 8, 16, 32
F_GHOST = 128


class _Params(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64),
        ("threads", C.c_int32),
        ("domains", C.c_int32),
        ("dt", C.c_double),
        ("k", C.c_double),
        ("max_disp", C.c_double),
        ("threshold", C.c_double),
        ("fixed_box", C.c_double),
        ("sorting_frequency", C.c_uint64),
        ("detect_static", C.c_int32),
        ("model", C.c_int32),
        ("mp", C.c_double * 8),
        ("env", C.c_int32),
        ("pad", C.c_int32),
    ]


@dataclass
class OracleParams:
    """Mirror of SimulationParams (params.hpp:17-52) restricted to the hot path."""

    seed: int = 42
    threads: int = 1
    domains: int = 1
    dt: float = 0.1
    k: float = 2.0
    max_disp: float = 3.0
    threshold: float = 0.0
    fixed_box: float = 0.0
    sorting_frequency: int = 0
    detect_static: bool = False
    model: int = MODEL_NONE
    mp: list = field(default_factory=lambda: [0.0] * 8)
    env: int = 0  # EnvironmentKind (params.hpp:9): 0 uniform grid, 1 brute force, 2 kd-tree (reference only)

    def to_c(self) -> _Params:
        p = _Params()
        p.seed = self.seed
        p.threads = self.threads
        p.domains = self.domains
        p.dt = self.dt
        p.k = self.k
        p.max_disp = self.max_disp
        p.threshold = self.threshold
        p.fixed_box = self.fixed_box
        p.sorting_frequency = self.sorting_frequency
        p.detect_static = 1 if self.detect_static else 0
        p.model = self.model
        p.env = self.env
        mp = list(self.mp) + [0.0] * (8 - len(self.mp))
        for i in range(8):
            p.mp[i] = float(mp[i])
        return p


def build(ref: bool = True) -> None:
    """Compile the C port (always) and the reference (when its sources exist)."""
    targets = ["port"]
    if ref and os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-j8", "-C", HERE, *targets], check=True)


def _ptr(a, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


_D = C.POINTER(C.c_double)
_U64 = C.POINTER(C.c_uint64)
_U32 = C.POINTER(C.c_uint32)
_U8 = C.POINTER(C.c_uint8)


class _Sim:
    prefix = ""
    _lib = None

    @classmethod
    def lib(cls):
        raise NotImplementedError

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib()[f"{self.prefix}last_error"]().decode())

    def __init__(self, params: OracleParams, x, y, z, d, mask=None):
        lib = self.lib()
        self.params = params
        x, y, z, d = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, y, z, d))
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        self._p = params.to_c()
        self.h = lib[f"{self.prefix}create"](C.byref(self._p), len(x), _ptr(x, C.c_double),
                                             _ptr(y, C.c_double), _ptr(z, C.c_double),
                                             _ptr(d, C.c_double), _ptr(m, C.c_uint8))
        if not self.h:
            raise RuntimeError(lib[f"{self.prefix}last_error"]().decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib()[f"{self.prefix}destroy"](self.h)
            self.h = None

    def __del__(self):
        self.close()

    def simulate(self, iterations: int):
        self._check(self.lib()[f"{self.prefix}simulate"](self.h, iterations))

    def counts(self) -> dict:
        out = np.zeros(8, np.uint64)
        self._counts(out)
        keys = ["agents", "uid_count", "iterations", "force_evaluations", "force_skips",
                "agents_added", "agents_removed", "agents_sorted"]
        return {k: int(v) for k, v in zip(keys, out)}

    def dump(self) -> dict:
        n = self.counts()["agents"]
        out = {
            "uid": np.zeros(n, np.uint64),
            "x": np.zeros(n), "y": np.zeros(n), "z": np.zeros(n), "d": np.zeros(n),
            "fx": np.zeros(n), "fy": np.zeros(n), "fz": np.zeros(n),
            "partners": np.zeros(n, np.uint32), "flags": np.zeros(n, np.uint8),
            "volume": np.zeros(n),
        }
        self._check(self.lib()[f"{self.prefix}dump"](
            self.h, _ptr(out["uid"], C.c_uint64), *(_ptr(out[k], C.c_double) for k in
                                                    ("x", "y", "z", "d", "fx", "fy", "fz")),
            _ptr(out["partners"], C.c_uint32), _ptr(out["flags"], C.c_uint8),
            _ptr(out["volume"], C.c_double)))
        return out

    def env_update(self) -> dict:
        g = np.zeros(5)
        dims = np.zeros(3, np.uint32)
        idx = C.c_uint64(0)
        self._check(self.lib()[f"{self.prefix}env_update"](self.h, _ptr(g, C.c_double),
                                                           _ptr(dims, C.c_uint32), C.byref(idx)))
        return {"origin": g[:3].copy(), "box": float(g[3]), "dmax": float(g[4]),
                "dims": dims.copy(), "indexed": int(idx.value)}

    def cell_ids(self) -> np.ndarray:
        n = self.counts()["agents"]
        out = np.zeros(n, np.uint64)
        self._check(self.lib()[f"{self.prefix}cell_ids"](self.h, _ptr(out, C.c_uint64)))
        return out

    def neighbors(self):
        """(offsets[n+1], uids) CSR of sorted force-query neighbour uids, storage order."""
        n = self.counts()["agents"]
        offsets = np.zeros(n + 1, np.uint64)
        cap = max(64, 64 * n)
        while True:
            uids = np.zeros(cap, np.uint64)
            tot = self.lib()[f"{self.prefix}neighbors"](self.h, _ptr(offsets, C.c_uint64),
                                                        _ptr(uids, C.c_uint64), cap)
            if tot == -2:
                cap = int(offsets[-1]) + 1
                continue
            if tot < 0:
                self._check(-1)
            return offsets, uids[:tot].copy()

    def sort(self) -> int:
        moved = C.c_uint64(0)
        self._check(self.lib()[f"{self.prefix}sort"](self.h, C.byref(moved)))
        return int(moved.value)

    def set_tags(self, tags):
        """Agent::set_tag per agent, storage order (agent.hpp:35-36)."""
        t = np.ascontiguousarray(tags, np.uint32)
        self._check(self.lib()[f"{self.prefix}set_tags"](self.h, _ptr(t, C.c_uint32)))

    def tags(self) -> np.ndarray:
        out = np.zeros(self.counts()["agents"], np.uint32)
        self._check(self.lib()[f"{self.prefix}tags"](self.h, _ptr(out, C.c_uint32)))
        return out

    def rng_counters(self) -> np.ndarray:
        """Agent::rng_counter per agent, storage order (agent.hpp:145)."""
        out = np.zeros(self.counts()["agents"], np.uint64)
        self._check(self.lib()[f"{self.prefix}rng_counters"](self.h, _ptr(out, C.c_uint64)))
        return out


def _bind(lib, prefix, ref_style):
    lib[f"{prefix}last_error"].restype = C.c_char_p
    lib[f"{prefix}create"].restype = C.c_void_p
    lib[f"{prefix}create"].argtypes = [C.c_void_p, C.c_uint64, _D, _D, _D, _D, _U8]
    lib[f"{prefix}destroy"].argtypes = [C.c_void_p]
    lib[f"{prefix}simulate"].argtypes = [C.c_void_p, C.c_uint64]
    lib[f"{prefix}dump"].argtypes = [C.c_void_p, _U64] + [_D] * 7 + [_U32, _U8, _D]
    lib[f"{prefix}env_update"].argtypes = [C.c_void_p, _D, _U32, _U64]
    lib[f"{prefix}cell_ids"].argtypes = [C.c_void_p, _U64]
    lib[f"{prefix}neighbors"].restype = C.c_int64
    lib[f"{prefix}neighbors"].argtypes = [C.c_void_p, _U64, _U64, C.c_uint64]
    lib[f"{prefix}sort"].argtypes = [C.c_void_p, _U64]
    lib[f"{prefix}set_tags"].argtypes = [C.c_void_p, _U32]
    lib[f"{prefix}tags"].argtypes = [C.c_void_p, _U32]
    lib[f"{prefix}rng_counters"].argtypes = [C.c_void_p, _U64]
    if ref_style:
        lib[f"{prefix}counts"].argtypes = [C.c_void_p, _U64, _D]
    else:
        lib[f"{prefix}counts"].argtypes = [C.c_void_p, _U64]


class _LibDict:
    def __init__(self, cdll):
        self.cdll = cdll

    def __getitem__(self, name):
        return getattr(self.cdll, name)


class RefSim(_Sim):
    """The unmodified reference engine through its public API."""

    prefix = "ref_"

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref`")
            d = _LibDict(C.CDLL(REF_SO))
            _bind(d, "ref_", True)
            d["ref_create_builtin"].restype = C.c_void_p
            d["ref_create_builtin"].argtypes = [C.c_void_p, C.c_char_p, C.c_uint64]
            cls._lib = d
        return cls._lib

    def neighbor_counts(self, threads: int = 0) -> np.ndarray:
        """Per-agent force-query neighbour counts (storage order), multithreaded;
        call after env_update()."""
        lib = self.lib().cdll
        lib.ref_neighbor_counts.argtypes = [C.c_void_p, _U32, C.c_int]
        out = np.zeros(self.counts()["agents"], np.uint32)
        if lib.ref_neighbor_counts(self.h, _ptr(out, C.c_uint32), threads or os.cpu_count()) != 0:
            raise RuntimeError(lib.ref_last_error().decode())
        return out

    @classmethod
    def builtin(cls, params: OracleParams, name: str, n: int) -> "RefSim":
        self = cls.__new__(cls)
        self.params = params
        self._p = params.to_c()
        self.h = cls.lib()["ref_create_builtin"](C.byref(self._p), name.encode(), n)
        if not self.h:
            raise RuntimeError(cls.lib()["ref_last_error"]().decode())
        return self

    def _counts(self, out):
        wall = C.c_double(0)
        self._check(self.lib()["ref_counts"](self.h, _ptr(out, C.c_uint64), C.byref(wall)))
        self.wall_ms = wall.value


class PortSim(_Sim):
    """The C restatement (oracle/absim_oracle.c)."""

    prefix = "orc_"

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(PORT_SO):
                build(ref=False)
            d = _LibDict(C.CDLL(PORT_SO))
            _bind(d, "orc_", False)
            d["orc_remove"].argtypes = [C.c_void_p, _U32, C.c_uint32]
            d["orc_set_rng_counters"].argtypes = [C.c_void_p, _U64]
            d["orc_set_grid_override"].argtypes = [C.c_void_p, _D, _U32]
            d["orc_dump_beh"].argtypes = [C.c_void_p, _U8, _U32]
            d["orc_sir_counts"].argtypes = [C.c_void_p, _U64]
            d["orc_load"].argtypes = [C.c_void_p, C.c_uint64, _U64, _D, _D, _D, _D, _U8, _U32, _D, _U8,
                                      C.c_uint64, C.c_uint64]
            d["orc_morton_encode3"].argtypes = [C.c_uint32] * 3 + [_U64]
            d["orc_morton_decode3"].argtypes = [C.c_uint64, _U32]
            d["orc_offsets_table"].restype = C.c_int64
            d["orc_offsets_table"].argtypes = [_U32, _U64, _U64, C.c_uint64]
            d["orc_exclusive_scan"].restype = C.c_uint64
            d["orc_exclusive_scan"].argtypes = [_U64, C.c_uint64]
            cls._lib = d
        return cls._lib

    def _counts(self, out):
        self._check(self.lib()["orc_counts"](self.h, _ptr(out, C.c_uint64)))

    def set_grid_override(self, grid=None, dims=None):
        """Force the global grid (origin[3], box, dmax) + dims; None clears."""
        if grid is None:
            self._check(self.lib()["orc_set_grid_override"](self.h, None, None))
            return
        g = np.ascontiguousarray(grid, np.float64)
        dm = np.ascontiguousarray(dims, np.uint32)
        self._check(self.lib()["orc_set_grid_override"](self.h, _ptr(g, C.c_double), _ptr(dm, C.c_uint32)))

    def load(self, st: dict, uid_count: int, iteration: int):
        """Replace the population with a full state dict (dump() layout + 'beh')."""
        n = len(st["x"])
        a = {k: np.ascontiguousarray(st[k]) for k in ("x", "y", "z", "d")}
        uid = np.ascontiguousarray(st["uid"], np.uint64)
        fl = np.ascontiguousarray(st["flags"], np.uint8)
        pa = np.ascontiguousarray(st["partners"], np.uint32)
        vo = np.ascontiguousarray(st["volume"], np.float64)
        be = np.ascontiguousarray(st.get("beh", np.zeros(n, np.uint8)), np.uint8)
        self._check(self.lib()["orc_load"](self.h, n, _ptr(uid, C.c_uint64),
                                           *(_ptr(a[k], C.c_double) for k in ("x", "y", "z", "d")),
                                           _ptr(fl, C.c_uint8), _ptr(pa, C.c_uint32), _ptr(vo, C.c_double),
                                           _ptr(be, C.c_uint8), uid_count, iteration))

    def sir_state(self):
        """(state per agent [0 S, 1 I, 2 R], infection iteration), storage order."""
        n = self.counts()["agents"]
        st = np.zeros(n, np.uint8)
        ti = np.zeros(n, np.uint32)
        self._check(self.lib()["orc_dump_beh"](self.h, _ptr(st, C.c_uint8), _ptr(ti, C.c_uint32)))
        return st, ti

    def sir_counts(self):
        out = np.zeros(3, np.uint64)
        self._check(self.lib()["orc_sir_counts"](self.h, _ptr(out, C.c_uint64)))
        return [int(v) for v in out]

    def remove(self, slots):
        s = np.ascontiguousarray(slots, dtype=np.uint32)
        self._check(self.lib()["orc_remove"](self.h, _ptr(s, C.c_uint32), len(s)))

    def set_rng_counters(self, c):
        v = np.ascontiguousarray(c, np.uint64)
        self._check(self.lib()["orc_set_rng_counters"](self.h, _ptr(v, C.c_uint64)))


class RefSirSim:
    """Config 5 (SIR, periodic cube) through the UNMODIFIED reference engine:
    ghost images at the faces + public agent / standalone operations
    (ref_harness.cpp, RefSir). Same interface as PortSim's SIR subset."""

    def __init__(self, params: OracleParams, x, y, z):
        lib = RefSim.lib().cdll
        lib.ref_sir_create.restype = C.c_void_p
        lib.ref_sir_create.argtypes = [C.c_void_p, C.c_uint64, _D, _D, _D]
        lib.ref_sir_destroy.argtypes = [C.c_void_p]
        lib.ref_sir_simulate.argtypes = [C.c_void_p, C.c_uint64]
        lib.ref_sir_counts.restype = C.c_int64
        lib.ref_sir_counts.argtypes = [C.c_void_p, _U64, C.c_uint64]
        lib.ref_sir_dump.argtypes = [C.c_void_p, _U64, _D, _D, _D, _U8, _U32]
        lib.ref_sir_agents.restype = C.c_uint64
        lib.ref_sir_agents.argtypes = [C.c_void_p]
        self.lib = lib
        x, y, z = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, y, z))
        self._p = params.to_c()
        self.h = lib.ref_sir_create(C.byref(self._p), len(x), _ptr(x, C.c_double), _ptr(y, C.c_double),
                                    _ptr(z, C.c_double))
        if not self.h:
            raise RuntimeError(lib.ref_last_error().decode())
        self.iterations = 0

    def close(self):
        if getattr(self, "h", None):
            self.lib.ref_sir_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def simulate(self, iterations: int):
        if self.lib.ref_sir_simulate(self.h, iterations) != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        self.iterations += iterations

    def count_history(self) -> np.ndarray:
        out = np.zeros((max(self.iterations, 1), 3), np.uint64)
        n = self.lib.ref_sir_counts(self.h, _ptr(out, C.c_uint64), self.iterations)
        return out[:n]

    def sir_counts(self):
        return [int(v) for v in self.count_history()[-1]]

    def agents(self) -> int:
        return int(self.lib.ref_sir_agents(self.h))

    def counts(self) -> dict:
        return {"agents": self.agents(), "iterations": self.iterations}

    def dump(self) -> dict:
        n = self.agents()
        out = {"uid": np.zeros(n, np.uint64), "x": np.zeros(n), "y": np.zeros(n), "z": np.zeros(n),
               "state": np.zeros(n, np.uint8), "t": np.zeros(n, np.uint32)}
        if self.lib.ref_sir_dump(self.h, _ptr(out["uid"], C.c_uint64), _ptr(out["x"], C.c_double),
                                 _ptr(out["y"], C.c_double), _ptr(out["z"], C.c_double),
                                 _ptr(out["state"], C.c_uint8), _ptr(out["t"], C.c_uint32)) != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return out


def morton_encode3(x: int, y: int, z: int) -> int:
    out = C.c_uint64(0)
    if PortSim.lib()["orc_morton_encode3"](x, y, z, C.byref(out)) != 0:
        raise ValueError(PortSim.lib()["orc_last_error"]().decode())
    return int(out.value)


def morton_decode3(code: int):
    out = np.zeros(3, np.uint32)
    PortSim.lib()["orc_morton_decode3"](code, _ptr(out, C.c_uint32))
    return tuple(int(v) for v in out)


def offsets_table(dims):
    d = np.ascontiguousarray(dims, dtype=np.uint32)
    cap = 4096
    st = np.zeros(cap, np.uint64)
    of = np.zeros(cap, np.uint64)
    n = PortSim.lib()["orc_offsets_table"](_ptr(d, C.c_uint32), _ptr(st, C.c_uint64),
                                           _ptr(of, C.c_uint64), cap)
    if n < 0:
        raise ValueError(PortSim.lib()["orc_last_error"]().decode())
    assert n <= cap
    return [(int(a), int(b)) for a, b in zip(st[:n], of[:n])]


def exclusive_scan(values):
    v = np.ascontiguousarray(values, dtype=np.uint64).copy()
    total = PortSim.lib()["orc_exclusive_scan"](_ptr(v, C.c_uint64), len(v))
    return v, int(total)
