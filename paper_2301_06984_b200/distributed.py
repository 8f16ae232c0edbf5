"""Slab domain decomposition of the mechanical step across ranks.

The reference scales only inside one shared-memory node (NUMA domains +
work stealing); this is the multi-GPU form of the same
data-parallel step. One process per GPU, `torch.distributed` for the
exchange (NCCL on GPUs, gloo for the CPU tests). Per iteration:

1. **Global grid.** Each rank reduces the bounds of its owned agents; an
   all-reduce(MAX) over [-lo, hi, dmax] (7 doubles, exact) gives every rank
   the single-domain grid (uniform_grid.cpp:74-141): origin, box length,
   dims. Cell ids and box geometry therefore match the one-process
   reference bit for bit.
2. **Ownership by box layer.** Rank r owns the agents whose reference box z
   index lies in [L_r, L_{r+1}) (equal split of dims[2]; z is the
   Morton-major axis, morton.hpp:9-11). Agents whose layer changed migrate
   to the owning rank (max displacement << box, so only to r-1/r+1).
3. **Ghost halo.** Each rank sends its bottom layer to r-1 and its top layer
   to r+1; received agents are loaded flagged ABS_FLAG_GHOST: they are
   binned and serve as candidates (27-box neighbourhood complete for every
   owned agent) but are never stepped.
4. **Step** with the global grid forced (abs_gpu_set_grid_override), then
   keep the owned agents.

Models that add agents (config 2) need a global daughter-uid ranking and are
not decomposed yet (NotImplementedError).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

FLAG_GHOST = 128
FIELDS_F = ["x", "y", "z", "d", "volume", "fx", "fy", "fz"]
FIELDS_I = ["uid", "flags", "partners", "beh"]


def _empty_state():
    st = {k: np.zeros(0) for k in FIELDS_F}
    st.update({"uid": np.zeros(0, np.uint64), "flags": np.zeros(0, np.uint8),
               "partners": np.zeros(0, np.uint32), "beh": np.zeros(0, np.uint8)})
    return st


def _take(st, idx):
    return {k: v[idx] for k, v in st.items()}


def _concat(states):
    out = {}
    for k in states[0]:
        out[k] = np.concatenate([s[k] for s in states])
    return out


def pack(st) -> np.ndarray:
    """Agents -> (n, 12) float64 records (uids < 2^53 are exact)."""
    n = len(st["x"])
    rec = np.empty((n, 12), np.float64)
    for j, k in enumerate(FIELDS_F):
        rec[:, j] = st[k]
    for j, k in enumerate(FIELDS_I):
        rec[:, 8 + j] = st[k].astype(np.float64)
    return rec


def unpack(rec: np.ndarray):
    st = {k: np.ascontiguousarray(rec[:, j]) for j, k in enumerate(FIELDS_F)}
    st["uid"] = rec[:, 8].astype(np.uint64)
    st["flags"] = rec[:, 9].astype(np.uint8)
    st["partners"] = rec[:, 10].astype(np.uint32)
    st["beh"] = rec[:, 11].astype(np.uint8)
    return st


@dataclass
class GlobalGrid:
    origin: np.ndarray
    box: float
    dmax: float
    dims: np.ndarray

    def as_override(self):
        return np.array([*self.origin, self.box, self.dmax]), self.dims.astype(np.uint32)


def global_grid(bounds7: np.ndarray, fixed_box_length: float = 0.0) -> GlobalGrid:
    """uniform_grid.cpp:112-141 on all-reduced bounds (same IEEE ops)."""
    lo, hi, dmax = bounds7[:3], bounds7[3:6], float(bounds7[6])
    if not (np.isfinite(lo).all() and np.isfinite(hi).all()):
        raise RuntimeError("agent positions are not finite")
    if fixed_box_length > 0.0:
        if dmax > fixed_box_length:
            raise RuntimeError("fixed box length is smaller than the largest agent diameter")
        box = fixed_box_length
    else:
        box = dmax
    dims = np.array([max(1, int(math.floor((hi[k] - lo[k]) / box)) + 1) for k in range(3)], np.int64)
    if int(np.prod(dims)) > (1 << 31):
        raise RuntimeError("grid would exceed the box budget")
    return GlobalGrid(lo.copy(), box, dmax, dims)


def box_layer(z: np.ndarray, g: GlobalGrid) -> np.ndarray:
    """Reference box z-coordinate (uniform_grid.cpp:28-37)."""
    rel = (z - g.origin[2]) / g.box
    return np.clip(np.floor(rel), 0, g.dims[2] - 1).astype(np.int64)


def layer_bounds(dims_z: int, world: int) -> np.ndarray:
    return np.array([(r * dims_z) // world for r in range(world + 1)], np.int64)


class SlabDecomposition:
    """Drives one rank. `engine` implements load/set_grid_override/step/dump/
    counters (see GpuRankEngine / tests' OracleRankEngine)."""

    def __init__(self, engine, dist, rank: int, world: int, state: dict, uid_count: int,
                 fixed_box_length: float = 0.0, device=None):
        self.e, self.dist, self.rank, self.world = engine, dist, rank, world
        self.state = state  # owned agents only
        self.uid_count = uid_count
        self.iteration = 0
        self.fixed_box_length = fixed_box_length
        self.device = device
        self.evals = 0
        self.skips = 0

    # -- collectives (torch.distributed) ----------------------------------
    def _t(self, a):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(a))
        return t.to(self.device) if self.device is not None else t

    def _allreduce_max(self, a: np.ndarray) -> np.ndarray:
        t = self._t(a.astype(np.float64))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.cpu().numpy()

    def _allreduce_sum(self, a: np.ndarray) -> np.ndarray:
        t = self._t(a.astype(np.int64))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t.cpu().numpy()

    def _exchange(self, to_prev: np.ndarray, to_next: np.ndarray):
        """Send record blocks to r-1 / r+1, receive theirs (no wrap-around)."""
        import torch
        ops, recv = [], {}
        r, w = self.rank, self.world
        peers = [(p, blk) for p, blk in ((r - 1, to_prev), (r + 1, to_next)) if 0 <= p < w]
        counts = {}
        for p, blk in peers:  # sizes first
            cs = self._t(np.array([len(blk)], np.int64))
            cr = self._t(np.zeros(1, np.int64))
            ops.append(self.dist.isend(cs, p))
            ops.append(self.dist.irecv(cr, p))
            counts[p] = cr
        for o in ops:
            o.wait()
        ops = []
        for p, blk in peers:
            n_in = int(counts[p].cpu().item())
            if len(blk):
                ops.append(self.dist.isend(self._t(blk), p))
            buf = self._t(np.zeros((n_in, 12), np.float64))
            if n_in:
                ops.append(self.dist.irecv(buf, p))
            recv[p] = buf
        for o in ops:
            o.wait()
        got = [recv[p].cpu().numpy() if isinstance(recv[p], torch.Tensor) else recv[p] for p, _ in peers]
        return got

    # -- one iteration ------------------------------------------------------
    def step(self):
        st = self.state
        n = len(st["x"])
        b = np.array([np.inf] * 3 + [-np.inf] * 3 + [0.0])
        if n:
            b[:3] = [st["x"].min(), st["y"].min(), st["z"].min()]
            b[3:6] = [st["x"].max(), st["y"].max(), st["z"].max()]
            b[6] = st["d"].max()
        red = self._allreduce_max(np.concatenate([-b[:3], b[3:]]))
        bounds = np.concatenate([-red[:3], red[3:]])
        g = global_grid(bounds, self.fixed_box_length)
        L = layer_bounds(int(g.dims[2]), self.world)
        lay = box_layer(st["z"], g)
        lo_l, hi_l = L[self.rank], L[self.rank + 1]
        down, up = lay < lo_l, lay >= hi_l
        if self.rank > 0 and (lay < L[self.rank - 1]).any() or self.rank + 1 < self.world and (lay >= L[self.rank + 2]).any():
            raise RuntimeError("an agent moved more than one slab in one iteration")
        keep = ~(down | up)
        mig = self._exchange(pack(_take(st, down)), pack(_take(st, up)))
        owned = _concat([_take(st, keep)] + [unpack(m) for m in mig])
        lay = box_layer(owned["z"], g)
        bottom, top = lay == lo_l, lay == hi_l - 1
        halo = self._exchange(pack(_take(owned, bottom)), pack(_take(owned, top)))
        ghosts = [unpack(h) for h in halo if len(h)]
        for gh in ghosts:
            gh["flags"] = gh["flags"] | FLAG_GHOST
        n_owned = len(owned["x"])
        full = _concat([owned] + ghosts) if ghosts else owned
        origin_box, dims = g.as_override()
        self.e.load(full, self.uid_count, self.iteration)
        self.e.set_grid_override(origin_box, dims)
        c0 = self.e.counters()
        self.e.step()
        c1 = self.e.counters()
        out = self.e.dump()
        mine = (out["flags"] & FLAG_GHOST) == 0
        self.state = _take(out, np.nonzero(mine)[0])
        if len(self.state["x"]) != n_owned:
            raise RuntimeError("owned agent count changed inside a step")
        tot = self._allreduce_sum(np.array([c1[0] - c0[0], c1[1] - c0[1]], np.int64))
        self.evals += int(tot[0])
        self.skips += int(tot[1])
        self.iteration += 1
        return g

    def simulate(self, iterations: int):
        for _ in range(iterations):
            self.step()


class GpuRankEngine:
    """Rank engine over the B200 C ABI (one context per GPU)."""

    def __init__(self, params, device: int = 0):
        from .engine import Simulation
        if params.model == 1:
            raise NotImplementedError("agent additions across ranks need a global daughter-uid ranking")
        self.sim = Simulation(params, device=device)

    def load(self, st, uid_count, iteration):
        self.sim.add_agents(st["x"], st["y"], st["z"], st["d"], behaviour_mask=st["beh"], uid=st["uid"],
                            volume=st["volume"], flags=st["flags"], partners=st["partners"],
                            uid_count=uid_count)
        self.sim.set_iteration(iteration)

    def set_grid_override(self, grid, dims):
        self.sim.set_grid_override(grid, dims)

    def step(self):
        self.sim.simulate(1)

    def counters(self):
        r = self.sim.report()
        return r.force_evaluations, r.force_skips

    def dump(self):
        a = self.sim.agents()
        uid = a["uid"]
        a["beh"] = self._beh(uid)
        return a

    def _beh(self, uid):
        return np.zeros(len(uid), np.uint8) if self.beh_by_uid is None else self.beh_by_uid[uid.astype(np.int64)]

    beh_by_uid = None


def sir_grid(L: float, r: float) -> GlobalGrid:
    """Config 5's periodic grid, as abs_gpu_create builds it: D = max(3,
    floor(L / r)) boxes of L / D per axis, origin 0."""
    D = max(3, int(math.floor(L / r)))
    return GlobalGrid(np.zeros(3), L / D, r, np.array([D, D, D], np.int64))


def initial_partition(x, y, z, d, world: int, rank: int, fixed_box_length=0.0, mask=None, grid=None):
    """The owned slice of a population for `rank` (box layers of the initial
    grid, or of `grid` when given — e.g. the periodic grid of config 5)."""
    n = len(x)
    st = {"x": np.asarray(x, np.float64), "y": np.asarray(y, np.float64), "z": np.asarray(z, np.float64),
          "d": np.asarray(d, np.float64), "volume": np.zeros(n), "fx": np.zeros(n), "fy": np.zeros(n),
          "fz": np.zeros(n), "uid": np.arange(n, dtype=np.uint64), "flags": np.zeros(n, np.uint8),
          "partners": np.zeros(n, np.uint32),
          "beh": np.zeros(n, np.uint8) if mask is None else np.asarray(mask, np.uint8)}
    if grid is None:
        b = np.array([st["x"].min(), st["y"].min(), st["z"].min(), st["x"].max(), st["y"].max(),
                      st["z"].max(), st["d"].max()])
        g = global_grid(b, fixed_box_length)
    else:
        g = grid
    L = layer_bounds(int(g.dims[2]), world)
    lay = box_layer(st["z"], g)
    return _take(st, np.nonzero((lay >= L[rank]) & (lay < L[rank + 1]))[0])


class DeviceSlabDecomposition:
    """The same decomposition with a device-resident population: agents stay
    in the rank's HBM; per iteration only the 7-double bounds, migrants and
    the two boundary layers (packed 96-byte records, ABS_RECORD_BYTES) move.
    transport="nccl": CUDA tensors straight through torch.distributed (NCCL
    over NVLink); transport="host": staged through host tensors (gloo) — used
    to test several ranks sharing one GPU."""

    RECORD = 96

    def __init__(self, sim, dist, rank: int, world: int, fixed_box_length: float = 0.0,
                 transport: str = "nccl", cap: int = 1 << 20):
        import torch
        self.sim, self.dist, self.rank, self.world = sim, dist, rank, world
        self.fixed_box_length = fixed_box_length
        self.transport = transport
        self.torch = torch
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self._alloc(cap)
        self._r0 = sim.report()
        self.iteration = 0
        # additions (config 2): daughters are committed only after the ranks
        # have summed their division marks, so uids match the single domain
        from ._native import MODEL_GROW_DIVIDE, MODEL_PROLIFERATION, MODEL_SIR
        self.additions = sim.params.model in (MODEL_PROLIFERATION, MODEL_GROW_DIVIDE)
        self._marks = None
        if self.additions:
            sim.set_defer_commit(True)
        # config 5: the periodic cube's fixed grid (abs_gpu_create: box L / D,
        # D = max(3, floor(L / r))); slabs form a ring of z layers
        self.periodic = sim.params.model == MODEL_SIR
        if self.periodic:
            self._fixed = sir_grid(float(sim.params.model_params[0]), float(sim.params.model_params[1]))
        # NCCL: the first P2P batch must not be a communicator's first call
        self.dist.barrier()

    def _alloc(self, cap):
        t = self.torch
        self.cap = cap
        self.buf = {k: t.empty(cap * self.RECORD, dtype=t.uint8, device=self.dev)
                    for k in ("send_lo", "send_hi", "recv_lo", "recv_hi")}

    # -- collectives -----------------------------------------------------------
    def _coll_tensor(self, a):
        t = self.torch.from_numpy(np.ascontiguousarray(a))
        return t.to(self.dev) if self.transport == "nccl" else t

    def _allreduce(self, a, op):
        t = self._coll_tensor(a)
        self.dist.all_reduce(t, op=op)
        return t.cpu().numpy()

    def _peers(self):
        """(lo peer, hi peer); None at an open slab end. Periodic: a ring."""
        r, w = self.rank, self.world
        if w == 1:
            return None, None
        if self.periodic:
            return (r - 1) % w, (r + 1) % w
        return (r - 1 if r > 0 else None), (r + 1 if r < w - 1 else None)

    def _p2p(self, sends, recvs):
        """One batched round of point-to-point transfers (a single NCCL group,
        so paired sends/receives cannot deadlock). sends/recvs: lists of
        (tensor, peer, tag). Messages to one peer are posted lo-side first and
        received hi-side first on every rank, so at world 2 on a ring (both
        peers the same rank) the in-order matching of NCCL pairs each message
        with the right buffer; the tags do the same for gloo."""
        d = self.dist
        ops = [d.P2POp(d.isend, t, p, tag=tag) for t, p, tag in sends]
        ops += [d.P2POp(d.irecv, t, p, tag=tag) for t, p, tag in recvs]
        if ops:
            for w in d.batch_isend_irecv(ops):
                w.wait()

    def _exchange(self, n_lo: int, n_hi: int):
        """Send send_lo[:n_lo] to the lo peer and send_hi[:n_hi] to the hi peer;
        returns the received record counts (from lo peer, from hi peer) into
        recv_lo / recv_hi. Tag 1: travels to the receiver's hi side, tag 0: to
        its lo side."""
        t = self.torch
        lo_p, hi_p = self._peers()
        sends, recvs, cnt = [], [], {}
        if lo_p is not None:
            sends.append((self._coll_tensor(np.array([n_lo], np.int64)), lo_p, 1))
        if hi_p is not None:
            sends.append((self._coll_tensor(np.array([n_hi], np.int64)), hi_p, 0))
        if hi_p is not None:
            cnt["hi"] = self._coll_tensor(np.zeros(1, np.int64))
            recvs.append((cnt["hi"], hi_p, 1))
        if lo_p is not None:
            cnt["lo"] = self._coll_tensor(np.zeros(1, np.int64))
            recvs.append((cnt["lo"], lo_p, 0))
        self._p2p(sends, recvs)
        got = {k: int(v.cpu().item()) for k, v in cnt.items()}
        need = max([n_lo if lo_p is not None else 0, n_hi if hi_p is not None else 0] + list(got.values()) + [0])
        if need > self.cap:
            raise RuntimeError("halo larger than the exchange buffers")
        staged = []

        def buf(key, nbytes, incoming):
            if self.transport == "nccl":
                return self.buf[key][:nbytes]
            if not incoming:
                return self.buf[key][:nbytes].cpu()
            host = t.empty(nbytes, dtype=t.uint8)
            staged.append((key, host))
            return host
        sends, recvs = [], []
        if lo_p is not None and n_lo:
            sends.append((buf("send_lo", n_lo * self.RECORD, False), lo_p, 1))
        if hi_p is not None and n_hi:
            sends.append((buf("send_hi", n_hi * self.RECORD, False), hi_p, 0))
        if got.get("hi", 0):
            recvs.append((buf("recv_hi", got["hi"] * self.RECORD, True), hi_p, 1))
        if got.get("lo", 0):
            recvs.append((buf("recv_lo", got["lo"] * self.RECORD, True), lo_p, 0))
        self._p2p(sends, recvs)
        for key, host in staged:
            self.buf[key][:host.numel()].copy_(host.to(self.dev))
        # the engine consumes the buffers on its own CUDA stream: make the
        # received bytes (NCCL / staging copies on torch's stream) visible first
        t.cuda.current_stream().synchronize()
        return got.get("lo", 0), got.get("hi", 0)

    # -- one iteration -------------------------------------------------------------
    def _export(self, g, lo, hi, mode):
        from . import _native as N
        import ctypes as C
        if self.periodic:
            mode |= 2
        grid, dims = g.as_override()
        grid = np.ascontiguousarray(grid)
        dims = np.ascontiguousarray(dims, np.uint32)
        a, b = C.c_uint64(0), C.c_uint64(0)
        rc = N.load().abs_gpu_export_layers(self.sim._ctx, grid.ctypes.data_as(C.POINTER(C.c_double)),
                                            dims.ctypes.data_as(C.POINTER(C.c_uint32)), int(lo), int(hi), mode,
                                            self.buf["send_lo"].data_ptr(), self.buf["send_hi"].data_ptr(),
                                            self.cap, C.byref(a), C.byref(b))
        N.check(rc, self.sim._ctx)
        return int(a.value), int(b.value)

    def _import(self, key, count, ghost):
        from . import _native as N
        if count:
            N.check(N.load().abs_gpu_import(self.sim._ctx, self.buf[key].data_ptr(), count, 1 if ghost else 0),
                    self.sim._ctx)

    def step(self):
        from . import _native as N
        if self.periodic:  # fixed grid, already forced at context creation
            g = self._fixed
        else:
            b = self.sim.local_bounds()
            red = self._allreduce(np.concatenate([-b[:3], b[3:]]), self.dist.ReduceOp.MAX)
            g = global_grid(np.concatenate([-red[:3], red[3:]]), self.fixed_box_length)
        L = layer_bounds(int(g.dims[2]), self.world)
        lo, hi = L[self.rank], L[self.rank + 1]
        n_lo, n_hi = self._export(g, lo, hi, 0)            # migrants leave
        got_lo, got_hi = self._exchange(n_lo, n_hi)
        self._import("recv_lo", got_lo, False)
        self._import("recv_hi", got_hi, False)
        n_lo, n_hi = self._export(g, lo, hi, 1)            # boundary layers
        got_lo, got_hi = self._exchange(n_lo, n_hi)
        self._import("recv_lo", got_lo, True)
        self._import("recv_hi", got_hi, True)
        if not self.periodic:
            grid, dims = g.as_override()
            self.sim.set_grid_override(grid, dims)
        self.sim.simulate(1)
        if self.additions:
            self._commit_additions()
        N.check(N.load().abs_gpu_drop_ghosts(self.sim._ctx), self.sim._ctx)
        self.iteration += 1
        return g

    def _commit_additions(self):
        """Sum the ranks' uid-indexed division marks (every uid divides on at
        most one rank) and commit: daughter uid = uid_count + rank of the
        parent among all dividers (commit.cpp:186-222)."""
        t = self.torch
        length = self.sim.division_marks()  # uid_count: identical on every rank
        if self._marks is None or self._marks.numel() < max(length, 1):
            self._marks = t.zeros(max(int(length * 1.5), 1024), dtype=t.int32, device=self.dev)
        self.sim.division_marks(self._marks.data_ptr(), self._marks.numel())
        view = self._marks[:length]
        if self.transport == "nccl":
            self.dist.all_reduce(view, op=self.dist.ReduceOp.SUM)
        else:
            host = view.cpu()
            self.dist.all_reduce(host, op=self.dist.ReduceOp.SUM)
            view.copy_(host.to(self.dev))
        t.cuda.current_stream().synchronize()  # the engine reads the sum on its own stream
        self.sim.commit(view.data_ptr(), length)

    def sir_counts(self):
        """Config 5: S/I/R over all ranks after the last iteration."""
        c = self._allreduce(np.array(self.sim.sir_counts(), np.int64), self.dist.ReduceOp.SUM)
        return [int(v) for v in c]

    def totals(self):
        """Force evaluations and static skips summed over ranks since this
        decomposition was created (one all-reduce; ghosts never count)."""
        r = self.sim.report()
        tot = self._allreduce(np.array([r.force_evaluations - self._r0.force_evaluations,
                                        r.force_skips - self._r0.force_skips], np.int64), self.dist.ReduceOp.SUM)
        return int(tot[0]), int(tot[1])

    def simulate(self, iterations: int):
        for _ in range(iterations):
            self.step()
