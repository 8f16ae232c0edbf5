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


HIST_BINS, MIN_LAYERS = 4096, 2  # decomp.cuh kHistBins / kMinLayers


def balanced_bounds(layer_counts: np.ndarray, world: int, min_layers: int = MIN_LAYERS) -> np.ndarray:
    """Slab edges with equal agent counts (the host mirror of decomp.cuh's
    k_layer_bounds, integer for integer): layers coarsened into <= 4096 bins,
    edge r = first bin edge whose prefix exceeds r * total / world, every
    slab >= min_layers layers (the analogue of sort_balance.cpp:61-77)."""
    D = len(layer_counts)
    if D < world * min_layers:
        raise RuntimeError("fewer than 2 z box layers per rank")
    cz = (D + HIST_BINS - 1) // HIST_BINS
    nb = (D + cz - 1) // cz
    hist = np.zeros(nb, np.int64)
    np.add.at(hist, np.arange(D) // cz, np.asarray(layer_counts, np.int64))
    total = int(hist.sum())
    lb = np.zeros(world + 1, np.int64)
    lb[world] = D
    run, b = 0, 0
    for r in range(1, world):
        target = (total * r) // world
        while b < nb and run + int(hist[b]) <= target:
            run += int(hist[b])
            b += 1
        e = b * cz if total else (D * r) // world
        lo_ok = int(lb[r - 1]) + min_layers
        hi_ok = D - (world - r) * min_layers
        lb[r] = min(max(e, lo_ok), hi_ok)
    return lb


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


def initial_partition(x, y, z, d, world: int, rank: int, fixed_box_length=0.0, mask=None, grid=None,
                      balanced=False):
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
    lay = box_layer(st["z"], g)
    if balanced:  # the device driver's equal-count edges (DeviceSlabDecomposition)
        L = balanced_bounds(np.bincount(lay, minlength=int(g.dims[2])), world)
    else:
        L = layer_bounds(int(g.dims[2]), world)
    return _take(st, np.nonzero((lay >= L[rank]) & (lay < L[rank + 1]))[0])


class DeviceSlabDecomposition:
    """The library's own slab decomposition (csrc/decomp.cuh,
    abs_gpu_simulate_decomposed): agents stay in the rank's HBM; per
    iteration a device all-reduce of the bounds gives the single-domain grid,
    an all-reduced z-layer histogram gives equal-count slab edges
    (balanced_bounds), and one export pass + one exchange move emigrants
    (owned records) and boundary layers (ghosts, ABS_RECORD_BYTES each).
    transport="nccl": the library's NCCL communicator (abs_gpu_comm_init; rank
    0 draws the unique id, torch.distributed shares it). transport="host": the
    same driver with collectives supplied here through torch.distributed
    (gloo, staged through host memory) — used to test several ranks sharing
    one GPU."""

    RECORD = 96

    def __init__(self, sim, dist, rank: int, world: int, fixed_box_length: float = 0.0,
                 transport: str = "nccl", cap: int = 1 << 20):
        import ctypes as C

        import torch

        from . import _native as N
        self.sim, self.dist, self.rank, self.world = sim, dist, rank, world
        self.transport = transport
        self.torch = torch
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self._r0 = sim.report()
        self.iteration = 0
        from ._native import MODEL_SIR
        self.periodic = sim.params.model == MODEL_SIR
        if fixed_box_length != sim.params.fixed_box_length:
            raise ValueError("fixed_box_length is the context's (SimulationParams.fixed_box_length)")
        lib = N.load()
        if transport == "nccl":
            uid = torch.zeros(128, dtype=torch.uint8)
            if rank == 0:
                N.check(lib.abs_gpu_nccl_unique_id(uid.data_ptr()))
            box = uid.to(self.dev) if dist.get_backend() == "nccl" else uid
            dist.broadcast(box, 0)
            uid = box.cpu()
            N.check(lib.abs_gpu_comm_init(sim._ctx, uid.data_ptr(), rank, world), sim._ctx)
        else:
            self._tr = N.Transport(None, N.ALLREDUCE_FN(self._cb_allreduce), N.COUNTS_FN(self._cb_counts),
                                   N.RECORDS_FN(self._cb_records))
            N.check(lib.abs_gpu_comm_set_transport(sim._ctx, C.byref(self._tr), rank, world), sim._ctx)
        N.check(lib.abs_gpu_comm_reserve(sim._ctx, cap), sim._ctx)
        self.dist.barrier()

    # -- host transport (torch.distributed, staged through host memory) ------------
    def _peers(self):
        r, w = self.rank, self.world
        if w == 1:
            return None, None
        if self.periodic:
            return (r - 1) % w, (r + 1) % w
        return (r - 1 if r > 0 else None), (r + 1 if r < w - 1 else None)

    def _copy(self, dst, src, nbytes, stream):
        from . import _native as N
        return N.load().abs_gpu_memcpy(dst, src, nbytes, stream)

    def _cb_allreduce(self, user, dev, count, dtype, stream):
        try:
            t = self.torch
            from . import _native as N
            dt = {N.DT_F64_MAX: t.float64, N.DT_U64_SUM: t.int64, N.DT_U32_SUM: t.int32}[dtype]
            host = t.empty(count, dtype=dt)
            nbytes = count * host.element_size()
            if self._copy(host.data_ptr(), dev, nbytes, stream):
                return 1
            self.dist.all_reduce(host, op=self.dist.ReduceOp.MAX if dtype == N.DT_F64_MAX else self.dist.ReduceOp.SUM)
            return 1 if self._copy(dev, host.data_ptr(), nbytes, stream) else 0
        except Exception:  # a callback must not raise through C
            import traceback
            traceback.print_exc()
            return 1

    def _p2p(self, sends, recvs):
        """One batched round (paired sends/receives cannot deadlock). Messages
        to one peer are posted lo-side first and received hi-side first, with
        direction tags, so a two-rank ring (both peers the same rank) matches."""
        d = self.dist
        ops = [d.P2POp(d.isend, t, p, tag=tag) for t, p, tag in sends]
        ops += [d.P2POp(d.irecv, t, p, tag=tag) for t, p, tag in recvs]
        if ops:
            for w in d.batch_isend_irecv(ops):
                w.wait()

    def _cb_counts(self, user, n_lo, n_hi, got_lo, got_hi, stream):
        try:
            t = self.torch
            lo_p, hi_p = self._peers()
            sends, recvs, cnt = [], [], {}
            if lo_p is not None:
                sends.append((t.tensor([n_lo], dtype=t.int64), lo_p, 1))
            if hi_p is not None:
                sends.append((t.tensor([n_hi], dtype=t.int64), hi_p, 0))
            if hi_p is not None:
                cnt["hi"] = t.zeros(1, dtype=t.int64)
                recvs.append((cnt["hi"], hi_p, 1))
            if lo_p is not None:
                cnt["lo"] = t.zeros(1, dtype=t.int64)
                recvs.append((cnt["lo"], lo_p, 0))
            self._p2p(sends, recvs)
            got_lo[0] = int(cnt["lo"].item()) if "lo" in cnt else 0
            got_hi[0] = int(cnt["hi"].item()) if "hi" in cnt else 0
            return 0
        except Exception:
            import traceback
            traceback.print_exc()
            return 1

    def _cb_records(self, user, send_lo, n_lo, send_hi, n_hi, recv_lo, got_lo, recv_hi, got_hi, stream):
        try:
            t = self.torch
            R = self.RECORD
            lo_p, hi_p = self._peers()
            sends, recvs, land = [], [], []
            for ptr, cnt_, peer, tag in ((send_lo, n_lo, lo_p, 1), (send_hi, n_hi, hi_p, 0)):
                if peer is not None and cnt_:
                    host = t.empty(cnt_ * R, dtype=t.uint8)
                    if self._copy(host.data_ptr(), ptr, cnt_ * R, stream):
                        return 1
                    sends.append((host, peer, tag))
            for ptr, cnt_, peer, tag in ((recv_hi, got_hi, hi_p, 1), (recv_lo, got_lo, lo_p, 0)):
                if peer is not None and cnt_:
                    host = t.empty(cnt_ * R, dtype=t.uint8)
                    recvs.append((host, peer, tag))
                    land.append((ptr, host))
            self._p2p(sends, recvs)
            for ptr, host in land:
                if self._copy(ptr, host.data_ptr(), host.numel(), stream):
                    return 1
            return 0
        except Exception:
            import traceback
            traceback.print_exc()
            return 1

    # -- driving ---------------------------------------------------------------------
    def simulate(self, iterations: int):
        from . import _native as N
        N.check(N.load().abs_gpu_simulate_decomposed(self.sim._ctx, iterations), self.sim._ctx)
        self.iteration += iterations

    def step(self):
        self.simulate(1)

    def info(self):
        """(slab edges of the last iteration as z-layers, owned agents)."""
        import ctypes as C

        from . import _native as N
        lb = (C.c_int64 * (self.world + 1))()
        owned = C.c_uint64(0)
        N.check(N.load().abs_gpu_decomp_info(self.sim._ctx, lb, C.byref(owned)), self.sim._ctx)
        return np.array(lb[:], np.int64), int(owned.value)

    def _allreduce(self, a, op):
        t = self.torch.from_numpy(np.ascontiguousarray(a))
        if self.dist.get_backend() == "nccl":
            t = t.to(self.dev)
        self.dist.all_reduce(t, op=op)
        return t.cpu().numpy()

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
