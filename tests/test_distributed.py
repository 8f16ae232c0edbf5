"""CPU, world_size 2/3 over gloo: the slab decomposition
(paper_2301_06984_b200/distributed.py) with the C oracle as each rank's
engine reproduces the single-domain run: same evals/skips totals, same
per-uid flags and partners, positions within 1e-9."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from _util import assert_close, by_uid
from paper_2301_06984_b200 import configs as CF
from paper_2301_06984_b200 import distributed as D


class OracleRankEngine:
    def __init__(self, O, params, beh_by_uid):
        self.sim = O.PortSim(params, np.zeros(1), np.zeros(1), np.zeros(1), np.ones(1))
        self.beh_by_uid = beh_by_uid

    def load(self, st, uid_count, iteration):
        self.sim.load(st, uid_count, iteration)

    def set_grid_override(self, grid, dims):
        self.sim.set_grid_override(grid, dims)

    def step(self):
        self.sim.simulate(1)

    def counters(self):
        c = self.sim.counts()
        return c["force_evaluations"], c["force_skips"]

    def dump(self):
        d = self.sim.dump()
        d["beh"] = self.beh_by_uid[d["uid"].astype(np.int64)]
        return d


def _oparams(O, wl):
    prm = wl.params
    return O.OracleParams(seed=prm.get("seed", 42), dt=prm.get("simulation_time_step", 0.1),
                          detect_static=prm.get("detect_static_agents", False),
                          model=prm.get("model", 0), mp=prm.get("model_params", [0.0] * 8))


def _make(case):
    if case == "c1":
        return CF.c1_relaxation(3000, seed=1), 6
    if case == "c2":
        return CF.c2_proliferation(side=6, seed=0), 50
    if case == "c5":
        return CF.c5_sir(4000, seed=1), 26
    if case == "gd":  # the reference's own GrowDivide lattice
        return CF.ref_proliferation(343), 12
    if case == "c3":
        return CF.c3_spheroid(3000, seed=2), 5
    return CF.c4_large_uniform(3000, seed=3), 4


def _worker(rank, world, port, case, outdir):
    import torch.distributed as dist
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl, steps = _make(case)
    mask = wl.mask if wl.mask is not None else np.zeros(wl.n, np.uint8)
    beh = mask.astype(np.uint8) if wl.params.get("model", 0) else np.zeros(wl.n, np.uint8)
    st = D.initial_partition(wl.x, wl.y, wl.z, wl.d, world, rank, mask=beh)
    eng = OracleRankEngine(O, _oparams(O, wl), beh)
    dec = D.SlabDecomposition(eng, dist, rank, world, st, uid_count=wl.n)
    dec.simulate(steps)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), evals=dec.evals, skips=dec.skips, **dec.state)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,case", [(2, "c1"), (3, "c1"), (2, "c3"), (3, "c4")])
def test_slab_decomposition_matches_single_domain(oracle_mod, world, case):
    O = oracle_mod
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _free_port(), case, tmp), nprocs=world, join=True)
        parts = [dict(np.load(os.path.join(tmp, f"r{r}.npz"))) for r in range(world)]
    evals = int(parts[0]["evals"])
    skips = int(parts[0]["skips"])
    assert all(int(p["evals"]) == evals for p in parts)
    keys = ["uid", "x", "y", "z", "d", "fx", "fy", "fz", "partners", "flags"]
    got = by_uid({k: np.concatenate([p[k] for p in parts]) for k in keys})
    assert all(len(p["uid"]) > 0 for p in parts), "a rank owned nothing"

    wl, steps = _make(case)
    ref = O.PortSim(_oparams(O, wl), wl.x, wl.y, wl.z, wl.d, wl.mask)
    if wl.tags is not None:
        ref.set_tags(wl.tags)
        ref.set_rng_counters(wl.rng_counters)
    ref.simulate(steps)
    o = by_uid(ref.dump())
    if wl.tags is not None:  # tags and RandomStream counters travel with the agents
        ge = by_uid({"uid": np.concatenate([p["uid"] for p in parts]),
                     "tag": np.concatenate([p["tag"] for p in parts]),
                     "rngc": np.concatenate([p["rngc"] for p in parts])})
        oe = by_uid({"uid": ref.dump()["uid"], "tag": ref.tags(), "rngc": ref.rng_counters()})
        assert np.array_equal(ge["tag"], oe["tag"]) and np.array_equal(ge["rngc"], oe["rngc"])
    assert np.array_equal(got["uid"], o["uid"])
    for k in ("x", "y", "z", "d"):
        assert_close(got[k], o[k], 1e-9, 1.0, k)
    for k in ("fx", "fy", "fz"):
        assert_close(got[k], o[k], 1e-9, 2.0, k)
    assert np.array_equal(got["partners"], o["partners"])
    assert np.array_equal(got["flags"], o["flags"])
    c = ref.counts()
    assert (evals, skips) == (c["force_evaluations"], c["force_skips"])


def test_balanced_slab_edges():
    """Equal-count edges (decomp.cuh k_layer_bounds mirror): a dense middle
    (the c3 spheroid's profile) gets thin slabs, the ends thick ones, and no
    slab is thinner than 2 layers."""
    prof = np.array([1] * 20 + [50] * 20 + [1] * 20)
    lb = D.balanced_bounds(prof, 4)
    assert lb[0] == 0 and lb[-1] == 60 and (np.diff(lb) >= 2).all()
    share = [prof[lb[r]:lb[r + 1]].sum() for r in range(4)]
    assert max(share) <= 1.25 * sum(share) / 4  # one 50-agent layer is 19 % of a share
    assert list(D.balanced_bounds(np.zeros(12, np.int64), 4)) == [0, 3, 6, 9, 12]
    with pytest.raises(RuntimeError):
        D.balanced_bounds(np.ones(5), 3)
    # c3 at 8 ranks: equal-count slabs keep the largest share within 5 % of the mean
    wl = CF.c3_spheroid(60000, seed=0)
    b = np.array([wl.x.min(), wl.y.min(), wl.z.min(), wl.x.max(), wl.y.max(), wl.z.max(), wl.d.max()])
    g = D.global_grid(b)
    counts = np.bincount(D.box_layer(wl.z, g), minlength=int(g.dims[2]))
    lb = D.balanced_bounds(counts, 8)
    share = np.array([counts[lb[r]:lb[r + 1]].sum() for r in range(8)])
    eq = D.layer_bounds(int(g.dims[2]), 8)
    share_eq = np.array([counts[eq[r]:eq[r + 1]].sum() for r in range(8)])
    assert share.max() / share.mean() < share_eq.max() / share_eq.mean()


def test_grid_and_layers_helpers():
    b = np.array([0.0, 0.0, 0.0, 100.0, 50.0, 95.0, 10.0])
    g = D.global_grid(b)
    assert list(g.dims) == [11, 6, 10] and g.box == 10.0
    assert list(D.layer_bounds(10, 3)) == [0, 3, 6, 10]
    assert list(D.box_layer(np.array([0.0, 9.99, 10.0, 95.0]), g)) == [0, 0, 1, 9]
    st = D._empty_state()
    rec = D.pack(st)
    assert rec.shape == (0, 12)
    with pytest.raises(RuntimeError, match="fixed box"):
        D.global_grid(b, fixed_box_length=5.0)


def _gpu_worker(rank, world, port, case, outdir):
    import torch.distributed as dist

    import paper_2301_06984_b200 as E
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl, steps = _make(case)
    mask = wl.mask if wl.mask is not None else np.zeros(wl.n, np.uint8)
    beh = mask.astype(np.uint8) if wl.params.get("model", 0) else np.zeros(wl.n, np.uint8)
    st = D.initial_partition(wl.x, wl.y, wl.z, wl.d, world, rank, mask=beh)
    eng = D.GpuRankEngine(E.SimulationParams(**wl.params), device=0)
    eng.beh_by_uid = beh
    dec = D.SlabDecomposition(eng, dist, rank, world, st, uid_count=wl.n)
    dec.simulate(steps)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), evals=dec.evals, skips=dec.skips, **dec.state)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,case", [(2, "c1"), (2, "c3")])
def test_gpu_ranks_match_single_domain(oracle_mod, world, case):
    """Two processes, one GPU each (here both on device 0): the B200 engine
    with ghost halo + global grid override reproduces the single-domain run."""
    O = oracle_mod
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_gpu_worker, args=(world, _free_port(), case, tmp), nprocs=world, join=True)
        parts = [dict(np.load(os.path.join(tmp, f"r{r}.npz"))) for r in range(world)]
    keys = ["uid", "x", "y", "z", "d", "fx", "fy", "fz", "partners", "flags"]
    got = by_uid({k: np.concatenate([p[k] for p in parts]) for k in keys})
    wl, steps = _make(case)
    ref = O.PortSim(_oparams(O, wl), wl.x, wl.y, wl.z, wl.d, wl.mask)
    ref.simulate(steps)
    o = by_uid(ref.dump())
    assert np.array_equal(got["uid"], o["uid"])
    for k in ("x", "y", "z", "d"):
        assert_close(got[k], o[k], 1e-9, 1.0, k)
    assert np.array_equal(got["partners"], o["partners"])
    assert np.array_equal(got["flags"], o["flags"])
    c = ref.counts()
    assert (int(parts[0]["evals"]), int(parts[0]["skips"])) == (c["force_evaluations"], c["force_skips"])
    if case == "c5":  # SIR on the periodic ring: states and counts bit-exact
        gs = by_uid({"uid": got["uid"], "state": np.concatenate([p["state"] for p in parts]),
                     "t": np.concatenate([p["t"] for p in parts])})
        os_, ot = ref.sir_state()
        od = by_uid({"uid": ref.dump()["uid"], "state": os_, "t": ot})
        assert np.array_equal(gs["state"], od["state"]) and np.array_equal(gs["t"], od["t"])
        assert list(parts[0]["sir"]) == list(ref.sir_counts())
        assert ref.sir_counts()[1] + ref.sir_counts()[2] > 40  # the epidemic spread


def _dev_worker(rank, world, port, case, outdir):
    import torch
    import torch.distributed as dist

    import paper_2301_06984_b200 as E
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    wl, steps = _make(case)
    sir = wl.params.get("model") == E.MODEL_SIR
    mask = wl.mask if wl.mask is not None else np.ones(wl.n, np.uint8)  # None = behaviour on every agent
    grid = D.sir_grid(wl.params["model_params"][0], wl.params["model_params"][1]) if sir else None
    st = D.initial_partition(wl.x, wl.y, wl.z, wl.d, world, rank, mask=mask, grid=grid, balanced=True)
    sim = E.Simulation(E.SimulationParams(**wl.params), device=0)
    sim.add_agents(st["x"], st["y"], st["z"], st["d"], behaviour_mask=None if sir else st["beh"], uid=st["uid"],
                   uid_count=wl.n)  # SIR: initial states from (seed, uid), as in one domain
    if wl.tags is not None:
        sim.set_agent_ext(wl.tags[st["uid"]], wl.rng_counters[st["uid"]])
    dec = D.DeviceSlabDecomposition(sim, dist, rank, world, transport="host", cap=1 << 14)
    dec.simulate(steps)
    a = sim.agents()
    evals, skips = dec.totals()
    extra = {}
    extra["tag"], extra["rngc"] = sim.agent_ext()
    if dec.periodic:
        extra["state"], extra["t"] = sim.sir_state()
        extra["sir"] = np.array(dec.sir_counts())
    np.savez(os.path.join(outdir, f"r{rank}.npz"), evals=evals, skips=skips, **a, **extra)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,case", [(2, "c1"), (3, "c4"), (2, "c3"), (2, "c2"), (3, "c2"), (2, "c5"),
                                        (3, "c5"), (2, "gd")])
def test_device_exchange_matches_single_domain(oracle_mod, world, case):
    """Device-resident exchange (export/import kernels, packed records): the
    union of the ranks' populations equals the single-domain run."""
    O = oracle_mod
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_dev_worker, args=(world, _free_port(), case, tmp), nprocs=world, join=True)
        parts = [dict(np.load(os.path.join(tmp, f"r{r}.npz"))) for r in range(world)]
    keys = ["uid", "x", "y", "z", "d", "volume", "partners", "flags"]
    got = by_uid({k: np.concatenate([p[k] for p in parts]) for k in keys})
    wl, steps = _make(case)
    ref = O.PortSim(_oparams(O, wl), wl.x, wl.y, wl.z, wl.d, wl.mask)
    ref.simulate(steps)
    o = by_uid(ref.dump())
    assert np.array_equal(got["uid"], o["uid"])
    for k in ("x", "y", "z", "d", "volume"):
        assert_close(got[k], o[k], 1e-9, 1.0, k)
    assert np.array_equal(got["partners"], o["partners"])
    assert np.array_equal(got["flags"], o["flags"])
    c = ref.counts()
    assert (int(parts[0]["evals"]), int(parts[0]["skips"])) == (c["force_evaluations"], c["force_skips"])
