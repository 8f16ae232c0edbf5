"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle on
identical seeded inputs.

Bars: bit-exact for grid params, cell ids, neighbour sets
(sorted uid lists), static flags, partners and agent counts; fp64 positions
within |g-o| <= 1e-9 max(|o|, 1) and forces within 1e-9 max(|o|, k) per
component. Integer outputs are also checked teacher-forced (both sides fed
the oracle's step-t state) so a 1-ulp drift in free-running positions cannot
flip a floor() or <= decision.
"""
import math

import numpy as np
import pytest

from _util import assert_close, by_uid, contact_cases
from paper_2301_06984_b200 import configs as CF

pytestmark = pytest.mark.gpu

K = 2.0


def _oparams(O, prm, **kw):
    p = O.OracleParams(seed=prm.get("seed", 42), dt=prm.get("simulation_time_step", 0.1),
                       detect_static=prm.get("detect_static_agents", False),
                       model=prm.get("model", 0), mp=prm.get("model_params", [0.0] * 8),
                       sorting_frequency=prm.get("sorting_frequency", 0),
                       threshold=prm.get("force_threshold", 0.0),
                       fixed_box=prm.get("fixed_box_length", 0.0))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def _gpu(E, prm, wl=None, bins=1, **kw):
    p = E.SimulationParams(**{**prm, **kw})
    p.bins_per_box = bins
    sim = E.Simulation(p)
    if wl is not None:
        sim.add_agents(wl.x, wl.y, wl.z, wl.d, behaviour_mask=wl.mask)
    return sim


def compare_state(g, o, ints=True, what=""):
    g, o = by_uid(g), by_uid(o)
    assert np.array_equal(g["uid"], o["uid"]), f"{what}: uid sets differ"
    for k in ("x", "y", "z", "d", "volume"):
        assert_close(g[k], o[k], 1e-9, 1.0, f"{what} {k}")
    for k in ("fx", "fy", "fz"):
        assert_close(g[k], o[k], 1e-9, K, f"{what} {k}")
    if ints:
        assert np.array_equal(g["partners"], o["partners"]), f"{what}: partners"
        assert np.array_equal(g["flags"], o["flags"]), f"{what}: flags"


def compare_env(sim, orc, what=""):
    env = sim.environment()
    env.update()
    og = orc.env_update()
    assert np.array_equal(env.origin(), og["origin"]), what
    assert env.box_length() == og["box"] and env.largest_agent_diameter() == og["dmax"], what
    assert np.array_equal(env.dims(), og["dims"]), what
    ga = sim.agents()
    gid = dict(zip(ga["uid"].tolist(), env.cell_ids().tolist()))
    od = orc.dump()
    oid = dict(zip(od["uid"].tolist(), orc.cell_ids().tolist()))
    assert gid == oid, f"{what}: cell ids"
    go, gu = env.neighbors()
    oo, ou = orc.neighbors()
    gn = {int(u): tuple(gu[go[i]:go[i + 1]].tolist()) for i, u in enumerate(ga["uid"])}
    on = {int(u): tuple(ou[oo[i]:oo[i + 1]].tolist()) for i, u in enumerate(od["uid"])}
    assert gn == on, f"{what}: neighbour sets"


def teacher_force(sim, orc, mask_by_uid=None):
    """Upload the oracle's current state into the GPU context."""
    o = orc.dump()
    c = orc.counts()
    m = None if mask_by_uid is None else mask_by_uid(o["uid"])
    sim.add_agents(o["x"], o["y"], o["z"], o["d"], behaviour_mask=m, uid=o["uid"], volume=o["volume"],
                   flags=o["flags"], partners=o["partners"], uid_count=c["uid_count"])
    sim.set_iteration(c["iterations"])


# ---------------------------------------------------------------- configs
@pytest.mark.parametrize("bins", [1, 2])
def test_c1_free_running(engine, oracle_mod, bins):
    wl = CF.c1_relaxation(4096, seed=0)
    sim = _gpu(engine, wl.params, wl, bins)
    orc = oracle_mod.PortSim(_oparams(oracle_mod, wl.params), wl.x, wl.y, wl.z, wl.d)
    compare_env(sim, orc, "c1 t=0")
    for step in range(3):
        sim.simulate(4)
        orc.simulate(4)
        compare_state(sim.agents(), orc.dump(), what=f"c1 after {4 * (step + 1)}")
        r, c = sim.report(), orc.counts()
        assert r.force_evaluations == c["force_evaluations"]
        assert r.final_agent_count == c["agents"]


def test_c1_teacher_forced_integers(engine, oracle_mod):
    wl = CF.c1_relaxation(3000, seed=5)
    sim = _gpu(engine, wl.params, wl, 2)
    orc = oracle_mod.PortSim(_oparams(oracle_mod, wl.params), wl.x, wl.y, wl.z, wl.d)
    for step in range(8):
        teacher_force(sim, orc)
        compare_env(sim, orc, f"c1 tf step {step}")
        e0 = orc.counts()["force_evaluations"]
        sim.simulate(1)
        orc.simulate(1)
        compare_state(sim.agents(), orc.dump(), what=f"c1 tf step {step}")
        assert sim.report().force_evaluations == orc.counts()["force_evaluations"] - e0


def test_c2_proliferation(engine, oracle_mod):
    wl = CF.c2_proliferation(side=4, seed=0)
    sim = _gpu(engine, wl.params, wl, 1)
    orc = oracle_mod.PortSim(_oparams(oracle_mod, wl.params), wl.x, wl.y, wl.z, wl.d)
    for chunk in range(6):
        sim.simulate(10)
        orc.simulate(10)
        r, c = sim.report(), orc.counts()
        assert r.final_agent_count == c["agents"] and r.uid_count == c["uid_count"]
        assert r.agents_added == c["agents_added"]
        compare_state(sim.agents(), orc.dump(), what=f"c2 after {10 * (chunk + 1)}")
    assert sim.report().final_agent_count == 64 * 4  # two synchronous doublings by step 60


def test_c3_static_spheroid(engine, oracle_mod):
    wl = CF.c3_spheroid(4000, seed=0)
    sim = _gpu(engine, wl.params, wl, 1)
    orc = oracle_mod.PortSim(_oparams(oracle_mod, wl.params), wl.x, wl.y, wl.z, wl.d, wl.mask)
    for chunk in range(3):
        sim.simulate(3)
        orc.simulate(3)
        r, c = sim.report(), orc.counts()
        assert (r.force_evaluations, r.force_skips) == (c["force_evaluations"], c["force_skips"])
        compare_state(sim.agents(), orc.dump(), what=f"c3 after {3 * (chunk + 1)}")
    static = (sim.agents()["flags"] & 1).mean()
    assert static > 0.85


def test_c4_shape_small(engine, oracle_mod):
    wl = CF.c4_large_uniform(6000, seed=3)
    sim = _gpu(engine, wl.params, wl, 2)
    orc = oracle_mod.PortSim(_oparams(oracle_mod, wl.params), wl.x, wl.y, wl.z, wl.d)
    compare_env(sim, orc, "c4 t=0")
    sim.simulate(12)
    orc.simulate(12)
    compare_state(sim.agents(), orc.dump(), what="c4 after 12")
    assert sim.report().force_evaluations == orc.counts()["force_evaluations"]


@pytest.mark.parametrize("byz,bx", [(1, 2), (2, 1), (2, 2), (2, 3), (2, 4), (3, 3), (4, 4)])
def test_bin_geometries_exact(engine, oracle_mod, byz, bx):
    """Every sub-bin geometry (fp32-classified walk) visits exactly the
    reference's candidates: force evaluations, partners and positions."""
    wl = CF.c4_large_uniform(5000, seed=8)
    prm = {**wl.params, "sorting_frequency": 0}
    sim = _gpu(engine, prm, wl, byz, bins_per_box_x=bx)
    orc = oracle_mod.PortSim(_oparams(oracle_mod, prm), wl.x, wl.y, wl.z, wl.d)
    for step in range(2):
        teacher_force(sim, orc)
        e0 = orc.counts()["force_evaluations"]
        sim.simulate(2)
        orc.simulate(2)
        assert sim.report().force_evaluations == orc.counts()["force_evaluations"] - e0
        compare_state(sim.agents(), orc.dump(), what=f"bins {byz}x{bx} step {step}")


def test_large_extent_margin_band(engine, oracle_mod):
    """A domain with a large extent (slack ~ 16 E 2^-24 grows) and clusters of
    touching agents: the fp32 margin band falls back to the exact fp64 test."""
    rng = np.random.default_rng(21)
    centres = rng.uniform(0, 1.0, size=(60, 3)) * np.array([2.0e5, 150.0, 150.0])  # within the box budget
    pts = centres[rng.integers(0, 60, 6000)] + rng.normal(0, 9.0, size=(6000, 3))
    d = np.exp(np.log(10.0) + 0.1 * rng.standard_normal(6000))
    prm = dict(seed=3, simulation_time_step=0.01)
    sim = _gpu(engine, prm, None, 2, bins_per_box_x=3)
    sim.add_agents(pts[:, 0], pts[:, 1], pts[:, 2], d)
    orc = oracle_mod.PortSim(_oparams(oracle_mod, prm), pts[:, 0], pts[:, 1], pts[:, 2], d)
    compare_env(sim, orc, "large extent t=0")
    for step in range(3):
        teacher_force(sim, orc)
        e0 = orc.counts()["force_evaluations"]
        sim.simulate(1)
        orc.simulate(1)
        assert sim.report().force_evaluations == orc.counts()["force_evaluations"] - e0
        compare_state(sim.agents(), orc.dump(), what=f"large extent step {step}")


def test_against_reference_engine(engine, oracle_mod, have_ref):
    """The GPU against the unmodified reference (not only the C port)."""
    if not have_ref:
        pytest.skip("reference build unavailable")
    wl = CF.c1_relaxation(2048, seed=9)
    sim = _gpu(engine, wl.params, wl, 1)
    ref = oracle_mod.RefSim(_oparams(oracle_mod, wl.params), wl.x, wl.y, wl.z, wl.d)
    compare_env(sim, ref, "ref t=0")
    sim.simulate(5)
    ref.simulate(5)
    compare_state(sim.agents(), ref.dump(), what="vs reference")


# ---------------------------------------------------------------- known answers
def _lattice(s, spacing):
    pts = [(x * spacing, y * spacing, z * spacing) for x in range(s) for y in range(s) for z in range(s)]
    return [np.array(v, dtype=float) for v in zip(*pts)]


def test_static_lattice_known_answer(engine):
    """test_scheduler.cpp:464-488."""
    x, y, z = _lattice(3, 10.0)
    sim = engine.Simulation(engine.SimulationParams(detect_static_agents=True))
    sim.add_agents(x, y, z, np.full(27, 10.0))
    sim.simulate(1)
    r = sim.report()
    assert (r.force_evaluations, r.force_skips) == (108, 0)
    sim.simulate(1)
    r = sim.report()
    assert (r.force_evaluations, r.force_skips) == (108, 27)
    sim.simulate(1)
    assert sim.report().force_skips == 54
    assert (sim.agents()["flags"] & 1).sum() == 27


def test_cancelling_triple_known_answer(engine):
    """test_scheduler.cpp:490-519."""
    sim = engine.Simulation(engine.SimulationParams(detect_static_agents=True, force_threshold=10.0))
    sim.add_agents([0.0, 10.0, 20.0], [0.0] * 3, [0.0] * 3, [12.0] * 3)
    sim.simulate(1)
    assert (sim.report().force_evaluations, sim.report().force_skips) == (4, 0)
    sim.simulate(2)
    assert (sim.report().force_evaluations, sim.report().force_skips) == (8, 4)
    a = by_uid(sim.agents())
    assert [int(u) for u, f in zip(a["uid"], a["flags"]) if f & 1] == [0, 2]
    assert list(a["x"]) == [0.0, 10.0, 20.0]


def test_static_front_known_answer(engine):
    """test_scheduler.cpp:521-534 (reference Grow behaviour on one column)."""
    x, y, z = _lattice(3, 10.0)
    mask = np.array([1 if (i // 9 == 0 and (i // 3) % 3 == 1) else 0 for i in range(27)], np.uint8)
    sim = engine.Simulation(engine.SimulationParams(detect_static_agents=True, model=engine.MODEL_GROW,
                                                    model_params=[0.5, 20.0]))
    sim.add_agents(x, y, z, np.full(27, 10.0), behaviour_mask=mask)
    sim.simulate(3)
    a = by_uid(sim.agents())
    assert [int(u) for u, f in zip(a["uid"], a["flags"]) if f & 1] == [18, 19, 20, 24, 25, 26]


def test_static_on_off_same_trajectory(engine):
    """test_scheduler.cpp:536-558: static skipping does not change positions."""
    x, y, z = _lattice(3, 10.0)
    mask = np.array([1 if (i // 9 == 0 and (i // 3) % 3 == 1) else 0 for i in range(27)], np.uint8)
    out = []
    for detect in (True, False):
        sim = engine.Simulation(engine.SimulationParams(detect_static_agents=detect,
                                                        model=engine.MODEL_GROW, model_params=[0.5, 20.0]))
        sim.add_agents(x, y, z, np.full(27, 10.0), behaviour_mask=mask)
        sim.simulate(6)
        out.append((by_uid(sim.agents()), sim.report()))
    (a, ra), (b, rb) = out
    for k in "xyz":
        assert np.max(np.abs(a[k] - b[k])) <= 1e-12
    assert ra.force_skips > 0 and rb.force_skips == 0
    assert ra.force_evaluations < rb.force_evaluations


def test_grid_known_answers(engine):
    """test_grid.cpp:68-86 floor/clamp; :108-120 inclusive radius; :214-227 box = dmax."""
    sim = engine.Simulation(engine.SimulationParams(fixed_box_length=20.0))
    sim.add_agents([0.0, 100.0, 19.999, 100.0], [0.0, 100.0, 20.0, 100.0], [0.0, 100.0, 39.9, 100.0],
                   [10.0] * 4)
    env = sim.environment()
    env.update()
    assert list(env.dims()) == [6, 6, 6] and list(env.origin()) == [0, 0, 0]
    ids = dict(zip(sim.agents()["uid"].tolist(), env.cell_ids().tolist()))
    assert ids[2] == 0 + 6 * (1 + 6 * 1) and ids[3] == 215 and ids[1] == 215
    sim2 = engine.Simulation(engine.SimulationParams())
    sim2.add_agents([0.0, 15.0], [0.0, 0.0], [0.0, 0.0], [15.0, 15.0])
    sim2.environment().update()
    off, u = sim2.environment().neighbors()  # r = 0.5 (15 + 15) = 15 = separation
    assert list(off) == [0, 1, 2] and sorted(u.tolist()) == [0, 1]
    sim3 = engine.Simulation(engine.SimulationParams())
    sim3.add_agents([0.0, 40.0], [0.0, 0.0], [0.0, 0.0], [8.0, 17.5])
    sim3.environment().update()
    assert sim3.environment().box_length() == 17.5 == sim3.environment().largest_agent_diameter()


# ---------------------------------------------------------------- edge cases
def test_empty_population(engine):
    sim = engine.Simulation(engine.SimulationParams(detect_static_agents=True))
    sim.simulate(10)
    r = sim.report()
    assert r.iterations == 10 and r.final_agent_count == 0 and r.force_evaluations == 0
    sim.environment().update()
    assert list(sim.environment().dims()) == [1, 1, 1]
    sim.simulate(0)
    assert sim.report().iterations == 10


def test_single_agent_and_degenerate_volume(engine):
    sim = engine.Simulation(engine.SimulationParams())
    sim.add_agents([5.0], [5.0], [5.0], [10.0])
    sim.simulate(2)
    assert sim.report().force_evaluations == 0
    a = sim.agents()
    assert (a["x"][0], a["y"][0], a["z"][0]) == (5.0, 5.0, 5.0)
    # three coincident agents (test_acceptance.cpp:154-170 instance 7) and the coincident-centre
    # force of magnitude k * overlap (test_mechanics.cpp:55-72)
    sim = engine.Simulation(engine.SimulationParams(simulation_time_step=0.01))
    sim.add_agents([3.0] * 3, [3.0] * 3, [3.0] * 3, [10.0] * 3)
    env = sim.environment()
    env.update()
    off, u = env.neighbors()
    assert list(np.diff(off)) == [2, 2, 2]
    sim.simulate(1)
    a = sim.agents()
    for i in range(3):
        f = math.sqrt(a["fx"][i] ** 2 + a["fy"][i] ** 2 + a["fz"][i] ** 2)
        assert f > 0.0
    sim2 = engine.Simulation(engine.SimulationParams())
    sim2.add_agents([5.0, 5.0], [5.0, 5.0], [5.0, 5.0], [10.0, 10.0])
    sim2.simulate(1)
    b = by_uid(sim2.agents())
    f0 = np.array([b["fx"][0], b["fy"][0], b["fz"][0]])
    f1 = np.array([b["fx"][1], b["fy"][1], b["fz"][1]])
    assert abs(np.linalg.norm(f0) - 20.0) < 1e-12 and np.array_equal(f0, -f1)


@pytest.mark.parametrize("static", [False, True])
def test_contact_boundaries_match_oracle(engine, oracle_mod, static):
    """Exact decision boundaries (coincident, touching, d2 == r^2, box faces)
    against the oracle: cell ids and neighbour sets bit-exact, forces and
    positions within 1e-9, partner counts and evaluation totals exact."""
    x, y, z, d = contact_cases()
    prm = dict(seed=3, simulation_time_step=0.01, detect_static_agents=static)
    sim = engine.Simulation(engine.SimulationParams(**prm))
    sim.add_agents(x, y, z, d)
    orc = oracle_mod.PortSim(_oparams(oracle_mod, prm), x, y, z, d)
    compare_env(sim, orc, "contacts t=0")
    env = sim.environment()
    assert env.box_length() == 14.0
    for step in range(4):
        teacher_force(sim, orc)
        compare_env(sim, orc, f"contacts tf step {step}")
        e0 = orc.counts()["force_evaluations"]
        sim.simulate(1)
        orc.simulate(1)
        compare_state(sim.agents(), orc.dump(), what=f"contacts step {step}")
        assert sim.report().force_evaluations == orc.counts()["force_evaluations"] - e0
    # the touching pairs stay put with zero force, the coincident ones separate
    g = by_uid(sim.agents())
    f = np.sqrt(g["fx"] ** 2 + g["fy"] ** 2 + g["fz"] ** 2)
    assert np.all(f[8:16] == 0.0) and np.all(f[0:8] > 0.0)


def test_errors(engine):
    with pytest.raises(ValueError):
        engine.Simulation(engine.SimulationParams(simulation_time_step=0.0))
    sim = engine.Simulation(engine.SimulationParams(fixed_box_length=5.0))
    sim.add_agents([0.0, 1.0], [0.0, 0.0], [0.0, 0.0], [10.0, 10.0])
    with pytest.raises(engine.AbsimError, match="fixed box"):
        sim.simulate(1)
    sim = engine.Simulation(engine.SimulationParams())
    sim.add_agents([0.0, math.inf], [0.0, 0.0], [0.0, 0.0], [10.0, 10.0])
    with pytest.raises(engine.AbsimError, match="not finite"):
        sim.simulate(1)
    sim = engine.Simulation(engine.SimulationParams())
    with pytest.raises(ValueError, match="diameter"):
        sim.add_agents([0.0], [0.0], [0.0], [0.0])
    with pytest.raises(ValueError, match="uid_count"):
        sim.add_agents([0.0, 20.0], [0.0, 0.0], [0.0, 0.0], [10.0, 10.0], uid=[3, 7], uid_count=5)
    sim.add_agents([0.0, 20.0], [0.0, 0.0], [0.0, 0.0], [10.0, 10.0], uid=[3, 7], uid_count=8)
    sim.add_agents([0.0, 20.0], [0.0, 0.0], [0.0, 0.0], [10.0, 10.0], uid=[3, 7])  # derived
    assert sorted(sim.agents()["uid"].tolist()) == [3, 7]
    assert sim.report().uid_count == 8


def test_download_components_pinned(engine):
    """abs_gpu_download straight into page-locked caller arrays, any subset."""
    import torch
    wl = CF.c1_relaxation(5000, seed=2)
    sim = _gpu(engine, wl.params, wl, 1)
    sim.simulate(2)
    a = sim.agents()
    out = [torch.empty(wl.n, dtype=torch.float64).pin_memory().numpy() for _ in range(3)]
    assert sim.positions(*out) == wl.n
    for k, arr in zip("xyz", out):
        assert np.array_equal(arr, a[k])


def test_sort_matches_reference_order(engine, oracle_mod, have_ref):
    """sort_and_balance order (sort_balance.cpp:88-128) from a storage order
    equal to the reference's (fresh upload)."""
    wl = CF.c1_relaxation(3000, seed=4)
    sim = _gpu(engine, wl.params, wl, 1)
    sim.sort()
    got = sim.agents()["uid"]
    orc = oracle_mod.PortSim(_oparams(oracle_mod, wl.params), wl.x, wl.y, wl.z, wl.d)
    orc.env_update()
    orc.sort()
    assert np.array_equal(got, orc.dump()["uid"])
    if have_ref:
        ref = oracle_mod.RefSim(_oparams(oracle_mod, wl.params), wl.x, wl.y, wl.z, wl.d)
        ref.sort()
        assert np.array_equal(got, ref.dump()["uid"])


def test_inloop_sort_frequency(engine, oracle_mod):
    """sorting_frequency (simulation.cpp:246-247): the Morton sort runs inside
    the iteration loop on the device; results match the oracle that sorts at
    the same iterations."""
    wl = CF.c1_relaxation(2500, seed=6)
    prm = {**wl.params, "sorting_frequency": 2}
    sim = _gpu(engine, prm, wl, 2)
    orc = oracle_mod.PortSim(_oparams(oracle_mod, prm), wl.x, wl.y, wl.z, wl.d)
    for step in range(3):
        sim.simulate(3)
        orc.simulate(3)
        compare_state(sim.agents(), orc.dump(), what=f"sorted c1 after {3 * (step + 1)}")
        assert sim.report().force_evaluations == orc.counts()["force_evaluations"]


def test_sort_order_flat_layout(engine, oracle_mod):
    """2-D Morton table (morton.cpp:124-129, dims[2] == 1): a flat sheet."""
    rng = np.random.default_rng(11)
    n = 1500
    x, y = rng.uniform(0, 300, n), rng.uniform(0, 120, n)
    z, d = np.zeros(n), rng.uniform(8, 12, n)
    prm = dict(seed=1, simulation_time_step=0.01)
    sim = _gpu(engine, prm)
    sim.add_agents(x, y, z, d)
    sim.sort()
    orc = oracle_mod.PortSim(_oparams(oracle_mod, prm), x, y, z, d)
    orc.env_update()
    orc.sort()
    assert np.array_equal(sim.agents()["uid"], orc.dump()["uid"])


def test_removal_worked_example(engine):
    """test_commit.cpp:99-119 on a freshly uploaded (reference-ordered) store."""
    sim = engine.Simulation(engine.SimulationParams())
    sim.add_agents(np.arange(7, dtype=float) * 20, np.zeros(7), np.zeros(7), np.ones(7))
    sim.remove_agents([1, 4, 6])
    assert list(sim.agents()["uid"][np.argsort(sim.storage_keys())]) == [0, 5, 2, 3]
    assert sim.report().agents_removed == 3
    with pytest.raises(ValueError, match="unknown uid"):
        sim.remove_agents([1])  # no longer alive
    sim.simulate(2)
    assert sim.report().final_agent_count == 4


def test_removal_large_unordered(engine, oracle_mod):
    """remove_agents_parallel survivor order (commit.cpp:14-106) for a large
    unordered removal list; slots are looked up on the device."""
    rng = np.random.default_rng(5)
    n = 20000
    x = rng.uniform(0, 400, n)
    y = rng.uniform(0, 400, n)
    z = rng.uniform(0, 400, n)
    d = rng.uniform(8, 12, n)
    rem = rng.choice(n, 3000, replace=False)
    sim = engine.Simulation(engine.SimulationParams())
    sim.add_agents(x, y, z, d)
    sim.remove_agents(rem.astype(np.uint64))
    orc = oracle_mod.PortSim(oracle_mod.OracleParams(), x, y, z, d)
    orc.remove(rem.astype(np.uint32))  # fresh upload: slot == uid
    # the device compacts in O(removed) moves of its own; the reference's
    # survivor slots are the storage keys it carries
    keys = sim.storage_keys()
    assert np.array_equal(np.sort(keys), np.arange(n - len(rem)))
    assert np.array_equal(sim.agents()["uid"][np.argsort(keys)], orc.dump()["uid"])
    with pytest.raises(engine.AbsimError, match="twice"):
        sim.remove_agents([int(sim.agents()["uid"][0])] * 2)


@pytest.mark.parametrize("k,max_disp,threshold", [(5.0, 0.5, 0.0), (2.0, 3.0, 4.0), (0.5, 0.05, 1.0)])
def test_mechanics_parameters(engine, oracle_mod, k, max_disp, threshold):
    """Non-default repulsion_coefficient, max_displacement (the clamp of
    agent.hpp:115-133 active for most agents at dt 0.1) and force_threshold
    (simulation.cpp:485-487: forces at or below it do not move the agent)
    against the oracle, teacher-forced one step at a time."""
    wl = CF.c1_relaxation(3000, seed=11)
    prm = dict(seed=11, simulation_time_step=0.1, repulsion_coefficient=k,
               max_displacement=max_disp, force_threshold=threshold)
    sim = engine.Simulation(engine.SimulationParams(**prm))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    op = oracle_mod.OracleParams(seed=11, dt=0.1, k=k, max_disp=max_disp, threshold=threshold)
    orc = oracle_mod.PortSim(op, wl.x, wl.y, wl.z, wl.d)
    x0 = by_uid(orc.dump())
    for step in range(3):
        teacher_force(sim, orc)
        e0 = orc.counts()["force_evaluations"]
        sim.simulate(1)
        orc.simulate(1)
        compare_state(sim.agents(), orc.dump(), what=f"k={k} max={max_disp} thr={threshold} step {step}")
        assert sim.report().force_evaluations == orc.counts()["force_evaluations"] - e0
    g = by_uid(sim.agents())
    moved = np.sqrt((g["x"] - x0["x"]) ** 2 + (g["y"] - x0["y"]) ** 2 + (g["z"] - x0["z"]) ** 2)
    assert moved.max() <= 3 * max_disp * (1 + 1e-12)


def test_grid_growth_retry(engine, oracle_mod):
    """Agents spreading far beyond the initial grid force a bin-table regrow
    (device-side retry) without changing results."""
    rng = np.random.default_rng(3)
    n = 400
    x, y, z = rng.uniform(0, 30, (3, n))
    d = np.full(n, 10.0)
    prm = dict(simulation_time_step=0.05, max_displacement=3.0)
    sim = engine.Simulation(engine.SimulationParams(**prm))
    sim.add_agents(x, y, z, d)
    orc = oracle_mod.PortSim(oracle_mod.OracleParams(dt=0.05), x, y, z, d)
    for _ in range(6):
        # teacher-forced: free-running strong repulsion is chaotic over tens of
        # steps, so compare one step at a time from the oracle's state
        teacher_force(sim, orc)
        sim.simulate(10)
        orc.simulate(10)
        compare_state(sim.agents(), orc.dump(), ints=False, what="spreading")
    assert sim.environment().dims().prod() > 4 * 4 * 4


def test_reupload_with_growing_population(engine, oracle_mod):
    """Re-uploading a larger population (capacity regrowth) after a step must
    not leak the previous cell table into the next binning."""
    wl = CF.c1_relaxation(3000, seed=1)
    sim = _gpu(engine, wl.params, None, 2)
    for n in (600, 1500, 3000):
        sim.add_agents(wl.x[:n], wl.y[:n], wl.z[:n], wl.d[:n])
        sim.simulate(2)
        orc = oracle_mod.PortSim(_oparams(oracle_mod, wl.params), wl.x[:n], wl.y[:n], wl.z[:n], wl.d[:n])
        orc.simulate(2)
        compare_state(sim.agents(), orc.dump(), what=f"reupload n={n}")


def test_phase_report_categories(engine):
    """SimulationReport wall-time categories (report.hpp:12-23) from device
    events; they add up to the per-iteration times and export in the
    reference bench's schema."""
    from paper_2301_06984_b200 import report as R
    wl = CF.c1_relaxation(4000, seed=3)
    sim = _gpu(engine, {**wl.params, "sorting_frequency": 2}, wl, 1)
    sim.simulate(1)
    sim.reset_timers(True)
    sim.simulate(5)
    r = sim.phase_report()
    assert len(r.per_iteration_ms) == 5
    parts = r.env_update_ms + r.sorting_ms + r.agent_ops_ms + r.setup_teardown_ms
    assert abs(parts - sum(r.per_iteration_ms)) < 1e-3 * max(parts, 1.0)
    assert r.env_update_ms > 0 and r.agent_ops_ms > 0 and r.sorting_ms > 0
    assert r.total_wall_ms > 0 and r.peak_rss_bytes > 0
    j = R.report_json(R.RunOptions(model="c1", agents=wl.n, iterations=6, sorting_frequency=2), r)
    assert j["report"]["per_iteration_ms"] == r.per_iteration_ms
